cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
CMD="python tools/phase_bench.py C4 --reps 1"
timeout 600 $CMD > gpurun_out/c4_plain.json 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:p2p_kernel -s 1 -c 1 -o gpurun_out/prof_c4 $CMD > gpurun_out/ncu_c4.log 2>&1
echo "ncu rc=$?"
