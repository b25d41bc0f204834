cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"p2p_warp|s2l_kernel" -s 0 -c 2 \
   -o gpurun_out/prof_c4 python tools/phase_bench.py C4 --reps 1 > gpurun_out/ncu_c4.log 2>&1; echo "rc=$?"
