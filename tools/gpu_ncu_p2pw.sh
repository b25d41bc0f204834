cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"p2p" -s 2 -c 1 \
   -o gpurun_out/p2pw_c2 python tools/phase_bench.py C2 --reps 1 > gpurun_out/ncu_p2pw.log 2>&1; echo "rc=$?"
CYLFMM_P2P_VARIANT=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"p2p" -s 2 -c 1 \
   -o gpurun_out/p2p_c2 python tools/phase_bench.py C2 --reps 1 > gpurun_out/ncu_p2p.log 2>&1; echo "rc=$?"
