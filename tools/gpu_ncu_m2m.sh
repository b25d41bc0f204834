cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"m2m_kernel|l2l_kernel|prescale" -s 12 -c 4 \
   -o gpurun_out/prof_m2m python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_m2m.log 2>&1; echo "rc=$?"
