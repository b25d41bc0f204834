cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
   --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-s2l_kernel|p2p_kernel|tensor_seed|tensor_fill}" -s 12 -c 4 \
   -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu2 rc=$?"
