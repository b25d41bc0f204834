#!/bin/bash
# tools/gpu_g.sh <tag>: all GPU tests + smoke, then C4 (adaptive tree, as bench.py runs it): launch
# list of the bench command and --set full of its S2L and near-field kernels (raw pages as CSV:
# the reports of 20 launches exceed what gpurun copies back)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
TAG=$1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/${TAG}_launch_c4.csv python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_launch_c4.log 2>&1; echo "ncu launch rc=$?"
for k in "s2l_batch_units:1:1" "p2p_warp:0:12"; do
  IFS=: read KR SK N <<< "$k"
  timeout 900 ncu --set full --clock-control none -k regex:"$KR" -s $SK -c $N \
     -o /tmp/${TAG}_full_${KR}_C4 -f python tools/solve_once.py C4 --adaptive 11 224 > gpurun_out/${TAG}_full_${KR}_C4.log 2>&1; echo "ncu full $KR rc=$?"
  ncu -i /tmp/${TAG}_full_${KR}_C4.ncu-rep --page raw --csv > gpurun_out/${TAG}_full_${KR}_C4.csv 2>/dev/null
done
du -sh gpurun_out
