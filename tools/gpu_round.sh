#!/bin/bash
# Round evidence in one gpurun call: GPU tests, smoke, bench lines (C5 headline, C2), the ncu
# launch list of the C5 bench command, and --set full captures of the two top C5 kernels.
#   tools/gpu_round.sh <tag>
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-r}
nvidia-smi > gpurun_out/${TAG}_nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
bash tools/gpu_bench.sh ${TAG}
for k in "p2p_warp:2" "s2l_batch:1"; do
  KR=${k%%:*}; N=${k##*:}
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$KR" -s $N -c $N \
     -o gpurun_out/${TAG}_full_${KR}_C5 -f python tools/solve_once.py C5 > gpurun_out/${TAG}_full_${KR}_C5.log 2>&1; echo "ncu full $KR rc=$?"
done
