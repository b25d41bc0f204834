#!/bin/bash
# --set full captures of chosen kernels: tools/gpu_ncu.sh <tag> <config>:<kernel regex>:<skip> ...
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=$1; shift
for spec in "$@"; do
  IFS=: read CFG KR SKIP <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KR" -s ${SKIP:-1} -c 1 \
     -o gpurun_out/${TAG}_${CFG}_${KR} -f python tools/solve_once.py $CFG > gpurun_out/${TAG}_${CFG}_${KR}.log 2>&1
  echo "ncu $CFG $KR rc=$?"
done
