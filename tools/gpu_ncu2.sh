#!/bin/bash
# --set full capture of N consecutive launches of one kernel: tools/gpu_ncu2.sh <tag> <config> <regex> <skip> <count>
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$3" -s $4 -c $5 \
   -o gpurun_out/$1_$2_$3 -f python tools/solve_once.py $2 > gpurun_out/$1_$2_$3.log 2>&1
echo "ncu rc=$?"
