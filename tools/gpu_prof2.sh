#!/bin/bash
# ncu --set full of N launches of one kernel in one solve of a config.
#   tools/gpu_prof2.sh <kernel-regex> <tag> <config> [count]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
KR=$1; TAG=$2; C=$3; N=${4:-1}
timeout 300 python tools/solve_once.py $C > /dev/null 2>&1 || { echo "$C plain run failed"; exit 1; }
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$KR" -s $N -c $N \
   -o gpurun_out/${TAG}_full_$C -f python tools/solve_once.py $C > gpurun_out/${TAG}_full_$C.log 2>&1; echo "$C full rc=$?"
