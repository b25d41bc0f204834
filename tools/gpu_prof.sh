#!/bin/bash
# ncu launch lists of one solve per config, plus a --set full capture of one kernel.
#   tools/gpu_prof.sh <kernel-regex> <tag> configs...
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
KR=$1; TAG=$2; shift 2
for c in "$@"; do
  timeout 300 python tools/solve_once.py $c > /dev/null 2>&1 || { echo "$c plain run failed"; continue; }
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
     --log-file gpurun_out/${TAG}_launch_$c.csv python tools/solve_once.py $c --warm 0 > /dev/null 2>&1; echo "$c launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KR" -s 1 -c 1 \
     -o gpurun_out/${TAG}_full_$c -f python tools/solve_once.py $c > gpurun_out/${TAG}_full_$c.log 2>&1; echo "$c full rc=$?"
done
