#!/bin/bash
# bench lines (C5 default, C2, C3, C4 adaptive and uniform) and the ncu launch list of the C5 bench command.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-b}
timeout 900 python bench.py > gpurun_out/${TAG}_bench_c5.json 2> gpurun_out/${TAG}_bench_c5.err; echo "bench C5 rc=$?"
tail -c 3000 gpurun_out/${TAG}_bench_c5.json; tail -3 gpurun_out/${TAG}_bench_c5.err
for c in C2 C3 C4; do
timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_bench_${c,,}.json 2> gpurun_out/${TAG}_bench_${c,,}.err; echo "bench $c rc=$?"
done
timeout 600 python bench.py --config C4 --adaptive 0 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_c4_uniform.json 2> gpurun_out/${TAG}_bench_c4_uniform.err; echo "bench C4 uniform rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/${TAG}_launch_c5.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "ncu launch rc=$?"
