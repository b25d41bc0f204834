#!/bin/bash
# One gpurun call: GPU tests, the C5 diagnostic, a bench line, the ncu launch list, one --set
# full capture of the top kernels, and the C2..C5 full-size configs with oracle parity.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/cfg_*.json
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
   --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"s2l_kernel|p2p_warp" -s 6 -c 2 \
   -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu2 rc=$?"
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python tools/direct_speedup.py C2 C3 > gpurun_out/speedup.jsonl 2> gpurun_out/speedup.err
for c in C2 C3 C4 C5; do
  timeout 1200 python tools/run_config.py $c --sample 96 > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err; echo "$c rc=$?"
done
