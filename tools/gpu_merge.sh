#!/bin/bash
# S2L merged (di,-3)/(di,+3) offsets: GPU tests, per-phase times C2..C5, bench line.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a gpurun_out/pytest_gpu.log
for c in C2 C3 C4 C5; do timeout 600 python tools/phase_bench.py $c --reps 5; done > gpurun_out/phase_merge.jsonl 2> gpurun_out/phase_merge.err
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
