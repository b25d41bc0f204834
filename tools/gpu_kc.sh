#!/bin/bash
# S2L depth-chunk (KC) variants at p = 12 / 16: per-phase times.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for v in 0 1 2; do
  for c in C3 C4; do CYLFMM_S2L_VARIANT=$v timeout 600 python tools/phase_bench.py $c --reps 5; done
done > gpurun_out/kc.jsonl 2> gpurun_out/kc.err
