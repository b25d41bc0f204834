#!/bin/bash
# S2L tiling variants at p = 16: per-phase times (C4, C5) and the parity tests under the variant.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for v in 0 2; do
  for c in C4 C5; do CYLFMM_S2L_VARIANT=$v timeout 600 python tools/phase_bench.py $c --reps 3; done
done > gpurun_out/kc.jsonl 2> gpurun_out/kc.err
CYLFMM_S2L_VARIANT=2 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fmm" > gpurun_out/kc_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/kc_pytest.log
