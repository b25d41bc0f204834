cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
rm -f gpurun_out/seed.txt
for t in 128 64 128 64; do
  CYLFMM_SEED_THREADS=$t timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tensor" > gpurun_out/pytest_p$t.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_p$t.log
  CYLFMM_SEED_THREADS=$t timeout 300 python tools/phase_bench.py C2 --reps 4 > gpurun_out/f.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/f.json')); print('threads=$t', d['config'], d['ms_tensor'])" >> gpurun_out/seed.txt
  CYLFMM_SEED_THREADS=$t timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('threads=$t bench', d['ms_per_step'])" >> gpurun_out/seed.txt
done
