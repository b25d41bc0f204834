cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
rm -f gpurun_out/m2m.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fmm_small or tensor" > gpurun_out/pytest_p.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_p.log
for t in 256 128 64 256 128 64; do
  CYLFMM_M2M_THREADS=$t timeout 300 python tools/phase_bench.py C2 --reps 4 > gpurun_out/f.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/f.json')); print('threads=$t', d['config'], d['ms_m2m'])" >> gpurun_out/m2m.txt
  CYLFMM_M2M_THREADS=$t timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('threads=$t bench', d['ms_per_step'])" >> gpurun_out/m2m.txt
done
for t in 256 128; do CYLFMM_M2M_THREADS=$t timeout 300 python tools/phase_bench.py C4 --reps 2 > gpurun_out/f.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/f.json')); print('threads=$t', d['config'], d['ms_m2m'])" >> gpurun_out/m2m.txt; done
