cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
rm -f gpurun_out/ord.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fmm" > gpurun_out/pytest_p.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_p.log
for v in 1 0 1 0; do
  for c in C2 C3 C4; do CYLFMM_S2L_ASC=$v timeout 300 python tools/phase_bench.py $c --reps 3 > gpurun_out/f.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/f.json')); print('asc=$v', d['config'], d['ms_s2l'])" >> gpurun_out/ord.txt; done
  CYLFMM_S2L_ASC=$v timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('asc=$v bench', d['ms_per_step'])" >> gpurun_out/ord.txt
done
