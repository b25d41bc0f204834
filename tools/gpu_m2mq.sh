cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
rm -f gpurun_out/m2mq.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for c in C2 C3 C4; do timeout 300 python tools/phase_bench.py $c --reps 3 > gpurun_out/f.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/f.json')); print(d['config'], 'm2m', d['ms_m2m'], 'l2l', d['ms_l2l'])" >> gpurun_out/m2mq.txt; done
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('bench', d['ms_per_step'])" >> gpurun_out/m2mq.txt; done
