cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
rm -f gpurun_out/reuse.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for c in C2 C3 C4; do timeout 300 python tools/phase_bench.py $c --reps 3 > gpurun_out/f.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/f.json')); print(d['config'], 's2l', d['ms_s2l'])" >> gpurun_out/reuse.txt; done
for i in 1 2 3; do timeout 300 python bench.py --no-cpu-baseline --steps 40 > gpurun_out/b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('bench', d['ms_per_step'], d['roofline']['frac'])" >> gpurun_out/reuse.txt; done
timeout 600 python tools/run_config.py C2 --sample 96 > gpurun_out/cfg_C2.json 2> gpurun_out/cfg_C2.err
