cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
rm -f gpurun_out/needq.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for i in 1 2 3; do timeout 300 python bench.py --no-cpu-baseline --steps 40 > gpurun_out/b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('bench', d['ms_per_step'], d['e2e']['ms_per_step'])" >> gpurun_out/needq.txt; done
timeout 900 python tools/run_config.py C5 --sample 48 > gpurun_out/cfg_C5.json 2> gpurun_out/cfg_C5.err
