cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
rm -f gpurun_out/sortq.txt
for it in 8 1 2 4 8 1 2 4; do CYLFMM_SORT_ITEMS=$it timeout 300 python bench.py --no-cpu-baseline --steps 40 > gpurun_out/b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('items=$it bench', d['ms_per_step'], d['phase_ms']['ms_tree'])" >> gpurun_out/sortq.txt; done
