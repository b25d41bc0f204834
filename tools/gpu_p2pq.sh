cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
rm -f gpurun_out/p2pq.jsonl
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fmm or near or greens or direct" > gpurun_out/pytest_p.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_p.log
for c in C2 C3 C4 C5; do timeout 600 python tools/phase_bench.py $c --reps 4 >> gpurun_out/p2pq.jsonl 2>>gpurun_out/p2pq.err; done
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --steps 40 > gpurun_out/b.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('bench', d['ms_per_step'])" >> gpurun_out/p2pq.jsonl; done
