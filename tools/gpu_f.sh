#!/bin/bash
# iteration: all GPU tests, then quick bench phase lines.   tools/gpu_f.sh <tag> <configs...>
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
TAG=$1; shift
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
for c in "$@"; do
  if [ "$c" = "C1" ]; then
    timeout 300 python bench.py --config C1 --no-cpu-baseline > gpurun_out/${TAG}_bench_C1.json 2> gpurun_out/${TAG}_bench_C1.err; echo "bench C1 rc=$?"
    python -c "
import json; d=json.loads(open('gpurun_out/${TAG}_bench_C1.json').read().strip().splitlines()[-1])
print('C1', d['ms_per_step'], d['ms_per_step_l2_flushed'], d['ms_per_call_synchronous_api'], d['roofline']['frac'])"
    continue
  fi
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err; echo "bench $c rc=$?"
  python - "$TAG" "$c" <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/{sys.argv[1]}_bench_{sys.argv[2]}.json").read().strip().splitlines()[-1])
print(sys.argv[2], round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['phase_ms'].items()})
PY
done
