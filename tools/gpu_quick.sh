#!/bin/bash
# Quick iteration: GPU tests matching a -k expression (optional) and bench phase lines.
#   tools/gpu_quick.sh <tag> "<pytest -k expr or ''>" <configs...>
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=$1; K=$2; shift 2
if [ -n "$K" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
fi
for c in "$@"; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err; echo "bench $c rc=$?"
  python - "$TAG" "$c" <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/{sys.argv[1]}_bench_{sys.argv[2]}.json").read().strip().splitlines()[-1])
print(sys.argv[2], round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['phase_ms'].items()}, (d.get('fixed_geometry') or {}).get('ms_per_step_cuda_graph'))
PY
done
