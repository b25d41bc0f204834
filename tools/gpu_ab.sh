#!/bin/bash
# A/B of two builds in one call: ab_old/ (a checkout of an earlier commit with its own .so) vs the tree.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for c in "$@"; do
  for w in old new old new; do
    d=.; [ $w = old ] && d=ab_old
    (cd $d && timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 2>/dev/null | tail -1 > /tmp/ab.json; python -c "
import json; d=json.loads(open('/tmp/ab.json').read()); print('$c $w', round(d['ms_per_step'],3), {k:round(v,2) for k,v in d['phase_ms'].items() if k in ('ms_p2m','ms_l2p','ms_p2p','ms_s2l')})")
  done
done
