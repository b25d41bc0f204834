#!/usr/bin/env python
"""Per-phase solve timings (median over reps) for one config at a chosen depth / mode chunk;
used to compare builds on the GPU box.  Prints one JSON line."""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="C2")
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--depth", type=int, default=0)
    ap.add_argument("--chunk", type=int, default=0)
    a = ap.parse_args()
    import torch
    import paper_2301_01179_b200 as g
    from paper_2301_01179_b200.inputs import CONFIGS
    pr = CONFIGS[a.config]()
    dev = torch.device("cuda", 0)
    t = lambda x: torch.as_tensor(x, device=dev)  # noqa: E731
    sr, sz, S, fr, fz = t(pr.sr), t(pr.sz), t(pr.S), t(pr.fr), t(pr.fz)
    plan = g.Plan(g.FMMConfig(n_modes=pr.K, order=pr.p, depth=a.depth or pr.depth, L=pr.L,
                              z0=pr.z0, mode_chunk=a.chunk))
    out = torch.empty((len(pr.fr), pr.K), dtype=torch.complex128, device=dev)
    recs = []
    for i in range(a.reps + 2):
        _, tm = plan.solve(sr, sz, S, fr, fz, out=out, timings=True)
        if i >= 2:
            recs.append(tm)
    med = {k: round(statistics.median(r[k] for r in recs), 4) for k in recs[0] if k.startswith("ms_")}
    print(json.dumps({"config": a.config, "env": {k: v for k, v in os.environ.items()
                                                   if k.startswith("CYLFMM_")}, **med}), flush=True)
    plan.close()


if __name__ == "__main__":
    main()
