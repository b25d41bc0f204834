#!/usr/bin/env python
"""Measured solve time against tree depth at each config's order, beside the cost model of
cylfmm_select_params (R#25): checks that the modelled argmin is the measured one (or close).
Prints one JSON line per (config, depth)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2301_01179_b200 as g
    from paper_2301_01179_b200.inputs import CONFIGS
    for name in (sys.argv[1:] or ["C2", "C3"]):
        pr = CONFIGS[name]()
        dev = torch.device("cuda", 0)
        t = lambda x: torch.as_tensor(x, device=dev)  # noqa: E731
        sr, sz, S, fr, fz = t(pr.sr), t(pr.sz), t(pr.S), t(pr.fr), t(pr.fz)
        dmin, dmax = max(pr.depth - 2, 2), min(pr.depth + 2, 11)
        cfg, info = g.select_params(pr.sr, pr.sz, pr.fr, pr.fz, pr.K, 1e-3, L=pr.L, z0=pr.z0,
                                    depth_min=dmin, depth_max=dmax)
        # the model at the config's own order (select_params picks the order from tol; re-run
        # with the tol whose order is pr.p so est_ms is at that order)
        tol = 0.1 * 10.0 ** (-0.4 * pr.p)
        cfg, info = g.select_params(pr.sr, pr.sz, pr.fr, pr.fz, pr.K, tol * (1 + 1e-9), L=pr.L,
                                    z0=pr.z0, depth_min=dmin, depth_max=dmax)
        out = torch.empty((len(pr.fr), pr.K), dtype=torch.complex128, device=dev)
        for q, d in enumerate(info["depths"]):
            plan = g.Plan(g.FMMConfig(n_modes=pr.K, order=pr.p, depth=int(d), L=pr.L, z0=pr.z0))
            reps = 10 if pr.K * len(pr.fr) < 1e7 else 3
            for _ in range(2):
                plan.solve(sr, sz, S, fr, fz, out=out)
            torch.cuda.synchronize()
            ts = []
            for _ in range(reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                plan.solve(sr, sz, S, fr, fz, out=out)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            plan.close()
            print(json.dumps({"config": name, "order": pr.p, "depth": int(d),
                              "ms_measured": round(min(ts), 3),
                              "ms_model": round(float(info["est_ms"][q]), 3),
                              "near_pairs": int(info["near_pairs"][q]),
                              "s2l_pairs": int(info["s2l_pairs"][q]),
                              "model_choice": cfg.depth, "config_depth": pr.depth}), flush=True)


if __name__ == "__main__":
    main()
