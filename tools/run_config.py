#!/usr/bin/env python
"""Run one BASELINE config (C2..C5) through the GPU FMM with per-phase timings, then check a
seeded sample of field points against the oracle FMM (parity, 1e-12) and the GPU direct sum
(eps vs direct, the paper's metric P:697-703).  Diagnostic tool (GPU box); prints one JSON line.

  python tools/run_config.py C4 [--sample 128] [--depth D] [--adaptive SIGMA] [--chunk KW] [--no-oracle]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def eps(A, B):
    return np.abs(A - B).max(axis=0) / np.maximum(np.abs(B).max(axis=0), 1e-300)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--sample", type=int, default=128)
    ap.add_argument("--depth", type=int, default=0)
    ap.add_argument("--chunk", type=int, default=0)
    ap.add_argument("--adaptive", type=int, default=0, help="adaptive source tree leaf size (R#26)")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--no-oracle", action="store_true")
    a = ap.parse_args()
    import torch
    import paper_2301_01179_b200 as g
    from paper_2301_01179_b200.inputs import CONFIGS
    t0 = time.time()
    pr = CONFIGS[a.config]()
    d = a.depth or pr.depth
    rec = {"config": a.config, "n_src": len(pr.sr), "n_fld": len(pr.fr), "K": pr.K, "p": pr.p,
           "depth": d, "adaptive_leaf": a.adaptive, "gen_s": round(time.time() - t0, 1)}
    dev = torch.device("cuda", 0)
    sr, sz = torch.as_tensor(pr.sr, device=dev), torch.as_tensor(pr.sz, device=dev)
    S = torch.as_tensor(pr.S, device=dev)
    fr, fz = torch.as_tensor(pr.fr, device=dev), torch.as_tensor(pr.fz, device=dev)
    plan = g.Plan(g.FMMConfig(n_modes=pr.K, order=pr.p, depth=d, L=pr.L, z0=pr.z0,
                              mode_chunk=a.chunk, adaptive_leaf=a.adaptive))
    out, tm = plan.solve(sr, sz, S, fr, fz, timings=True)
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.solve(sr, sz, S, fr, fz, out=out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    rec["ms_solve"] = min(ts)
    rec["phase_ms"] = {k: round(v, 3) for k, v in tm.items() if k.startswith("ms_")}
    rec.update({k: tm[k] for k in ("n_near_pairs", "n_skipped", "n_s2l_pairs", "kernel_launches")})
    rec["mem_gb"] = round(torch.cuda.max_memory_allocated() / 1e9, 2)
    rng = np.random.default_rng(1234)
    idx = np.sort(rng.choice(len(pr.fr), size=min(a.sample, len(pr.fr)), replace=False))
    F = out.cpu().numpy()[idx]
    D = g.direct(sr, sz, S, fr[torch.as_tensor(idx, device=dev)],
                 fz[torch.as_tensor(idx, device=dev)]).cpu().numpy()
    rec["eps_vs_direct"] = [float(f"{v:.3g}") for v in eps(F, D)]
    if not a.no_oracle:
        import oracle
        oracle.build()
        t0 = time.time()
        O, sk = oracle.fmm(pr.sr, pr.sz, pr.S, pr.fr[idx], pr.fz[idx], pr.p, d, pr.L, pr.z0,
                           leaf_src=a.adaptive)
        rec["oracle_s"] = round(time.time() - t0, 1)
        e = eps(F, O)
        rec["eps_vs_oracle_fmm_max"] = float(e.max())
        Od, _ = oracle.direct(pr.sr, pr.sz, pr.S, pr.fr[idx], pr.fz[idx])
        rec["gpu_direct_vs_oracle_direct_max"] = float(eps(D, Od).max())
    print(json.dumps(rec), flush=True)
    plan.close()


if __name__ == "__main__":
    main()
