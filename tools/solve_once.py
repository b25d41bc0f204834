#!/usr/bin/env python
"""Profiling driver: build one BASELINE config, run `--warm` solves then one more (device inputs,
no timings), so that ncu can skip the warm-up launches.   python tools/solve_once.py C3 [--warm 1]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--warm", type=int, default=1)
    ap.add_argument("--adaptive", type=int, nargs=2, metavar=("DEPTH", "LEAF"),
                    help="adaptive source tree (bench.py's C4: 11 224)")
    a = ap.parse_args()
    import torch
    import paper_2301_01179_b200 as g
    from paper_2301_01179_b200.inputs import CONFIGS
    pr = CONFIGS[a.config]()
    dev = torch.device("cuda", 0)
    sr, sz = torch.as_tensor(pr.sr, device=dev), torch.as_tensor(pr.sz, device=dev)
    S = torch.as_tensor(pr.S, device=dev)
    if pr.fields_are_sources:
        fr, fz = sr, sz
    else:
        fr, fz = torch.as_tensor(pr.fr, device=dev), torch.as_tensor(pr.fz, device=dev)
    depth, leaf = a.adaptive if a.adaptive else (pr.depth, 0)
    plan = g.Plan(g.FMMConfig(n_modes=pr.K, order=pr.p, depth=depth, L=pr.L, z0=pr.z0,
                              adaptive_leaf=leaf))
    out = torch.empty((len(pr.fr), pr.K), dtype=torch.complex128, device=dev)
    for _ in range(a.warm + 1):
        plan.solve(sr, sz, S, fr, fz, out=out)
    torch.cuda.synchronize()
    plan.close()


if __name__ == "__main__":
    main()
