#!/usr/bin/env python
"""FMM solve vs the GPU direct modal sum on the same B200 (the paper's 'speedup over direct
evaluation', as context).  Prints one JSON line per config."""
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
        plan = g.Plan(g.FMMConfig(n_modes=pr.K, order=pr.p, depth=pr.depth, L=pr.L, z0=pr.z0))
        out = torch.empty((len(pr.fr), pr.K), dtype=torch.complex128, device=dev)

        def timed(fn, reps):
            for _ in range(2):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / reps

        t_fmm = timed(lambda: plan.solve(sr, sz, S, fr, fz, out=out), 10)
        t_dir = min(timed(lambda: g.direct(sr, sz, S, fr, fz), 1) for _ in range(3))
        plan.close()
        print(json.dumps({"config": name, "ms_fmm": round(t_fmm, 3), "ms_direct": round(t_dir, 3),
                          "speedup": round(t_dir / t_fmm, 1)}), flush=True)


if __name__ == "__main__":
    main()
