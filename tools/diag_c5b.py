"""C5 diagnostic at run_config's sample: both near-field kernels vs the oracle FMM per mode."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2301_01179_b200 as g
from paper_2301_01179_b200.inputs import CONFIGS
import oracle
pr = CONFIGS["C5"]()
dev = torch.device("cuda", 0)
t = lambda x: torch.as_tensor(x, device=dev)
rng = np.random.default_rng(1234)
idx = np.sort(rng.choice(len(pr.fr), size=96, replace=False))
O, _ = oracle.fmm(pr.sr, pr.sz, pr.S, pr.fr[idx], pr.fz[idx], pr.p, pr.depth, pr.L, pr.z0)
mx = np.abs(O).max(axis=0)
for v in ["0", "1"]:
    os.environ["CYLFMM_P2P_VARIANT"] = v
    plan = g.Plan(g.FMMConfig(n_modes=pr.K, order=pr.p, depth=pr.depth, L=pr.L, z0=pr.z0))
    F = plan.solve(t(pr.sr), t(pr.sz), t(pr.S), t(pr.fr), t(pr.fz))[t(idx)].cpu().numpy()
    plan.close()
    d = np.abs(F - O)
    e = d.max(axis=0) / mx
    m = int(np.argmax(e)); pt = int(np.argmax(d[:, m]))
    print("variant", v, "max eps", e.max(), "mode", m, "point", int(idx[pt]), pr.fr[idx[pt]], pr.fz[idx[pt]],
          "F", F[pt, m], "O", O[pt, m], "max|O| mode", mx[m])
    print(np.array2string(e, precision=1))
