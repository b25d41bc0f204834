"""C5 diagnostic: near-field kernels (warp-task vs CTA) against each other and the oracle FMM."""
import os, sys, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2301_01179_b200 as g
from paper_2301_01179_b200.inputs import CONFIGS
import oracle
pr = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C5"]()
dev = torch.device("cuda", 0)
t = lambda x: torch.as_tensor(x, device=dev)
outs = {}
for v in ["0", "1"]:
    os.environ["CYLFMM_P2P_VARIANT"] = v
    plan = g.Plan(g.FMMConfig(n_modes=pr.K, order=pr.p, depth=pr.depth, L=pr.L, z0=pr.z0))
    outs[v] = plan.solve(t(pr.sr), t(pr.sz), t(pr.S), t(pr.fr), t(pr.fz))
    torch.cuda.synchronize()
    plan.close()
A, B = outs["0"], outs["1"]
d = (A - B).abs()
mx = B.abs().amax(dim=0)
eps = (d.amax(dim=0) / mx).cpu().numpy()
print("eps(warp vs cta) per mode:", np.array2string(eps, precision=2))
arg = d.argmax(dim=0).cpu().numpy()
worst = int(arg[int(np.argmax(eps))])
print("worst mode", int(np.argmax(eps)), "field", worst, "r,z", pr.fr[worst], pr.fz[worst])
idx = np.unique(np.concatenate([arg[np.argsort(eps)[-6:]], [worst]]))
O, _ = oracle.fmm(pr.sr, pr.sz, pr.S, pr.fr[idx], pr.fz[idx], pr.p, pr.depth, pr.L, pr.z0)
mxc = mx.cpu().numpy()
for v in ["0", "1"]:
    Fv = outs[v][t(idx)].cpu().numpy()
    e = np.abs(Fv - O).max(axis=0) / mxc
    print("variant", v, "eps vs oracle at worst points per mode:", np.array2string(e, precision=2))
for i in idx:
    print("field", int(i), "r,z", pr.fr[i], pr.fz[i])
