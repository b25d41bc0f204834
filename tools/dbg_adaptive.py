import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2301_01179_b200 as g
from paper_2301_01179_b200.inputs import CONFIGS
pr = CONFIGS["C4"]()
sigma, d = int(sys.argv[1]), int(sys.argv[2])
dev = torch.device("cuda", 0)
t = lambda a: torch.as_tensor(a, device=dev)
plan = g.Plan(g.FMMConfig(n_modes=pr.K, order=pr.p, depth=d, L=pr.L, z0=pr.z0, adaptive_leaf=sigma))
sr, sz, S = t(pr.sr), t(pr.sz), t(pr.S)
for i in range(2):
    out, tm = plan.solve(sr, sz, S, sr, sz, timings=True)
    torch.cuda.synchronize()
    print(i, 'ok', tm['n_near_pairs'], tm['n_s2l_pairs'], flush=True)
