"""C5 point (0.2549, 1.3083), mode 64: per-pair G^(n) GPU vs oracle for the near sources."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2301_01179_b200 as g
from paper_2301_01179_b200.inputs import CONFIGS
import oracle
pr = CONFIGS["C5"]()
i0 = 1068347
r0, z0 = pr.fr[i0], pr.fz[i0]
h = pr.L / 2**pr.depth
ix, iz = int(r0 / h), int((z0 - pr.z0) / h)
bx = np.minimum((pr.sr / h).astype(int), 2**pr.depth - 1)
bz = np.minimum(((pr.sz - pr.z0) / h).astype(int), 2**pr.depth - 1)
near = np.where((np.abs(bx - ix) <= 1) & (np.abs(bz - iz) <= 1))[0]
print("near sources", len(near))
sr, sz, S = pr.sr[near], pr.sz[near], pr.S[near]
K = pr.K
Gg = g.greens_batch(np.full(len(near), r0), sr, np.full(len(near), z0) - sz, K).cpu().numpy()
Go = np.array([oracle.greens(r0, a, z0 - b, K - 1) for a, b in zip(sr, sz)])
rel = np.abs(Gg - Go) / np.abs(Go).max(axis=0)
chi = (r0**2 + sr**2 + (z0 - sz)**2) / (2 * r0 * sr)
for n in [0, 16, 32, 48, 64]:
    k = int(np.argmax(rel[:, n]))
    print(f"n={n} max rel (per-mode max-normalised) {rel[k, n]:.2e} at chi-1={chi[k]-1:.3e} G={Go[k,n]:.6e} r1={sr[k]!r} x={z0-sz[k]!r}")
# contributions
cg = (S * Gg).sum(axis=0); co = (S * Go).sum(axis=0)
print("near-field sum mode 64 gpu", cg[64], "oracle", co[64], "diff", abs(cg[64] - co[64]))
D = g.direct(sr, sz, S, np.array([r0]), np.array([z0])).cpu().numpy()[0]
Do, _ = oracle.direct(sr, sz, S, np.array([r0]), np.array([z0]))
print("direct kernel mode 64", D[64], "oracle", Do[0, 64], "diff", abs(D[64] - Do[0, 64]))
np.save("gpurun_out/c5pairs.npy", np.stack([sr, sz, chi, rel[:, 64]], axis=1))
