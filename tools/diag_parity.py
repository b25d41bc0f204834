"""Diagnostics: per-mode / per-order GPU-vs-oracle errors for the conditioning-limited cases."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_2301_01179_b200 as g
from paper_2301_01179_b200.inputs import uniform_rings
np.set_printoptions(precision=2, linewidth=200)
rng = np.random.default_rng(513 * 7 + 129)
sr, sz, S = uniform_rings(rng, 513, 80)
fr, fz, _ = uniform_rings(rng, 129, 1)
ref, _ = oracle.direct(sr, sz, S, fr, fz)
out = g.direct(sr, sz, S, fr, fz).cpu().numpy()
e = np.abs(out - ref).max(0) / np.abs(ref).max(0)
print("direct K=80 eps per mode:\n", e)
for p, K in [(8, 17), (12, 9), (16, 5)]:
    geo = [(2.5, 0.5, 0.0), (3.5, 1.5, 2.0), (10.5, 10.5, 2.0), (16.5, 13.5, 3.0),
           (1.3, 0.7, 0.9), (0.8, 0.8, 0.5), (5.5, 3.5, 1.0)]
    r, r1, x = (np.array(v) for v in zip(*geo))
    T = g.tensor_batch(r, r1, x, K, p).cpu().numpy()
    a = np.arange(p + 1)[:, None, None]; b = np.arange(p + 1)[None, :, None]; c = np.arange(2 * p + 1)[None, None, :]
    order = a + b + c
    for q in range(len(r)):
        R = oracle.tensor(r[q], r1[q], x[q], K - 1, p)
        tab = np.zeros((K, 2 * p + 1))
        for n in range(K):
            for t in range(2 * p + 1):
                m = order == t
                den = np.abs(R[n][m]).max()
                tab[n, t] = np.abs(T[q, n][m] - R[n][m]).max() / den if den > 0 else 0
        print(f"p={p} K={K} geo={geo[q]} max over modes per order:", tab.max(0))
