#!/usr/bin/env python
"""GPU tensor (cylfmm_tensor_batch) vs oracle tensor at normalised FMM station geometries
(i_in + dI + 1/2, i_in + 1/2, dJ): worst weighted error per station.  Diagnostic (GPU box)."""
import sys, os, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle
import paper_2301_01179_b200 as g

p, K = int(sys.argv[1]) if len(sys.argv) > 1 else 16, int(sys.argv[2]) if len(sys.argv) > 2 else 65
cls = [(0, 2), (0, 3), (1, 2), (1, 3), (2, 0), (2, 1), (2, 2), (2, 3), (3, 0), (3, 1), (3, 2), (3, 3)]
ii = list(range(0, 48)) + [63, 100, 127, 255, 300, 511, 700, 1023]
geo = [(i + dI + 0.5, i + 0.5, float(dJ)) for i in ii for (dI, dJ) in cls]
r, r1, x = (np.array(v) for v in zip(*geo))
oracle.build()
T = g.tensor_batch(r, r1, x, K, p).cpu().numpy()
a = np.arange(p + 1)[:, None, None]; b = np.arange(p + 1)[None, :, None]; c = np.arange(2 * p + 1)[None, None, :]
w = 2.0 ** -(a + b) * ((a + b + c) <= 2 * p)
worst = []
for q in range(len(geo)):
    ref = oracle.tensor(r[q], r1[q], x[q], K - 1, p)
    e = [float(np.abs((T[q, n] - ref[n]) * w).max() / np.abs(ref[n] * w).max()) for n in range(K)]
    worst.append((max(e), geo[q], int(np.argmax(e))))
worst.sort(reverse=True)
print(json.dumps({"p": p, "K": K, "worst": worst[:15], "n_bad_1e12": sum(1 for w_ in worst if w_[0] > 1e-12)}))
