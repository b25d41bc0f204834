"""High-precision (mpmath, 50 digits) evaluation of the paper's derivative-tensor recursions
(P:904-1065 with R#6/R#7), used only to measure the ROUNDING error of the two FP64 codes (oracle
and GPU) where the recursion is ill-conditioned (high modes, SURVEY APP-E).  It is a test-side
accuracy yardstick, not a pin of the oracle (the oracle's pins are mpmath derivatives of
Q_{n-1/2} in tests/test_oracle_tensor.py)."""
import mpmath as mp
import numpy as np


def hp_tensor(r, r1, x, nmax, p, dps=50):
    mp.mp.dps = dps
    r, r1, x = mp.mpf(r), mp.mpf(r1), mp.mpf(x)
    Ni = max(nmax, 1)
    C = 2 * p
    half = mp.mpf(1) / 2
    chi = (r * r + r1 * r1 + x * x) / (2 * r * r1)
    G = [mp.re(mp.legenq(n - half, 0, chi, type=3)) / (2 * mp.pi * mp.sqrt(r * r1))
         for n in range(Ni + 1)]
    t, u, v, us = {}, {}, {}, {}
    for s, (a, b) in enumerate([(r + r1, r1 + r), (r - r1, r1 - r)]):
        z, zs = 1 / mp.mpc(x, -a), 1 / mp.mpc(x, -b)
        w, ws = z, zs
        for q in range(C + 2):
            t[s, q] = mp.re(w)
            u[s, q] = (-1 if q == 0 else 0) + 2 * r * mp.im(w)
            v[s, q] = (1 if s == 0 else -1) * 2 * r * (q + 1) * mp.re(w * z)
            us[s, q] = (-1 if q == 0 else 0) + 2 * r1 * mp.im(ws)
            w, ws = -w * z, -ws * zs
    Z = mp.mpf(0)
    g00 = [[Z] * (C + 1) for _ in range(Ni + 1)]
    g10 = [[Z] * (C + 1) for _ in range(Ni + 1)]
    g01 = [[Z] * (C + 1) for _ in range(Ni + 1)]
    g11 = [[Z] * (C + 1) for _ in range(Ni + 1)]
    mm = lambda n: 1 if n == 0 else n - 1  # noqa: E731  (G^(-1) == G^(1))
    for n in range(Ni + 1):
        g00[n][0] = G[n]
    for k in range(C):
        for n in range(Ni + 1):
            m = mm(n)
            s = sum((g00[n][k - q] + g00[m][k - q]) * t[0, q] + (g00[n][k - q] - g00[m][k - q]) * t[1, q]
                    for q in range(k + 1))
            g00[n][k + 1] = (n - half) * s / (k + 1)
    for n in range(Ni + 1):
        m = mm(n)
        for k in range(C):
            gp = [g00[n][k - q] + g00[m][k - q] for q in range(k + 1)]
            gd = [g00[n][k - q] - g00[m][k - q] for q in range(k + 1)]
            s1 = sum(gp[q] * u[0, q] + gd[q] * u[1, q] for q in range(k + 1))
            s2 = sum(gp[q] * us[0, q] + gd[q] * us[1, q] for q in range(k + 1))
            g10[n][k] = (-g00[n][k] + (n - half) * s1) / (2 * r)
            g01[n][k] = (-g00[n][k] + (n - half) * s2) / (2 * r1)
    for n in range(Ni + 1):
        m = mm(n)
        for k in range(C - 1):
            s = sum((g00[n][k - q] + g00[m][k - q]) * v[0, q] + (g01[n][k - q] + g01[m][k - q]) * u[0, q]
                    + (g00[n][k - q] - g00[m][k - q]) * v[1, q] + (g01[n][k - q] - g01[m][k - q]) * u[1, q]
                    for q in range(k + 1))
            g11[n][k] = (-g01[n][k] + (n - half) * s) / (2 * r)
    out = np.zeros((nmax + 1, p + 1, p + 1, C + 1))
    for n in range(nmax + 1):
        T = {}
        for c in range(C + 1):
            T[0, 0, c] = g00[n][c]
        for c in range(C):
            T[1, 0, c], T[0, 1, c] = g10[n][c], g01[n][c]
        for c in range(C - 1):
            T[1, 1, c] = g11[n][c]
        get = lambda a, b, c: T.get((a, b, c), Z)  # noqa: E731
        for b in range(2):
            for a in range(p - 1):
                for c in range(C + 1 - a - 2 - b):
                    lap = r * r * get(a, b, c + 2) + 2 * r * get(a - 1, b, c + 2) + get(a - 2, b, c + 2)
                    num = r * (a + 1) * (2 * a + 1) * get(a + 1, b, c) + (a * a - n * n) * get(a, b, c) \
                        + (c + 1) * (c + 2) * lap
                    T[a + 2, b, c] = -num / (r * r * (a + 1) * (a + 2))
        for b in range(p - 1):
            for a in range(p + 1):
                for c in range(C + 1 - a - b - 2):
                    lap = r1 * r1 * get(a, b, c + 2) + 2 * r1 * get(a, b - 1, c + 2) + get(a, b - 2, c + 2)
                    num = r1 * (b + 1) * (2 * b + 1) * get(a, b + 1, c) + (b * b - n * n) * get(a, b, c) \
                        + (c + 1) * (c + 2) * lap
                    T[a, b + 2, c] = -num / (r1 * r1 * (b + 1) * (b + 2))
        for (a, b, c), val in T.items():
            if a >= 0 and b >= 0 and a <= p and b <= p and a + b + c <= C:
                out[n, a, b, c] = float(val)
    return out
