"""Pins for the oracle's derivative tensor (oracle/tensor.c, P:876-1065 with reading R#6/R#7)
against mpmath's numerical differentiation of Q_{n-1/2} (independent code), the exchange,
parity and scaling symmetries of G, and Taylor reconstruction of G at a
displaced geometry."""
import math

import mpmath as mp
import numpy as np
import pytest


def _G_mp(n):
    def f(r, r1, x):
        chi = (r * r + r1 * r1 + x * x) / (2 * r * r1)
        return mp.re(mp.legenq(n - mp.mpf(1) / 2, 0, chi, type=3)) / (2 * mp.pi * mp.sqrt(r * r1))
    return f


@pytest.mark.parametrize("geom", [(1.3, 0.7, 0.9), (0.8, 0.8, 0.5), (2.5, 0.5, 0.0)])
def test_tensor_vs_mpmath_derivatives(orc, geom):
    mp.mp.dps = 40
    r, r1, x = geom
    p = 3
    T = orc.tensor(r, r1, x, 5, p)
    for n in [0, 1, 2, 5]:
        f = _G_mp(n)
        for a in range(p + 1):
            for b in range(p + 1):
                for c in range(0, 2 * p + 1 - a - b):
                    if a + b + c > 4:
                        continue
                    ref = mp.diff(f, (mp.mpf(r), mp.mpf(r1), mp.mpf(x)), (a, b, c)) / (
                        mp.factorial(a) * mp.factorial(b) * mp.factorial(c))
                    scale = max(abs(float(ref)), abs(T[n, 0, 0, 0]) * 1e-3)
                    assert abs(T[n, a, b, c] - float(ref)) <= 1e-13 * scale, (n, a, b, c)


def test_tensor_high_order_entries_vs_mpmath(orc):
    # spot-check entries reached only through both Laplace passes (a >= 2 and b >= 2, c > 0)
    mp.mp.dps = 40
    r, r1, x = 1.9, 1.1, 0.6
    T = orc.tensor(r, r1, x, 3, 4)
    for (n, a, b, c) in [(0, 2, 2, 1), (3, 3, 2, 0), (1, 2, 3, 1), (2, 4, 2, 0)]:
        ref = mp.diff(_G_mp(n), (mp.mpf(r), mp.mpf(r1), mp.mpf(x)), (a, b, c)) / (
            mp.factorial(a) * mp.factorial(b) * mp.factorial(c))
        assert T[n, a, b, c] == pytest.approx(float(ref), rel=1e-12)


def _order_max(T, p):
    """max |entry| per total order a+b+c, per mode."""
    K = T.shape[0]
    out = np.zeros((K, 2 * p + 1))
    for a in range(p + 1):
        for b in range(p + 1):
            for c in range(2 * p + 1 - a - b):
                out[:, a + b + c] = np.maximum(out[:, a + b + c], np.abs(T[:, a, b, c]))
    return out


def test_tensor_swap_parity_scaling(orc):
    p, N = 8, 6
    r, r1, x = 1.75, 1.25, 0.5  # a well-separated box-centre geometry in units of h
    T = orc.tensor(r, r1, x, N, p)
    Ts = orc.tensor(r1, r, x, N, p)
    Tn = orc.tensor(r, r1, -x, N, p)
    T2 = orc.tensor(2 * r, 2 * r1, 2 * x, N, p)
    om = _order_max(T, p)
    for a in range(p + 1):
        for b in range(p + 1):
            for c in range(2 * p + 1 - a - b):
                tol = 1e-12 * om[:, a + b + c]
                # exchange r <-> r1 swaps a <-> b (G symmetric in r, r1); this compares the
                # r-Laplace path with the r1-Laplace path, which are different computations
                assert np.all(np.abs(Ts[:, b, a, c] - T[:, a, b, c]) <= tol)
                assert np.all(np.abs(Tn[:, a, b, c] - (-1) ** c * T[:, a, b, c]) <= tol)
                s = 2.0 ** -(1 + a + b + c)  # G(s r, s r1, s x) = G / s
                assert np.all(np.abs(T2[:, a, b, c] - s * T[:, a, b, c]) <= s * tol)


def test_tensor_taylor_reconstruction(orc):
    # G(r+dr, r1+dr1, x+dx) = sum Gbar_abc dr^a dr1^b dx^c, geometric convergence
    r, r1, x = 2.5, 0.5, 1.0
    dr, dr1, dx = 0.11, -0.09, 0.07
    N = 4
    exact = orc.greens(r + dr, r1 + dr1, x + dx, N)
    errs = []
    for p in [4, 8, 12, 16]:
        T = orc.tensor(r, r1, x, N, p)
        approx = np.zeros(N + 1)
        for a in range(p + 1):
            for b in range(p + 1):
                for c in range(2 * p + 1 - a - b):
                    approx += T[:, a, b, c] * dr ** a * dr1 ** b * dx ** c
        errs.append(np.max(np.abs(approx - exact) / exact))
    assert errs[-1] < 1e-13
    assert errs[0] > errs[1] > errs[2]


def test_rational_tables_vs_mpmath_taylor(orc):
    mp.mp.dps = 30
    r, r1, x = 1.0, 1.0, 1.0
    tab = orc.rational_tables(r, r1, x, 6)
    assert tab[0, 0] == pytest.approx(0.2, rel=1e-15)  # x / rho_+^2 at (1,1,1) = 1/5
    for (r, r1, x) in [(1.3, 0.7, 0.9), (0.8, 0.8, 0.5)]:
        tab = orc.rational_tables(r, r1, x, 8)
        R, R1 = mp.mpf(r), mp.mpf(r1)
        fns = []
        for s in (+1, -1):
            fns.append(lambda xx, s=s: xx / ((R + s * R1) ** 2 + xx ** 2))
        for s in (+1, -1):
            fns.append(lambda xx, s=s: (R ** 2 - R1 ** 2 - xx ** 2) / ((R + s * R1) ** 2 + xx ** 2))
        for s in (+1, -1):  # d/dr1 of the previous pair
            fns.append(lambda xx, s=s: mp.diff(lambda q: (R ** 2 - q ** 2 - xx ** 2) / ((R + s * q) ** 2 + xx ** 2), R1))
        for s in (+1, -1):  # exchanged r <-> r1
            fns.append(lambda xx, s=s: (R1 ** 2 - R ** 2 - xx ** 2) / ((R1 + s * R) ** 2 + xx ** 2))
        for t, f in enumerate(fns):
            ref = mp.taylor(f, mp.mpf(x), 8)
            for q in range(9):
                assert tab[t, q] == pytest.approx(float(ref[q]), rel=1e-12, abs=1e-14), (t, q)


def test_tensor_laplace_residual(orc):
    # every stored Gbar satisfies the Laplace equation in (r, x) and in (r1, x)
    p, N = 6, 4
    r, r1, x = 1.5, 0.5, 2.0
    T = orc.tensor(r, r1, x, N, p)
    om = _order_max(T, p)
    for n in range(N + 1):
        for a in range(p - 1):
            for b in range(p + 1):
                for c in range(2 * p - 1 - a - b):
                    def g(i, cc):
                        return T[n, i, b, cc] if i >= 0 else 0.0
                    res = (r * r * (a + 1) * (a + 2) * g(a + 2, c) + r * (a + 1) * (2 * a + 1) * g(a + 1, c)
                           + (a * a - n * n) * g(a, c)
                           + (c + 1) * (c + 2) * (r * r * g(a, c + 2) + 2 * r * g(a - 1, c + 2) + g(a - 2, c + 2)))
                    assert abs(res) <= 1e-11 * om[n, a + b + c] * (1 + a + c) ** 2 * r * r


@pytest.mark.parametrize("geom", [(6.5, 3.5, 3.0), (2.5, 0.5, 1.0)])
def test_tensor_high_mode_x_derivatives_vs_mpmath(orc, geom):
    """Step 2b (reading R#22): Gbar^n_{00c} for modes far above the derivative order, against
    mpmath's differentiation of Q_{n-1/2}(chi(x)) in x (the definition).  The
    paper's cross-mode x-recursion alone fails this by many orders of magnitude at n = 40."""
    mp.mp.dps = 60
    r, r1, x = geom
    p = 6
    T = orc.tensor(r, r1, x, 40, p)
    for n in (2, 17, 40):
        f = _G_mp(n)
        cs = list(range(0, 2 * p + 1, 3))
        refs = [float(mp.diff(lambda t: f(mp.mpf(r), mp.mpf(r1), t), mp.mpf(x), c) / mp.factorial(c))
                for c in cs]
        # per-mode scale: the largest coefficient checked (isolated entries can vanish by
        # symmetry, e.g. Re (x + i a)^-6 = 0 at x = a, so entry-wise relative error is no measure)
        scale = max(abs(v) for v in refs)
        for c, ref in zip(cs, refs):
            assert abs(T[n, 0, 0, c] - ref) <= 1e-12 * scale, (n, c, T[n, 0, 0, c], ref)


@pytest.mark.parametrize("geom", [(130.5, 128.5, 2.0), (20.5, 17.5, 3.0), (3.5, 1.5, 2.0),
                                  (10.5, 10.5, 2.0), (11.5, 10.5, 2.0)])
def test_tensor_all_modes_vs_exact_recursion(orc, geom):
    """The whole tensor for K = 49 modes at p = 12 against the same recursions evaluated with
    100 significant digits (tests/hp_tensor.py), where their rounding amplification (up to
    ~1e22 at high modes) is harmless: the 100-digit values are the exact Taylor coefficients to
    far below FP64 rounding.  Per mode, in the S2L weighting (entry (a, b, c) scaled by 2^-(a+b))."""
    from tests.hp_tensor import hp_tensor
    r, r1, x = geom
    p, nmax = 12, 48
    E = hp_tensor(r, r1, x, nmax, p, dps=100)
    O = orc.tensor(r, r1, x, nmax, p)
    a = np.arange(p + 1)[:, None, None]
    b = np.arange(p + 1)[None, :, None]
    c = np.arange(2 * p + 1)[None, None, :]
    w = 2.0 ** -(a + b) * ((a + b + c) <= 2 * p)
    for n in range(nmax + 1):
        err = np.abs((O[n] - E[n]) * w).max() / np.abs(E[n] * w).max()
        assert err <= 2e-12, (n, err)


def _x_taylor_by_quadrature(r, r1, x, n, cmax, npts=None, dps=30):
    """Gbar^n_{00c} = (1/c!) d^c G^(n)/dx^c for c = 0..cmax from the DEFINITION
    G^(n) = int_0^2pi cos(n t) / (4 pi R) dt, R^2 = s^2 + ..., by the Legendre
    generating function: 1 / sqrt(s^2 + 2 x h + h^2) = sum_c P_c(-x / s) h^c / s^(c+1) with
    s^2 = r^2 + r1^2 - 2 r r1 cos t + x^2.  Trapezoid rule over t (spectrally accurate for
    separated rings), mpmath at `dps` digits.  Independent of the tensor recursions."""
    if npts is None:   # trapezoid error ~ exp(-alpha N), alpha ~ (closest distance) / sqrt(r r1)
        alpha = math.hypot(r - r1, x) / math.sqrt(r * r1)
        npts = max(512, 256 * math.ceil(44.0 / alpha / 256))
    mp.mp.dps = dps
    r, r1, x = mp.mpf(r), mp.mpf(r1), mp.mpf(x)
    acc = [mp.mpf(0)] * (cmax + 1)
    for k in range(npts):
        t = 2 * mp.pi * k / npts
        s = mp.sqrt(r * r + r1 * r1 - 2 * r * r1 * mp.cos(t) + x * x)
        u = -x / s
        w = mp.cos(n * t) / (4 * mp.pi * s)
        p0, p1 = mp.mpf(1), u            # Legendre P_c(u) by the three-term recursion
        for c in range(cmax + 1):
            pc = p0 if c == 0 else p1
            acc[c] += w * pc
            w /= s
            if c >= 1:
                p0, p1 = p1, ((2 * c + 1) * u * p1 - c * p0) / (c + 1)
    return [float(a * 2 * mp.pi / npts) for a in acc]


@pytest.mark.parametrize("geom", [(300.5, 298.5, 2.0), (50.5, 47.5, 3.0), (10.5, 10.5, 2.0)])
def test_tensor_x_derivatives_c5_regime_vs_definition(orc, geom):
    """Step 2b (reading R#22) in the C5 regime -- K = 65 modes, p = 16 (x-derivatives to order
    2p = 32) at normalised stations of the C5 tree (far from the axis, mid, and same-column) --
    against the definition of G^(n) as an angular integral of the 3-D kernel, whose
    x-Taylor coefficients follow from the Legendre generating function
    (_x_taylor_by_quadrature): an independent method, not the paper's recursions.  Per mode,
    relative to the largest coefficient of that mode."""
    r, r1, x = geom
    p, nmax = 16, 64
    T = orc.tensor(r, r1, x, nmax, p)
    for n in (2, 17, 33, 48, 64):
        ref = _x_taylor_by_quadrature(r, r1, x, n, 2 * p)
        scale = max(abs(v) for v in ref)
        err = max(abs(T[n, 0, 0, c] - ref[c]) for c in range(2 * p + 1)) / scale
        assert err <= 1e-12, (geom, n, err)
