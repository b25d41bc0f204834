"""Pins for the potential gradients of the oracle (P:36-40, 83-86 motivate
them): the first-order derivative relations of G^(n) (P:917-923 in x, P:958-966 in r) against
mpmath's differentiation of Q_{n-1/2} (the definition), the direct-sum gradients against central
finite differences of the direct sum, and FMM gradients converging to the direct ones in p."""
import mpmath as mp
import numpy as np
import pytest

from tests.inputs import uniform_rings


def _G_mp(n):
    def f(r, r1, x):
        chi = (r * r + r1 * r1 + x * x) / (2 * r * r1)
        return mp.re(mp.legenq(n - mp.mpf(1) / 2, 0, chi, type=3)) / (2 * mp.pi * mp.sqrt(r * r1))
    return f


@pytest.mark.parametrize("geom", [(0.7, 0.6, 0.05), (1.3, 0.4, 0.9), (0.2, 0.9, -0.3), (2.0, 1.9, 0.0)])
def test_greens_gradient_vs_mpmath(orc, geom):
    mp.mp.dps = 30
    r, r1, x = geom
    nmax = 12
    G, Gr, Gx = orc.greens_grad(r, r1, x, nmax)
    for n in (0, 1, 2, 7, 12):
        f = _G_mp(n)
        pt = (mp.mpf(r), mp.mpf(r1), mp.mpf(x))
        dr = float(mp.diff(f, pt, (1, 0, 0)))
        dx = float(mp.diff(f, pt, (0, 0, 1)))
        scale = max(abs(dr), abs(dx), abs(G[n]) / abs(r - r1 + 1e-300))
        assert abs(Gr[n] - dr) <= 1e-12 * scale, (n, Gr[n], dr)
        assert abs(Gx[n] - dx) <= 1e-12 * scale + 1e-300, (n, Gx[n], dx)


def test_direct_gradient_vs_finite_differences(orc):
    rng = np.random.default_rng(3)
    sr, sz, S = uniform_rings(rng, 60, 6)
    fr, fz, _ = uniform_rings(rng, 7, 1)
    fr = 0.1 + 0.8 * fr
    fz = 0.1 + 0.8 * fz
    P, Gr, Gz, _ = orc.direct_grad(sr, sz, S, fr, fz)
    P0, _ = orc.direct(sr, sz, S, fr, fz)
    assert np.array_equal(P, P0)
    h = 1e-6   # central differences: truncation ~1e-8 here (error scales as h^2: 5e-7 at 1e-5)
    Pp, _ = orc.direct(sr, sz, S, fr + h, fz)
    Pm, _ = orc.direct(sr, sz, S, fr - h, fz)
    Qp, _ = orc.direct(sr, sz, S, fr, fz + h)
    Qm, _ = orc.direct(sr, sz, S, fr, fz - h)
    fd_r = (Pp - Pm) / (2 * h)
    fd_z = (Qp - Qm) / (2 * h)
    assert np.max(np.abs(fd_r - Gr)) <= 1e-7 * np.max(np.abs(Gr))
    assert np.max(np.abs(fd_z - Gz)) <= 1e-7 * np.max(np.abs(Gz))


def test_fmm_gradient_converges_to_direct(orc):
    rng = np.random.default_rng(5)
    sr, sz, S = uniform_rings(rng, 1200, 3)
    fr, fz, _ = uniform_rings(rng, 150, 1)
    _, Dr, Dz, _ = orc.direct_grad(sr, sz, S, fr, fz)
    err = {}
    for p in (4, 8, 12):
        F, Fr, Fz, _ = orc.fmm(sr, sz, S, fr, fz, p, 4, 1.0, grad=True)
        err[p] = max(orc.eps_per_mode(Fr, Dr).max(), orc.eps_per_mode(Fz, Dz).max())
    assert err[4] > err[8] > err[12], err
    assert err[12] < 1e-5, err
