"""Pins for the oracle's special functions (oracle/specfun.c) against things other than itself:
closed forms, the Legendre relation, mpmath's independent implementations of K, E and Q_nu,
numerical quadrature of the defining integral, harmonicity and the
symmetry / scaling identities."""
import math

import mpmath as mp
import numpy as np
import pytest

pytestmark = pytest.mark.filterwarnings("ignore")


def test_carlson_closed_forms(orc):
    # R_F(x,x,x) = x^-1/2, R_D(x,x,x) = x^-3/2, R_F(0,1,1) = pi/2 (textbook special cases)
    for x in [0.3, 1.0, 7.5]:
        assert orc.carlson_rf(x, x, x) == pytest.approx(x ** -0.5, rel=2e-16 * 8)
        assert orc.carlson_rd(x, x, x) == pytest.approx(x ** -1.5, rel=2e-16 * 8)
    assert orc.carlson_rf(0.0, 1.0, 1.0) == pytest.approx(math.pi / 2, rel=1e-15)
    # against mpmath's own Carlson implementation
    mp.mp.dps = 30
    for (x, y, z) in [(0.0, 0.2, 1.0), (0.5, 2.0, 3.0), (1e-9, 1.0, 1.0)]:
        assert orc.carlson_rf(x, y, z) == pytest.approx(float(mp.elliprf(x, y, z)), rel=1e-15)
        assert orc.carlson_rd(x, y, z) == pytest.approx(float(mp.elliprd(x, y, z)), rel=1e-15)


def test_ke_special_values_and_legendre_relation(orc):
    K, E = orc.ellip_ke(1.0)  # k = 0
    assert K == pytest.approx(math.pi / 2, rel=1e-16 * 4)
    assert E == pytest.approx(math.pi / 2, rel=1e-16 * 4)
    # Legendre relation E K' + E' K - K K' = pi/2, with K' = K(k'), i.e. complementary parameter k^2
    for m in [1e-8, 0.01, 0.3, 0.5, 0.77, 0.999]:
        K, E = orc.ellip_ke(1.0 - m)
        Kp, Ep = orc.ellip_ke(m)
        assert E * Kp + Ep * K - K * Kp == pytest.approx(math.pi / 2, rel=1e-14)


def test_ke_vs_mpmath_near_singular(orc):
    mp.mp.dps = 40
    # K, E of parameter m = 1 - kp2, fed the complementary parameter directly (R#2)
    for kp2 in [1e-14, 1e-10, 1e-6, 1e-3, 0.1, 0.9]:
        K, E = orc.ellip_ke(kp2)
        m = 1 - mp.mpf(kp2)
        assert K == pytest.approx(float(mp.ellipk(m)), rel=1e-15)
        assert E == pytest.approx(float(mp.ellipe(m)), rel=1e-15)


def _q_ref(chi, nmax):
    mp.mp.dps = 40
    return [mp.re(mp.legenq(n - mp.mpf(1) / 2, 0, mp.mpf(chi), type=3)) for n in range(nmax + 1)]


def _geom_for_chi(chi):
    """(r, r1, x) with r = r1 = 1 exactly and the resulting chi reproduced exactly enough."""
    x = math.sqrt(2 * chi - 2)
    return 1.0, 1.0, x, (2.0 + x * x) / 2.0


@pytest.mark.parametrize("chi,tol", [
    (1.0005, 5e-13), (1.004, 5e-12),            # forward branch (chi < 1.008): loses lambda^2n
    (1.0081, 1e-14), (1.02, 1e-14), (1.3, 1e-14), (3.0, 1e-14), (47.0, 1e-14),
    (1e3, 1e-14), (1e6, 1e-14), (3e7, 1e-14),  # Miller branch, accurate start, rescaled
])
def test_q_sequence_vs_mpmath(orc, chi, tol):
    r, r1, x, chi = _geom_for_chi(chi)
    nmax = 32
    G = orc.greens(r, r1, x, nmax)
    Q = G * (2 * math.pi * math.sqrt(r * r1))
    ref = _q_ref(chi, nmax)
    for n in range(nmax + 1):
        if abs(ref[n]) < 1e-300:
            continue
        assert abs(Q[n] - float(ref[n])) <= tol * abs(float(ref[n])) * (1 + n / 8), (n, Q[n], ref[n])


def test_q_forward_branch_amplification_at_switch(orc):
    # Finding 6: the paper's forward recursion just below chi = 1.008 loses ~lambda^(2n) ~ 1e8 at
    # n = 64 (paper mode pins that the literal rule is kept there); the accurate mode narrows the
    # forward branch for large N (R#3) and is accurate at the same point.
    r, r1, x, chi = _geom_for_chi(1.0079999)
    ref = _q_ref(chi, 64)
    for miller, lo, hi in [(orc.MILLER_PAPER, 1e-11, 1e-7), (orc.MILLER_ACCURATE, 0.0, 1e-13)]:
        Q = orc.greens(r, r1, x, 64, miller=miller) * 2 * math.pi
        rel = max(abs(Q[n] - float(ref[n])) / float(ref[n]) for n in range(65))
        assert lo <= rel < hi, (miller, rel)


@pytest.mark.parametrize("geom", [
    (0.2548828125, 0.2549105212934298, 1.8260273504377977e-06),   # C5, chi - 1 = 5.9e-9
    (1.0, 1.0, 2e-5), (1.0, 1.0, 1.4e-3), (0.7, 0.7000003, 1e-7),
])
def test_q_forward_near_coincident_high_modes(orc, geom):
    # R#24: the forward recursion evaluated with chi = 1 + delta, delta from k'^2,
    # keeps near-coincident rings (chi - 1 down to 1e-10) accurate to ~1e-14 up to n = 64; with a
    # rounded chi it lost 4e-13 at n = 64 for the C5 pair.  Reference: mpmath legenq, 40 digits.
    r, r1, x = geom
    mp.mp.dps = 40
    chi = (mp.mpf(r) ** 2 + mp.mpf(r1) ** 2 + mp.mpf(x) ** 2) / (2 * mp.mpf(r) * mp.mpf(r1))
    assert chi - 1 < 1.2e-4                                         # forward branch at N = 64
    G = orc.greens(r, r1, x, 64)
    c = 2 * mp.pi * mp.sqrt(mp.mpf(r) * mp.mpf(r1))
    for n in range(65):
        ref = mp.re(mp.legenq(n - mp.mpf(1) / 2, 0, chi, type=3)) / c
        assert abs(G[n] - float(ref)) <= 6e-14 * abs(float(ref)), (n, G[n], ref)


def test_forward_switch_rule(orc):
    # R#3: the paper's chi < 1.008 in the paper mode and for N <= 16; beyond, in the
    # accurate mode, the switch t_N satisfies lambda(1 + t_N)^(2N) = 64 exactly (closed form).
    for n in (0, 1, 5, 16):
        assert orc.forward_coef(n, orc.MILLER_ACCURATE) == 0.016
    for n in (17, 32, 64, 100, 255):
        assert orc.forward_coef(n, orc.MILLER_PAPER) == 0.016
        t = orc.forward_coef(n, orc.MILLER_ACCURATE) / 2
        assert t < 0.008
        chi = mp.mpf(1) + t
        lam = chi + mp.sqrt(chi * chi - 1)
        assert float(lam ** (2 * n)) == pytest.approx(64.0, rel=1e-9)


def test_miller_paper_mode_contamination(orc):
    # P:868-874 start at N+80: contamination lambda^-160 ~ 1.6e-9 near chi = 1.008+ (finding 3);
    # the accurate mode (R#4) removes it.  Pins that the paper mode really starts at N+80.
    r, r1, x, chi = _geom_for_chi(1.0082)
    nmax = 16
    ref = np.array([float(v) for v in _q_ref(chi, nmax)])
    Qp = orc.greens(r, r1, x, nmax, miller=orc.MILLER_PAPER) * 2 * math.pi
    Qa = orc.greens(r, r1, x, nmax, miller=orc.MILLER_ACCURATE) * 2 * math.pi
    lam = chi + math.sqrt(chi * chi - 1)
    ep = np.max(np.abs(Qp - ref) / ref)
    ea = np.max(np.abs(Qa - ref) / ref)
    assert 0.05 * lam ** -160 < ep < 20 * lam ** -160
    assert ea < 1e-14


def test_greens_vs_definition_quadrature(orc):
    # G^(n)(r, r1, x) = int_0^2pi cos(n t) / (4 pi R) dt, adaptive quadrature
    for (r, r1, x) in [(0.7, 0.4, 0.3), (1.2, 0.8, 0.5), (0.3, 0.31, 0.02), (0.05, 0.9, 0.0),
                       (1.0, 1.0, 3.0)]:
        G = orc.greens(r, r1, x, 12)
        mp.mp.dps = 25
        for n in range(13):
            f = lambda t: mp.cos(n * t) / (4 * mp.pi * mp.sqrt(r * r + r1 * r1 - 2 * r * r1 * mp.cos(t) + x * x))
            val = float(2 * mp.quad(f, [0, 0.01, 0.1, 0.5, mp.pi]))
            assert abs(G[n] - val) <= 1e-12 * abs(G[0]), (r, r1, x, n, G[n], val)


def test_greens_axisymmetric_closed_form(orc):
    # G^(0) = K(k) / (pi rho_+), k^2 = 4 r r1 / rho_+^2 (textbook ring potential)
    mp.mp.dps = 30
    for (r, r1, x) in [(0.7, 0.4, 0.3), (0.5, 0.5, 1e-3), (2.0, 0.01, 0.7)]:
        rp2 = (mp.mpf(r) + r1) ** 2 + mp.mpf(x) ** 2
        ref = mp.ellipk(4 * mp.mpf(r) * r1 / rp2) / (mp.pi * mp.sqrt(rp2))
        assert orc.greens(r, r1, x, 0)[0] == pytest.approx(float(ref), rel=2e-15)
    # far field: G^(0) -> 1/(2|x|)
    assert orc.greens(0.5, 0.4, 1e4, 0)[0] == pytest.approx(1 / (2e4), rel=1e-8)


def test_greens_recursion_symmetry_scaling(orc):
    r, r1, x = 0.83, 0.37, 0.21
    N = 24
    G = orc.greens(r, r1, x, N)
    chi = (r * r + r1 * r1 + x * x) / (2 * r * r1)
    for n in range(2, N + 1):  # (2n-3) G^(n-2) = 4(n-1) chi G^(n-1) - (2n-1) G^(n)
        lhs = (2 * n - 3) * G[n - 2]
        rhs = 4 * (n - 1) * chi * G[n - 1] - (2 * n - 1) * G[n]
        assert abs(lhs - rhs) <= 1e-13 * abs(lhs)
    assert np.all(G > 0) and np.all(np.diff(G) < 0)
    np.testing.assert_allclose(orc.greens(r1, r, x, N), G, rtol=1e-15)
    np.testing.assert_allclose(orc.greens(r, r1, -x, N), G, rtol=0)
    np.testing.assert_allclose(orc.greens(2 * r, 2 * r1, 2 * x, N), G / 2, rtol=1e-14)


def test_greens_harmonic(orc):
    # Each mode satisfies G_rr + G_r / r - n^2 G / r^2 + G_xx = 0; 4th-order FD
    r, r1, x = 0.9, 0.5, 0.35
    h = 1e-3
    for n in [0, 1, 3, 8]:
        g = lambda rr, xx: orc.greens(rr, r1, xx, n)[n]
        c = [-1 / 12, 4 / 3, -5 / 2, 4 / 3, -1 / 12]
        d1 = [1 / 12, -2 / 3, 0, 2 / 3, -1 / 12]
        off = [-2, -1, 0, 1, 2]
        grr = sum(ci * g(r + o * h, x) for ci, o in zip(c, off)) / h ** 2
        gr = sum(ci * g(r + o * h, x) for ci, o in zip(d1, off)) / h
        gxx = sum(ci * g(r, x + o * h) for ci, o in zip(c, off)) / h ** 2
        g0 = g(r, x)
        res = grr + gr / r - n * n * g0 / (r * r) + gxx
        scale = abs(grr) + abs(gr / r) + abs(n * n * g0 / r / r) + abs(gxx)
        assert abs(res) <= 1e-6 * scale
