"""Pins for the oracle direct sum (oracle/direct.c) and reference FMM (oracle/fmm.c):
brute-force 3-D quadrature of 1/(4 pi |x - x'|) over discretised rings, linearity,
self-exclusion, binomial exactness of P2M/M2M/L2L/L2P,
S2L reductions and convergence, tree box assignment by brute force
(R#11), and FMM-vs-direct convergence ~0.4 decade per order
plus agreement with an independently-assembled "direct-expansion" form (R#21)."""
import math

import numpy as np
import pytest

from tests.inputs import uniform_rings


def _brute_3d(sr, sz, S, fr, fz, M=1024):
    """Rings discretised into M points carrying s(t) = sum_{n>=0} S^(n) e^{i n t}; field rings
    sampled at M angles; potential by plain 3-D summation of 1/(4 pi R) (2 pi / M), then the
    modal amplitudes by FFT over the field angle.  Spectrally accurate for separated rings."""
    K = S.shape[1]
    th = 2 * np.pi * np.arange(M) / M
    out = np.zeros((len(fr), K), dtype=np.complex128)
    for j in range(len(fr)):
        fx, fy = fr[j] * np.cos(th), fr[j] * np.sin(th)
        phi = np.zeros(M, dtype=np.complex128)
        for i in range(len(sr)):
            s = sum(S[i, n] * np.exp(1j * n * th) for n in range(K))  # density on source ring
            sx, sy = sr[i] * np.cos(th), sr[i] * np.sin(th)
            R = np.sqrt((fx[:, None] - sx[None, :]) ** 2 + (fy[:, None] - sy[None, :]) ** 2
                        + (fz[j] - sz[i]) ** 2)
            phi += (1.0 / (4 * np.pi * R)) @ s * (2 * np.pi / M)
        out[j] = np.fft.fft(phi)[:K] / M  # phi(theta) = sum_n Phi^(n) e^{i n theta}
    return out


def test_direct_vs_3d_quadrature(orc):
    rng = np.random.default_rng(11)
    sr = np.array([0.3, 0.9, 0.55, 1.4])
    sz = np.array([0.1, 0.4, 0.9, 0.0])
    fr = np.array([0.7, 0.2, 1.1])
    fz = np.array([0.6, -0.3, 0.45])
    K = 5
    S = rng.standard_normal((4, K)) + 1j * rng.standard_normal((4, K))
    D, sk = orc.direct(sr, sz, S, fr, fz)
    B = _brute_3d(sr, sz, S, fr, fz)
    assert sk == 0
    assert np.max(np.abs(D - B)) <= 1e-12 * np.max(np.abs(B))


def test_direct_linearity_and_self_exclusion(orc):
    sr, sz, S = uniform_rings(np.random.default_rng(3), 200, 7)
    fr, fz, _ = uniform_rings(np.random.default_rng(4), 50, 1)
    D1, _ = orc.direct(sr[:120], sz[:120], S[:120], fr, fz)
    D2, _ = orc.direct(sr[120:], sz[120:], S[120:], fr, fz)
    D, _ = orc.direct(sr, sz, S, fr, fz)
    np.testing.assert_allclose(D, D1 + D2, rtol=0, atol=1e-13 * np.abs(D).max())
    D3, _ = orc.direct(sr, sz, 2.5 * S, fr, fz)
    np.testing.assert_allclose(D3, 2.5 * D, rtol=1e-14)
    # fields = sources: skipping coincident pairs equals dropping the i == j term
    Ds, sk = orc.direct(sr, sz, S, sr, sz)
    assert sk == 200
    j = 17
    mask = np.arange(200) != j
    Dj, _ = orc.direct(sr[mask], sz[mask], S[mask], sr[j:j + 1], sz[j:j + 1])
    np.testing.assert_allclose(Ds[j], Dj[0], rtol=1e-14)
    # mode independence: zeroing mode m zeroes output m only
    S0 = S.copy()
    S0[:, 3] = 0
    Dz, _ = orc.direct(sr, sz, S0, fr, fz)
    assert np.all(Dz[:, 3] == 0)
    np.testing.assert_array_equal(Dz[:, [0, 1, 2, 4, 5, 6]], D[:, [0, 1, 2, 4, 5, 6]])


def test_p2m_m2m_l2l_l2p_exactness(orc):
    rng = np.random.default_rng(5)
    p, K = 7, 3
    r = 0.5 + 0.1 * rng.random(6)
    z = 0.2 + 0.1 * rng.random(6)
    S = rng.standard_normal((6, K)) + 1j * rng.standard_normal((6, K))
    # single source offset (a, b): S_ij = S a^i b^j
    M1 = orc.p2m(r[:1], z[:1], S[:1], p, 0.5, 0.2)
    a, b = r[0] - 0.5, z[0] - 0.2
    for i in range(p + 1):
        for j in range(p + 1 - i):
            np.testing.assert_allclose(M1[:, orc.tri_idx(i, j, p)], S[0] * a ** i * b ** j, rtol=1e-14)
    # M2M: shifted child moments == moments computed directly about the parent centre
    Mc = orc.p2m(r, z, S, p, 0.55, 0.25)
    Mp = orc.m2m(Mc, p, 0.55 - 0.6, 0.25 - 0.3)
    Md = orc.p2m(r, z, S, p, 0.6, 0.3)
    np.testing.assert_allclose(Mp, Md, rtol=1e-12, atol=1e-15)
    # L2L exact for a polynomial field of degree <= p; L2P reproduces it
    Lp = rng.standard_normal((K, orc.tri_size(p))) + 1j * rng.standard_normal((K, orc.tri_size(p)))
    Lc = orc.l2l(Lp, p, 0.03, -0.02)
    for (rr, zz) in [(0.51, 0.19), (0.53, 0.18)]:
        v_parent = orc.l2p(Lp, p, 0.5, 0.2, rr, zz)
        v_child = orc.l2p(Lc, p, 0.53, 0.18, rr, zz)
        np.testing.assert_allclose(v_child, v_parent, rtol=1e-12)
    # P2M conserves S00 through M2M
    np.testing.assert_allclose(Mp[:, 0], S.sum(axis=0), rtol=1e-14)


def test_s2l_point_source_and_convergence(orc):
    rng = np.random.default_rng(7)
    h = 1.0 / 32
    K = 4
    # point source at a box centre: Phi_00 = S G(target centre, source centre)
    for (si, sj, ti, tj) in [(10, 10, 12, 10), (10, 12, 13, 9), (12, 12, 10, 10), (13, 9, 10, 12), (0, 10, 2, 10)]:
        rs, zs = (si + 0.5) * h, (sj + 0.5) * h
        rt, zt = (ti + 0.5) * h, (tj + 0.5) * h
        S = rng.standard_normal(K) + 1j * rng.standard_normal(K)
        M = orc.p2m([rs], [zs], S[None, :], 4, rs, zs)
        L = orc.s2l(M, 4, rs, zs, rt, zt)
        G = orc.greens(rt, rs, zt - zs, K - 1)
        np.testing.assert_allclose(L[:, 0], S * G, rtol=1e-13)
    # random sources in the source box, targets in the target box: S2L+L2P -> direct, geometric in p;
    # all four variants FO, BO, FI, BI
    for (si, sj, ti, tj) in [(10, 10, 12, 10), (10, 12, 12, 10), (12, 9, 10, 12), (12, 12, 10, 10)]:
        rs, zs = (si + 0.5) * h, (sj + 0.5) * h
        rt, zt = (ti + 0.5) * h, (tj + 0.5) * h
        n = 8
        r = rs + (rng.random(n) - 0.5) * h
        z = zs + (rng.random(n) - 0.5) * h
        S = rng.standard_normal((n, K)) + 1j * rng.standard_normal((n, K))
        tr = rt + (rng.random(5) - 0.5) * h
        tz = zt + (rng.random(5) - 0.5) * h
        D, _ = orc.direct(r, z, S, tr, tz)
        errs = []
        for p in [4, 8, 12]:
            M = orc.p2m(r, z, S, p, rs, zs)
            L = orc.s2l(M, p, rs, zs, rt, zt)
            F = np.array([orc.l2p(L, p, rt, zt, tr[k], tz[k]) for k in range(5)])
            errs.append(np.max(np.abs(F - D)) / np.max(np.abs(D)))
        assert errs[2] < 1e-5 and errs[0] > errs[1] > errs[2], errs


def test_tree_keys_bruteforce(orc):
    rng = np.random.default_rng(9)
    n, d, L, z0 = 3000, 5, 2.0, 0.0
    r = L * (1 - rng.random(n))
    z = L * rng.random(n)
    r[:5] = L  # closed last box (R#11)
    z[5:10] = L
    key, perm = orc.tree_keys(r, z, d, L, z0)
    nb = 2 ** d
    ix = np.minimum(np.floor(r * nb / L), nb - 1).astype(np.int64)
    iz = np.minimum(np.floor((z - z0) * nb / L), nb - 1).astype(np.int64)
    ref = np.zeros(n, dtype=np.int64)
    for b in range(d):
        ref |= ((ix >> b) & 1) << (2 * b)
        ref |= ((iz >> b) & 1) << (2 * b + 1)
    np.testing.assert_array_equal(key.astype(np.int64), ref)
    np.testing.assert_array_equal(perm, np.argsort(ref, kind="stable"))


def _interaction_lists(ix, iz, level):
    """brute force, from the definition: children of the parent's neighbours, not neighbours"""
    nb = 2 ** level
    out = []
    for a in range(nb):
        for c in range(nb):
            if max(abs(a // 2 - ix // 2), abs(c // 2 - iz // 2)) <= 1 and max(abs(a - ix), abs(c - iz)) >= 2:
                out.append((a, c))
    return out


def test_interaction_list_partition(orc):
    # every pair of leaves is covered exactly once: neighbours at level d, or an S2L pair of the
    # same-level ancestors at exactly one level 2..d; 27 / 12 classes
    d = 4
    nb = 2 ** d
    classes = set()
    for tx in range(nb):
        for tz in range(nb):
            count = np.zeros((nb, nb), dtype=int)
            for a in range(nb):
                for c in range(nb):
                    if max(abs(a - tx), abs(c - tz)) <= 1:
                        count[a, c] += 1
            for lvl in range(2, d + 1):
                sh = d - lvl
                lst = _interaction_lists(tx >> sh, tz >> sh, lvl)
                assert len(lst) <= 27
                if 2 <= (tx >> sh) < 2 ** lvl - 3 and 2 <= (tz >> sh) < 2 ** lvl - 3:
                    assert len(lst) == 27
                for (a, c) in lst:
                    classes.add((abs(a - (tx >> sh)), abs(c - (tz >> sh))))
                    count[a << sh:(a + 1) << sh, c << sh:(c + 1) << sh] += 1
            assert np.all(count == 1)
    assert len(classes) == 12


def test_fmm_converges_to_direct(orc):
    # geometric convergence ~0.4 decade per order (read as C 10^(-0.4 M), R#17)
    sr, sz, S = uniform_rings(np.random.default_rng(2), 1024, 5)
    D, _ = orc.direct(sr, sz, S, sr, sz)
    eps = {}
    for p in [4, 8, 12, 16]:
        F, sk = orc.fmm(sr, sz, S, sr, sz, p, 3, 1.0)
        assert sk == 1024
        eps[p] = orc.eps_per_mode(F, D)
    slope = np.log10(eps[4][0] / eps[16][0]) / 12
    assert 0.25 < slope < 0.6, slope
    assert np.all(eps[16] < 1e-7) and eps[16][0] < 1e-8
    for p in [4, 8, 12]:
        assert np.all(eps[p] > eps[p + 4])


@pytest.mark.parametrize("p,pl", [(6, 6), (5, 8), (8, 4)])
def test_fmm_equals_direct_expansion_form(orc, p, pl):
    """Algorithm 1 (with M2M and L2L) vs the direct-expansion form assembled here from the same
    single-box operators: moments of each S2L-list box taken directly from its sources, S2L to
    the target's ancestor at each level, evaluated at the target; plus the near field (R#21).
    M2M and L2L are exact re-centrings, so the two agree to rounding."""
    rng = np.random.default_rng(21)
    sr, sz, S = uniform_rings(rng, 400, 3)
    fr, fz, _ = uniform_rings(rng, 12, 1)
    d, L = 3, 1.0
    F, _ = orc.fmm(sr, sz, S, fr, fz, p, d, L, pl=pl)
    nb = 2 ** d
    six = np.minimum(np.floor(sr * nb / L), nb - 1).astype(int)
    siz = np.minimum(np.floor(sz * nb / L), nb - 1).astype(int)
    out = np.zeros_like(F)
    for t in range(len(fr)):
        tx = min(int(math.floor(fr[t] * nb / L)), nb - 1)
        tz = min(int(math.floor(fz[t] * nb / L)), nb - 1)
        for lvl in range(2, d + 1):
            sh = d - lvl
            h = L / 2 ** lvl
            ax, az = tx >> sh, tz >> sh
            rt, zt = (ax + 0.5) * h, (az + 0.5) * h
            for (a, c) in _interaction_lists(ax, az, lvl):
                sel = ((six >> sh) == a) & ((siz >> sh) == c)
                if not np.any(sel):
                    continue
                rs, zs = (a + 0.5) * h, (c + 0.5) * h
                M = orc.p2m(sr[sel], sz[sel], S[sel], p, rs, zs)
                Lc = orc.s2l(M, p, rs, zs, rt, zt, pl=pl)
                out[t] += orc.l2p(Lc, pl, rt, zt, fr[t], fz[t])
        near = (np.abs(six - tx) <= 1) & (np.abs(siz - tz) <= 1)
        Dn, _ = orc.direct(sr[near], sz[near], S[near], fr[t:t + 1], fz[t:t + 1])
        out[t] += Dn[0]
    assert np.max(np.abs(out - F)) <= 1e-13 * np.max(np.abs(F))


def test_s2l_separate_orders_converge(orc):
    """Independent source and local orders: S2L from moments of
    order p to a local of order pl, evaluated in the target box, converges to the direct field as
    min(p, pl) grows, and raising one order alone is bounded by the other."""
    rng = np.random.default_rng(17)
    h, K = 1.0 / 16, 3
    rs, zs, rt, zt = 6.5 * h, 5.5 * h, 8.5 * h, 7.5 * h
    r = rs + (rng.random(10) - 0.5) * h
    z = zs + (rng.random(10) - 0.5) * h
    S = rng.standard_normal((10, K)) + 1j * rng.standard_normal((10, K))
    tr = rt + (rng.random(6) - 0.5) * h
    tz = zt + (rng.random(6) - 0.5) * h
    D, _ = orc.direct(r, z, S, tr, tz)

    def err(p, pl):
        M = orc.p2m(r, z, S, p, rs, zs)
        Lc = orc.s2l(M, p, rs, zs, rt, zt, pl=pl)
        F = np.array([orc.l2p(Lc, pl, rt, zt, tr[k], tz[k]) for k in range(6)])
        return np.max(np.abs(F - D)) / np.max(np.abs(D))

    assert err(10, 10) < err(6, 10) and err(10, 10) < err(10, 6)
    assert err(6, 12) < 10 * err(6, 6) and err(12, 6) < 10 * err(6, 6)
    assert err(12, 12) < 1e-6


@pytest.mark.parametrize("p", [2, 3, 4, 5, 6, 7])
def test_s2l_truncation_order_by_scaling(orc, p):
    """External pin of the S2L truncation boundary (R#8), single (i+j+k+l <= p) and double
    (i+j <= p, k+l <= p): S2L + L2P is a truncated Taylor expansion of G^(n)(r_t, r_s, z_t - z_s)
    in the source offset (r_s, z_s) - c_s and the target offset (r_t, z_t) - c_t.  In
    both truncations the lowest dropped terms have total degree p + 1, so shrinking BOTH offsets
    by a factor 2 must shrink the error against the exact G (oracle.greens, pinned to mpmath
    legenq in test_oracle_specfun) by 2^(p+1): a '>=' for '>' slip (one degree too few) gives
    2^p, one degree too many 2^(p+2).  Generic box pairs (no row / diagonal symmetry, which can
    cancel the leading term), outward and inward, forward and backward.  Single truncation drops
    terms double truncation keeps, so its error is the larger (SURVEY APP-F: 3x-30x)."""
    h = 1.0 / 32
    K = 4
    S = np.array([1.0 + 0.5j, -0.7 + 0.2j, 0.3 - 0.9j, 0.8 + 0.1j])
    for (si, sj, ti, tj) in [(10, 12, 13, 9), (13, 9, 10, 12), (9, 11, 12, 8), (12, 8, 9, 11)]:
        cs = ((si + 0.5) * h, (sj + 0.5) * h)
        ct = ((ti + 0.5) * h, (tj + 0.5) * h)
        errs = {0: [], 1: []}
        for lam in (0.5, 0.25, 0.125):
            rs, zs = cs[0] + lam * 0.31 * h, cs[1] - lam * 0.42 * h
            rt, zt = ct[0] - lam * 0.37 * h, ct[1] + lam * 0.26 * h
            exact = orc.greens(rt, rs, zt - zs, K - 1) * S
            M = orc.p2m([rs], [zs], S[None, :], p, cs[0], cs[1])
            for trunc in (0, 1):
                L = orc.s2l(M, p, cs[0], cs[1], ct[0], ct[1], truncation=trunc)
                F = orc.l2p(L, p, ct[0], ct[1], rt, zt)
                errs[trunc].append(np.abs(F - exact).max() / np.abs(exact).max())
        for trunc, tol in ((1, 0.25), (0, 0.5)):
            if trunc == 0 and p > 6:
                continue   # double truncation at p = 7 reaches rounding at the smallest offset
            e = errs[trunc]
            rates = [math.log2(e[k] / e[k + 1]) for k in range(2)]
            assert all(abs(r - (p + 1)) < tol for r in rates), ((si, sj, ti, tj), p, trunc, e, rates)
        assert all(a > b for a, b in zip(errs[1], errs[0])), (errs[1], errs[0])


# ---- adaptive source tree (reading R#26) ------------------------------------
def _clustered(n, K, seed):
    from tests.inputs import config_c4
    pr = config_c4(n=n, K=K, p=8, depth=6, seed=seed, clusters=8)
    return pr.sr, pr.sz, pr.S


def test_adaptive_sigma0_is_uniform(orc):
    """leaf_src = 0 is the uniform tree, operation for operation (bitwise)."""
    sr, sz, S = _clustered(1600, 3, 31)
    A, sa = orc.fmm(sr, sz, S, sr, sz, 6, 5, 1.0)
    B, sb = orc.fmm(sr, sz, S, sr, sz, 6, 5, 1.0, leaf_src=0)
    assert sa == sb and np.array_equal(A, B)


@pytest.mark.parametrize("leaf_src", [8, 40])
def test_adaptive_converges_to_direct(orc, leaf_src):
    """Pinned against the plain direct sum: with the adaptive lists every (target,
    source) pair must be covered exactly once -- a missing or doubled pair would leave an O(1)
    error floor -- so the error falls geometrically with the order (~0.4 decade per order, P:680,
    714-718) to the uniform tree's level; clustered C4-like input, depth 6."""
    sr, sz, S = _clustered(2400, 3, 32)
    D, _ = orc.direct(sr, sz, S, sr, sz)
    eps, uni = {}, {}
    for p in [4, 8, 12, 16]:
        F, sk = orc.fmm(sr, sz, S, sr, sz, p, 6, 1.0, leaf_src=leaf_src)
        assert sk >= 2400
        eps[p] = orc.eps_per_mode(F, D)
        U, _ = orc.fmm(sr, sz, S, sr, sz, p, 6, 1.0)
        uni[p] = orc.eps_per_mode(U, D)
    slope = np.log10(eps[4].max() / eps[16].max()) / 12
    assert 0.25 < slope < 0.8, slope
    for p in [4, 8, 12]:
        assert np.all(eps[p] > eps[p + 4])
    # same accuracy class as the uniform tree (the direct sums it adds are exact)
    assert np.all(eps[16] < 1e-8), eps[16]
    assert eps[16].max() < 10 * uni[16].max()


def test_adaptive_all_leaves_at_level2(orc):
    """leaf_src >= N: every level-2 source box is a leaf, so every target sums its level-2
    neighbourhood directly and takes S2L only from the non-adjacent level-2 boxes:
    the FMM equals that split, assembled here from the direct sum and single-box operators."""
    rng = np.random.default_rng(33)
    sr, sz, S = uniform_rings(rng, 300, 2)
    fr, fz, _ = uniform_rings(rng, 9, 1)
    p, d, L = 8, 4, 1.0
    F, _ = orc.fmm(sr, sz, S, fr, fz, p, d, L, leaf_src=10 ** 6)
    six = np.minimum(np.floor(sr * 4 / L), 3).astype(int)
    siz = np.minimum(np.floor(sz * 4 / L), 3).astype(int)
    h = L / 4
    out = np.zeros_like(F)
    for t in range(len(fr)):
        tx, tz = min(int(fr[t] * 4 / L), 3), min(int(fz[t] * 4 / L), 3)
        rt, zt = (tx + 0.5) * h, (tz + 0.5) * h
        for a in range(4):
            for c in range(4):
                sel = (six == a) & (siz == c)
                if not np.any(sel):
                    continue
                if abs(a - tx) <= 1 and abs(c - tz) <= 1:
                    Dn, _ = orc.direct(sr[sel], sz[sel], S[sel], fr[t:t + 1], fz[t:t + 1])
                    out[t] += Dn[0]
                else:
                    rs, zs = (a + 0.5) * h, (c + 0.5) * h
                    M = orc.p2m(sr[sel], sz[sel], S[sel], p, rs, zs)
                    Lc = orc.s2l(M, p, rs, zs, rt, zt)
                    # the level-2 local reaches the leaf by exact L2L re-centrings
                    out[t] += orc.l2p(Lc, p, rt, zt, fr[t], fz[t])
    assert np.max(np.abs(out - F)) <= 1e-12 * np.max(np.abs(F))
