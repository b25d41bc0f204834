"""Error-driven order and depth selection (cylfmm_select_params, host-only; SURVEY 8(f) item 2,
R#25).  CPU: the per-depth near-field and S2L pair counts against brute force over point pairs
and box pairs, the order rule, the argmin, the error codes.  GPU: the counts equal what a solve
at the chosen depth reports, and the chosen order meets the requested tolerance against the
direct sum (the paper's per-mode error)."""
import numpy as np
import pytest

import paper_2301_01179_b200 as cyl
from tests.inputs import uniform_rings

EPS_C = 0.1   # CYLFMM_EPS_C, include/cylfmm.h


def _boxes(r, z, d, L, z0):
    nb = 1 << d
    ix = np.minimum(np.floor(r * nb / L).astype(np.int64), nb - 1)
    iz = np.minimum(np.floor((z - z0) * nb / L).astype(np.int64), nb - 1)
    return ix, iz


def _brute_counts(sr, sz, fr, fz, d, L, z0):
    """near(d): (field, source) point pairs whose depth-d leaves touch (|di|, |dj| <= 1);
    s2l(d): over levels 2..d, (non-empty target box, non-empty source box) pairs whose parents
    touch and which do not touch themselves."""
    six, siz = _boxes(sr, sz, d, L, z0)
    fix, fiz = _boxes(fr, fz, d, L, z0)
    near = int(np.sum((np.abs(fix[:, None] - six[None, :]) <= 1) &
                      (np.abs(fiz[:, None] - siz[None, :]) <= 1)))
    s2l = 0
    for l in range(2, d + 1):
        S = np.array(sorted(set(zip(*_boxes(sr, sz, l, L, z0)))))
        T = np.array(sorted(set(zip(*_boxes(fr, fz, l, L, z0)))))
        if len(S) == 0 or len(T) == 0:
            continue
        dx = np.abs(T[:, None, 0] - S[None, :, 0])
        dz = np.abs(T[:, None, 1] - S[None, :, 1])
        px = np.abs(T[:, None, 0] // 2 - S[None, :, 0] // 2)
        pz = np.abs(T[:, None, 1] // 2 - S[None, :, 1] // 2)
        s2l += int(np.sum((px <= 1) & (pz <= 1) & ((dx >= 2) | (dz >= 2))))
    return near, s2l


def _problem(seed=5, ns=400, nf=300):
    rng = np.random.default_rng(seed)
    sr, sz, _ = uniform_rings(rng, ns, 1)
    # a clustered field set (half on a short segment) so the counts are not uniform
    fr, fz, _ = uniform_rings(rng, nf, 1)
    k = nf // 2
    fr[:k] = 0.30 + 0.05 * rng.random(k)
    fz[:k] = 0.62 + 0.01 * rng.random(k)
    return sr, sz, fr, fz


def test_select_counts_match_brute_force():
    sr, sz, fr, fz = _problem()
    cfg, info = cyl.select_params(sr, sz, fr, fz, n_modes=5, tol=1e-4, depth_min=2, depth_max=6)
    for q, d in enumerate(info["depths"]):
        near, s2l = _brute_counts(sr, sz, fr, fz, int(d), 1.0, 0.0)
        assert info["near_pairs"][q] == near, d
        assert info["s2l_pairs"][q] == s2l, d
    assert cfg.depth == int(info["depths"][np.argmin(info["est_ms"])])


def test_select_counts_shifted_domain_and_sources_as_fields():
    rng = np.random.default_rng(9)
    sr, sz, _ = uniform_rings(rng, 350, 1)
    sr, sz = 2.0 * sr, 2.0 * sz - 1.0          # domain [0, 2] x [-1, 1]
    cfg, info = cyl.select_params(sr, sz, sr, sz, n_modes=3, tol=1e-3, L=2.0, z0=-1.0,
                                  depth_min=3, depth_max=5)
    for q, d in enumerate(info["depths"]):
        near, s2l = _brute_counts(sr, sz, sr, sz, int(d), 2.0, -1.0)
        assert (info["near_pairs"][q], info["s2l_pairs"][q]) == (near, s2l)


def test_select_order_rule():
    sr, sz, fr, fz = _problem(ns=50, nf=40)
    prev = 0
    for tol in [1e-1, 3e-2, 1e-3, 1e-5, 1e-6, 1e-8, 1e-12]:
        cfg, info = cyl.select_params(sr, sz, fr, fz, n_modes=2, tol=tol, depth_min=2, depth_max=3)
        p = cfg.order
        eps = lambda q: EPS_C * 10.0 ** (-0.4 * q)   # noqa: E731
        if p < 16:
            assert eps(p) <= tol and (p == 1 or eps(p - 1) > tol), tol
        else:
            assert p == 16 and (eps(15) > tol)
        assert info["eps_model"] == pytest.approx(eps(p), rel=1e-14)
        assert p >= prev and cfg.order_local == 0
        prev = p


def test_select_depth_outside_range_and_errors():
    sr, sz, fr, fz = _problem(ns=60, nf=50)
    cfg, info = cyl.select_params(sr, sz, fr, fz, n_modes=2, tol=1e-4, depth_min=0, depth_max=3)
    assert list(info["near_pairs"][:2]) == [-1, -1] and list(info["est_ms"][:2]) == [-1.0, -1.0]
    assert 2 <= cfg.depth <= 3
    with pytest.raises(cyl.CylFMMError):
        cyl.select_params(sr, sz, fr, fz, n_modes=2, tol=0.0)
    with pytest.raises(cyl.CylFMMError):
        cyl.select_params(sr, sz, fr, fz, n_modes=2, tol=1e-4, depth_min=5, depth_max=4)
    with pytest.raises(cyl.CylFMMError):
        cyl.select_params(sr, sz, fr, fz, n_modes=2, tol=1e-4, depth_min=12, depth_max=14)
    with pytest.raises(cyl.CylFMMError):
        cyl.select_params(np.array([1.5]), np.array([0.5]), fr, fz, n_modes=2, tol=1e-4)


def test_select_model_prefers_shallower_tree_for_few_points():
    # a handful of points: the near field is cheap at any depth, the far field only grows
    sr, sz, fr, fz = _problem(ns=30, nf=30)
    cfg, info = cyl.select_params(sr, sz, fr, fz, n_modes=4, tol=1e-4, depth_min=2, depth_max=8)
    assert cfg.depth == 2
    assert np.all(np.diff(info["s2l_pairs"]) >= 0) and np.all(np.diff(info["near_pairs"]) <= 0)


@pytest.mark.gpu
def test_select_counts_equal_solve_counters():
    import torch
    from paper_2301_01179_b200.inputs import CONFIGS
    pr = CONFIGS["C2"]()
    cfg, info = cyl.select_params(pr.sr, pr.sz, pr.fr, pr.fz, pr.K, 1e-4, L=pr.L, z0=pr.z0,
                                  depth_min=3, depth_max=7)
    dev = lambda a: torch.as_tensor(a, device="cuda")   # noqa: E731
    for q, d in enumerate(info["depths"]):
        c = cyl.FMMConfig(n_modes=pr.K, order=4, depth=int(d), L=pr.L, z0=pr.z0)
        _, tm = cyl.Plan(c).solve(dev(pr.sr), dev(pr.sz), dev(pr.S), dev(pr.fr), dev(pr.fz),
                                  timings=True)
        assert tm["n_near_pairs"] + tm["n_skipped"] == info["near_pairs"][q], d
        assert tm["n_s2l_pairs"] == info["s2l_pairs"][q], d


@pytest.mark.gpu
@pytest.mark.parametrize("name,tol", [("C2", 1e-4), ("C2", 1e-6), ("C2", 1e-7), ("C3", 1e-6)])
def test_selected_order_meets_tolerance(orc, name, tol):
    """The selected (order, depth) solve of a config's inputs meets tol against the oracle direct
    sum on 64 sampled field points, per mode."""
    import torch
    from paper_2301_01179_b200.inputs import CONFIGS
    pr = CONFIGS[name]()
    cfg, info = cyl.select_params(pr.sr, pr.sz, pr.fr, pr.fz, pr.K, tol, L=pr.L, z0=pr.z0,
                                  depth_min=3, depth_max=8)
    dev = lambda a: torch.as_tensor(a, device="cuda")   # noqa: E731
    out = cyl.Plan(cfg).solve(dev(pr.sr), dev(pr.sz), dev(pr.S), dev(pr.fr), dev(pr.fz)).cpu().numpy()
    idx = np.random.default_rng(2).choice(len(pr.fr), 64, replace=False)
    ref, _ = orc.direct(pr.sr, pr.sz, pr.S, pr.fr[idx], pr.fz[idx])
    eps = np.abs(out[idx] - ref).max(axis=0) / np.abs(ref).max(axis=0)
    assert eps.max() <= tol, (cfg, eps.max())
