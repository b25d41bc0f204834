"""Seeded synthetic input generators for the BASELINE.json configurations C1..C5.

This module holds NO arithmetic of the method (no Green's functions, expansions or trees):
it only draws ring positions and modal coefficients.  It is the one module shared by the
tests (oracle side), the product bench and the GPU parity tests.

Recipe: numpy ``default_rng(seed)``, seed = config index; draw order
source r, source z, Re S, Im S, then field r, field z.  The paper's own workload is synthetic
uniform random rings; BASELINE.json's configs stand in for it.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Problem:
    name: str
    sr: np.ndarray            # source radii, float64 [Ns]
    sz: np.ndarray            # source axial positions, float64 [Ns]
    S: np.ndarray             # complex128 [Ns, K] modal coefficients S^(n), n = 0..K-1
    fr: np.ndarray            # field radii [Nf]
    fz: np.ndarray            # field axial positions [Nf]
    p: int = 0                # expansion order (0 = direct only)
    depth: int = 0            # tree depth d
    L: float = 1.0            # square domain [0, L] x [z0, z0 + L]
    z0: float = 0.0
    fields_are_sources: bool = False

    @property
    def K(self) -> int:
        return self.S.shape[1]


def uniform_rings(rng, n, K, rmax=1.0, zmax=1.0, decay=False):
    """r = rmax (1 - U) in (0, rmax], z = zmax U, S = (a + i b) [/(1+n)], a, b ~ N(0,1)."""
    r = rmax * (1.0 - rng.random(n))
    z = zmax * rng.random(n)
    S = rng.standard_normal((n, K)) + 1j * rng.standard_normal((n, K))
    if decay:
        S = S / (1.0 + np.arange(K))[None, :]
    return r, z, S


def config_c1(n=1000, K=9, seed=1) -> Problem:
    """C1: direct modal sum, N = M = 1000, n = 0..8, independent field draws."""
    rng = np.random.default_rng(seed)
    sr, sz, S = uniform_rings(rng, n, K)
    fr = 1.0 - rng.random(n)
    fz = rng.random(n)
    return Problem("C1-direct", sr, sz, S, fr, fz)


def config_c2(n=16384, K=17, p=8, depth=5, seed=2) -> Problem:
    """C2: FMM, N = M = 16384 uniform in (0,1]x[0,1], n = 0..16, p = 8, fields = sources."""
    rng = np.random.default_rng(seed)
    sr, sz, S = uniform_rings(rng, n, K)
    return Problem("C2-fmm-uniform", sr, sz, S, sr, sz, p=p, depth=depth, L=1.0,
                   fields_are_sources=True)


def config_c3(n=131072, K=33, p=12, depth=7, seed=3) -> Problem:
    """C3: FMM, N = M = 131072 in (0,1]x[0,2], n = 0..32, S /(1+n), p = 12, L = 2."""
    rng = np.random.default_rng(seed)
    sr, sz, S = uniform_rings(rng, n, K, rmax=1.0, zmax=2.0, decay=True)
    return Problem("C3-fmm-uniform", sr, sz, S, sr, sz, p=p, depth=depth, L=2.0,
                   fields_are_sources=True)


def config_c4(n=1048576, K=17, p=16, depth=8, seed=4, clusters=16) -> Problem:
    """C4: 16 Gaussian clusters (sigma 0.02), 25% of centres at r < 0.05; r clamped to
    [1e-6, 1], z to [0, 1]; fields = sources (reading: SURVEY 8(d))."""
    rng = np.random.default_rng(seed)
    nax = clusters // 4
    rc = np.concatenate([0.05 * (1.0 - rng.random(nax)), 0.05 + 0.95 * rng.random(clusters - nax)])
    zc = rng.random(clusters)
    per = n // clusters
    idx = np.repeat(np.arange(clusters), per)
    r = rc[idx] + 0.02 * rng.standard_normal(n)
    z = zc[idx] + 0.02 * rng.standard_normal(n)
    r = np.clip(r, 1e-6, 1.0)
    z = np.clip(z, 0.0, 1.0)
    S = rng.standard_normal((n, K)) + 1j * rng.standard_normal((n, K))
    return Problem("C4-fmm-clustered", r, z, S, r, z, p=p, depth=depth, L=1.0,
                   fields_are_sources=True)


def surface_sources(n):
    """Uniform arc-length points on a torus generating circle (centre (0.5, 0.5), radius 0.2)
    followed by a sphere generating semicircle (centre (0, 1), radius 0.4)."""
    ltor, lsph = 2 * np.pi * 0.2, np.pi * 0.4
    s = (np.arange(n) + 0.5) * (ltor + lsph) / n
    tor = s < ltor
    ang = s[tor] / 0.2
    psi = (s[~tor] - ltor) / 0.4
    r = np.concatenate([0.5 + 0.2 * np.cos(ang), 0.4 * np.sin(psi)])
    z = np.concatenate([0.5 + 0.2 * np.sin(ang), 1.0 - 0.4 * np.cos(psi)])
    return r, z


def config_c5(n=4194304, grid=2048, K=65, p=16, depth=10, seed=5) -> Problem:
    """C5: sources on torus + sphere generating curves, fields on a grid x grid tensor grid
    r_i = i / grid (i = 1..grid), z_j = 2 j / (grid - 1) (j = 0..grid-1), r-major; L = 2."""
    rng = np.random.default_rng(seed)
    sr, sz = surface_sources(n)
    S = rng.standard_normal((n, K)) + 1j * rng.standard_normal((n, K))
    ri = np.arange(1, grid + 1) / grid
    zj = 2.0 * np.arange(grid) / (grid - 1)
    fr = np.repeat(ri, grid)
    fz = np.tile(zj, grid)
    return Problem("C5-fmm-surface", sr, sz, S, fr, fz, p=p, depth=depth, L=2.0)


CONFIGS = {"C1": config_c1, "C2": config_c2, "C3": config_c3, "C4": config_c4, "C5": config_c5}
