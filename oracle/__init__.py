"""Oracle: plain, slow, obviously-correct FP64 CPU reference (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2301_01179_b200``/``libcylfmm.so``) never imports, links or executes it, and the two
share no code.  The C sources in this directory cite PAPER.md line numbers (P:n) and the
DESIGN.md readings (R#k) they follow.

This module is argument marshalling only: every number is computed by ``liboracle.so``
(plain C, -O2, no fast-math, no FMA contraction, OpenMP over independent outputs).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_SOURCES = ["specfun.c", "tensor.c", "direct.c", "fmm.c"]

MILLER_ACCURATE = 0
MILLER_PAPER = 1
TRUNC_DOUBLE = 0
TRUNC_SINGLE = 1


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C, no fast-math, no FP contraction)."""
    srcs = [os.path.join(_HERE, s) for s in _SOURCES]
    hdr = os.path.join(_HERE, "oracle.h")
    if not force and os.path.exists(_LIB_PATH):
        newest = max(os.path.getmtime(p) for p in srcs + [hdr])
        if os.path.getmtime(_LIB_PATH) >= newest:
            return _LIB_PATH
    cmd = ["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
           "-fno-fast-math", "-Wall", "-o", _LIB_PATH + ".tmp"] + srcs + ["-lm"]
    subprocess.check_call(cmd)
    os.replace(_LIB_PATH + ".tmp", _LIB_PATH)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        d, i, i64 = ctypes.c_double, ctypes.c_int, ctypes.c_int64
        P = ctypes.POINTER
        pd = P(d)
        L.or_carlson_rf.restype = d
        L.or_carlson_rf.argtypes = [d, d, d]
        L.or_carlson_rd.restype = d
        L.or_carlson_rd.argtypes = [d, d, d]
        L.or_ellip_ke.restype = None
        L.or_ellip_ke.argtypes = [d, pd, pd]
        L.or_legendre_q.restype = i
        L.or_legendre_q.argtypes = [d, d, i, i, i, pd]
        L.or_forward_coef.restype = d
        L.or_forward_coef.argtypes = [i, i]
        L.or_greens.restype = i
        L.or_greens.argtypes = [d, d, d, i, i, pd]
        L.or_rational_tables.restype = None
        L.or_rational_tables.argtypes = [d, d, d, i, pd]
        L.or_tensor.restype = i
        L.or_tensor.argtypes = [d, d, d, i, i, i, pd]
        L.or_direct.restype = i64
        L.or_direct.argtypes = [pd, pd, pd, i64, pd, pd, i64, i, i, i, pd, i]
        L.or_tree_keys.restype = None
        L.or_tree_keys.argtypes = [pd, pd, i64, i, d, d, P(ctypes.c_uint32), P(i64)]
        L.or_p2m.restype = None
        L.or_p2m.argtypes = [pd, pd, pd, i64, i, i, d, d, pd]
        L.or_m2m.restype = None
        L.or_m2m.argtypes = [pd, i, i, d, d, pd]
        L.or_l2l.restype = None
        L.or_l2l.argtypes = [pd, i, i, d, d, pd]
        L.or_l2p.restype = None
        L.or_l2p.argtypes = [pd, i, i, d, d, d, d, pd]
        L.or_s2l.restype = i
        L.or_s2l.argtypes = [pd, i, i, i, d, d, d, d, i, i, pd]
        L.or_fmm.restype = i64
        L.or_fmm.argtypes = [pd, pd, pd, i64, pd, pd, i64, i, i, i, i, d, d, i, i, pd, pd, pd, i, i64]
        L.or_greens_grad.restype = i
        L.or_greens_grad.argtypes = [d, d, d, i, i, pd, pd, pd]
        L.or_direct_grad.restype = i64
        L.or_direct_grad.argtypes = [pd, pd, pd, i64, pd, pd, i64, i, i, i, pd, pd, pd, i]
        _lib = L
    return _lib


def _pd(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)


def tri_size(p: int) -> int:
    return (p + 1) * (p + 2) // 2


def tri_idx(i: int, j: int, p: int) -> int:
    return i * (p + 1) - i * (i - 1) // 2 + j


def carlson_rf(x, y, z) -> float:
    return lib().or_carlson_rf(x, y, z)


def carlson_rd(x, y, z) -> float:
    return lib().or_carlson_rd(x, y, z)


def ellip_ke(kp2: float):
    K, E = ctypes.c_double(), ctypes.c_double()
    lib().or_ellip_ke(kp2, ctypes.byref(K), ctypes.byref(E))
    return K.value, E.value


def legendre_q(chi: float, kp2: float, forward: bool, nmax: int, miller: int = MILLER_ACCURATE):
    out = np.zeros(nmax + 1)
    rc = lib().or_legendre_q(chi, kp2, int(forward), nmax, miller, _pd(out))
    if rc != 0:
        raise ValueError("or_legendre_q failed")
    return out


def forward_coef(nmax: int, miller: int = MILLER_ACCURATE) -> float:
    return lib().or_forward_coef(nmax, miller)


def greens(r: float, r1: float, x: float, nmax: int, miller: int = MILLER_ACCURATE):
    out = np.zeros(nmax + 1)
    if lib().or_greens(r, r1, x, nmax, miller, _pd(out)) != 0:
        raise ValueError("or_greens: domain error")
    return out


def rational_tables(r, r1, x, qmax):
    out = np.zeros(8 * (qmax + 1))
    lib().or_rational_tables(r, r1, x, qmax, _pd(out))
    return out.reshape(8, qmax + 1)


def tensor(r, r1, x, nmax, p, miller: int = MILLER_ACCURATE):
    out = np.zeros((nmax + 1, p + 1, p + 1, 2 * p + 1))
    if lib().or_tensor(r, r1, x, nmax, p, miller, _pd(out)) != 0:
        raise ValueError("or_tensor failed")
    return out


def direct(sr, sz, S, fr, fz, miller: int = MILLER_ACCURATE, exclude_coincident: bool = True,
           nthreads: int = 0):
    sr, sz, fr, fz = _f64(sr), _f64(sz), _f64(fr), _f64(fz)
    S = _c128(S)
    ns, K = S.shape
    nf = fr.shape[0]
    Phi = np.zeros((nf, K), dtype=np.complex128)
    sk = lib().or_direct(_pd(sr), _pd(sz), _pd(S.view(np.float64)), ns, _pd(fr), _pd(fz), nf, K,
                         miller, int(exclude_coincident), _pd(Phi.view(np.float64)), nthreads)
    if sk < 0:
        raise ValueError("or_direct: domain error or unexcluded coincident pair")
    return Phi, int(sk)


def greens_grad(r, r1, x, nmax, miller: int = MILLER_ACCURATE):
    """G^(n), dG/dr, dG/dx (field point) for n = 0..nmax."""
    G, Gr, Gx = (np.zeros(nmax + 1) for _ in range(3))
    if lib().or_greens_grad(r, r1, x, nmax, miller, _pd(G), _pd(Gr), _pd(Gx)) != 0:
        raise ValueError("or_greens_grad failed")
    return G, Gr, Gx


def direct_grad(sr, sz, S, fr, fz, miller: int = MILLER_ACCURATE, exclude_coincident: bool = True,
                nthreads: int = 0):
    """Direct sum with field gradients: (Phi, dPhi/dr, dPhi/dz, skipped)."""
    sr, sz, fr, fz = _f64(sr), _f64(sz), _f64(fr), _f64(fz)
    S = _c128(S)
    ns, K = S.shape
    nf = fr.shape[0]
    out = [np.zeros((nf, K), dtype=np.complex128) for _ in range(3)]
    sk = lib().or_direct_grad(_pd(sr), _pd(sz), _pd(S.view(np.float64)), ns, _pd(fr), _pd(fz), nf,
                              K, miller, int(exclude_coincident),
                              *[_pd(o.view(np.float64)) for o in out], nthreads)
    if sk < 0:
        raise ValueError("or_direct_grad: domain error or unexcluded coincident pair")
    return out[0], out[1], out[2], int(sk)


def tree_keys(r, z, depth, L, z0):
    r, z = _f64(r), _f64(z)
    n = r.shape[0]
    key = np.zeros(n, dtype=np.uint32)
    perm = np.zeros(n, dtype=np.int64)
    lib().or_tree_keys(_pd(r), _pd(z), n, depth, L, z0,
                       key.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
                       perm.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    return key, perm


def p2m(r, z, S, p, rc, zc):
    r, z, S = _f64(r), _f64(z), _c128(S)
    n, K = S.shape
    M = np.zeros((K, tri_size(p)), dtype=np.complex128)
    lib().or_p2m(_pd(r), _pd(z), _pd(S.view(np.float64)), n, K, p, rc, zc, _pd(M.view(np.float64)))
    return M


def m2m(Mc, p, dr, dz):
    Mc = _c128(Mc)
    out = np.zeros_like(Mc)
    lib().or_m2m(_pd(Mc.view(np.float64)), Mc.shape[0], p, dr, dz, _pd(out.view(np.float64)))
    return out


def l2l(Lp, p, dr, dz):
    Lp = _c128(Lp)
    out = np.zeros_like(Lp)
    lib().or_l2l(_pd(Lp.view(np.float64)), Lp.shape[0], p, dr, dz, _pd(out.view(np.float64)))
    return out


def l2p(Lc, p, rc, zc, r, z):
    Lc = _c128(Lc)
    out = np.zeros(Lc.shape[0], dtype=np.complex128)
    lib().or_l2p(_pd(Lc.view(np.float64)), Lc.shape[0], p, rc, zc, r, z, _pd(out.view(np.float64)))
    return out


def s2l(M, p, rs, zs, rt, zt, truncation=TRUNC_DOUBLE, miller=MILLER_ACCURATE, pl=None):
    """Source moments M [K, P(p)] -> local contribution [K, P(pl)] (pl defaults to p)."""
    M = _c128(M)
    pl = p if pl is None else pl
    out = np.zeros((M.shape[0], tri_size(pl)), dtype=np.complex128)
    rc = lib().or_s2l(_pd(M.view(np.float64)), M.shape[0], p, pl, rs, zs, rt, zt, truncation,
                      miller, _pd(out.view(np.float64)))
    if rc != 0:
        raise ValueError("or_s2l failed")
    return out


def fmm(sr, sz, S, fr, fz, p, depth, L, z0=0.0, truncation=TRUNC_DOUBLE,
        miller=MILLER_ACCURATE, nthreads: int = 0, pl=None, grad=False, leaf_src: int = 0):
    """Algorithm 1: source/moment order p, local order pl (default p).
    grad=True also returns the field gradients dPhi/dr, dPhi/dz: (Phi, dPr, dPz, skipped).
    leaf_src > 0: the adaptive source tree of R#26 (a source box with <= leaf_src sources is a
    leaf); 0 = the uniform tree."""
    sr, sz, fr, fz = _f64(sr), _f64(sz), _f64(fr), _f64(fz)
    S = _c128(S)
    ns, K = S.shape
    nf = fr.shape[0]
    Phi = np.zeros((nf, K), dtype=np.complex128)
    grad = bool(grad)
    Gr = np.zeros((nf, K), dtype=np.complex128) if grad else None
    Gz = np.zeros((nf, K), dtype=np.complex128) if grad else None
    nul = ctypes.POINTER(ctypes.c_double)()
    sk = lib().or_fmm(_pd(sr), _pd(sz), _pd(S.view(np.float64)), ns, _pd(fr), _pd(fz), nf, K, p,
                      0 if pl is None else pl, depth, L, z0, truncation, miller,
                      _pd(Phi.view(np.float64)), _pd(Gr.view(np.float64)) if grad else nul,
                      _pd(Gz.view(np.float64)) if grad else nul, nthreads, int(leaf_src))
    if sk < 0:
        raise ValueError("or_fmm: invalid input")
    return (Phi, Gr, Gz, int(sk)) if grad else (Phi, int(sk))


def eps_per_mode(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """The paper's error metric: max_j |A-B| / max_j |B| per mode."""
    num = np.abs(A - B).max(axis=0)
    den = np.abs(B).max(axis=0)
    return num / np.where(den > 0, den, 1.0)
