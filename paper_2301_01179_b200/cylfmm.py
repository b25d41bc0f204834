"""Thin Python binding of libcylfmm.so (include/cylfmm.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels of ``csrc/``; PyTorch supplies device
memory and the current stream.  There is no CPU fallback: if the shared library is missing
or no CUDA device is present, the calls raise.
"""
from __future__ import annotations

import ctypes
import os
import re
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_PATH = os.path.join(HERE, "libcylfmm.so")
HEADER = os.path.join(ROOT, "include", "cylfmm.h")

OK, EINVAL, EDOMAIN, ENUMERIC, ECUDA, ENCCL, ENOMEM = range(7)
MILLER_ACCURATE, MILLER_PAPER = 0, 1
TRUNC_DOUBLE, TRUNC_SINGLE = 0, 1


class CylFMMError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: status {status} ({detail})")
        self.status = status


class Params(ctypes.Structure):
    _fields_ = [("n_modes", ctypes.c_int), ("order", ctypes.c_int), ("depth", ctypes.c_int),
                ("truncation", ctypes.c_int), ("miller", ctypes.c_int),
                ("exclude_coincident", ctypes.c_int), ("domain_z0", ctypes.c_double),
                ("domain_L", ctypes.c_double), ("mode_chunk", ctypes.c_int),
                ("order_local", ctypes.c_int), ("adaptive_leaf", ctypes.c_int)]


class Timings(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("ms_tree", "ms_p2m", "ms_m2m", "ms_tensor", "ms_s2l",
                                                "ms_l2l", "ms_l2p", "ms_p2p", "ms_total")] + \
               [(n, ctypes.c_int64) for n in ("n_near_pairs", "n_skipped", "n_s2l_pairs",
                                              "kernel_launches")] + \
               [(n, ctypes.c_double) for n in ("ms_sort", "ms_lists", "ms_unpermute", "ms_allgather")] + \
               [(n, ctypes.c_int64) for n in ("n_solves", "n_forward", "n_far", "n_miller",
                                              "miller_steps")] + \
               [("ms_seeds", ctypes.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None


def header_functions() -> list[str]:
    """Names of the functions declared in include/cylfmm.h."""
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return re.findall(r"\b(cylfmm_[a-z_]+)\s*\(", txt)


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libcylfmm.so not built ({LIB_PATH}); run __graft_entry__.build()")
    L = ctypes.CDLL(LIB_PATH)
    d, i, i64, vp = ctypes.c_double, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p
    L.cylfmm_status_string.restype = ctypes.c_char_p
    L.cylfmm_status_string.argtypes = [i]
    L.cylfmm_last_error.restype = ctypes.c_char_p
    L.cylfmm_last_error.argtypes = []
    L.cylfmm_version.restype = ctypes.c_char_p
    L.cylfmm_version.argtypes = []
    L.cylfmm_direct.restype = i
    L.cylfmm_direct.argtypes = [vp, vp, vp, i64, vp, vp, i64, i, i, i, vp, vp]
    L.cylfmm_direct_workspace_bytes.restype = i
    L.cylfmm_direct_workspace_bytes.argtypes = [i64, i64, i, ctypes.POINTER(i64)]
    L.cylfmm_direct_enqueue.restype = i
    L.cylfmm_direct_enqueue.argtypes = [vp, vp, vp, i64, vp, vp, i64, i, i, i, vp, vp, i64, vp]
    L.cylfmm_plan_create.restype = i
    L.cylfmm_plan_create.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(Params)]
    L.cylfmm_plan_destroy.restype = None
    L.cylfmm_plan_destroy.argtypes = [vp]
    L.cylfmm_plan_sync.restype = i
    L.cylfmm_plan_sync.argtypes = [vp]
    L.cylfmm_comm_unique_id.restype = i
    L.cylfmm_comm_unique_id.argtypes = [vp]
    L.cylfmm_plan_create_dist.restype = i
    L.cylfmm_plan_create_dist.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(Params), i, i, vp]
    L.cylfmm_fmm_solve_dist.restype = i
    L.cylfmm_fmm_solve_dist.argtypes = [vp, vp, vp, vp, i64, vp, vp, i64, vp, vp,
                                         ctypes.POINTER(Timings)]
    L.cylfmm_plan_set_geometry_cache.restype = i
    L.cylfmm_plan_set_geometry_cache.argtypes = [vp, i]
    L.cylfmm_plan_set_profiling.restype = i
    L.cylfmm_plan_set_profiling.argtypes = [vp, i]
    L.cylfmm_plan_read_timings.restype = i
    L.cylfmm_plan_read_timings.argtypes = [vp, ctypes.POINTER(Timings)]
    L.cylfmm_fmm_solve.restype = i
    L.cylfmm_fmm_solve.argtypes = [vp, vp, vp, vp, i64, vp, vp, i64, vp, vp,
                                   ctypes.POINTER(Timings)]
    L.cylfmm_fmm_solve_host.restype = i
    L.cylfmm_fmm_solve_host.argtypes = L.cylfmm_fmm_solve.argtypes
    L.cylfmm_fmm_solve_host_async.restype = i
    L.cylfmm_fmm_solve_host_async.argtypes = [vp, vp, vp, vp, i64, vp, vp, i64, vp, vp]
    L.cylfmm_fmm_solve_grad.restype = i
    L.cylfmm_fmm_solve_grad.argtypes = [vp, vp, vp, vp, i64, vp, vp, i64, vp, vp, vp, vp,
                                        ctypes.POINTER(Timings)]
    L.cylfmm_greens_batch.restype = i
    L.cylfmm_greens_batch.argtypes = [vp, vp, vp, i64, i, i, vp, vp]
    L.cylfmm_tensor_batch.restype = i
    L.cylfmm_tensor_batch.argtypes = [vp, vp, vp, i64, i, i, i, vp, vp]
    L.cylfmm_tree_sort.restype = i
    L.cylfmm_tree_sort.argtypes = [vp, vp, i64, i, d, d, vp, vp, vp]
    L.cylfmm_partition_fields.restype = i
    L.cylfmm_partition_fields.argtypes = [vp, vp, i64, vp, vp, i64, ctypes.POINTER(Params), i,
                                          vp, vp]
    L.cylfmm_select_params.restype = i
    L.cylfmm_select_params.argtypes = [vp, vp, i64, vp, vp, i64, d, i, i, ctypes.POINTER(Params),
                                       vp, vp, vp, vp]
    _lib = L
    return L


def _check(st: int, where: str):
    if st != OK:
        L = lib()
        raise CylFMMError(st, where, f"{L.cylfmm_status_string(st).decode()}: "
                                     f"{L.cylfmm_last_error().decode()}")


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("cylfmm: no CUDA device (there is no CPU fallback)")
    return torch


def _dev_f64(t, torch):
    t = torch.as_tensor(t, dtype=torch.float64, device="cuda")
    return t.contiguous()


def _dev_c128(t, torch):
    t = torch.as_tensor(t, dtype=torch.complex128, device="cuda")
    return t.contiguous()


def _stream(torch):
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None and t.numel() > 0 else ctypes.c_void_p(0)


def direct(src_r, src_z, src_S, fld_r, fld_z, miller=MILLER_ACCURATE, exclude_coincident=True,
           out=None):
    """Direct modal sum on the GPU (cylfmm_direct).  Returns complex128 [n_fld, K] (cuda)."""
    torch = _torch()
    sr, sz, fr, fz = (_dev_f64(a, torch) for a in (src_r, src_z, fld_r, fld_z))
    S = _dev_c128(src_S, torch)
    ns, K = S.shape
    nf = fr.shape[0]
    if out is None:
        out = torch.empty((nf, K), dtype=torch.complex128, device="cuda")
    _check(lib().cylfmm_direct(_ptr(sr), _ptr(sz), _ptr(S), ns, _ptr(fr), _ptr(fz), nf, K, miller,
                               int(bool(exclude_coincident)), _ptr(out), _stream(torch)),
           "cylfmm_direct")
    return out


def direct_workspace_bytes(n_src, n_fld, n_modes):
    """Bytes of caller-owned device workspace cylfmm_direct_enqueue needs."""
    n = ctypes.c_int64(0)
    _check(lib().cylfmm_direct_workspace_bytes(n_src, n_fld, n_modes, ctypes.byref(n)),
           "cylfmm_direct_workspace_bytes")
    return n.value


def direct_enqueue(src_r, src_z, src_S, fld_r, fld_z, out, workspace, miller=MILLER_ACCURATE,
                   exclude_coincident=True):
    """cylfmm_direct_enqueue: the direct sum as launches only (CUDA-graph capturable).  All
    arguments are CUDA tensors; `workspace` is a uint8 tensor of direct_workspace_bytes(...)
    bytes whose first int32 is the error flag after completion.  Returns `out`."""
    torch = _torch()
    ns, K = src_S.shape
    nf = fld_r.shape[0]
    _check(lib().cylfmm_direct_enqueue(_ptr(src_r), _ptr(src_z), _ptr(src_S), ns, _ptr(fld_r),
                                       _ptr(fld_z), nf, K, miller, int(bool(exclude_coincident)),
                                       _ptr(out), _ptr(workspace), workspace.numel(),
                                       _stream(torch)), "cylfmm_direct_enqueue")
    return out


def greens_batch(r, r1, x, n_modes, miller=MILLER_ACCURATE):
    torch = _torch()
    r, r1, x = (_dev_f64(a, torch) for a in (r, r1, x))
    n = r.shape[0]
    out = torch.empty((n, n_modes), dtype=torch.float64, device="cuda")
    _check(lib().cylfmm_greens_batch(_ptr(r), _ptr(r1), _ptr(x), n, n_modes, miller, _ptr(out),
                                     _stream(torch)), "cylfmm_greens_batch")
    return out


def tensor_batch(r, r1, x, n_modes, p, miller=MILLER_ACCURATE):
    torch = _torch()
    r, r1, x = (_dev_f64(a, torch) for a in (r, r1, x))
    n = r.shape[0]
    out = torch.empty((n, n_modes, p + 1, p + 1, 2 * p + 1), dtype=torch.float64, device="cuda")
    _check(lib().cylfmm_tensor_batch(_ptr(r), _ptr(r1), _ptr(x), n, n_modes, p, miller,
                                     _ptr(out), _stream(torch)), "cylfmm_tensor_batch")
    return out


def tree_sort(r, z, depth, L, z0=0.0):
    torch = _torch()
    r, z = _dev_f64(r, torch), _dev_f64(z, torch)
    n = r.shape[0]
    key = torch.empty(n, dtype=torch.int32, device="cuda")
    perm = torch.empty(n, dtype=torch.int32, device="cuda")
    _check(lib().cylfmm_tree_sort(_ptr(r), _ptr(z), n, depth, float(L), float(z0), _ptr(key),
                                  _ptr(perm), _stream(torch)), "cylfmm_tree_sort")
    return key, perm


@dataclass
class FMMConfig:
    n_modes: int
    order: int
    depth: int
    L: float = 1.0
    z0: float = 0.0
    truncation: int = TRUNC_DOUBLE
    miller: int = MILLER_ACCURATE
    exclude_coincident: bool = True
    mode_chunk: int = 0
    order_local: int = 0      # local-expansion order (0: = order)
    adaptive_leaf: int = 0    # adaptive source tree: leaf if <= this many sources (0: uniform)


def comm_unique_id() -> bytes:
    """An NCCL unique id for cylfmm_plan_create_dist (cylfmm_comm_unique_id), 128 bytes."""
    buf = ctypes.create_string_buffer(128)
    _check(lib().cylfmm_comm_unique_id(buf), "cylfmm_comm_unique_id")
    return buf.raw


class Plan:
    """An FMM plan (cylfmm_plan_create); owns its device workspace.  With dist=(nranks, rank,
    unique_id) the plan also owns an NCCL communicator (cylfmm_plan_create_dist, collective) and
    solve_dist runs the multi-device solve."""

    def __init__(self, cfg: FMMConfig, dist=None):
        _torch()
        self.cfg = cfg
        prm = Params(cfg.n_modes, cfg.order, cfg.depth, cfg.truncation, cfg.miller,
                     int(bool(cfg.exclude_coincident)), float(cfg.z0), float(cfg.L),
                     cfg.mode_chunk, cfg.order_local, cfg.adaptive_leaf)
        h = ctypes.c_void_p()
        if dist is None:
            _check(lib().cylfmm_plan_create(ctypes.byref(h), ctypes.byref(prm)), "cylfmm_plan_create")
        else:
            nranks, rank, uid = dist
            ub = ctypes.create_string_buffer(bytes(uid), 128)
            _check(lib().cylfmm_plan_create_dist(ctypes.byref(h), ctypes.byref(prm), int(nranks),
                                                 int(rank), ub), "cylfmm_plan_create_dist")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().cylfmm_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def solve(self, src_r, src_z, src_S, fld_r, fld_z, out=None, timings=False):
        """Device solve (cylfmm_fmm_solve).  Returns out (complex128 [n_fld, K], cuda) and the
        timings dict if requested (that path synchronises)."""
        torch = _torch()
        sr, sz, fr, fz = (_dev_f64(a, torch) for a in (src_r, src_z, fld_r, fld_z))
        S = _dev_c128(src_S, torch)
        ns = S.shape[0]
        nf = fr.shape[0]
        if out is None:
            out = torch.empty((nf, self.cfg.n_modes), dtype=torch.complex128, device="cuda")
        tm = Timings() if timings else None
        _check(lib().cylfmm_fmm_solve(self._h, _ptr(sr), _ptr(sz), _ptr(S), ns, _ptr(fr), _ptr(fz),
                                      nf, _ptr(out), _stream(torch),
                                      ctypes.byref(tm) if tm is not None else None),
               "cylfmm_fmm_solve")
        return (out, tm.as_dict()) if timings else out

    def solve_dist(self, src_r, src_z, src_S, fld_r, fld_z, out=None, timings=False):
        """Collective multi-device solve (cylfmm_fmm_solve_dist): this rank's source shard and
        field points in, the potentials of all sources at its field points out (cuda)."""
        torch = _torch()
        sr, sz, fr, fz = (_dev_f64(a, torch) for a in (src_r, src_z, fld_r, fld_z))
        S = _dev_c128(src_S, torch)
        ns, nf = S.shape[0], fr.shape[0]
        if out is None:
            out = torch.empty((nf, self.cfg.n_modes), dtype=torch.complex128, device="cuda")
        tm = Timings() if timings else None
        _check(lib().cylfmm_fmm_solve_dist(self._h, _ptr(sr), _ptr(sz), _ptr(S), ns, _ptr(fr),
                                           _ptr(fz), nf, _ptr(out), _stream(torch),
                                           ctypes.byref(tm) if tm is not None else None),
               "cylfmm_fmm_solve_dist")
        return (out, tm.as_dict()) if timings else out

    def solve_grad(self, src_r, src_z, src_S, fld_r, fld_z, timings=False):
        """Device solve with potential gradients (cylfmm_fmm_solve_grad): returns (Phi, dPhi/dr,
        dPhi/dz), complex128 [n_fld, K] each (cuda), and the timings dict if requested."""
        torch = _torch()
        sr, sz, fr, fz = (_dev_f64(a, torch) for a in (src_r, src_z, fld_r, fld_z))
        S = _dev_c128(src_S, torch)
        ns, nf = S.shape[0], fr.shape[0]
        outs = [torch.empty((nf, self.cfg.n_modes), dtype=torch.complex128, device="cuda")
                for _ in range(3)]
        tm = Timings() if timings else None
        _check(lib().cylfmm_fmm_solve_grad(self._h, _ptr(sr), _ptr(sz), _ptr(S), ns, _ptr(fr),
                                           _ptr(fz), nf, *[_ptr(o) for o in outs], _stream(torch),
                                           ctypes.byref(tm) if tm is not None else None),
               "cylfmm_fmm_solve_grad")
        return (tuple(outs), tm.as_dict()) if timings else tuple(outs)

    def solve_host(self, src_r, src_z, src_S, fld_r, fld_z, out=None, timings=False):
        """Host-buffer solve (cylfmm_fmm_solve_host): numpy in, numpy out, copies included."""
        torch = _torch()
        sr, sz, fr, fz = (np.ascontiguousarray(a, dtype=np.float64) for a in (src_r, src_z, fld_r, fld_z))
        S = np.ascontiguousarray(src_S, dtype=np.complex128)
        ns, nf = S.shape[0], fr.shape[0]
        if out is None:
            out = np.empty((nf, self.cfg.n_modes), dtype=np.complex128)
        tm = Timings() if timings else None
        p = lambda a: ctypes.c_void_p(a.ctypes.data) if a.size else ctypes.c_void_p(0)  # noqa: E731
        _check(lib().cylfmm_fmm_solve_host(self._h, p(sr), p(sz), p(S), ns, p(fr), p(fz), nf, p(out),
                                           _stream(torch),
                                           ctypes.byref(tm) if tm is not None else None),
               "cylfmm_fmm_solve_host")
        return (out, tm.as_dict()) if timings else out

    def solve_host_async(self, src_r, src_z, src_S, fld_r, fld_z, out):
        """Pipelined host-buffer solve (cylfmm_fmm_solve_host_async): queues the upload, the solve
        and the download and returns; `out` (and the inputs, which must stay unmodified) are
        valid after sync().  Arrays must be C-contiguous float64 / complex128, ideally pinned."""
        torch = _torch()
        arrs = (src_r, src_z, src_S, fld_r, fld_z, out)
        for a in arrs:
            if not (isinstance(a, np.ndarray) and a.flags.c_contiguous):
                raise ValueError("solve_host_async: C-contiguous numpy arrays required")
        ns, nf = src_S.shape[0], fld_r.shape[0]
        p = lambda a: ctypes.c_void_p(a.ctypes.data) if a.size else ctypes.c_void_p(0)  # noqa: E731
        _check(lib().cylfmm_fmm_solve_host_async(self._h, p(src_r), p(src_z), p(src_S), ns,
                                                 p(fld_r), p(fld_z), nf, p(out), _stream(torch)),
               "cylfmm_fmm_solve_host_async")
        return out

    def sync(self):
        _check(lib().cylfmm_plan_sync(self._h), "cylfmm_plan_sync")

    def set_geometry_cache(self, on: bool):
        """Reuse the coordinate-only work of the previous solve when the coordinate arrays are the
        same (cylfmm_plan_set_geometry_cache): sync-free, graph-capturable solves."""
        _check(lib().cylfmm_plan_set_geometry_cache(self._h, int(bool(on))),
               "cylfmm_plan_set_geometry_cache")

    def set_profiling(self, on: bool):
        """Record phase events in the following (asynchronous) solves (cylfmm_plan_set_profiling)."""
        _check(lib().cylfmm_plan_set_profiling(self._h, int(bool(on))), "cylfmm_plan_set_profiling")

    def read_timings(self) -> dict:
        """Phase times averaged over the profiled solves since the last read
        (cylfmm_plan_read_timings; synchronises their events)."""
        tm = Timings()
        _check(lib().cylfmm_plan_read_timings(self._h, ctypes.byref(tm)), "cylfmm_plan_read_timings")
        return tm.as_dict()


def partition_fields(src_r, src_z, fld_r, fld_z, cfg: "FMMConfig", n_parts: int):
    """Cost-weighted Morton partition of the field points over n_parts GPUs
    (cylfmm_partition_fields, host-only: no device needed).  Returns (part int32 [n_fld],
    estimated flops per part float64 [n_parts])."""
    a = [np.ascontiguousarray(v, dtype=np.float64) for v in (src_r, src_z, fld_r, fld_z)]
    part = np.empty(a[2].shape[0], dtype=np.int32)
    cost = np.empty(n_parts, dtype=np.float64)
    prm = Params(cfg.n_modes, cfg.order, cfg.depth, cfg.truncation, cfg.miller,
                 int(bool(cfg.exclude_coincident)), float(cfg.z0), float(cfg.L), cfg.mode_chunk,
                 cfg.order_local, cfg.adaptive_leaf)
    p = lambda x: ctypes.c_void_p(x.ctypes.data) if x.size else ctypes.c_void_p(0)  # noqa: E731
    _check(lib().cylfmm_partition_fields(p(a[0]), p(a[1]), a[0].shape[0], p(a[2]), p(a[3]),
                                         a[2].shape[0], ctypes.byref(prm), int(n_parts), p(part),
                                         p(cost)), "cylfmm_partition_fields")
    return part, cost


def select_params(src_r, src_z, fld_r, fld_z, n_modes: int, tol: float, L: float = 1.0,
                  z0: float = 0.0, depth_min: int = 2, depth_max: int = 11):
    """Error-driven order and depth (cylfmm_select_params, host-only): the smallest order whose
    modelled error CYLFMM_EPS_C 10^(-0.4 p) meets tol (R#25), and the depth in
    [depth_min, depth_max] minimising the modelled solve time.  Returns (FMMConfig, info) with
    info = {"eps_model", "depths", "near_pairs", "s2l_pairs", "est_ms"} (per-depth arrays)."""
    a = [np.ascontiguousarray(v, dtype=np.float64) for v in (src_r, src_z, fld_r, fld_z)]
    nd = max(depth_max - depth_min + 1, 0)
    near = np.zeros(nd, dtype=np.int64)
    s2l = np.zeros(nd, dtype=np.int64)
    ms = np.zeros(nd, dtype=np.float64)
    eps = ctypes.c_double(0.0)
    prm = Params(int(n_modes), 1, 2, TRUNC_DOUBLE, MILLER_ACCURATE, 1, float(z0), float(L), 0, 0)
    p = lambda x: ctypes.c_void_p(x.ctypes.data) if x.size else ctypes.c_void_p(0)  # noqa: E731
    _check(lib().cylfmm_select_params(p(a[0]), p(a[1]), a[0].shape[0], p(a[2]), p(a[3]),
                                      a[2].shape[0], float(tol), int(depth_min), int(depth_max),
                                      ctypes.byref(prm), p(near), p(s2l), p(ms),
                                      ctypes.byref(eps)), "cylfmm_select_params")
    cfg = FMMConfig(n_modes=int(n_modes), order=prm.order, depth=prm.depth, L=float(L), z0=float(z0))
    info = {"eps_model": eps.value, "depths": np.arange(depth_min, depth_max + 1),
            "near_pairs": near, "s2l_pairs": s2l, "est_ms": ms}
    return cfg, info
