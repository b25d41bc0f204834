"""Host-side checks of the C-ABI boundary (no GPU needed): libcylfmm.so builds for sm_100a,
loads, exports every function include/cylfmm.h declares, and the product path fails loudly
(no CPU fallback) when no CUDA device is present."""
import ctypes
import os
import shutil

import pytest

from paper_2301_01179_b200 import cylfmm
from paper_2301_01179_b200.build import LIB, build


@pytest.fixture(scope="module")
def libso():
    if not os.path.exists(LIB):
        if shutil.which(os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")) is None:
            pytest.skip("nvcc not available and libcylfmm.so not built")
        build()
    return ctypes.CDLL(LIB)


def test_header_declares_the_boundary():
    names = set(cylfmm.header_functions())
    for f in ("cylfmm_direct", "cylfmm_direct_enqueue", "cylfmm_direct_workspace_bytes", "cylfmm_plan_create", "cylfmm_fmm_solve", "cylfmm_fmm_solve_host",
              "cylfmm_plan_sync", "cylfmm_plan_destroy", "cylfmm_greens_batch",
              "cylfmm_tensor_batch", "cylfmm_tree_sort", "cylfmm_status_string",
              "cylfmm_last_error", "cylfmm_version"):
        assert f in names


def test_library_exports_every_header_symbol(libso):
    for f in cylfmm.header_functions():
        assert hasattr(libso, f), f


def test_library_is_sm100a(libso):
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {LIB} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out


def test_host_only_entry_points(libso):
    L = cylfmm.lib()
    assert L.cylfmm_status_string(0) == b"ok"
    assert b"domain" in L.cylfmm_status_string(2)
    assert b"sm_100a" in L.cylfmm_version()


def test_invalid_arguments_rejected_before_any_work(libso):
    L = cylfmm.lib()
    # negative sizes / bad mode counts are argument errors, detected on the host
    st = L.cylfmm_direct(None, None, None, -1, None, None, 0, 3, 0, 1, None, None)
    assert st == cylfmm.EINVAL
    st = L.cylfmm_direct_enqueue(None, None, None, 4, None, None, 4, 3, 0, 1, None, None, 0, None)
    assert st == cylfmm.EINVAL
    assert L.cylfmm_direct_workspace_bytes(4, 4, 0, None) == cylfmm.EINVAL
    st = L.cylfmm_greens_batch(None, None, None, 4, 0, 0, None, None)
    assert st == cylfmm.EINVAL
    prm = cylfmm.Params(3, 0, 4, 0, 0, 1, 0.0, 1.0, 0)   # order 0 is invalid
    h = ctypes.c_void_p()
    assert L.cylfmm_plan_create(ctypes.byref(h), ctypes.byref(prm)) == cylfmm.EINVAL
    assert b"bad parameters" in L.cylfmm_last_error()


def test_no_cpu_fallback_without_gpu(libso):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        cylfmm.direct([0.5], [0.1], [[1.0 + 0j]], [0.7], [0.2])
    L = cylfmm.lib()
    prm = cylfmm.Params(3, 4, 4, 0, 0, 1, 0.0, 1.0, 0)
    h = ctypes.c_void_p()
    assert L.cylfmm_plan_create(ctypes.byref(h), ctypes.byref(prm)) == cylfmm.ECUDA
