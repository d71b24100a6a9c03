"""ctypes binding of the product's native library (libtoc_b200.so, built in-tree for sm_100a).

The library exports the C ABI declared in include/toc_b200.h.  There is no fallback: if the
library is missing or no CUDA device is present, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# TOC_LIB (tests only): load another build of the library, e.g. the bounds-checked one
# (libtoc_b200_checked.so, `make checked`).
LIB_PATH = os.environ.get("TOC_LIB") or os.path.join(_HERE, "libtoc_b200.so")

TOC_OK, TOC_E_BAD_MAGIC, TOC_E_BAD_VERSION, TOC_E_TRUNCATED, TOC_E_FORMAT = 0, 1, 2, 3, 4
TOC_E_CORRUPT, TOC_E_INPUT, TOC_E_CUDA, TOC_E_ARG = 5, 6, 7, 8
TOC_MATVEC, TOC_VECMAT = 1, 2

(D_NONE, D_WIDTH, D_PAIR_COUNT, D_CODE_COUNT, D_TRAILING, D_OFFS_COUNT, D_OFFS_SPAN, D_OFFS_MONO,
 D_REF_RANGE, D_PAIR_COL, D_PAIR_VAL, D_CODE_LT1, D_UNDEF, D_MAGIC, D_VERSION, D_TRUNC) = range(16)

# numpy mirror of TocBlockMeta (include/toc_b200.h), 68 bytes
META_DTYPE = np.dtype([
    ("n_rows", "<u4"), ("n_cols", "<u4"), ("n_uniques", "<u4"), ("n_pairs", "<u4"),
    ("n_codes", "<u4"), ("n_derived", "<u4"), ("off_uniques", "<u4"), ("off_cols", "<u4"),
    ("off_refs", "<u4"), ("off_codes", "<u4"), ("off_offsets", "<u4"),
    ("w_cols", "u1"), ("w_refs", "u1"), ("w_codes", "u1"), ("w_offsets", "u1"),
    ("status", "<i4"), ("corrupt", "<i4"), ("detail", "<u4"), ("detail_a", "<u4"), ("detail_b", "<u4"),
])
assert META_DTYPE.itemsize == 68


class TocPlan(ctypes.Structure):
    _fields_ = [("threads", ctypes.c_int32), ("ctas", ctypes.c_int32), ("smem_bytes", ctypes.c_int32),
                ("wide", ctypes.c_int32), ("vec_in_smem", ctypes.c_int32), ("n_cols", ctypes.c_int32),
                ("max_rows", ctypes.c_int32), ("global_tables", ctypes.c_int32),
                ("scratch_bytes", ctypes.c_int64)]


class TocSweepChunk(ctypes.Structure):
    _fields_ = [("byte_lo", ctypes.c_int64), ("byte_hi", ctypes.c_int64), ("d_arena", ctypes.c_void_p),
                ("d_block_off", ctypes.c_void_p), ("d_block_len", ctypes.c_void_p), ("d_meta", ctypes.c_void_p),
                ("d_row_base", ctypes.c_void_p), ("d_scratch", ctypes.c_void_p), ("n_blocks", ctypes.c_int64),
                ("b0", ctypes.c_int64), ("row0", ctypes.c_int64), ("n_rows", ctypes.c_int64), ("plan", TocPlan),
                ("ev_upload", ctypes.c_void_p), ("ev_operands", ctypes.c_void_p), ("ev_done", ctypes.c_void_p)]


class NativeError(RuntimeError):
    """A native call failed for a reason that is not a data error (CUDA error, bad argument)."""


_lib = None
P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64


def lib():
    """Load libtoc_b200.so.  Raises ImportError when it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    L.toc_version.restype = ctypes.c_char_p
    L.toc_sizeof_meta.restype = ctypes.c_int
    L.toc_sizeof_plan.restype = ctypes.c_int
    L.toc_device_info.argtypes = [P, P, P]
    L.toc_index_blocks.argtypes = [P, P, P, I64, P, P]
    L.toc_plan.argtypes = [P, I64, I32, ctypes.POINTER(TocPlan)]
    L.toc_linalg.argtypes = [P, P, P, P, I64, ctypes.POINTER(TocPlan), I32, P, P, P, P, P, P]
    L.toc_tree_offsets.argtypes = [P, I64, I32, P]
    L.toc_build_trees.argtypes = [P, P, P, I64, ctypes.POINTER(TocPlan), P, P, P, P]
    L.toc_linalg_trees.argtypes = [P, P, P, P, I64, ctypes.POINTER(TocPlan), I32, P, P, P, P, P, P, P, P]
    L.toc_matmat.argtypes = [P, P, P, P, P, I64, I32, I32, I32, P, P, P, I64, P]
    L.toc_matmat_scratch.argtypes = [P, I64, I32, I32, I32, ctypes.POINTER(ctypes.c_int64)]
    L.toc_decode_counts.argtypes = [P, P, P, P, I64, ctypes.POINTER(TocPlan), P, P, P]
    L.toc_decode_rows.argtypes = [P, P, P, P, I64, ctypes.POINTER(TocPlan), P, P, P, P, P]
    L.toc_sweep_upload.argtypes = [P, P, P, I64, I64, P]
    L.toc_sweep_events.argtypes = [P, I64]
    L.toc_exact_matvec.argtypes = [P, P, P, P, P, I32, P, P, I32, P, P, P, P]
    L.toc_exact_vecmat.argtypes = [P, P, I32, P, P, I32, P, P, P, P, P, P, I32, P, P, P, P]
    L.toc_sweep_events_free.argtypes = [P, I64]
    L.toc_sweep_operands.argtypes = [P, I64, I32, P, P, P, P, P]
    L.toc_sweep_compute.argtypes = [P, I64, I32, P, P, P, P, P, P, P, P, P]
    L.toc_linalg32.argtypes = [P, P, P, P, I64, ctypes.POINTER(TocPlan), I32, P, P, P, P, P, P, P]
    L.toc_matcache_offsets.argtypes = [P, I64, P]
    L.toc_matcache_build.argtypes = [P, P, P, I64, ctypes.POINTER(TocPlan), P, P, P, P]
    L.toc_matcache_right.argtypes = [P, P, P, I64, I64, I32, I32, P, P, P]
    L.toc_matcache_left_scratch.argtypes = [P, I32, I32, ctypes.POINTER(ctypes.c_int64)]
    L.toc_matcache_left.argtypes = [P, P, I32, I32, P, P, P, I64, P]
    L.toc_mlp_scratch.argtypes = [I32, I32, I32, I32, ctypes.POINTER(ctypes.c_int64)]
    L.toc_mlpcache_offsets.argtypes = [P, I64, P]
    L.toc_mlpcache_build.argtypes = [P, P, P, I64, ctypes.POINTER(TocPlan), P, P, P, P]
    L.toc_mlp_epoch.argtypes = [P, P, P, P, P, P, I64, I32, I32, I32, P, P, P, P, P, ctypes.c_double, I32, P, I64,
                                P]
    L.toc_mlp_risk.argtypes = [P, P, P, P, P, P, I64, I32, I32, I32, P, P, P, P, P, I32, P, P, I64, P]
    L.toc_mlp_set_pdl.argtypes = [I32]
    L.toc_mlp_step_grad.argtypes = [P, P, P, P, P, P, I64, I64, I32, I32, I32, P, P, P, P, P, I32, P, P, I64, P]
    L.toc_levels_build.restype = P
    L.toc_levels_build.argtypes = [P, P, P, I64, I32]
    L.toc_levels_info.argtypes = [P, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int32),
                                  ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]
    L.toc_levels_copy.argtypes = [P, P, P]
    L.toc_levels_free.restype = None
    L.toc_levels_free.argtypes = [P]
    L.toc_levels_smem.restype = I64
    L.toc_levels_smem.argtypes = [I32, I32, I32, I32, I32]
    L.toc_linalg_levels.argtypes = [P, I64, I32, I32, I32, I32, I32, P, P, P, P, P, P, P]
    L.toc_linalg_levels32.argtypes = [P, I64, I32, I32, I32, I32, I32, P, P, P, P, P, P, P]
    L.toc_levels_set_trace.argtypes = [P]
    L.toc_tree_arrays.argtypes = [P, P, P, I64, ctypes.POINTER(TocPlan), P, P, P, P, P, P, P, P]
    L.toc_dense_matvec.argtypes = [P, I64, I64, P, P, P]
    L.toc_dense_vecmat.argtypes = [P, P, I64, I64, P, P]
    L.toc_dense_matmat.argtypes = [P, P, I64, I64, I64, P, P]
    L.toc_csr_matvec.argtypes = [P, P, P, I64, P, P, P]
    L.toc_csc_vecmat.argtypes = [P, P, P, I64, P, P, P]
    L.toc_csr_matmat_right.argtypes = [P, P, P, I64, P, I64, P, P]
    L.toc_csc_matmat_left.argtypes = [P, P, P, I64, P, I64, I64, P, P]
    for name in EXPORTS:
        getattr(L, name).restype = getattr(L, name).restype or ctypes.c_int
    if (L.toc_sizeof_meta() != META_DTYPE.itemsize or L.toc_sizeof_plan() != ctypes.sizeof(TocPlan)
            or L.toc_sizeof_sweep_chunk() != ctypes.sizeof(TocSweepChunk)):
        raise ImportError("libtoc_b200.so ABI mismatch with the Python binding")
    _lib = L
    return L


# Every symbol include/toc_b200.h declares (tests check the library exports all of them).
EXPORTS = ["toc_index_blocks", "toc_plan", "toc_linalg", "toc_linalg_trees", "toc_build_trees", "toc_tree_offsets",
           "toc_version", "toc_device_info", "toc_sizeof_meta", "toc_sizeof_plan"]


def check(rc: int, what: str) -> None:
    if rc != TOC_OK:
        raise NativeError(f"{what} failed with status {rc}")


def device_info():
    """(sm_count, max dynamic shared memory per CTA, L2 bytes) of the current device."""
    sm, smem, l2 = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int64()
    check(lib().toc_device_info(ctypes.byref(sm), ctypes.byref(smem), ctypes.byref(l2)), "toc_device_info")
    return sm.value, smem.value, l2.value


def require_cuda():
    """The compute path needs a CUDA device; fail loudly instead of falling back."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_1702_06943_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    return torch


def stream_handle(torch_mod=None):
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
