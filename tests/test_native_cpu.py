"""CPU-side checks of the product's native library and host logic (no GPU needed): the in-tree
library loads, exports every symbol include/toc_b200.h declares, agrees on the struct layouts,
and the product package never imports the oracle."""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "toc_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int64_t|int|void\s*\*|void|const char\s*\*)\s*(toc_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_1702_06943_b200 import _native as N

    lib = ctypes.CDLL(N.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s


def test_abi_struct_sizes_and_binding():
    from paper_1702_06943_b200 import _native as N
    from paper_1702_06943_b200.codec import INFO_DTYPE

    L = N.lib()
    assert L.toc_sizeof_meta() == N.META_DTYPE.itemsize == 68
    assert L.toc_sizeof_plan() == ctypes.sizeof(N.TocPlan) == 40
    assert L.toc_sizeof_batch_info() == INFO_DTYPE.itemsize == 48
    assert L.toc_sizeof_sweep_chunk() == ctypes.sizeof(N.TocSweepChunk) == 160
    assert b"sm_100a" in L.toc_version()


def test_plan_is_host_only():
    """toc_plan works from host metadata without a device (B200 figures as defaults)."""
    from paper_1702_06943_b200 import _native as N

    meta = np.zeros(3, N.META_DTYPE)
    meta["n_rows"] = 250
    meta["n_cols"] = 784
    meta["n_pairs"] = [11308, 11680, 11333]
    meta["n_derived"] = [23985, 24481, 23705]
    meta["n_uniques"] = 255
    p = N.TocPlan()
    assert N.lib().toc_plan(meta.ctypes.data_as(ctypes.c_void_p), 3, 3, ctypes.byref(p)) == 0
    assert p.wide == 0 and p.global_tables == 0 and p.smem_bytes <= 232448
    assert p.ctas == 3 and p.threads == 1024


def test_encode_sizes_host_only():
    from paper_1702_06943_b200 import _native as N
    from paper_1702_06943_b200.codec import TocEncodeSizes, _bind

    eb = np.array([0, 100, 100, 5000], np.int64)
    s = TocEncodeSizes()
    assert _bind().toc_encode_sizes(3, eb.ctypes.data_as(ctypes.c_void_p), ctypes.byref(s)) == 0
    assert s.n_elems == 5000 and s.hash_slots >= 3 * 32 and s.work_bytes > 0


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1702_06943_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"(from|import)\s+oracle|liboracle|toc_oracle|oracle\.py|\bor_\w+\(", text), f


def test_compute_fails_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_1702_06943_b200.matrix import SparseRowMatrix
    from paper_1702_06943_b200 import codec

    with pytest.raises(RuntimeError, match="CUDA"):
        codec.encode(SparseRowMatrix(2, [[(0, 1.0)]]))


def test_matrix_containers_validate():
    from paper_1702_06943_b200.matrix import DenseMatrix, SparseRowMatrix, as_vector, dense_to_sparse, sparse_to_dense

    with pytest.raises(ValueError, match="strictly increasing"):
        SparseRowMatrix(3, [[(1, 1.0), (1, 2.0)]])
    with pytest.raises(ValueError, match="out of range"):
        SparseRowMatrix(3, [[(3, 1.0)]])
    with pytest.raises(ValueError, match="explicit zero"):
        SparseRowMatrix(3, [[(0, 0.0)]])
    with pytest.raises(ValueError, match="non-finite"):
        SparseRowMatrix(3, [[(0, float("nan"))]])
    with pytest.raises(ValueError, match="5"):
        as_vector([1.0] * 4, 5, "vector")
    s = SparseRowMatrix(4, [[(0, 1.5), (3, -2.0)], [], [(2, 7.0)]])
    assert s.rows == [[(0, 1.5), (3, -2.0)], [], [(2, 7.0)]]
    assert dense_to_sparse(sparse_to_dense(s)) == s
    assert s.take_rows([2, 0]).rows == [[(2, 7.0)], [(0, 1.5), (3, -2.0)]]
    with pytest.raises(ValueError, match="finite"):
        DenseMatrix([[float("inf")]])


def test_train_config_validation():
    from paper_1702_06943_b200.training import TrainConfig

    for kwargs, match in [(dict(loss_kind="absolute"), "loss_kind"), (dict(execution="gpu"), "execution"),
                          (dict(batch_size=0), "batch_size"), (dict(epochs=0), "epochs"),
                          (dict(learning_rate=0.0), "learning_rate"), (dict(learning_rate=float("nan")), "learning_rate"),
                          (dict(loss_kind="nn_mse", hidden_units=0), "hidden_units")]:
        base = dict(loss_kind="squared", batch_size=4, learning_rate=0.1, epochs=2)
        base.update(kwargs)
        with pytest.raises(ValueError, match=match):
            TrainConfig(**base)


def test_shuffle_matches_stdlib():
    import random

    from paper_1702_06943_b200.training import shuffle_order

    order = list(range(20))
    random.Random(7).shuffle(order)
    assert shuffle_order(20, 7).tolist() == order


def test_physical_host_helpers():
    import struct

    from paper_1702_06943_b200.physical import BlockFormatError, TruncatedBlockError, pack_ints, unpack_ints

    for largest, width in [(0, 1), (255, 1), (256, 2), (65535, 2), (65536, 3), (2**24, 4), (2**32 - 1, 4)]:
        assert pack_ints([largest])[4] == width
    assert pack_ints([]) == struct.pack("<IB", 0, 1)
    assert pack_ints([0x010203])[5:] == b"\x03\x02\x01"
    assert unpack_ints(b"junk" + pack_ints([7, 8]), 4) == ([7, 8], 4 + 5 + 2)
    with pytest.raises(ValueError, match="negative"):
        pack_ints([-1])
    with pytest.raises(ValueError, match="four bytes"):
        pack_ints([2**32])
    with pytest.raises(TruncatedBlockError, match="offset 5"):
        unpack_ints(pack_ints([1, 2, 3])[:-1])
    with pytest.raises(BlockFormatError, match="1..4"):
        unpack_ints(struct.pack("<IB", 1, 5) + b"\x00" * 5)
