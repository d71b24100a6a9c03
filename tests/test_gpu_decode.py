"""GPU parity: device decode (reference codec.py:262-292) and the DecodeTree arrays
(codec.py:194-259) -- bit-exact against the reference's golden fixtures (tests/golden) and the
oracle; decode is lossless on the configs' batches; corrupt encodings raise the reference's
CorruptEncodingError; CompressedMatrix.tree keeps the once-only, lazy semantics
(reference tests/test_kernels.py:250-276)."""

from __future__ import annotations

import json
import os
import struct
import threading

import numpy as np
import pytest

from helpers import TOY_ROWS, random_alphabet_rows

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "golden.json")))


def rows_of(case):
    return [[(c, struct.unpack("<d", bytes.fromhex(x))[0]) for c, x in r] for r in case["rows"]]


def unhex(xs):
    return np.array([struct.unpack("<d", bytes.fromhex(x))[0] for x in xs], dtype=np.float64)


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def first_pairs(parent, column, value):
    """first_col / first_val of every node: follow parent links to the first layer (codec.py:230-251)."""
    fc, fv = [], []
    for x in range(len(parent)):
        if x == 0:
            fc.append(-1)
            fv.append(0.0)
            continue
        y = x
        while parent[y] != 0:
            y = parent[y]
        fc.append(column[y])
        fv.append(value[y])
    return fc, fv


@pytest.mark.parametrize("i", range(len(GOLD["cases"])))
def test_tree_and_decode_match_reference(i):
    from paper_1702_06943_b200.codec import build_prefix_tree, decode, encode
    from paper_1702_06943_b200.matrix import SparseRowMatrix

    case = GOLD["cases"][i]
    rows = rows_of(case)
    enc = encode(SparseRowMatrix(case["n_cols"], rows))
    t = build_prefix_tree(enc)
    assert t.parent == case["parent"] and t.column == case["column"]
    assert np.array_equal(bits(t.value), bits(unhex(case["value"])))
    fc, fv = first_pairs(t.parent, t.column, t.value)
    assert t.first_col == fc and np.array_equal(bits(t.first_val), bits(fv))
    assert len(t) == 1 + len(enc.pairs) + enc.derived_node_count()
    got = decode(enc).rows
    assert len(got) == len(rows)
    for g, w in zip(got, rows):
        assert [c for c, _ in g] == [c for c, _ in w]
        assert np.array_equal(bits([v for _, v in g]), bits([v for _, v in w]))


def _arena_roundtrip(oracle, n_cols, row_ptr, cols, vals, batch_row):
    from paper_1702_06943_b200.codec import compress_csr

    arena = compress_csr(n_cols, row_ptr, cols, vals, batch_row)
    rp, c, v = arena.decode()
    assert np.array_equal(rp.cpu().numpy(), row_ptr)
    assert np.array_equal(c.cpu().numpy(), cols)
    assert np.array_equal(bits(v.cpu().numpy()), bits(vals))
    return arena


def test_decode_cfg1_bit_exact(oracle):
    from paper_1702_06943_b200 import synth

    rp, c, v = synth.dense_to_csr(synth.cfg1_dense(0))
    arena = _arena_roundtrip(oracle, 128, rp, c, v, np.array([0, 256], np.int64))
    t = arena.decode_trees()[0]
    parent, column, value = oracle.Tree.from_encoding(oracle.encode_csr(128, rp, c, v)).arrays()
    assert t.parent == parent.tolist() and t.column == column.tolist()
    assert np.array_equal(bits(t.value), bits(value))


def test_decode_cfg2_many_batches(oracle):
    from paper_1702_06943_b200 import synth

    dense = [synth.cfg2_batch_dense(0, b) for b in range(6)]
    parts = [synth.dense_to_csr(d) for d in dense]
    rp = np.concatenate([[0], np.cumsum(np.concatenate([np.diff(p[0]) for p in parts]))]).astype(np.int64)
    c = np.concatenate([p[1] for p in parts])
    v = np.concatenate([p[2] for p in parts])
    _arena_roundtrip(oracle, 784, rp, c, v, np.arange(0, 1501, 250, dtype=np.int64))


def test_decode_ragged_empty_and_wide(oracle):
    """Empty rows, a short last batch, and a > 65536-node tree (32-bit ids, global tables)."""
    from paper_1702_06943_b200.arena import BlockArena

    rng = np.random.default_rng(7)
    rows = random_alphabet_rows(rng, 97, 50, 0.4) + [[]] * 3 + [[(49, 1.5)]]
    rp, c, v = oracle.rows_to_csr(rows, 50)
    _arena_roundtrip(oracle, 50, rp, c, v, np.array([0, 37, 74, 101], np.int64))
    base = random_alphabet_rows(rng, 30, 400, 0.9, 64)
    wide = [base[i % 30] if i % 3 else random_alphabet_rows(rng, 1, 400, 0.9, 64)[0] for i in range(600)]
    enc = oracle.encode_rows(400, wide)
    assert enc.tree_length() > 65536
    arena = BlockArena.from_bytes([oracle.serialize(enc)])
    rp2, c2, v2 = arena.decode()
    wrp, wc, wv = oracle.rows_to_csr(wide, 400)
    assert np.array_equal(rp2.cpu().numpy(), wrp) and np.array_equal(c2.cpu().numpy(), wc)
    assert np.array_equal(bits(v2.cpu().numpy()), bits(wv))
    t = arena.decode_trees()[0]
    parent, column, value = oracle.Tree.from_encoding(enc).arrays()
    assert t.parent == parent.tolist() and t.column == column.tolist()
    assert np.array_equal(bits(t.value), bits(value))


def test_corrupt_encoding_raises():
    from paper_1702_06943_b200.codec import LogicalEncoding, build_prefix_tree, decode
    from paper_1702_06943_b200.errors import CorruptEncodingError

    enc = LogicalEncoding(n_rows=1, n_cols=2, pairs=[(0, 1.0), (1, 2.0)], rows=[[1, 7]])
    with pytest.raises(CorruptEncodingError):
        build_prefix_tree(enc)
    with pytest.raises(CorruptEncodingError):
        decode(enc)


def test_compressed_matrix_tree_is_lazy_and_once(oracle):
    from paper_1702_06943_b200.kernels import CompressedMatrix
    from paper_1702_06943_b200.matrix import SparseRowMatrix

    cm = CompressedMatrix.from_sparse(SparseRowMatrix(5, TOY_ROWS))
    assert cm._tree is None
    assert cm.tree is cm.tree
    assert cm.tree.parent == [-1, 0, 0, 0, 0, 0, 0, 0, 1, 2, 3, 4, 6, 7, 10]  # test_codec.py toy tree
    assert cm.decode().rows == [list(r) for r in TOY_ROWS]

    cm2 = CompressedMatrix.from_sparse(SparseRowMatrix(5, TOY_ROWS))
    seen = []
    threads = [threading.Thread(target=lambda: seen.append(cm2.tree)) for _ in range(8)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert len(seen) == 8 and all(t is seen[0] for t in seen)


# ---- sparse-safe rewrites (reference kernels.py:87-112, tests/test_kernels.py:98-130) -------------
def _toy():
    from paper_1702_06943_b200.kernels import CompressedMatrix
    from paper_1702_06943_b200.matrix import SparseRowMatrix

    return CompressedMatrix.from_sparse(SparseRowMatrix(5, TOY_ROWS))


def test_scalar_multiply_scales_values():
    from paper_1702_06943_b200.kernels import scalar_multiply
    from paper_1702_06943_b200.matrix import SparseRowMatrix, sparse_to_dense

    cm = _toy()
    scaled = scalar_multiply(cm, 2.5)
    assert np.array_equal(sparse_to_dense(scaled.decode()).values, sparse_to_dense(SparseRowMatrix(5, TOY_ROWS)).values * 2.5)
    assert scaled.encoding.rows is cm.encoding.rows
    assert cm._tree is None and scaled._tree is None


def test_rewrites_match_host_serialization(oracle):
    """The device-rebuilt block equals serialize_block of the rewritten logical encoding, byte for byte
    (value index rebuilt: scaling by 0 collapses every unique into one)."""
    from paper_1702_06943_b200.kernels import CompressedMatrix, elementwise_power, scalar_multiply
    from paper_1702_06943_b200.matrix import SparseRowMatrix

    rng = np.random.default_rng(11)
    rows = random_alphabet_rows(rng, 120, 30, 0.5)
    cm = CompressedMatrix.from_sparse(SparseRowMatrix(30, rows))
    from paper_1702_06943_b200.physical import serialize_block

    for out in (scalar_multiply(cm, -1.75), scalar_multiply(cm, 0.0), elementwise_power(cm, 2.0),
                elementwise_power(cm, 3.0), elementwise_power(cm, -1.0)):
        enc = out.encoding
        oenc = oracle.Encoding(enc.n_rows, 30, np.array([c for c, _ in enc.pairs], np.int32),
                               np.array([v for _, v in enc.pairs], np.float64),
                               np.array([c for r in enc.rows for c in r], np.uint32),
                               np.concatenate([[0], np.cumsum([len(r) for r in enc.rows])]).astype(np.int64))
        got = bytes(out.arena.data[: int(out.arena.block_len[0])].cpu().numpy())
        assert got == oracle.serialize(oenc)
        assert got == serialize_block(enc)
        assert out._tree is None


def test_scale_by_zero_keeps_structure():
    from paper_1702_06943_b200.kernels import scalar_multiply

    cm = _toy()
    zeroed = scalar_multiply(cm, 0.0)
    assert all(v == 0.0 for _, v in zeroed.encoding.pairs)
    got = zeroed.decode()
    assert [[c for c, _ in r] for r in got.rows] == [[c for c, _ in r] for r in TOY_ROWS]
    assert all(v == 0.0 for r in got.rows for _, v in r)


def test_rewrite_rejects_non_finite():
    from paper_1702_06943_b200.kernels import elementwise_power, scalar_multiply

    cm = _toy()
    with pytest.raises(ValueError):
        scalar_multiply(cm, float("inf"))
    with pytest.raises(ValueError):
        scalar_multiply(cm, 1e308)  # overflows to inf
    neg = scalar_multiply(cm, -1.0)
    with pytest.raises(ValueError):
        elementwise_power(neg, 0.5)  # nan


def test_arena_rewrites_many_batches(oracle):
    """Arena-level rewrites (device map + rebuild) over config-2 batches: decode equals the mapped
    input bit for bit for multiply; within 2 ulp for pow."""
    from paper_1702_06943_b200 import synth
    from paper_1702_06943_b200.codec import compress_csr

    dense = [synth.cfg2_batch_dense(1, b) for b in range(4)]
    parts = [synth.dense_to_csr(d) for d in dense]
    rp = np.concatenate([[0], np.cumsum(np.concatenate([np.diff(p[0]) for p in parts]))]).astype(np.int64)
    c = np.concatenate([p[1] for p in parts])
    v = np.concatenate([p[2] for p in parts])
    arena = compress_csr(784, rp, c, v, np.arange(0, 1001, 250, dtype=np.int64))
    s = arena.scalar_multiply(-3.25)
    rp2, c2, v2 = s.decode()
    assert np.array_equal(c2.cpu().numpy(), c) and np.array_equal(bits(v2.cpu().numpy()), bits(v * -3.25))
    pw = arena.elementwise_power(2.0)
    _, _, v3 = pw.decode()
    assert np.array_equal(bits(v3.cpu().numpy()), bits(v * v))
    pw3 = arena.elementwise_power(1.5)
    _, _, v4 = pw3.decode()
    assert np.allclose(v4.cpu().numpy(), v ** 1.5, rtol=5e-16, atol=0)


def test_scalar_add_densifies():
    from paper_1702_06943_b200.kernels import scalar_add
    from paper_1702_06943_b200.matrix import SparseRowMatrix, sparse_to_dense

    got = scalar_add(_toy(), 0.5).values
    assert np.array_equal(got, sparse_to_dense(SparseRowMatrix(5, TOY_ROWS)).values + 0.5)
    with pytest.raises(ValueError):
        scalar_add(_toy(), float("nan"))
