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
