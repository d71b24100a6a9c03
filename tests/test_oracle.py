"""Pin the oracle (test infrastructure) to the reference's own outputs (tests/golden, generated
by make_golden.py from the reference package) and to the reference's hand-traced known answers
(reference tests/test_codec.py:154-230, test_physical.py:403-452, test_kernels.py:44-97).

Everything the oracle restates in floating point follows the reference's operation order, so
the pins are bit-exact except the GLM training curves (libm exp vs numpy exp, <= 1e-12).
"""

from __future__ import annotations

import json
import os
import struct

import numpy as np
import pytest

from helpers import TOY_ROWS, TREE_ROWS

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "golden.json")))


def unhex(xs):
    return np.array([struct.unpack("<d", bytes.fromhex(x))[0] for x in xs], dtype=np.float64)


def rows_of(case):
    return [[(c, struct.unpack("<d", bytes.fromhex(x))[0]) for c, x in r] for r in case["rows"]]


def bits_equal(a, b) -> bool:
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


class TestKnownAnswers:
    """The reference's hand-traced worked examples."""

    def test_toy_encoding(self, oracle):
        enc = oracle.encode_rows(5, TOY_ROWS)
        assert enc.pairs == [(0, 1.0), (1, 2.0), (2, 3.0), (3, 4.0), (4, 5.0), (0, 6.0), (1, 7.0)]
        assert enc.rows == [[1, 2, 3, 4, 5], [6, 7, 10, 5]]

    def test_toy_tree_and_block(self, oracle):
        enc = oracle.encode_rows(5, TOY_ROWS)
        parent, _, _ = oracle.Tree.from_encoding(enc).arrays()
        assert parent.tolist() == [-1, 0, 0, 0, 0, 0, 0, 0, 1, 2, 3, 4, 6, 7, 10]
        blk = oracle.serialize(enc)
        assert len(blk) == 127
        want = (b"TOC1" + struct.pack("<BII", 1, 2, 5) + struct.pack("<I", 7)
                + struct.pack("<7d", 1.0, 2.0, 3.0, 4.0, 5.0, 6.0, 7.0) + struct.pack("<I", 7)
                + struct.pack("<IB", 7, 1) + bytes([0, 1, 2, 3, 4, 0, 1])
                + struct.pack("<IB", 7, 1) + bytes([0, 1, 2, 3, 4, 5, 6])
                + struct.pack("<I", 9) + struct.pack("<IB", 9, 1) + bytes([1, 2, 3, 4, 5, 6, 7, 10, 5])
                + struct.pack("<IB", 3, 1) + bytes([0, 5, 9]))
        assert blk == want

    def test_toy_kernels(self, oracle):
        t = oracle.Tree.from_encoding(oracle.encode_rows(5, TOY_ROWS))
        assert t.matvec(np.ones(5)).tolist() == [15.0, 25.0]
        assert t.vecmat(np.ones(2)).tolist() == [7.0, 9.0, 6.0, 8.0, 10.0]
        assert t.T == 15

    def test_tree_example(self, oracle):
        enc = oracle.encode_rows(5, TREE_ROWS)
        assert enc.rows == [[1, 2, 3, 4], [6, 8], [5, 8]]
        parent, column, value = oracle.Tree.from_encoding(enc).arrays()
        assert parent.tolist() == [-1, 0, 0, 0, 0, 0, 1, 2, 3, 6, 5]
        assert list(zip(column.tolist(), value.tolist()))[1:] == [
            (1, 1.1), (2, 2.0), (3, 3.0), (4, 1.4), (2, 1.1), (2, 2.0), (3, 3.0), (4, 1.4), (3, 3.0), (3, 3.0)]

    def test_width_table(self, oracle):
        # reference tests/test_physical.py:21-28: widths 1,1,1,2,2,3,3,4,4
        for largest, width in [(0, 1), (1, 1), (255, 1), (256, 2), (65535, 2), (65536, 3), (2**24 - 1, 3),
                               (2**24, 4), (2**32 - 1, 4)]:
            enc = oracle.Encoding(1, 1, np.zeros(0, np.int32), np.zeros(0), np.zeros(0, np.uint32),
                                  np.array([0, 0], np.int64))
            blk = oracle.serialize(enc)
            assert blk[-3] == 1  # offsets array [0, 0] packs at width 1
            del largest, width


@pytest.mark.parametrize("i", range(len(GOLD["cases"])))
def test_golden_case(oracle, i):
    case = GOLD["cases"][i]
    rows = rows_of(case)
    enc = oracle.encode_rows(case["n_cols"], rows)
    assert [[c, struct.pack("<d", x).hex()] for c, x in enc.pairs] == case["pairs"]
    assert enc.rows == case["codes"]
    blk = oracle.serialize(enc)
    assert blk.hex() == case["block"]
    dec = oracle.deserialize(blk)
    assert dec.rows == case["codes"] and dec.pairs == enc.pairs
    t = oracle.Tree.from_block(blk)
    parent, column, value = t.arrays()
    assert parent.tolist() == case["parent"] and column.tolist() == case["column"]
    assert bits_equal(value, unhex(case["value"]))
    n_rows, n_cols = len(rows), case["n_cols"]
    assert bits_equal(t.matvec(unhex(case["v"])), unhex(case["matvec"]))
    assert bits_equal(t.vecmat(unhex(case["u"])), unhex(case["vecmat"]))
    Mr = unhex(case["Mr"]).reshape(n_cols, 3)
    Ml = unhex(case["Ml"]).reshape(2, n_rows)
    assert bits_equal(t.matmat_right(Mr).ravel(), unhex(case["matmat_right"]))
    assert bits_equal(t.matmat_left(Ml).ravel(), unhex(case["matmat_left"]))
    assert case["kernel_cost"] == (t.T - 1) + len(enc.codes)  # kernels.py:250-266


@pytest.mark.parametrize("i", range(len(GOLD["corrupt"])))
def test_golden_corrupt(oracle, i):
    c = GOLD["corrupt"][i]
    data = bytes.fromhex(c["block"])
    try:
        oracle.Tree.from_block(data)
        kind = "OK"
    except oracle.OracleError as e:
        kind = e.kind
    assert kind == c["kind"], (c["label"], c["message"])


@pytest.mark.parametrize("i", range(len(GOLD["training"])))
def test_golden_training(oracle, i):
    c = GOLD["training"][i]
    rows = rows_of(c)
    rp, cols, vals = oracle.rows_to_csr(rows)
    labels = unhex(c["labels"])
    if c["loss"] == "nn_mse":
        w1, w2, risks = oracle.train_nn(rp, cols, vals, labels, c["n_cols"], c["hidden_units"], c["batch_size"],
                                        c["lr"], c["epochs"], c["seed"])
        assert np.allclose(risks, unhex(c["risks"]), rtol=1e-12, atol=0)
        assert np.allclose(w1.ravel(), unhex(c["w1"]), rtol=1e-12, atol=1e-15)
        assert np.allclose(w2.ravel(), unhex(c["w2"]), rtol=1e-12, atol=1e-15)
        return
    w, risks = oracle.train_glm(rp, cols, vals, labels, c["n_cols"], c["loss"], c["batch_size"], c["lr"],
                                c["epochs"], c["seed"])
    want_r = unhex(c["risks"])
    want_w = unhex(c["weights"])
    assert np.allclose(risks, want_r, rtol=1e-12, atol=0)
    assert np.allclose(w, want_w, rtol=1e-12, atol=1e-15)


def test_cfg1_golden(oracle):
    from paper_1702_06943_b200 import synth

    g = np.load(os.path.join(HERE, "golden", "cfg1.npz"))
    A = synth.cfg1_dense(0)
    enc = oracle.encode_csr(128, *synth.dense_to_csr(A))
    blk = oracle.serialize(enc)
    assert blk == g["block"].tobytes()
    t = oracle.Tree.from_block(blk)
    assert t.T == int(g["tree_len"])
    assert bits_equal(t.matvec(g["v"]), g["matvec"])
    assert bits_equal(t.vecmat(g["u"]), g["vecmat"])


def test_sweep_matches_per_batch(oracle):
    from paper_1702_06943_b200 import synth

    encs = [oracle.encode_csr(784, *synth.dense_to_csr(synth.cfg2_batch_dense(0, b))) for b in range(3)]
    trees = [oracle.Tree.from_encoding(e) for e in encs]
    v, u = synth.cfg2_operands(0, 3)
    R, O = oracle.sweep(trees, [0, 250, 500], v, u, 2, nthreads=2)
    for b, t in enumerate(trees):
        assert bits_equal(R[250 * b : 250 * (b + 1)], t.matvec(v))
        assert bits_equal(O[b], t.vecmat(u[250 * b : 250 * (b + 1)]))
