"""GPU parity for A.M and M.A on compressed batches (reference kernels.py:177-234) vs the
reference's golden outputs and the oracle, within 1e-9 relative."""

from __future__ import annotations

import json
import os
import struct

import numpy as np
import pytest

from conftest import max_rel_err, within_rel

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "golden.json")))
REL = 1e-9


def unhex(xs):
    return np.array([struct.unpack("<d", bytes.fromhex(x))[0] for x in xs], dtype=np.float64)


@pytest.mark.parametrize("i", range(len(GOLD["cases"])))
def test_matmat_golden(i):
    from paper_1702_06943_b200.kernels import CompressedMatrix, OpCounter, kernel_cost, matmat_left, matmat_right
    from paper_1702_06943_b200.matrix import DenseMatrix, SparseRowMatrix

    case = GOLD["cases"][i]
    rows = [[(c, struct.unpack("<d", bytes.fromhex(x))[0]) for c, x in r] for r in case["rows"]]
    n_rows, n_cols = len(rows), case["n_cols"]
    cm = CompressedMatrix.from_sparse(SparseRowMatrix(n_cols, rows))
    Mr = unhex(case["Mr"]).reshape(n_cols, 3)
    Ml = unhex(case["Ml"]).reshape(2, n_rows)
    counter = OpCounter()
    got = matmat_right(cm, DenseMatrix(Mr), counter).values
    assert within_rel(got.ravel(), unhex(case["matmat_right"]), REL), max_rel_err(got.ravel(), unhex(case["matmat_right"]))
    assert counter.multiply_adds == kernel_cost(cm, "matmat_right", 3)
    counter = OpCounter()
    got = matmat_left(DenseMatrix(Ml), cm, counter).values
    assert within_rel(got.ravel(), unhex(case["matmat_left"]), REL), max_rel_err(got.ravel(), unhex(case["matmat_left"]))
    assert counter.multiply_adds == kernel_cost(cm, "matmat_left", 2)


@pytest.mark.parametrize("cached", [False, True])
@pytest.mark.parametrize("p", [1, 200, 300])
def test_matmat_batches_vs_oracle(oracle, p, cached):
    """Config-1 style batches widened to 784 columns (the config-5 input recipe), p up to 300;
    rebuilt tables (toc_matmat) and the node-record cache (toc_matcache_*), whole arena and per
    batch (the MLP step's call)."""
    import torch

    from paper_1702_06943_b200 import synth
    from paper_1702_06943_b200.codec import compress_csr

    rng = np.random.default_rng(p)
    blocks = [synth.dense_to_csr(synth.cfg1_dense(s, n_rows=250, n_cols=784)) for s in range(3)]
    rp = np.concatenate([[0]] + [b[0][1:] + sum(int(x[0][-1]) for x in blocks[:k]) for k, b in enumerate(blocks)])
    c = np.concatenate([b[1] for b in blocks])
    v = np.concatenate([b[2] for b in blocks])
    arena = compress_csr(784, rp, c, v, np.array([0, 250, 500, 750]))
    if cached:
        arena.build_matcache()
    M = rng.standard_normal((784, p))
    Mt = rng.standard_normal((750, p))  # rows of M^T are batch rows
    Md, Mtd = torch.from_numpy(M).cuda(), torch.from_numpy(Mt).cuda()
    R = arena.matmat(0, Md, p).cpu().numpy()
    L = arena.matmat(1, Mtd, p).cpu().numpy()
    for b, (brp, bc, bv) in enumerate(blocks):
        t = oracle.Tree.from_encoding(oracle.encode_csr(784, brp, bc, bv))
        want_r = t.matmat_right(M)
        assert within_rel(R[250 * b : 250 * (b + 1)], want_r, REL), max_rel_err(R[250 * b : 250 * (b + 1)], want_r)
        want_l = t.matmat_left(np.ascontiguousarray(Mt[250 * b : 250 * (b + 1)].T))
        assert within_rel(L[b], want_l, REL), max_rel_err(L[b], want_l)
        rb = arena.matmat(0, Md, p, batch=b).cpu().numpy()
        assert within_rel(rb, want_r, REL), max_rel_err(rb, want_r)
        lb = arena.matmat(1, Mtd[250 * b : 250 * (b + 1)].contiguous(), p, batch=b)[0].cpu().numpy()
        assert within_rel(lb, want_l, REL), max_rel_err(lb, want_l)


def test_matmat_dimension_errors():
    from paper_1702_06943_b200.kernels import CompressedMatrix, matmat_left, matmat_right
    from paper_1702_06943_b200.matrix import DenseMatrix, SparseRowMatrix

    from helpers import TOY_ROWS

    cm = CompressedMatrix.from_sparse(SparseRowMatrix(5, TOY_ROWS))
    with pytest.raises(ValueError, match="inner dimensions"):
        matmat_right(cm, DenseMatrix([[1.0], [2.0]]))
    with pytest.raises(ValueError, match="inner dimensions"):
        matmat_left(DenseMatrix([[1.0, 2.0, 3.0]]), cm)
    out = matmat_right(cm, DenseMatrix(np.eye(5)))  # identity recovers the matrix (test_kernels.py:89-91)
    assert np.array_equal(out.values, np.array([[1, 2, 3, 4, 5], [6, 7, 3, 4, 5]], dtype=float))


def test_matcache_wide_ragged(oracle):
    """Node-record cache on a > 65536-node tree, an empty row and a short batch."""
    import torch

    from helpers import random_alphabet_rows

    from paper_1702_06943_b200.arena import BlockArena

    rng = np.random.default_rng(31)
    base = random_alphabet_rows(rng, 30, 400, 0.9, 64)
    wide = [base[i % 30] if i % 3 else random_alphabet_rows(rng, 1, 400, 0.9, 64)[0] for i in range(600)]
    small = random_alphabet_rows(rng, 9, 400, 0.3) + [[]]
    encs = [oracle.encode_rows(400, wide), oracle.encode_rows(400, small)]
    assert encs[0].tree_length() > 65536
    arena = BlockArena.from_bytes([oracle.serialize(e) for e in encs]).build_matcache()
    M = rng.standard_normal((400, 40))
    Mt = rng.standard_normal((610, 40))
    R = arena.matmat(0, torch.from_numpy(M).cuda(), 40).cpu().numpy()
    L = arena.matmat(1, torch.from_numpy(Mt).cuda(), 40).cpu().numpy()
    base_r = 0
    for b, e in enumerate(encs):
        t = oracle.Tree.from_encoding(e)
        want_r = t.matmat_right(M)
        assert within_rel(R[base_r : base_r + e.n_rows], want_r, REL), max_rel_err(R[base_r : base_r + e.n_rows], want_r)
        want_l = t.matmat_left(np.ascontiguousarray(Mt[base_r : base_r + e.n_rows].T))
        assert within_rel(L[b], want_l, REL), max_rel_err(L[b], want_l)
        base_r += e.n_rows
