"""GPU checks of the reference-API mirror beyond the compressed kernels: the device dense / CSR
baselines (bit for bit against the reference's ascending-order loops, restated here in plain
Python), the per-batch training API, execution="dense" | "csr" and empirical_risk."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import within_rel
from helpers import random_alphabet_rows

pytestmark = pytest.mark.gpu


def _loops(rows, n_cols, v, u, M, L):
    """matrix.py:164-279's accumulation orders, in Python floats (the reference's own arithmetic)."""
    n = len(rows)
    dense = [[0.0] * n_cols for _ in range(n)]
    for i, r in enumerate(rows):
        for c, x in r:
            dense[i][c] = x
    mv = []
    for row in dense:
        acc = 0.0
        for j, x in enumerate(row):
            acc += x * v[j]
        mv.append(acc)
    vm = []
    for j in range(n_cols):
        acc = 0.0
        for i in range(n):
            acc += u[i] * dense[i][j]
        vm.append(acc)
    csr_mv = []
    for r in rows:
        acc = 0.0
        for c, x in r:
            acc += x * v[c]
        csr_mv.append(acc)
    csr_vm = [0.0] * n_cols
    for i, r in enumerate(rows):
        for c, x in r:
            csr_vm[c] += u[i] * x
    p = len(M[0])
    right = [[0.0] * p for _ in range(n)]
    for i, r in enumerate(rows):
        for j in range(p):
            acc = 0.0
            for c, x in r:
                acc += x * M[c][j]
            right[i][j] = acc
    q = len(L)
    left = [[0.0] * n_cols for _ in range(q)]
    for i, r in enumerate(rows):
        for c, x in r:
            for k in range(q):
                left[k][c] += L[k][i] * x
    return dense, mv, vm, csr_mv, csr_vm, right, left


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_dense_and_csr_baselines_bit_exact(seed):
    from paper_1702_06943_b200 import matrix as Mx

    rng = np.random.default_rng(seed)
    n, m = int(rng.integers(1, 40)), int(rng.integers(1, 30))
    rows = random_alphabet_rows(rng, n, m, float(rng.uniform(0.1, 0.9)))
    v, u = rng.standard_normal(m).tolist(), rng.standard_normal(n).tolist()
    M, L = rng.standard_normal((m, 3)).tolist(), rng.standard_normal((2, n)).tolist()
    dense, mv, vm, cmv, cvm, right, left = _loops(rows, m, v, u, M, L)
    s = Mx.SparseRowMatrix(m, rows)
    D = Mx.DenseMatrix(dense)
    assert Mx.dense_matvec(D, v).tobytes() == np.array(mv).tobytes()
    assert Mx.dense_vecmat(u, D).tobytes() == np.array(vm).tobytes()
    assert Mx.csr_matvec(s, v).tobytes() == np.array(cmv).tobytes()
    assert Mx.csr_vecmat(u, s).tobytes() == np.array(cvm).tobytes()
    assert Mx.csr_matmat_right(s, Mx.DenseMatrix(M)).values.tobytes() == np.array(right).tobytes()
    assert Mx.csr_matmat_left(Mx.DenseMatrix(L), s).values.tobytes() == np.array(left).tobytes()
    mm = [[sum_ordered(dense[i], [M[k][j] for k in range(m)]) for j in range(3)] for i in range(n)]
    assert Mx.dense_matmat(D, Mx.DenseMatrix(M)).values.tobytes() == np.array(mm).tobytes()


def sum_ordered(a, b):
    acc = 0.0
    for x, y in zip(a, b):
        acc += x * y
    return acc


def test_degenerate_shapes():
    from paper_1702_06943_b200 import matrix as Mx

    s = Mx.SparseRowMatrix(0, [[], []])
    assert Mx.csr_matvec(s, []).tolist() == [0.0, 0.0]
    assert Mx.csr_vecmat([1.0, 2.0], s).tolist() == []
    assert Mx.dense_matvec(Mx.DenseMatrix(np.zeros((2, 0))), []).tolist() == [0.0, 0.0]
    with pytest.raises(ValueError, match="inner dimensions"):
        Mx.dense_matmat(Mx.DenseMatrix([[1.0, 2.0]]), Mx.DenseMatrix([[1.0]]))


def _dataset(oracle, n=400, m=9, seed=31, sign=False):
    from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix

    rng = np.random.default_rng(seed)
    rows = random_alphabet_rows(rng, n, m, 0.6)
    w = rng.standard_normal(m)
    z = np.array([sum(x * w[c] for c, x in r) for r in rows])
    y = np.where(z >= 0, 1.0, -1.0) if sign else z
    return LabeledDataset(features=SparseRowMatrix(m, rows), labels=y), rows


@pytest.mark.parametrize("execution", ["dense", "csr"])
@pytest.mark.parametrize("loss", ["squared", "logistic", "hinge"])
def test_execution_layouts_match_compressed(oracle, execution, loss):
    """train(execution=dense|csr) runs the reference's per-batch loop on the device baselines; it
    agrees with the compressed epoch kernels (reference test_training.py:343-353) and the oracle."""
    from paper_1702_06943_b200.training import TrainConfig, train

    ds, _ = _dataset(oracle, sign=loss != "squared")
    lr = 1e-3 if loss == "squared" else 0.05
    base = TrainConfig(loss, 32, lr, 2)
    alt = TrainConfig(loss, 32, lr, 2, execution=execution)
    m0, t0 = train(ds, base)
    m1, t1 = train(ds, alt)
    assert within_rel(m1.weights, m0.weights, 1e-9)
    assert within_rel(t1.risks, t0.risks, 1e-9)
    rp, c, v = oracle.rows_to_csr(ds.features.rows)
    w_ref, risks_ref = oracle.train_glm(rp, c, v, ds.labels, 9, loss, 32, lr, 2, 0)
    assert within_rel(m1.weights, w_ref, 1e-9) and within_rel(t1.risks, risks_ref, 1e-9)


def test_empirical_risk_vs_oracle(oracle):
    from paper_1702_06943_b200.training import GlmModel, empirical_risk

    ds, _ = _dataset(oracle, sign=True)
    rp, c, v = oracle.rows_to_csr(ds.features.rows)
    w = np.random.default_rng(4).standard_normal(9) * 0.3
    for loss in ("squared", "logistic", "hinge"):
        got = empirical_risk(GlmModel(w), ds, loss)
        want = oracle.empirical_risk_glm(w, rp, c, v, ds.labels, loss)
        assert abs(got - want) <= 1e-12 * abs(want), (loss, got, want)


def test_glm_gradient_layouts_agree(oracle):
    from paper_1702_06943_b200.kernels import CompressedMatrix
    from paper_1702_06943_b200.matrix import sparse_to_dense
    from paper_1702_06943_b200.training import Batch, GlmModel, glm_gradient

    ds, _ = _dataset(oracle, n=60, sign=True)
    w = np.random.default_rng(6).standard_normal(9) * 0.2
    for loss in ("squared", "logistic", "hinge"):
        got = [glm_gradient(Batch(f, ds.labels), GlmModel(w), loss) for f in
               (ds.features, sparse_to_dense(ds.features), CompressedMatrix.from_sparse(ds.features))]
        assert within_rel(got[1], got[0], 1e-12) and within_rel(got[2], got[0], 1e-12)


def _exact_cases():
    from helpers import TOY_ROWS, TREE_ROWS

    rng = np.random.default_rng(17)
    out = [("toy", TOY_ROWS, 5), ("tree", TREE_ROWS, 5), ("empty_rows", [[], [(1, 2.0)], [], [(0, 1.0)], []], 3)]
    for k, (n, m, dens) in enumerate([(60, 40, 0.3), (300, 20, 0.9), (64, 200, 0.05)]):
        out.append((f"rand{k}", random_alphabet_rows(rng, n, m, dens, alphabet_size=4 + 3 * k), m))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["config1"] + [c[0] for c in _exact_cases()])
def test_single_matrix_products_bit_exact(oracle, case):
    """The reference-API matvec / vecmat (kernels.CompressedMatrix) run the reference's own operation
    order (toc_exact.cu) and equal it bit for bit: the oracle restates kernels.py:115-174 in that
    order and is pinned bit-exactly to the reference's goldens (tests/test_oracle.py)."""
    from paper_1702_06943_b200 import synth
    from paper_1702_06943_b200.kernels import CompressedMatrix, matvec, vecmat
    from paper_1702_06943_b200.matrix import SparseRowMatrix

    if case == "config1":
        rp, c, v = synth.dense_to_csr(synth.cfg1_dense(0))
        enc, m = oracle.encode_csr(128, rp, c, v), 128
        sp = SparseRowMatrix.from_csr(128, rp, c, v)
    else:
        name, rows, m = next(x for x in _exact_cases() if x[0] == case)
        enc = oracle.encode_rows(m, rows)
        r = [list(x) for x in rows]
        rp = np.r_[0, np.cumsum([len(x) for x in r])].astype(np.int64)
        sp = SparseRowMatrix.from_csr(m, rp, np.array([cc for x in r for cc, _ in x], np.int32),
                                      np.array([vv for x in r for _, vv in x], np.float64))
    a = CompressedMatrix.from_sparse(sp)
    t = oracle.Tree.from_encoding(enc)
    rng = np.random.default_rng(5)
    for _ in range(3):
        x, u = rng.standard_normal(m), rng.standard_normal(enc.n_rows) * 10.0 ** rng.uniform(-6, 6, enc.n_rows)
        assert np.array_equal(matvec(a, x), t.matvec(x))
        assert np.array_equal(vecmat(u, a), t.vecmat(u))
