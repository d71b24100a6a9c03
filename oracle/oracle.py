"""TEST INFRASTRUCTURE ONLY -- ctypes wrapper over the C oracle (oracle/toc_oracle.c).

The oracle is a CPU restatement of the reference TOC algorithm (reference package `toc`,
/root/reference/pkg/src/toc).  Only ``tests/``, ``__graft_entry__.smoke()`` and bench.py's CPU
baseline legs may use it; the product package never imports it.

Every entry point names the reference function it restates.  Rows are given in the reference's
own sparse form: a list (one per row) of (column, value) pairs with strictly increasing columns
(matrix.py:78-142).
"""

from __future__ import annotations

import ctypes
import os
import random
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

OR_OK, OR_BAD_MAGIC, OR_BAD_VERSION, OR_TRUNCATED, OR_FORMAT, OR_CORRUPT, OR_VALUE, OR_NOMEM = range(8)
ERROR_KIND = {
    OR_BAD_MAGIC: "BadMagicError",
    OR_BAD_VERSION: "UnsupportedVersionError",
    OR_TRUNCATED: "TruncatedBlockError",
    OR_FORMAT: "BlockFormatError",
    OR_CORRUPT: "CorruptEncodingError",
    OR_VALUE: "ValueError",
    OR_NOMEM: "MemoryError",
}


class OracleError(Exception):
    """An oracle call failed; ``kind`` names the reference exception class it stands for."""

    def __init__(self, kind: str, detail: int, where: int):
        super().__init__(f"{kind} (detail {detail}, at {where})")
        self.kind = kind
        self.detail = detail
        self.where = where


def build() -> str:
    """Compile the oracle (make -C oracle).  Returns the library path."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None

P = ctypes.c_void_p
I64 = ctypes.c_int64
PI64 = ctypes.POINTER(ctypes.c_int64)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.or_encode.argtypes = [I64, I64, P, P, P, PI64, P, P, PI64, P, P]
        L.or_serialize.argtypes = [I64, I64, I64, P, P, I64, P, P, P, PI64]
        L.or_deserialize.argtypes = [P, I64, P, P, P, P, P, PI64, PI64]
        L.or_tree_build.restype = P
        L.or_tree_build.argtypes = [I64, I64, I64, P, P, I64, P, P, ctypes.POINTER(ctypes.c_int), PI64, PI64]
        L.or_tree_from_block.restype = P
        L.or_tree_from_block.argtypes = [P, I64, ctypes.POINTER(ctypes.c_int), PI64, PI64]
        L.or_tree_free.argtypes = [P]
        L.or_tree_len.restype = I64
        L.or_tree_len.argtypes = [P]
        L.or_tree_arrays.argtypes = [P, P, P, P]
        L.or_matvec.argtypes = [P, P, P, P]
        L.or_vecmat.argtypes = [P, P, P, P]
        L.or_matmat_right.argtypes = [P, P, I64, P, P]
        L.or_matmat_left.argtypes = [P, P, I64, P, P]
        L.or_sweep.argtypes = [I64, P, P, P, P, P, P, ctypes.c_int, ctypes.c_int]
        L.or_max_threads.restype = ctypes.c_int
        L.or_csr_matvec.argtypes = [I64, P, P, P, P, P]
        L.or_glm_epoch.argtypes = [I64, P, P, P, P, ctypes.c_int, ctypes.c_double]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def rows_to_csr(rows, n_cols=None):
    """(row_ptr int64, cols int32, vals float64) from a list of (col, val) pair lists."""
    lens = np.fromiter((len(r) for r in rows), dtype=np.int64, count=len(rows))
    row_ptr = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum(lens, out=row_ptr[1:])
    nnz = int(row_ptr[-1])
    cols = np.empty(nnz, dtype=np.int32)
    vals = np.empty(nnz, dtype=np.float64)
    k = 0
    for r in rows:
        for c, v in r:
            cols[k] = c
            vals[k] = v
            k += 1
    return row_ptr, cols, vals


@dataclass
class Encoding:
    """Array form of the reference's LogicalEncoding (codec.py:142-174)."""

    n_rows: int
    n_cols: int
    I_cols: np.ndarray  # int32 [nI]
    I_vals: np.ndarray  # float64 [nI]
    codes: np.ndarray  # uint32 [C]
    offsets: np.ndarray  # int64 [n_rows + 1]

    @property
    def pairs(self):
        return [(int(c), float(v)) for c, v in zip(self.I_cols, self.I_vals)]

    @property
    def rows(self):
        o = self.offsets
        return [[int(x) for x in self.codes[o[i] : o[i + 1]]] for i in range(self.n_rows)]

    def tree_length(self) -> int:
        lens = np.diff(self.offsets)
        return 1 + len(self.I_cols) + int(np.sum(np.maximum(lens - 1, 0)))


def encode_csr(n_cols: int, row_ptr: np.ndarray, cols: np.ndarray, vals: np.ndarray) -> Encoding:
    """codec.encode (codec.py:177-191) on CSR input."""
    n_rows = len(row_ptr) - 1
    nnz = int(row_ptr[-1])
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int32)
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    I_cols = np.empty(max(nnz, 1), dtype=np.int32)
    I_vals = np.empty(max(nnz, 1), dtype=np.float64)
    codes = np.empty(max(nnz, 1), dtype=np.uint32)
    offsets = np.empty(n_rows + 1, dtype=np.int64)
    nI = ctypes.c_int64()
    C = ctypes.c_int64()
    rc = lib().or_encode(n_rows, n_cols, _ptr(row_ptr), _ptr(cols), _ptr(vals), ctypes.byref(nI),
                         _ptr(I_cols), _ptr(I_vals), ctypes.byref(C), _ptr(codes), _ptr(offsets))
    if rc:
        raise OracleError(ERROR_KIND[rc], 0, 0)
    return Encoding(n_rows, n_cols, I_cols[: nI.value].copy(), I_vals[: nI.value].copy(),
                    codes[: C.value].copy(), offsets)


def encode_rows(n_cols: int, rows) -> Encoding:
    return encode_csr(n_cols, *rows_to_csr(rows))


def serialize(enc: Encoding) -> bytes:
    """physical.serialize_block (physical.py:110-130)."""
    L = lib()
    n = ctypes.c_int64()
    args = [enc.n_rows, enc.n_cols, len(enc.I_cols), _ptr(np.ascontiguousarray(enc.I_cols, np.int32)),
            _ptr(np.ascontiguousarray(enc.I_vals, np.float64)), len(enc.codes),
            _ptr(np.ascontiguousarray(enc.codes, np.uint32)), _ptr(np.ascontiguousarray(enc.offsets, np.int64))]
    keep = args  # keep arrays alive
    rc = L.or_serialize(*keep, None, ctypes.byref(n))
    if rc:
        raise OracleError(ERROR_KIND[rc], 0, 0)
    out = np.empty(n.value, dtype=np.uint8)
    rc = L.or_serialize(*keep, _ptr(out), ctypes.byref(n))
    if rc:
        raise OracleError(ERROR_KIND[rc], 0, 0)
    return out.tobytes()


def deserialize(data: bytes) -> Encoding:
    """physical.deserialize_block (physical.py:138-186); raises OracleError(kind) on bad input."""
    L = lib()
    buf = np.frombuffer(data, dtype=np.uint8).copy() if len(data) else np.zeros(1, np.uint8)
    dims = np.zeros(4, dtype=np.int64)
    detail = ctypes.c_int64()
    where = ctypes.c_int64()
    rc = L.or_deserialize(_ptr(buf), len(data), _ptr(dims), None, None, None, None,
                          ctypes.byref(detail), ctypes.byref(where))
    if rc:
        raise OracleError(ERROR_KIND[rc], detail.value, where.value)
    n_rows, n_cols, nI, C = (int(x) for x in dims)
    I_cols = np.empty(max(nI, 1), np.int32)
    I_vals = np.empty(max(nI, 1), np.float64)
    codes = np.empty(max(C, 1), np.uint32)
    offsets = np.empty(n_rows + 1, np.int64)
    rc = L.or_deserialize(_ptr(buf), len(data), _ptr(dims), _ptr(I_cols), _ptr(I_vals), _ptr(codes),
                          _ptr(offsets), ctypes.byref(detail), ctypes.byref(where))
    if rc:
        raise OracleError(ERROR_KIND[rc], detail.value, where.value)
    return Encoding(n_rows, n_cols, I_cols[:nI].copy(), I_vals[:nI].copy(), codes[:C].copy(), offsets)


class Tree:
    """codec.build_prefix_tree (codec.py:215-259) held as a C object, plus the kernels of
    kernels.py:115-234 evaluated on it in the reference's exact order."""

    def __init__(self, handle, n_rows: int, n_cols: int):
        self._h = handle
        self.n_rows = n_rows
        self.n_cols = n_cols
        self.T = int(lib().or_tree_len(handle))

    @classmethod
    def from_encoding(cls, enc: Encoding) -> "Tree":
        rc = ctypes.c_int()
        bad_row = ctypes.c_int64()
        bad_code = ctypes.c_int64()
        arrs = [np.ascontiguousarray(enc.I_cols, np.int32), np.ascontiguousarray(enc.I_vals, np.float64),
                np.ascontiguousarray(enc.codes, np.uint32), np.ascontiguousarray(enc.offsets, np.int64)]
        h = lib().or_tree_build(enc.n_rows, enc.n_cols, len(arrs[0]), _ptr(arrs[0]), _ptr(arrs[1]),
                                len(arrs[2]), _ptr(arrs[2]), _ptr(arrs[3]), ctypes.byref(rc),
                                ctypes.byref(bad_row), ctypes.byref(bad_code))
        if not h:
            raise OracleError(ERROR_KIND.get(rc.value, "?"), bad_row.value, bad_code.value)
        return cls(h, enc.n_rows, enc.n_cols)

    @classmethod
    def from_block(cls, data: bytes) -> "Tree":
        buf = np.frombuffer(data, dtype=np.uint8).copy()
        rc = ctypes.c_int()
        d = ctypes.c_int64()
        w = ctypes.c_int64()
        h = lib().or_tree_from_block(_ptr(buf), len(data), ctypes.byref(rc), ctypes.byref(d), ctypes.byref(w))
        if not h:
            raise OracleError(ERROR_KIND.get(rc.value, "?"), d.value, w.value)
        n_rows = int.from_bytes(data[5:9], "little")
        n_cols = int.from_bytes(data[9:13], "little")
        return cls(h, n_rows, n_cols)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.or_tree_free(self._h)
            self._h = None

    def arrays(self):
        parent = np.empty(self.T, np.int32)
        column = np.empty(self.T, np.int32)
        value = np.empty(self.T, np.float64)
        lib().or_tree_arrays(self._h, _ptr(parent), _ptr(column), _ptr(value))
        return parent, column, value

    def matvec(self, v) -> np.ndarray:
        v = np.ascontiguousarray(v, np.float64)
        out = np.empty(self.n_rows, np.float64)
        h = np.empty(self.T, np.float64)
        lib().or_matvec(self._h, _ptr(v), _ptr(out), _ptr(h))
        return out

    def vecmat(self, u) -> np.ndarray:
        u = np.ascontiguousarray(u, np.float64)
        out = np.empty(self.n_cols, np.float64)
        h = np.empty(self.T, np.float64)
        lib().or_vecmat(self._h, _ptr(u), _ptr(out), _ptr(h))
        return out

    def matmat_right(self, M) -> np.ndarray:
        M = np.ascontiguousarray(M, np.float64)
        p = M.shape[1]
        out = np.empty((self.n_rows, p), np.float64)
        h = np.empty(self.T * p + 1, np.float64)
        lib().or_matmat_right(self._h, _ptr(M), p, _ptr(out), _ptr(h))
        return out

    def matmat_left(self, M) -> np.ndarray:
        M = np.ascontiguousarray(M, np.float64)
        p = M.shape[0]
        out = np.empty((p, self.n_cols), np.float64)
        h = np.empty(self.T * p + 1, np.float64)
        lib().or_matmat_left(self._h, _ptr(M), p, _ptr(out), _ptr(h))
        return out


def sweep(trees, row_base, v, u, kind: int, nthreads: int = 0):
    """Many batches with prebuilt trees (cli.py:299-383 conventions); kind 0/1/2 = matvec /
    vecmat / both.  Returns (R, O)."""
    n_b = len(trees)
    handles = (ctypes.c_void_p * n_b)(*[t._h for t in trees])
    row_base = np.ascontiguousarray(row_base, np.int64)
    n_total = int(row_base[-1] + trees[-1].n_rows) if n_b else 0
    m = trees[0].n_cols if n_b else 0
    R = np.zeros(max(n_total, 1), np.float64)
    O = np.zeros(max(n_b * m, 1), np.float64)
    v = np.ascontiguousarray(v, np.float64)
    u = np.ascontiguousarray(u, np.float64)
    rc = lib().or_sweep(n_b, handles, _ptr(row_base), _ptr(v), _ptr(u), _ptr(R), _ptr(O), kind, nthreads)
    if rc:
        raise OracleError(ERROR_KIND[rc], 0, 0)
    return R[:n_total], O[: n_b * m].reshape(n_b, m)


def max_threads() -> int:
    return int(lib().or_max_threads())


def csr_matvec(row_ptr, cols, vals, v) -> np.ndarray:
    """matrix.csr_matvec (matrix.py:225-239)."""
    n = len(row_ptr) - 1
    out = np.empty(n, np.float64)
    a = [np.ascontiguousarray(row_ptr, np.int64), np.ascontiguousarray(cols, np.int32),
         np.ascontiguousarray(vals, np.float64), np.ascontiguousarray(v, np.float64)]
    lib().or_csr_matvec(n, _ptr(a[0]), _ptr(a[1]), _ptr(a[2]), _ptr(a[3]), _ptr(out))
    return out


# ------------------------------------------------------------------------------------------
# Training (training.py:131-361), GLM losses, restated with the C epoch kernel.

LOSS_CODE = {"squared": 0, "logistic": 1, "hinge": 2}


def shuffle_order(n_rows: int, seed: int) -> np.ndarray:
    """shuffle_once's permutation (training.py:138-139): the stdlib Fisher-Yates."""
    order = list(range(n_rows))
    random.Random(seed).shuffle(order)
    return np.asarray(order, dtype=np.int64)


def _softplus(t):  # training.py:206-212
    out = np.empty_like(t)
    pos = t > 0
    out[pos] = t[pos] + np.log1p(np.exp(-t[pos]))
    out[~pos] = np.log1p(np.exp(t[~pos]))
    return out


def empirical_risk_glm(w, row_ptr, cols, vals, labels, loss_kind: str) -> float:
    """empirical_risk for GLMs (training.py:231-258) on the unshuffled CSR data."""
    z = csr_matvec(row_ptr, cols, vals, w)
    y = labels
    if loss_kind == "squared":
        losses = 0.5 * (y - z) ** 2
    elif loss_kind == "logistic":
        losses = _softplus(-y * z)
    else:
        losses = np.maximum(0.0, 1.0 - y * z)
    return float(np.mean(losses))


def make_batch_trees(row_ptr, cols, vals, n_cols, order, batch_size):
    """shuffle_once + make_batches(execution='compressed') (training.py:131-167): returns the
    per-batch trees, row bases and the shuffled labels index."""
    trees, bases = [], []
    n = len(order)
    lens = np.diff(row_ptr)
    for lo in range(0, n, batch_size):
        idx = order[lo : lo + batch_size]
        l = lens[idx]
        rp = np.zeros(len(idx) + 1, np.int64)
        np.cumsum(l, out=rp[1:])
        gather = np.concatenate([np.arange(row_ptr[i], row_ptr[i + 1]) for i in idx]) if rp[-1] else np.zeros(0, np.int64)
        enc = encode_csr(n_cols, rp, cols[gather], vals[gather])
        trees.append(Tree.from_encoding(enc))
        bases.append(lo)
    return trees, np.asarray(bases, np.int64)


def train_glm(row_ptr, cols, vals, labels, n_cols, loss_kind, batch_size, lr, epochs, seed=0,
              trees_cache=None):
    """training.train for GLM losses in compressed execution (training.py:336-361).
    Returns (weights, risks)."""
    order = shuffle_order(len(labels), seed)
    if trees_cache is None:
        trees, bases = make_batch_trees(row_ptr, cols, vals, n_cols, order, batch_size)
    else:
        trees, bases = trees_cache
    y_sh = np.ascontiguousarray(labels[order], np.float64)
    w = np.zeros(n_cols, np.float64)
    handles = (ctypes.c_void_p * len(trees))(*[t._h for t in trees])
    risks = []
    for _ in range(epochs):
        rc = lib().or_glm_epoch(len(trees), handles, _ptr(bases), _ptr(y_sh), _ptr(w),
                                LOSS_CODE[loss_kind], float(lr))
        if rc:
            raise OracleError(ERROR_KIND[rc], 0, 0)
        risks.append(empirical_risk_glm(w, row_ptr, cols, vals, labels, loss_kind))
    return w, risks


# ------------------------------------------------------------------------------------------
# The reference's one-hidden-layer network (training.py:81-98, 206-228, 284-293, 319-333).

def _sigmoid(z):  # training.py:215-221
    out = np.empty_like(z)
    pos = z >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-z[pos]))
    ez = np.exp(z[~pos])
    out[~pos] = ez / (1.0 + ez)
    return out


def csr_matmat_right(row_ptr, cols, vals, M):
    """matrix.csr_matmat_right (matrix.py:260-272): row-wise acc += val * M[col]."""
    n = len(row_ptr) - 1
    out = np.zeros((n, M.shape[1]))
    for i in range(n):
        acc = out[i]
        for e in range(row_ptr[i], row_ptr[i + 1]):
            acc += vals[e] * M[cols[e]]
    return out


def init_nn(n_cols, hidden, seed):  # training.py:327-333
    import math

    rng = np.random.default_rng(seed)
    s1 = 1.0 / math.sqrt(max(n_cols, 1))
    s2 = 1.0 / math.sqrt(hidden)
    return rng.uniform(-s1, s1, size=(n_cols, hidden)), rng.uniform(-s2, s2, size=(hidden, 1))


def train_nn(row_ptr, cols, vals, labels, n_cols, hidden, batch_size, lr, epochs, seed=0):
    """training.train with loss_kind='nn_mse', compressed execution.  Returns (w1, w2, risks)."""
    order = shuffle_order(len(labels), seed)
    trees, bases = make_batch_trees(row_ptr, cols, vals, n_cols, order, batch_size)
    y_sh = labels[order]
    w1, w2 = init_nn(n_cols, hidden, seed)
    risks = []
    for _ in range(epochs):
        for t, lo in zip(trees, bases):
            y = y_sh[lo : lo + t.n_rows]
            h1 = _sigmoid(t.matmat_right(w1))
            yhat = h1 @ w2
            err = yhat - y[:, None]
            g_w2 = h1.T @ err
            delta = (err @ w2.T) * h1 * (1.0 - h1)
            g_w1 = t.matmat_left(np.ascontiguousarray(delta.T)).T.copy()
            n = t.n_rows
            w1 = w1 - (lr / n) * g_w1
            w2 = w2 - (lr / n) * g_w2
        h1 = _sigmoid(csr_matmat_right(row_ptr, cols, vals, w1))
        yhat = h1 @ w2
        risks.append(float(np.mean(0.5 * (labels - yhat[:, 0]) ** 2)))
    return w1, w2, risks


def train_mlp(row_ptr, cols, vals, labels, n_cols, hidden, classes, batch_size, lr, epochs, seed=0):
    """CPU restatement of the config-5 MLP step (ReLU, softmax cross-entropy, biases, Xavier init)
    with the first layer through the oracle's matmat_right / matmat_left.  Not a reference
    function (the reference has no such model): parity for it is unpinned by reference outputs."""
    import math

    rng = np.random.default_rng(seed)
    l1 = math.sqrt(6.0 / (n_cols + hidden))
    l2 = math.sqrt(6.0 / (hidden + classes))
    w1 = rng.uniform(-l1, l1, size=(n_cols, hidden))
    b1 = np.zeros(hidden)
    w2 = rng.uniform(-l2, l2, size=(hidden, classes))
    b2 = np.zeros(classes)
    order = shuffle_order(len(labels), seed)
    trees, bases = make_batch_trees(row_ptr, cols, vals, n_cols, order, batch_size)
    y_sh = labels[order].astype(np.int64)
    risks = []

    def softmax(x):
        e = np.exp(x - x.max(axis=1, keepdims=True))
        return e / e.sum(axis=1, keepdims=True)

    for _ in range(epochs):
        for t, lo in zip(trees, bases):
            y = y_sh[lo : lo + t.n_rows]
            a1 = np.maximum(t.matmat_right(w1) + b1, 0.0)
            p = softmax(a1 @ w2 + b2)
            p[np.arange(len(y)), y] -= 1.0
            g_w2, g_b2 = a1.T @ p, p.sum(0)
            delta = (p @ w2.T) * (a1 > 0)
            g_b1 = delta.sum(0)
            g_w1 = t.matmat_left(np.ascontiguousarray(delta.T)).T
            s = lr / len(y)
            w1, b1, w2, b2 = w1 - s * g_w1, b1 - s * g_b1, w2 - s * g_w2, b2 - s * g_b2
        z = csr_matmat_right(row_ptr, cols, vals, w1)
        logits = np.maximum(z + b1, 0.0) @ w2 + b2
        lp = logits - logits.max(axis=1, keepdims=True)
        lp = lp - np.log(np.exp(lp).sum(axis=1, keepdims=True))
        risks.append(float(-np.mean(lp[np.arange(len(labels)), labels.astype(np.int64)])))
    return (w1, b1, w2, b2), risks
