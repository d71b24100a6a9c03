"""Matrix containers of the reference API (reference matrix.py:21-161), CSR-backed.

The reference stores a sparse matrix as a list of (column, value) pair lists.  Here the
canonical form is CSR (row_ptr int64, cols int32, vals float64) because that is what is uploaded
to the device; the reference's ``rows`` view is materialised on demand.  Validation follows the
reference contract (matrix.py:90-114): strictly increasing columns inside a row, columns in
[0, n_cols), values finite and non-zero.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

SparseRow = list


def as_vector(v: Sequence[float], expected: int, name: str) -> np.ndarray:
    """Finite float64 vector of the expected length (matrix.py:21-30 contract)."""
    arr = np.asarray(v, dtype=np.float64)
    if arr.ndim != 1:
        raise ValueError(f"{name} must be one-dimensional, got shape {arr.shape}")
    if arr.shape[0] != expected:
        raise ValueError(f"{name} has length {arr.shape[0]}, expected {expected}")
    if not np.all(np.isfinite(arr)):
        raise ValueError(f"{name} contains non-finite entries")
    return arr


class DenseMatrix:
    """Immutable row-major float64 matrix with finite entries (matrix.py:33-75)."""

    __slots__ = ("values",)

    def __init__(self, values):
        arr = np.array(values, dtype=np.float64)
        if arr.ndim != 2:
            raise ValueError(f"dense matrix needs a 2-d array, got shape {arr.shape}")
        if not np.all(np.isfinite(arr)):
            raise ValueError("dense matrix entries must be finite")
        arr = np.ascontiguousarray(arr)
        arr.setflags(write=False)
        self.values = arr

    @property
    def n_rows(self) -> int:
        return self.values.shape[0]

    @property
    def n_cols(self) -> int:
        return self.values.shape[1]

    def row_lists(self):
        return self.values.tolist()

    def __eq__(self, other):
        if not isinstance(other, DenseMatrix):
            return NotImplemented
        return self.values.shape == other.values.shape and bool(np.array_equal(self.values, other.values))

    __hash__ = None

    def __repr__(self):
        return f"DenseMatrix({self.n_rows}x{self.n_cols})"


def _check_csr(n_cols: int, row_ptr: np.ndarray, cols: np.ndarray, vals: np.ndarray) -> None:
    """Vectorised SparseRowMatrix validation; the first offending row is reported."""
    if len(cols) == 0:
        return
    row_of = np.repeat(np.arange(len(row_ptr) - 1), np.diff(row_ptr))
    first_in_row = np.zeros(len(cols), bool)
    first_in_row[row_ptr[:-1][np.diff(row_ptr) > 0]] = True
    prev = np.concatenate([[-1], cols[:-1]])
    bad_order = (~first_in_row) & (cols <= prev)
    checks = [
        (bad_order, lambda i: f"row {row_of[i]}: column {cols[i]} after {prev[i]}; columns must be strictly increasing"),
        ((cols < 0) | (cols >= n_cols), lambda i: f"row {row_of[i]}: column {cols[i]} out of range for n_cols={n_cols}"),
        (vals == 0.0, lambda i: f"row {row_of[i]}: explicit zero at column {cols[i]}"),
        (~np.isfinite(vals), lambda i: f"row {row_of[i]}: non-finite value at column {cols[i]}"),
    ]
    worst = None
    for mask, msg in checks:
        idx = np.flatnonzero(mask)
        if len(idx) and (worst is None or idx[0] < worst[0]):
            worst = (int(idx[0]), msg)
    if worst is not None:
        raise ValueError(worst[1](worst[0]))


class SparseRowMatrix:
    """Sparse rows of (column, value) pairs (matrix.py:78-142), stored as CSR."""

    __slots__ = ("n_cols", "row_ptr", "cols", "vals", "_rows")

    def __init__(self, n_cols: int, rows: Iterable[Iterable[tuple[int, float]]]):
        if n_cols < 0:
            raise ValueError(f"n_cols must be non-negative, got {n_cols}")
        ptr, cs, vs = [0], [], []
        for row in rows:
            for c, v in row:
                cs.append(int(c))
                vs.append(float(v))
            ptr.append(len(cs))
        row_ptr = np.asarray(ptr, np.int64)
        cols = np.asarray(cs, np.int64)
        vals = np.asarray(vs, np.float64)
        _check_csr(n_cols, row_ptr, cols, vals)
        self._init(n_cols, row_ptr, cols.astype(np.int32), vals)

    def _init(self, n_cols, row_ptr, cols, vals):
        self.n_cols = int(n_cols)
        self.row_ptr = np.ascontiguousarray(row_ptr, np.int64)
        self.cols = np.ascontiguousarray(cols, np.int32)
        self.vals = np.ascontiguousarray(vals, np.float64)
        self._rows = None

    @classmethod
    def from_csr(cls, n_cols: int, row_ptr, cols, vals, check: bool = True) -> "SparseRowMatrix":
        m = object.__new__(cls)
        row_ptr = np.asarray(row_ptr, np.int64)
        cols = np.asarray(cols)
        vals = np.asarray(vals, np.float64)
        if check:
            _check_csr(n_cols, row_ptr, cols.astype(np.int64), vals)
        m._init(n_cols, row_ptr, cols, vals)
        return m

    @classmethod
    def from_rows_unchecked(cls, n_cols: int, rows) -> "SparseRowMatrix":
        m = object.__new__(cls)
        ptr, cs, vs = [0], [], []
        for row in rows:
            for c, v in row:
                cs.append(c)
                vs.append(v)
            ptr.append(len(cs))
        m._init(n_cols, np.asarray(ptr, np.int64), np.asarray(cs, np.int32), np.asarray(vs, np.float64))
        return m

    @property
    def rows(self):
        if self._rows is None:
            rp, c, v = self.row_ptr, self.cols.tolist(), self.vals.tolist()
            self._rows = [list(zip(c[rp[i]:rp[i + 1]], v[rp[i]:rp[i + 1]])) for i in range(len(rp) - 1)]
        return self._rows

    @property
    def n_rows(self) -> int:
        return len(self.row_ptr) - 1

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def take_rows(self, idx) -> "SparseRowMatrix":
        """Rows idx (in that order) as a new matrix (used by shuffle_once / make_batches)."""
        idx = np.asarray(idx, np.int64)
        lens = np.diff(self.row_ptr)[idx]
        rp = np.zeros(len(idx) + 1, np.int64)
        np.cumsum(lens, out=rp[1:])
        if rp[-1]:
            starts = self.row_ptr[idx]
            gather = np.repeat(starts - rp[:-1], lens) + np.arange(rp[-1])
            cols, vals = self.cols[gather], self.vals[gather]
        else:
            cols, vals = np.zeros(0, np.int32), np.zeros(0)
        return SparseRowMatrix.from_csr(self.n_cols, rp, cols, vals, check=False)

    def __eq__(self, other):
        if not isinstance(other, SparseRowMatrix):
            return NotImplemented
        return (self.n_cols == other.n_cols and np.array_equal(self.row_ptr, other.row_ptr)
                and np.array_equal(self.cols, other.cols)
                and self.vals.tobytes() == other.vals.tobytes())

    __hash__ = None

    def __repr__(self):
        return f"SparseRowMatrix({self.n_rows}x{self.n_cols}, nnz={self.nnz})"


@dataclass
class LabeledDataset:
    """Features plus one label per row (matrix.py:145-161)."""

    features: SparseRowMatrix
    labels: np.ndarray = field(repr=False)

    def __post_init__(self):
        self.labels = as_vector(self.labels, self.features.n_rows, "labels")

    @property
    def n_rows(self) -> int:
        return self.features.n_rows

    @property
    def n_cols(self) -> int:
        return self.features.n_cols


def sparse_to_dense(s: SparseRowMatrix) -> DenseMatrix:
    out = np.zeros((s.n_rows, s.n_cols), dtype=np.float64)
    r = np.repeat(np.arange(s.n_rows), np.diff(s.row_ptr))
    out[r, s.cols] = s.vals
    return DenseMatrix(out)


def dense_to_sparse(a: DenseMatrix) -> SparseRowMatrix:
    """Drop exact zeros; surviving entries keep their bits (matrix.py:217-222)."""
    mask = a.values != 0.0
    rp = np.zeros(a.n_rows + 1, np.int64)
    np.cumsum(mask.sum(axis=1), out=rp[1:])
    r, c = np.nonzero(mask)
    return SparseRowMatrix.from_csr(a.n_cols, rp, c.astype(np.int32), a.values[r, c], check=False)


# ---- the reference's uncompressed baselines (matrix.py:164-279), on the device ------------------
# Same ascending accumulation order and separate multiply / add as the reference, one device
# thread per output element (csrc/toc_dense.cu): results equal the reference's bit for bit.  They
# back train(execution="dense" | "csr") and empirical_risk; the compressed hot path never uses them.

def _device():
    from . import _native as N

    torch = N.require_cuda()
    return torch, N


def _d(torch, a, dtype):
    return torch.from_numpy(np.array(a, dtype=dtype, order="C")).cuda()


def _inner(left_cols: int, right_rows: int) -> None:
    if left_cols != right_rows:
        raise ValueError(f"inner dimensions differ: left has {left_cols} columns, right has {right_rows} rows")


def _csc(torch, s: SparseRowMatrix):
    """The entries of s grouped by column, rows ascending within a column (stable sort by column
    of the row-major entries): the reference's row-order scatters become ordered column sums."""
    rows = np.repeat(np.arange(s.n_rows, dtype=np.int32), np.diff(s.row_ptr))
    order = np.argsort(s.cols, kind="stable")
    cp = np.zeros(s.n_cols + 1, np.int64)
    np.cumsum(np.bincount(s.cols, minlength=s.n_cols)[: s.n_cols], out=cp[1:])
    return _d(torch, cp, np.int64), _d(torch, rows[order], np.int32), _d(torch, s.vals[order], np.float64)


def _run(N, rc: int, what: str) -> None:
    N.check(rc, what)


def dense_matvec(a: DenseMatrix, v: Sequence[float]) -> np.ndarray:
    """A @ v, each row summed left to right (reference matrix.py:164-173)."""
    vec = as_vector(v, a.n_cols, "vector")
    if a.n_rows == 0:
        return np.zeros(0)
    torch, N = _device()
    A, x = _d(torch, a.values, np.float64), _d(torch, vec, np.float64)
    out = torch.empty(a.n_rows, dtype=torch.float64, device="cuda")
    _run(N, N.lib().toc_dense_matvec(A.data_ptr(), a.n_rows, a.n_cols, x.data_ptr(), out.data_ptr(),
                                     N.stream_handle()), "toc_dense_matvec")
    return out.cpu().numpy()


def dense_vecmat(v: Sequence[float], a: DenseMatrix) -> np.ndarray:
    """v @ A, each column summed over rows in ascending order (reference matrix.py:176-186)."""
    vec = as_vector(v, a.n_rows, "vector")
    if a.n_cols == 0:
        return np.zeros(0)
    torch, N = _device()
    A, x = _d(torch, a.values, np.float64), _d(torch, vec, np.float64)
    out = torch.empty(a.n_cols, dtype=torch.float64, device="cuda")
    _run(N, N.lib().toc_dense_vecmat(x.data_ptr(), A.data_ptr(), a.n_rows, a.n_cols, out.data_ptr(),
                                     N.stream_handle()), "toc_dense_vecmat")
    return out.cpu().numpy()


def dense_matmat(a: DenseMatrix, m: DenseMatrix) -> DenseMatrix:
    """A @ M with the inner dimension accumulated in ascending order (reference matrix.py:189-206)."""
    _inner(a.n_cols, m.n_rows)
    if a.n_rows * m.n_cols == 0:
        return DenseMatrix(np.zeros((a.n_rows, m.n_cols)))
    torch, N = _device()
    A, M = _d(torch, a.values, np.float64), _d(torch, m.values, np.float64)
    out = torch.empty((a.n_rows, m.n_cols), dtype=torch.float64, device="cuda")
    _run(N, N.lib().toc_dense_matmat(A.data_ptr(), M.data_ptr(), a.n_rows, a.n_cols, m.n_cols, out.data_ptr(),
                                     N.stream_handle()), "toc_dense_matmat")
    return DenseMatrix(out.cpu().numpy())


def csr_matvec(s: SparseRowMatrix, v: Sequence[float]) -> np.ndarray:
    """S @ v; bit-identical to dense_matvec of the densified matrix (reference matrix.py:225-239)."""
    vec = as_vector(v, s.n_cols, "vector")
    if s.n_rows == 0:
        return np.zeros(0)
    torch, N = _device()
    rp, c, x = _d(torch, s.row_ptr, np.int64), _d(torch, s.cols, np.int32), _d(torch, s.vals, np.float64)
    vd = _d(torch, vec, np.float64)
    out = torch.empty(s.n_rows, dtype=torch.float64, device="cuda")
    _run(N, N.lib().toc_csr_matvec(rp.data_ptr(), c.data_ptr(), x.data_ptr(), s.n_rows, vd.data_ptr(),
                                   out.data_ptr(), N.stream_handle()), "toc_csr_matvec")
    return out.cpu().numpy()


def csr_vecmat(v: Sequence[float], s: SparseRowMatrix) -> np.ndarray:
    """v @ S, each column accumulated over rows in ascending order (reference matrix.py:242-249)."""
    vec = as_vector(v, s.n_rows, "vector")
    if s.n_cols == 0:
        return np.zeros(0)
    torch, N = _device()
    cp, rows, x = _csc(torch, s)
    vd = _d(torch, vec, np.float64)
    out = torch.empty(s.n_cols, dtype=torch.float64, device="cuda")
    _run(N, N.lib().toc_csc_vecmat(cp.data_ptr(), rows.data_ptr(), x.data_ptr(), s.n_cols, vd.data_ptr(),
                                   out.data_ptr(), N.stream_handle()), "toc_csc_vecmat")
    return out.cpu().numpy()


def csr_matmat_right(s: SparseRowMatrix, m: DenseMatrix) -> DenseMatrix:
    """S @ M for sparse S and dense M (reference matrix.py:252-264)."""
    _inner(s.n_cols, m.n_rows)
    if s.n_rows * m.n_cols == 0:
        return DenseMatrix(np.zeros((s.n_rows, m.n_cols)))
    torch, N = _device()
    rp, c, x = _d(torch, s.row_ptr, np.int64), _d(torch, s.cols, np.int32), _d(torch, s.vals, np.float64)
    M = _d(torch, m.values, np.float64)
    out = torch.empty((s.n_rows, m.n_cols), dtype=torch.float64, device="cuda")
    _run(N, N.lib().toc_csr_matmat_right(rp.data_ptr(), c.data_ptr(), x.data_ptr(), s.n_rows, M.data_ptr(),
                                         m.n_cols, out.data_ptr(), N.stream_handle()), "toc_csr_matmat_right")
    return DenseMatrix(out.cpu().numpy())


def csr_matmat_left(m: DenseMatrix, s: SparseRowMatrix) -> DenseMatrix:
    """M @ S for dense M and sparse S (reference matrix.py:267-279)."""
    _inner(m.n_cols, s.n_rows)
    if m.n_rows * s.n_cols == 0:
        return DenseMatrix(np.zeros((m.n_rows, s.n_cols)))
    torch, N = _device()
    cp, rows, x = _csc(torch, s)
    M = _d(torch, m.values, np.float64)
    out = torch.empty((m.n_rows, s.n_cols), dtype=torch.float64, device="cuda")
    _run(N, N.lib().toc_csc_matmat_left(cp.data_ptr(), rows.data_ptr(), x.data_ptr(), s.n_cols, M.data_ptr(),
                                        m.n_rows, s.n_rows, out.data_ptr(), N.stream_handle()),
         "toc_csc_matmat_left")
    return DenseMatrix(out.cpu().numpy())
