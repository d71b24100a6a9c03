"""Seeded synthetic inputs standing in for BASELINE.json's configs (no datasets are available
offline; DESIGN.md "Synthetic inputs" records every choice made where BASELINE.json is silent).

All generators return CSR pieces (row_ptr int64, cols int32, vals float64) with strictly
increasing columns and no explicit zeros -- the reference's SparseRowMatrix contract
(matrix.py:78-114) -- so they can be fed to the encoder directly.
"""

from __future__ import annotations

import numpy as np


def dense_to_csr(A: np.ndarray):
    """Drop exact zeros row by row, keeping values bit for bit (matrix.py:217-222)."""
    mask = A != 0.0
    lens = mask.sum(axis=1).astype(np.int64)
    row_ptr = np.zeros(A.shape[0] + 1, np.int64)
    np.cumsum(lens, out=row_ptr[1:])
    r, c = np.nonzero(mask)
    return row_ptr, c.astype(np.int32), A[r, c].astype(np.float64)


def csr_rows(row_ptr, cols, vals):
    """Reference-style list of (col, value) pair lists."""
    return [[(int(c), float(v)) for c, v in zip(cols[row_ptr[i]:row_ptr[i + 1]], vals[row_ptr[i]:row_ptr[i + 1]])]
            for i in range(len(row_ptr) - 1)]


def _zipf_probs(k: int, s: float) -> np.ndarray:
    p = 1.0 / np.arange(1, k + 1, dtype=np.float64) ** s
    return p / p.sum()


# ---- config 1: single 256x128 mini-batch --------------------------------------------------
def cfg1_dense(seed: int = 0, n_rows: int = 256, n_cols: int = 128, n_templates: int = 32,
               vocab: int = 16, zipf_s: float = 1.2, mutate: float = 0.1) -> np.ndarray:
    """BASELINE.json configs[0]: rows copied from one of 32 seed-0 template rows, each element
    mutated with probability 0.1; values from a 16-value vocabulary U[-1,1] with Zipf(1.2)
    frequencies."""
    rng = np.random.default_rng(seed)
    words = rng.uniform(-1.0, 1.0, vocab)
    p = _zipf_probs(vocab, zipf_s)
    templates = words[rng.choice(vocab, size=(n_templates, n_cols), p=p)]
    A = templates[rng.integers(0, n_templates, size=n_rows)]
    mask = rng.random((n_rows, n_cols)) < mutate
    A[mask] = words[rng.choice(vocab, size=int(mask.sum()), p=p)]
    return A


def cfg1_operands(seed: int = 0, n_rows: int = 256, n_cols: int = 128):
    rng = np.random.default_rng(seed + 1)
    return rng.standard_normal(n_cols), rng.standard_normal(n_rows)


# ---- config 2: the matrix-op sweep ---------------------------------------------------------
def _cfg2_elements(rng, shape, p_zero):
    k = rng.integers(1, 256, size=shape)
    z = rng.random(shape) < p_zero
    return np.where(z, 0.0, k / 255.0)


def cfg2_batch_dense(seed: int, batch: int, n_rows: int = 250, n_cols: int = 784, n_templates: int = 64,
                     p_zero: float = 0.8, mutate: float = 0.05) -> np.ndarray:
    """BASELINE.json configs[1], one mini-batch: elements 0 w.p. 0.8 else k/255, k~U{1..255};
    rows copied from 64 per-batch templates with 5% per-element mutation (re-drawn from the same
    element distribution).  Batch b uses its own stream SeedSequence((seed, b)) so any shard of
    the 8192 batches can be generated independently on its rank."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, batch]))
    templates = _cfg2_elements(rng, (n_templates, n_cols), p_zero)
    A = templates[rng.integers(0, n_templates, size=n_rows)]
    mask = rng.random((n_rows, n_cols)) < mutate
    A[mask] = _cfg2_elements(rng, int(mask.sum()), p_zero)
    return A


def cfg2_batches_csr(seed: int, batches, n_rows: int = 250, n_cols: int = 784):
    """Concatenated CSR of the given batch indices, plus the per-batch row counts."""
    ptrs, cols, vals, counts = [], [], [], []
    base = 0
    for b in batches:
        rp, c, v = dense_to_csr(cfg2_batch_dense(seed, int(b), n_rows, n_cols))
        ptrs.append(rp[:-1] + base)
        base += int(rp[-1])
        cols.append(c)
        vals.append(v)
        counts.append(n_rows)
    row_ptr = np.concatenate(ptrs + [np.array([base], np.int64)])
    return row_ptr, np.concatenate(cols), np.concatenate(vals), np.asarray(counts, np.int64)


def cfg2_operands(seed: int, n_batches: int, n_rows: int = 250, n_cols: int = 784):
    """One shared v ~ N(0,1)[n_cols] and a per-batch slice of u ~ N(0,1) (cli.py:321-334)."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, 1 << 30]))
    return rng.standard_normal(n_cols), rng.standard_normal(n_rows * n_batches)
