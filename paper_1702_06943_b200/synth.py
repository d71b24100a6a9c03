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


# ---- config 3: logistic-regression MGD data -------------------------------------------------
def cfg3_dataset(n_rows: int = 2_000_000, n_cols: int = 68, seed: int = 3, n_levels: int = 16,
                 zipf_s: float = 1.5, flip: float = 0.05, chunk: int = 250_000):
    """BASELINE.json configs[2]: each column a categorical integer 0..15 with Zipf(1.5)
    frequencies (category k has weight (k+1)^-1.5, so 0 -- dropped by the sparse encoding -- is the
    most frequent), stored as float64.  Labels sign(x . w*) with w* ~ N(0,1)^68 (0 -> +1), then 5%
    flipped.  Returns (row_ptr, cols, vals, labels)."""
    rng = np.random.default_rng(seed)
    p = _zipf_probs(n_levels, zipf_s)
    w_star = rng.standard_normal(n_cols)
    ptrs, cols, vals, labels = [np.zeros(1, np.int64)], [], [], []
    base = 0
    for lo in range(0, n_rows, chunk):
        k = min(chunk, n_rows - lo)
        X = rng.choice(n_levels, size=(k, n_cols), p=p).astype(np.float64)
        z = X @ w_star
        y = np.where(z >= 0, 1.0, -1.0)
        y[rng.random(k) < flip] *= -1.0
        rp, c, v = dense_to_csr(X)
        ptrs.append(rp[1:] + base)
        base += int(rp[-1])
        cols.append(c)
        vals.append(v)
        labels.append(y)
    return np.concatenate(ptrs), np.concatenate(cols), np.concatenate(vals), np.concatenate(labels)


# ---- config 4: sparse high-dimensional hinge MGD data --------------------------------------
def cfg4_dataset(n_rows: int = 800_000, n_cols: int = 47_236, seed: int = 4, nnz: int = 75,
                 zipf_s: float = 1.1, levels: int = 1000, chunk: int = 50_000):
    """BASELINE.json configs[3]: ~75 distinct columns per row with Zipf(1.1) column popularity
    (drawn without replacement: 4x oversampling with replacement, de-duplicated, then a random 75
    of the distinct ones), raw values U(0,1], each row L2-normalised and THEN quantised to 1000
    levels in (0,1] (q = ceil(1000 x) / 1000) so the value alphabet stays small.
    Labels sign(x . w*) for a random sparse hyperplane w* (10% of columns N(0,1)), 0 -> +1."""
    rng = np.random.default_rng(seed)
    p = _zipf_probs(n_cols, zipf_s)
    perm = rng.permutation(n_cols)  # popularity rank -> column id
    cdf = np.cumsum(p)
    w_star = np.where(rng.random(n_cols) < 0.1, rng.standard_normal(n_cols), 0.0)
    ptrs, cols_out, vals_out, labels = [np.zeros(1, np.int64)], [], [], []
    base = 0
    for lo in range(0, n_rows, chunk):
        k = min(chunk, n_rows - lo)
        cand = perm[np.minimum(np.searchsorted(cdf, rng.random((k, 4 * nnz))), n_cols - 1)]
        cand.sort(axis=1)
        dup = np.zeros_like(cand, dtype=bool)
        dup[:, 1:] = cand[:, 1:] == cand[:, :-1]
        prio = rng.random(cand.shape)
        prio[dup] = 2.0  # duplicates last
        pick = np.argsort(prio, axis=1)[:, :nnz]
        chosen = np.take_along_axis(cand, pick, axis=1)
        ok = np.take_along_axis(prio, pick, axis=1) < 2.0
        chosen = np.where(ok, chosen, -1)
        chosen.sort(axis=1)
        raw = rng.random(chosen.shape)
        raw = np.where(chosen >= 0, raw, 0.0)
        raw /= np.sqrt((raw * raw).sum(axis=1, keepdims=True))
        q = np.where(chosen >= 0, np.maximum(np.ceil(raw * levels), 1.0) / levels, 0.0)
        keep = chosen >= 0
        lens = keep.sum(axis=1)
        rp = np.zeros(k + 1, np.int64)
        np.cumsum(lens, out=rp[1:])
        c = chosen[keep].astype(np.int32)
        v = q[keep]
        z = np.add.reduceat(v * w_star[c], rp[:-1]) if len(v) else np.zeros(k)
        z[lens == 0] = 0.0
        labels.append(np.where(z >= 0, 1.0, -1.0))
        ptrs.append(rp[1:] + base)
        base += int(rp[-1])
        cols_out.append(c)
        vals_out.append(v)
    return np.concatenate(ptrs), np.concatenate(cols_out), np.concatenate(vals_out), np.concatenate(labels)


# ---- config 5: MLP inputs ---------------------------------------------------------------------
def cfg5_teacher(n_in: int = 784, hidden: int = 200, classes: int = 10, seed: int = 5):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((n_in, hidden)) / np.sqrt(n_in), rng.standard_normal(hidden) * 0.1,
            rng.standard_normal((hidden, classes)) / np.sqrt(hidden))


def cfg5_batches(n_rows: int, seed: int = 5, batch: int = 250, n_cols: int = 784):
    """BASELINE.json configs[4] (decision): rows "generated as in config 1", widened to
    784 columns -- ONE 16-value Zipf(1.2) vocabulary U[-1,1] and 32 template rows for the whole
    dataset (config 1's recipe), each row a random template with 10% of its elements re-drawn --
    and raw teacher logits of a random 784-200-10 ReLU MLP.  Rows are generated in chunks of
    `batch` with their own seeded streams.  Yields (row_ptr, cols, vals, logits) per chunk."""
    W1, b1, W2 = cfg5_teacher(n_cols, seed=seed)
    rng = np.random.default_rng(np.random.SeedSequence([seed, 0x7e]))
    words = rng.uniform(-1.0, 1.0, 16)
    p = _zipf_probs(16, 1.2)
    templates = words[rng.choice(16, size=(32, n_cols), p=p)]
    for lo in range(0, n_rows, batch):
        k = min(batch, n_rows - lo)
        r = np.random.default_rng(np.random.SeedSequence([seed, lo]))
        A = templates[r.integers(0, 32, size=k)]
        mask = r.random((k, n_cols)) < 0.1
        A[mask] = words[r.choice(16, size=int(mask.sum()), p=p)]
        logits = np.maximum(A @ W1 + b1, 0.0) @ W2
        rp, c, v = dense_to_csr(A)
        yield rp, c, v, logits


def cfg5_dataset(n_rows: int, seed: int = 5):
    """The config-5 rows (cfg5_batches) with labels argmax of the teacher logits centred per class
    over the whole dataset (so the ten classes come out near uniform)."""
    ptrs, cols, vals, logits, base = [np.zeros(1, np.int64)], [], [], [], 0
    for rp, c, v, lg in cfg5_batches(n_rows, seed):
        ptrs.append(rp[1:] + base)
        base += int(rp[-1])
        cols.append(c)
        vals.append(v)
        logits.append(lg)
    lg = np.concatenate(logits) if logits else np.zeros((0, 10))
    labels = np.argmax(lg - lg.mean(axis=0), axis=1).astype(np.float64)
    return np.concatenate(ptrs), np.concatenate(cols), np.concatenate(vals), labels
