"""Input factories for the tests (numpy, seeded)."""

from __future__ import annotations

import numpy as np


def random_alphabet_rows(rng, n_rows, n_cols, density, alphabet_size=16, integer_alphabet=False):
    """Random sparse rows over a small value alphabet (the shape of the reference's own test
    factory, reference tests/conftest.py:45-67, written independently)."""
    if integer_alphabet:
        alphabet = np.arange(1, alphabet_size + 1, dtype=np.float64)
    else:
        alphabet = np.zeros(0)
        while len(np.unique(alphabet)) != alphabet_size:
            alphabet = np.round(rng.standard_normal(alphabet_size) * 4, 3)
            alphabet = alphabet[alphabet != 0.0]
    rows = []
    for _ in range(n_rows):
        cols = np.flatnonzero(rng.random(n_cols) < density)
        vals = rng.choice(alphabet, size=len(cols))
        rows.append([(int(c), float(v)) for c, v in zip(cols, vals)])
    return rows


TOY_ROWS = [
    [(0, 1.0), (1, 2.0), (2, 3.0), (3, 4.0), (4, 5.0)],
    [(0, 6.0), (1, 7.0), (2, 3.0), (3, 4.0), (4, 5.0)],
]
TREE_ROWS = [
    [(1, 1.1), (2, 2.0), (3, 3.0), (4, 1.4)],
    [(1, 1.1), (2, 2.0), (3, 3.0), (4, 1.4)],
    [(2, 1.1), (3, 3.0), (4, 1.4)],
]
