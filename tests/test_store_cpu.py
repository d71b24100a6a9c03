"""TOCS batch-store layout on the host: the writer reproduces the reference's bytes (golden
store.tocs from tests/golden/make_store_golden.py) and the structural parse applies the
reference's checks (store.py:87-129) in its order."""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "store.json")))
RAW = open(os.path.join(HERE, "golden", "store.tocs"), "rb").read()


def unhex(xs):
    return np.array([np.frombuffer(bytes.fromhex(x), "<f8")[0] for x in xs], dtype=np.float64)


def test_writer_reproduces_reference_bytes(tmp_path):
    from paper_1702_06943_b200.store import save_batch_store

    blocks = [bytes.fromhex(b) for b in GOLD["blocks"]]
    labels = unhex(GOLD["labels"])
    bs = GOLD["batch_size"]
    groups = [labels[i : i + bs] for i in range(0, len(labels), bs)]
    p = tmp_path / "s.tocs"
    save_batch_store(p, blocks, groups, bs, GOLD["n_cols"], GOLD["seed"])
    assert p.read_bytes() == RAW
    with pytest.raises(ValueError):
        save_batch_store(p, blocks, groups[:-1], bs, GOLD["n_cols"], GOLD["seed"])


def test_structural_index():
    from paper_1702_06943_b200.store import _index

    idx, pending = _index(RAW)
    assert pending is None
    assert (idx.batch_size, idx.n_cols, idx.seed, idx.total_rows) == (GOLD["batch_size"], GOLD["n_cols"], GOLD["seed"],
                                                                     len(GOLD["labels"]))
    assert [RAW[o : o + n].hex() for o, n in zip(idx.block_off, idx.block_len)] == GOLD["blocks"]
    assert idx.label_count.tolist() == [7, 7, 7, 3]


@pytest.mark.parametrize("name", sorted(GOLD["variants"]))
def test_structural_errors_match_reference(name):
    """Errors found before any block is decoded are raised by the parse itself; the rest are held
    back (pending) until the blocks before them have been validated on the device."""
    from paper_1702_06943_b200 import errors
    from paper_1702_06943_b200.store import _index

    v = GOLD["variants"][name]
    data = bytes.fromhex(v["data"])
    want = v["raises"]
    try:
        _, pending = _index(data)
    except Exception as e:  # noqa: BLE001
        assert type(e).__name__ == want
        return
    if want in ("BadMagicError", "UnsupportedVersionError") and name.startswith("inner"):
        return  # an inner block error: the device raises it (test_gpu_store.py)
    assert pending is not None and type(pending[1]).__name__ == want, (name, pending)
    assert isinstance(pending[1], getattr(errors, want))
