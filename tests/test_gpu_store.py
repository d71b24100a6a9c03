"""GPU parity for TOCS batch stores (reference store.py:59-129, cli.py:177-221): loading the
reference's golden store decodes to its rows and labels bit for bit; every damaged variant raises
the exception class the reference raised on it (tests/golden/store.json); streaming a store
through the device in chunks equals loading it whole; verify accepts a faithful store and names
the first mismatch otherwise."""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "store.json")))
RAW_PATH = os.path.join(HERE, "golden", "store.tocs")


def unhex(xs):
    return np.array([np.frombuffer(bytes.fromhex(x), "<f8")[0] for x in xs], dtype=np.float64)


def gold_rows():
    return [[(c, float(unhex([x])[0])) for c, x in r] for r in GOLD["rows"]]


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def test_load_golden_store():
    from paper_1702_06943_b200.codec import decode
    from paper_1702_06943_b200.store import load_batch_store

    st = load_batch_store(RAW_PATH)
    assert (st.batch_size, st.n_cols, st.seed, st.total_rows) == (7, 9, -5, 24)
    rows = [r for enc, _ in st.batches for r in decode(enc).rows]
    want = gold_rows()
    assert [[c for c, _ in r] for r in rows] == [[c for c, _ in r] for r in want]
    assert np.array_equal(bits([v for r in rows for _, v in r]), bits([v for r in want for _, v in r]))
    labels = np.concatenate([lab for _, lab in st.batches])
    assert labels.tobytes() == unhex(GOLD["labels"]).tobytes()


@pytest.mark.parametrize("name", sorted(GOLD["variants"]))
def test_damaged_store_raises_reference_class(tmp_path, name):
    from paper_1702_06943_b200.store import BatchStoreStream, load_batch_store

    v = GOLD["variants"][name]
    p = tmp_path / "d.tocs"
    p.write_bytes(bytes.fromhex(v["data"]))
    with pytest.raises(Exception) as ei:
        load_batch_store(p)
    assert type(ei.value).__name__ == v["raises"]
    with pytest.raises(Exception) as ei:  # the streaming reader agrees, for every chunk size
        with BatchStoreStream(p, chunk=2) as st:
            for _ in st:
                pass
    assert type(ei.value).__name__ == v["raises"]


def _cfg2_store(tmp_path, n_batches=23, seed=4):
    from paper_1702_06943_b200 import synth
    from paper_1702_06943_b200.codec import compress_csr
    from paper_1702_06943_b200.store import save_arena_store

    parts = [synth.dense_to_csr(synth.cfg2_batch_dense(seed, b)) for b in range(n_batches)]
    rp = np.concatenate([[0], np.cumsum(np.concatenate([np.diff(p[0]) for p in parts]))]).astype(np.int64)
    c = np.concatenate([p[1] for p in parts])
    v = np.concatenate([p[2] for p in parts])
    y = np.random.default_rng(seed).standard_normal(250 * n_batches)
    arena = compress_csr(784, rp, c, v, np.arange(0, 250 * n_batches + 1, 250, dtype=np.int64))
    path = tmp_path / "cfg2.tocs"
    save_arena_store(path, arena, y, 250, 17)
    return path, arena, rp, c, v, y


def test_stream_chunks_equal_whole(tmp_path):
    import torch

    from paper_1702_06943_b200.store import BatchStoreStream, decompress_store, load_batch_store

    path, arena, rp, c, v, y = _cfg2_store(tmp_path)
    st = load_batch_store(path)
    assert len(st.batches) == 23 and st.seed == 17
    seen = 0
    with BatchStoreStream(path, chunk=5) as s:
        for ch in s:
            a = ch.arena
            for b in range(a.n_blocks):
                got = a.data[int(a.block_off[b]) : int(a.block_off[b]) + int(a.block_len[b])]
                want = arena.data[int(arena.block_off[ch.first + b]) : int(arena.block_off[ch.first + b])
                                  + int(arena.block_len[ch.first + b])]
                assert torch.equal(got, want)
            assert ch.labels.cpu().numpy().tobytes() == y[250 * ch.first : 250 * (ch.first + a.n_blocks)].tobytes()
            seen += a.n_blocks
    assert seen == 23
    drp, dc, dv, dy = decompress_store(path)
    assert np.array_equal(drp, rp) and np.array_equal(dc, c) and np.array_equal(bits(dv), bits(v))
    assert dy.tobytes() == y.tobytes()


def test_stream_products_match_in_memory(tmp_path):
    """Out-of-core A.v / v^T.A: chunk by chunk from the store equals the in-memory arena."""
    import torch

    from paper_1702_06943_b200.store import BatchStoreStream

    path, arena, *_ = _cfg2_store(tmp_path, n_batches=9, seed=6)
    v = torch.randn(784, dtype=torch.float64, device="cuda")
    u = torch.randn(arena.n_rows_total, dtype=torch.float64, device="cuda")
    R, O = arena.linalg(3, v=v, u=u)
    with BatchStoreStream(path, chunk=4) as s:
        for ch in s:
            a = ch.arena
            r0 = 250 * ch.first
            Rc, Oc = a.linalg(3, v=v, u=u[r0 : r0 + a.n_rows_total].contiguous())
            assert torch.equal(Rc, R[r0 : r0 + a.n_rows_total])
            assert torch.equal(Oc, O[ch.first : ch.first + a.n_blocks])


def test_verify_store(tmp_path):
    from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix
    from paper_1702_06943_b200.store import VerificationError, verify_store

    path, arena, rp, c, v, y = _cfg2_store(tmp_path, n_batches=6, seed=8)
    ds = LabeledDataset(features=SparseRowMatrix.from_csr(784, rp, c, v), labels=y)
    assert verify_store(path, ds) == 1500
    y2 = y.copy()
    y2[777] += 1.0
    with pytest.raises(VerificationError, match="row 777: label differs"):
        verify_store(path, LabeledDataset(features=ds.features, labels=y2))
    v2 = v.copy()
    v2[rp[1203] + 2] = 0.5  # a value of dataset row 1203 (batch 4)
    with pytest.raises(VerificationError, match="batch 4, dataset row 1203: decoded row differs"):
        verify_store(path, LabeledDataset(features=SparseRowMatrix.from_csr(784, rp, c, v2), labels=y))
    with pytest.raises(VerificationError, match="columns"):
        verify_store(path, LabeledDataset(features=SparseRowMatrix.from_csr(785, rp, c, v), labels=y))


def test_train_from_store_matches_oracle(tmp_path, oracle):
    """Streaming MGD from a store (3 chunks of 7 batches) equals the oracle trainer: the store holds
    the seed-0 shuffled dataset's batches in order, exactly the batches train(seed=0) uses, and the
    mean risk does not depend on row order."""
    from conftest import max_rel_err, within_rel

    from paper_1702_06943_b200 import synth
    from paper_1702_06943_b200.codec import compress_csr
    from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix
    from paper_1702_06943_b200.store import save_arena_store
    from paper_1702_06943_b200.training import TrainConfig, shuffle_once, train_store

    rp, c, v, y = synth.cfg3_dataset(5_000, seed=41)
    ds = shuffle_once(LabeledDataset(features=SparseRowMatrix.from_csr(68, rp, c, v), labels=y), 0)
    s = ds.features
    arena = compress_csr(68, s.row_ptr, s.cols, s.vals, np.concatenate([np.arange(0, 5000, 250), [5000]]))
    path = tmp_path / "cfg3.tocs"
    save_arena_store(path, arena, ds.labels, 250, 0)
    m_store, t_store = train_store(path, TrainConfig("logistic", 250, 0.1, 3), chunk=7)
    w_ref, risks_ref = oracle.train_glm(rp, c, v, y, 68, "logistic", 250, 0.1, 3, 0)
    risks_ref = np.asarray(risks_ref)
    assert np.all(np.abs(np.array(t_store.risks) - risks_ref) <= 1e-6 * np.abs(risks_ref)), (t_store.risks, risks_ref)
    assert within_rel(m_store.weights, w_ref, 1e-6), max_rel_err(m_store.weights, w_ref)
    assert len(t_store.seconds) == 3
