"""GPU parity for the network trainers on compressed batches.

* nn_mse (the reference's own net): against the reference's golden curve and weights (1e-6).
* the config-5 MLP (784-200-10, ReLU, softmax-CE): against the oracle's CPU restatement (1e-6);
  the reference has no such model, so this one is not pinned to reference outputs.
"""

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
REL = 1e-6


def unhex(xs):
    return np.array([struct.unpack("<d", bytes.fromhex(x))[0] for x in xs], dtype=np.float64)


def test_nn_mse_matches_reference_curve():
    from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix
    from paper_1702_06943_b200.training import NnModel, TrainConfig, train

    c = [t for t in GOLD["training"] if t["loss"] == "nn_mse"][0]
    rows = [[(col, struct.unpack("<d", bytes.fromhex(x))[0]) for col, x in r] for r in c["rows"]]
    ds = LabeledDataset(features=SparseRowMatrix(c["n_cols"], rows), labels=unhex(c["labels"]))
    cfg = TrainConfig("nn_mse", c["batch_size"], c["lr"], c["epochs"], seed=c["seed"], hidden_units=c["hidden_units"])
    model, trace = train(ds, cfg)
    assert isinstance(model, NnModel)
    want = unhex(c["risks"])
    assert np.all(np.abs(np.array(trace.risks) - want) <= REL * np.abs(want)), (trace.risks, want)
    assert within_rel(model.w1.ravel(), unhex(c["w1"]), REL)
    assert within_rel(model.w2.ravel(), unhex(c["w2"]), REL)


def test_cfg5_mlp_vs_cpu_restatement(oracle):
    from paper_1702_06943_b200 import synth
    from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix
    from paper_1702_06943_b200.mlp import train_mlp

    rp, c, v, y = synth.cfg5_dataset(1000, seed=9)
    ds = LabeledDataset(features=SparseRowMatrix.from_csr(784, rp, c, v), labels=y)
    model, trace = train_mlp(ds, hidden=32, classes=10, batch_size=250, learning_rate=0.05, epochs=2, seed=0)
    (w1, b1, w2, b2), risks = oracle.train_mlp(rp, c, v, y, 784, 32, 10, 250, 0.05, 2, 0)
    assert np.all(np.abs(np.array(trace.risks) - np.array(risks)) <= REL * np.abs(risks)), (trace.risks, risks)
    for got, want in ((model.w1, w1), (model.b1, b1), (model.w2, w2), (model.b2, b2)):
        assert within_rel(got, want, REL), max_rel_err(got, want)


def test_matmat_per_batch_scratch_covers_every_batch(oracle):
    """Per-batch matmat (the MLP step's call) sizes its global-table scratch for the largest batch,
    not the first: a small first batch followed by a > 65536-node one."""
    import torch

    from helpers import random_alphabet_rows

    from paper_1702_06943_b200.arena import BlockArena

    rng = np.random.default_rng(12)
    small = oracle.encode_rows(400, random_alphabet_rows(rng, 5, 400, 0.5, 64))
    base = random_alphabet_rows(rng, 30, 400, 0.9, 64)
    big = oracle.encode_rows(400, [base[i % 30] if i % 3 else random_alphabet_rows(rng, 1, 400, 0.9, 64)[0]
                                   for i in range(600)])
    assert big.tree_length() > 65536
    arena = BlockArena.from_bytes([oracle.serialize(small), oracle.serialize(big)])
    M = torch.randn(400, 3, dtype=torch.float64, device="cuda")
    for b, enc in enumerate((small, big)):
        got = arena.matmat(0, M, 3, batch=b).cpu().numpy()
        want = oracle.Tree.from_encoding(enc).matmat_right(M.cpu().numpy())
        assert np.allclose(got, want, rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("n,batch,hidden", [(1000, 300, 200), (777, 250, 40), (500, 250, 13)])
def test_cfg5_native_epoch_vs_cpu_restatement(oracle, n, batch, hidden):
    """The native epoch (toc_mlp_epoch: DMMA first layer over decoded tiles, fused tail) against the
    oracle's step: ragged last batches, hidden sizes that leave partial 8-wide tiles."""
    from paper_1702_06943_b200 import synth
    from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix
    from paper_1702_06943_b200.mlp import train_mlp

    rp, c, v, y = synth.cfg5_dataset(n, seed=11)
    ds = LabeledDataset(features=SparseRowMatrix.from_csr(784, rp, c, v), labels=y)
    model, trace = train_mlp(ds, hidden=hidden, classes=10, batch_size=batch, learning_rate=0.05, epochs=2, seed=3)
    (w1, b1, w2, b2), risks = oracle.train_mlp(rp, c, v, y, 784, hidden, 10, batch, 0.05, 2, 3)
    assert np.all(np.abs(np.array(trace.risks) - np.array(risks)) <= REL * np.abs(risks)), (trace.risks, risks)
    for got, want in ((model.w1, w1), (model.b1, b1), (model.w2, w2), (model.b2, b2)):
        assert within_rel(got, want, REL), max_rel_err(got, want)


def test_cfg5_native_equals_per_step_path():
    """Both implementations of the step: the same curve and weights to fp64 rounding."""
    from paper_1702_06943_b200 import synth
    from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix
    from paper_1702_06943_b200.mlp import train_mlp

    rp, c, v, y = synth.cfg5_dataset(1500, seed=5)
    ds = LabeledDataset(features=SparseRowMatrix.from_csr(784, rp, c, v), labels=y)
    m1, t1 = train_mlp(ds, hidden=200, epochs=2, native=True)
    m2, t2 = train_mlp(ds, hidden=200, epochs=2, native=False)
    assert np.allclose(t1.risks, t2.risks, rtol=1e-9, atol=0)
    for a, b in zip((m1.w1, m1.b1, m1.w2, m1.b2), (m2.w1, m2.b1, m2.w2, m2.b2)):
        assert within_rel(a, b, 1e-9), max_rel_err(a, b)


@pytest.mark.parametrize("n_rows,batch", [(1000, 250), (1130, 250)])
def test_dp_mlp_world1_nccl(oracle, n_rows, batch):
    """The data-parallel config-5 trainer (toc_mlp_step_grad -> NCCL all-reduce -> update, one CUDA
    graph per epoch) on a one-rank NCCL group: graph == eager bit for bit, == the single-GPU native
    trainer to fp64 rounding, == the oracle's CPU restatement (1e-6); includes a short last batch."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_1702_06943_b200 import synth
    from paper_1702_06943_b200.distributed import train_mlp_data_parallel
    from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix
    from paper_1702_06943_b200.mlp import train_mlp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rp, c, v, y = synth.cfg5_dataset(n_rows, seed=9)
        ds = LabeledDataset(features=SparseRowMatrix.from_csr(784, rp, c, v), labels=y)
        kw = dict(hidden=40, classes=10, batch_size=batch, learning_rate=0.05, epochs=2, seed=0)
        mg, tg = train_mlp_data_parallel(ds, 1, 0, graph=True, **kw)
        me, te = train_mlp_data_parallel(ds, 1, 0, graph=False, **kw)
        assert tg.graph and not te.graph
        for a, b in ((mg.w1, me.w1), (mg.b1, me.b1), (mg.w2, me.w2), (mg.b2, me.b2)):
            assert np.array_equal(a, b)
        mn, tn = train_mlp(ds, **kw)
        for a, b in ((mg.w1, mn.w1), (mg.b1, mn.b1), (mg.w2, mn.w2), (mg.b2, mn.b2)):
            assert within_rel(a, b, 1e-9), max_rel_err(a, b)
        (w1, b1, w2, b2), risks = oracle.train_mlp(rp, c, v, y, 784, 40, 10, batch, 0.05, 2, 0)
        assert np.all(np.abs(np.array(tg.risks) - np.array(risks)) <= REL * np.abs(risks)), (tg.risks, risks)
        for got, want in ((mg.w1, w1), (mg.b1, b1), (mg.w2, w2), (mg.b2, b2)):
            assert within_rel(got, want, REL), max_rel_err(got, want)
    finally:
        dist.destroy_process_group()


def test_mlp_epoch_pdl_matches_plain_launches():
    """The native epoch with programmatic dependent launch (the default) equals the same epoch
    launched without it, bit for bit."""
    from paper_1702_06943_b200 import _native as N, synth
    from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix
    from paper_1702_06943_b200.mlp import train_mlp

    rp, c, v, y = synth.cfg5_dataset(1500, seed=4)
    ds = LabeledDataset(features=SparseRowMatrix.from_csr(784, rp, c, v), labels=y)
    kw = dict(hidden=40, classes=10, batch_size=250, learning_rate=0.05, epochs=2, seed=0)
    try:
        N.lib().toc_mlp_set_pdl(0)
        m0, t0 = train_mlp(ds, **kw)
    finally:
        N.lib().toc_mlp_set_pdl(1)
    m1, t1 = train_mlp(ds, **kw)
    for a, b in ((m0.w1, m1.w1), (m0.b1, m1.b1), (m0.w2, m1.w2), (m0.b2, m1.b2)):
        assert np.array_equal(a, b)
    assert t0.risks == t1.risks

