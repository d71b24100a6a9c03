"""GPU parity for MGD on compressed batches.

Bar (BASELINE.json north_star): per-epoch loss curves within 1e-6 relative of the reference
(here: the reference's own golden curves, tests/golden, and the oracle port on larger seeded
data); final weights within 1e-6 relative (max(1,|w|) scale).
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


def dataset_from_csr(n_cols, rp, c, v, y):
    from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix

    return LabeledDataset(features=SparseRowMatrix.from_csr(n_cols, rp, c, v), labels=y)


GLM_CASES = [i for i, t in enumerate(GOLD["training"]) if t["loss"] != "nn_mse"]  # nn_mse: test_gpu_mlp.py


@pytest.mark.parametrize("i", GLM_CASES)
def test_train_matches_reference_curves(i):
    from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix
    from paper_1702_06943_b200.training import TrainConfig, train

    c = GOLD["training"][i]
    rows = [[(col, struct.unpack("<d", bytes.fromhex(x))[0]) for col, x in r] for r in c["rows"]]
    ds = LabeledDataset(features=SparseRowMatrix(c["n_cols"], rows), labels=unhex(c["labels"]))
    cfg = TrainConfig(loss_kind=c["loss"], batch_size=c["batch_size"], learning_rate=c["lr"], epochs=c["epochs"],
                      seed=c["seed"])
    model, trace = train(ds, cfg)
    want = unhex(c["risks"])
    assert len(trace.risks) == c["epochs"] and len(trace.seconds) == c["epochs"]
    assert np.all(np.abs(np.array(trace.risks) - want) <= REL * np.abs(want)), (trace.risks, want)
    assert within_rel(model.weights, unhex(c["weights"]), REL), max_rel_err(model.weights, unhex(c["weights"]))


def _vs_oracle(oracle, n_cols, rp, c, v, y, loss, bs, lr, epochs, seed=0):
    from paper_1702_06943_b200.training import TrainConfig, train

    w_ref, risks_ref = oracle.train_glm(rp, c, v, y, n_cols, loss, bs, lr, epochs, seed)
    model, trace = train(dataset_from_csr(n_cols, rp, c, v, y),
                         TrainConfig(loss_kind=loss, batch_size=bs, learning_rate=lr, epochs=epochs, seed=seed))
    risks_ref = np.asarray(risks_ref)
    assert np.all(np.abs(np.array(trace.risks) - risks_ref) <= REL * np.abs(risks_ref)), (trace.risks, risks_ref)
    assert within_rel(model.weights, w_ref, REL), max_rel_err(model.weights, w_ref)
    assert within_pure_rel(model.weights, w_ref, REL), pure_rel_err(model.weights, w_ref)
    return trace


def within_pure_rel(got, want, rel):
    """Relative to each weight itself (no max(1, |w|) floor: config-4 weights are ~1e-5), with an
    absolute floor of 1e-12 of the largest weight for entries that are exactly zero in one run."""
    want = np.asarray(want)
    return bool(np.all(np.abs(got - want) <= rel * np.abs(want) + 1e-12 * np.max(np.abs(want), initial=0.0)))


def pure_rel_err(got, want):
    want = np.asarray(want)
    floor = 1e-12 * np.max(np.abs(want), initial=0.0)
    return float(np.max(np.abs(got - want) / (np.abs(want) + floor + 1e-300)))


def test_cfg3_logistic_vs_oracle(oracle):
    from paper_1702_06943_b200 import synth

    rp, c, v, y = synth.cfg3_dataset(20_000, seed=13)
    _vs_oracle(oracle, 68, rp, c, v, y, "logistic", 250, 0.1, 3)


def test_cfg4_hinge_large_m_vs_oracle(oracle):
    """47,236 columns: gradient accumulators and the touched-column set live in global memory."""
    from paper_1702_06943_b200 import synth

    rp, c, v, y = synth.cfg4_dataset(6_000, seed=14)
    _vs_oracle(oracle, 47_236, rp, c, v, y, "hinge", 250, 0.01, 2)


def test_squared_outlier_labels_vs_oracle(oracle):
    """Squared loss with a few labels ~1e6 among O(1) ones: the per-row weights s = z - y span six
    orders of magnitude, so the exact fixed-point gradient's quantum (set by the batch's sum |s|)
    is coarse for the batches holding an outlier -- curves and weights must still match."""
    from paper_1702_06943_b200 import synth

    rp, c, v, _ = synth.cfg3_dataset(20_000, seed=23)
    rng = np.random.default_rng(23)
    w_true = rng.standard_normal(68) * 0.05
    y = np.array([float(np.dot(v[rp[i] : rp[i + 1]], w_true[c[rp[i] : rp[i + 1]]])) for i in range(20_000)])
    y[rng.choice(20_000, 40, replace=False)] *= 1e6
    _vs_oracle(oracle, 68, rp, c, v, y, "squared", 250, 1e-5, 2)


def test_squared_short_last_batch(oracle):
    from helpers import random_alphabet_rows

    rng = np.random.default_rng(21)
    rows = random_alphabet_rows(rng, 1003, 9, 0.6)
    rp, c, v = oracle.rows_to_csr(rows)
    w = rng.standard_normal(9)
    y = np.array([sum(val * w[col] for col, val in r) for r in rows])
    _vs_oracle(oracle, 9, rp, c, v, y, "squared", 64, 1e-3, 3, seed=5)


def test_batch_gradients_vs_oracle(oracle):
    """toc_glm_grad: the summed per-batch gradient the data-parallel trainer all-reduces."""
    import torch

    from paper_1702_06943_b200 import synth
    from paper_1702_06943_b200.distributed import batch_gradients
    from paper_1702_06943_b200.training import DeviceBatches

    rp, c, v, y = synth.cfg3_dataset(3_000, seed=15)
    ds = dataset_from_csr(68, rp, c, v, y)
    batches = DeviceBatches(ds, 250)
    w = np.random.default_rng(1).standard_normal(68) * 0.1
    G = batch_gradients(batches, "logistic", torch.from_numpy(w).cuda()).cpu().numpy()
    for b in range(len(batches.batch_sizes)):
        lo, hi = 250 * b, min(250 * (b + 1), 3000)
        enc = oracle.encode_csr(68, rp[lo : hi + 1] - rp[lo], c[rp[lo] : rp[hi]], v[rp[lo] : rp[hi]])
        t = oracle.Tree.from_encoding(enc)
        z = t.matvec(w)
        s = -y[lo:hi] / (1.0 + np.exp(y[lo:hi] * z))
        want = t.vecmat(s)
        assert within_rel(G[b], want, 1e-9), max_rel_err(G[b], want)


def test_counter_charges_matvec_and_vecmat(oracle):
    from paper_1702_06943_b200 import synth
    from paper_1702_06943_b200.kernels import OpCounter
    from paper_1702_06943_b200.training import TrainConfig, train

    rp, c, v, y = synth.cfg3_dataset(1_000, seed=16)
    counter = OpCounter()
    train(dataset_from_csr(68, rp, c, v, y), TrainConfig("logistic", 250, 0.1, 1), counter)
    order = oracle.shuffle_order(1000, 0)
    want = 0
    for lo in range(0, 1000, 250):
        idx = order[lo : lo + 250]
        lens = np.diff(rp)[idx]
        brp = np.concatenate([[0], np.cumsum(lens)])
        g = np.concatenate([np.arange(rp[i], rp[i + 1]) for i in idx])
        enc = oracle.encode_csr(68, brp, c[g], v[g])
        want += 2 * ((enc.tree_length() - 1) + len(enc.codes))
    assert counter.multiply_adds == want


def _trainer(rp, c, v, y, n_cols, bs, loss, lr, mode, cluster=0):
    from paper_1702_06943_b200.training import DeviceBatches, GlmTrainer

    return GlmTrainer(DeviceBatches(dataset_from_csr(n_cols, rp, c, v, y), bs), loss, lr, mode=mode, cluster=cluster)


@pytest.mark.parametrize("loss,lr,cluster", [("logistic", 0.1, 1), ("logistic", 0.1, 2), ("logistic", 0.1, 4),
                                             ("logistic", 0.1, 8), ("hinge", 0.05, 8), ("squared", 1e-3, 1),
                                             ("squared", 1e-3, 4), ("logistic", 0.1, 16)])
def test_step_images_match_relay(loss, lr, cluster):
    """The cluster epoch over cached step images computes what the relay computes: the same fixed-
    point G per row set; only the per-column sums of value * G run in fp64 in (column, pair, CTA)
    order instead of a fixed-point scatter, so the weights agree to ~1e-15."""
    from paper_1702_06943_b200 import synth

    rp, c, v, y = synth.cfg3_dataset(6_000, seed=31)
    if loss == "squared":
        y = y * 0.5 + 0.25
    ti = _trainer(rp, c, v, y, 68, 250, loss, lr, "images", cluster)
    tr = _trainer(rp, c, v, y, 68, 250, loss, lr, "relay")
    assert ti.mode == "images" and tr.mode == "relay" and ti.cluster == cluster
    for _ in range(2):
        ti.epoch()
        tr.epoch()
        wi, wr = ti.weights(), tr.weights()
        assert within_rel(wi, wr, 1e-12), max_rel_err(wi, wr)
        assert ti.risk() == pytest.approx(tr.risk(), rel=1e-12)


def test_step_images_ragged_batches(oracle):
    """Short last batch, rows of very different lengths, a batch size that is not a multiple of 32."""
    from helpers import random_alphabet_rows

    rng = np.random.default_rng(33)
    rows = random_alphabet_rows(rng, 777, 40, 0.3) + [[(0, 1.0)], [], [(39, 2.0)]] * 5
    rp, c, v = oracle.rows_to_csr(rows)
    y = np.where(rng.random(len(rows)) < 0.5, -1.0, 1.0)
    t = _trainer(rp, c, v, y, 40, 37, "logistic", 0.2, "images")
    assert t.mode == "images" and t.image_build_seconds > 0
    from paper_1702_06943_b200.training import TrainConfig, train

    model, trace = train(dataset_from_csr(40, rp, c, v, y), TrainConfig("logistic", 37, 0.2, 2))
    w_ref, risks_ref = oracle.train_glm(rp, c, v, y, 40, "logistic", 37, 0.2, 2, 0)
    risks_ref = np.asarray(risks_ref)
    assert np.all(np.abs(np.array(trace.risks) - risks_ref) <= REL * np.abs(risks_ref)), (trace.risks, risks_ref)
    assert within_rel(model.weights, w_ref, REL), max_rel_err(model.weights, w_ref)


def test_large_m_uses_parts_and_squared_uses_relay():
    from paper_1702_06943_b200 import synth

    rp, c, v, y = synth.cfg4_dataset(1_000, seed=34)
    t = _trainer(rp, c, v, y, 47_236, 250, "hinge", 0.01, "auto")
    from paper_1702_06943_b200.training import parts_cluster

    assert t.mode == "parts" and t.cluster == parts_cluster() and t.cluster in (8, 16)
    with pytest.raises(ValueError):
        _trainer(rp, c, v, y, 47_236, 250, "hinge", 0.01, "images")
    ts = _trainer(rp, c, v, y * 0.5, 47_236, 250, "squared", 0.01, "auto")
    assert ts.mode == "relay"


@pytest.mark.parametrize("loss,lr,cluster", [("hinge", 0.01, 8), ("logistic", 0.05, 8), ("hinge", 0.01, 16)])
def test_parts_match_relay(loss, lr, cluster):
    """The large-n_cols cluster epoch (per-CTA part images, global fixed-point gradient) computes what
    the relay computes, up to the per-CTA rounding of the fixed-point contributions (~1e-15)."""
    from paper_1702_06943_b200 import synth

    rp, c, v, y = synth.cfg4_dataset(3_000, seed=35)
    tp = _trainer(rp, c, v, y, 47_236, 250, loss, lr, "parts", cluster)
    tr = _trainer(rp, c, v, y, 47_236, 250, loss, lr, "relay")
    assert tp.mode == "parts" and tp.cluster == cluster
    for _ in range(2):
        tp.epoch()
        tr.epoch()
        wp, wr = tp.weights(), tr.weights()
        assert within_rel(wp, wr, 1e-12), max_rel_err(wp, wr)
        assert tp.risk() == pytest.approx(tr.risk(), rel=1e-12)
    assert int(tp.gacc.abs().sum().item()) == 0  # the fixed-point gradient is left cleared


def test_parts_ragged_batches(oracle):
    """Parts with short / empty CTA row ranges: 13-row batches over an 8-CTA cluster, a short last batch."""
    from helpers import random_alphabet_rows

    rng = np.random.default_rng(36)
    rows = random_alphabet_rows(rng, 300, 40, 0.3) + [[], [(39, 1.0)]]
    rp, c, v = oracle.rows_to_csr(rows)
    y = np.where(rng.random(len(rows)) < 0.5, -1.0, 1.0)
    from paper_1702_06943_b200.training import DeviceBatches, GlmTrainer

    tp = GlmTrainer(DeviceBatches(dataset_from_csr(40, rp, c, v, y), 13), "hinge", 0.1, mode="parts", cluster=8)
    tr = GlmTrainer(DeviceBatches(dataset_from_csr(40, rp, c, v, y), 13), "hinge", 0.1, mode="relay")
    for _ in range(2):
        tp.epoch()
        tr.epoch()
    assert within_rel(tp.weights(), tr.weights(), 1e-12), max_rel_err(tp.weights(), tr.weights())


@pytest.mark.parametrize("loss", ["logistic", "hinge", "squared"])
def test_dp_epoch_graph_world1_nccl(oracle, loss):
    """The device DP-MGD epoch (toc_glm_grad -> NCCL all-reduce -> update per step, one CUDA graph
    per epoch) on a one-rank NCCL group equals the eager sequence and the oracle trainer."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    from paper_1702_06943_b200 import synth
    from paper_1702_06943_b200.distributed import train_data_parallel
    from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix
    from paper_1702_06943_b200.training import TrainConfig, train

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rp, c, v, y = synth.cfg3_dataset(4000, seed=21)
        if loss == "squared":
            y = y * 0.5 + 0.1
        ds = LabeledDataset(features=SparseRowMatrix.from_csr(68, rp, c, v), labels=y)
        cfg = TrainConfig(loss, 250, 0.05, 2)
        m_g, t_g = train_data_parallel(ds, cfg, 1, 0, graph=True, fused=False)
        m_e, t_e = train_data_parallel(ds, cfg, 1, 0, graph=False, fused=False)
        assert t_g.graph and not t_e.graph and t_g.mode == ("grad" if loss == "squared" else "parts")
        assert np.array_equal(m_g.weights, m_e.weights)
        # the exchange fused into the cluster epoch kernel (NVLink peer memory): at world 1 the very
        # same arithmetic as the single-GPU cluster epoch, so bit-identical to train()
        m_f, t_f = train_data_parallel(ds, cfg, 1, 0)
        assert t_f.mode == "fused"
        m_1, t_1 = train(ds, cfg)
        assert np.array_equal(m_f.weights, m_1.weights)
        assert np.allclose(m_f.weights, m_g.weights, rtol=1e-9, atol=1e-12)
        w_ref, risks = oracle.train_glm(rp, c, v, y, 68, loss, 250, 0.05, 2, 0)
        assert np.allclose(m_g.weights, w_ref, rtol=1e-9, atol=1e-12), np.max(np.abs(m_g.weights - w_ref))
        assert np.allclose(t_g.risks, risks, rtol=1e-6)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("loss,world", [("logistic", 2), ("hinge", 2), ("logistic", 4)])
def test_dp_fused_exchange_emulated_ranks(oracle, loss, world):
    """The fused NVLink gradient exchange of toc_glm_epoch_images_dp with `world` ranks, run on one
    GPU as one cooperative launch of `world` clusters (rank = cluster; receive slots and flags in
    device memory).  Every rank's weights after 3 back-to-back epochs (the receive slot alternates
    with the global step sequence, no host barrier between epochs) equal the reference trainer at
    the global batch size 250 * world, and equal each other bit for bit."""
    from paper_1702_06943_b200 import synth
    from paper_1702_06943_b200.distributed import EmulatedDPEpochs
    from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix

    n = 250 * world * 10 - 100  # last global step short (the last rank holds 150 rows)
    rp, c, v, y = synth.cfg3_dataset(n, seed=41)
    ds = LabeledDataset(features=SparseRowMatrix.from_csr(68, rp, c, v), labels=y)
    lr, epochs = 0.05, 3
    run = EmulatedDPEpochs(ds, 250, world, loss, lr, seed=0)
    for _ in range(epochs):
        ws = run.epoch()
    got = [w.cpu().numpy()[:68] for w in ws]
    w_ref, _ = oracle.train_glm(rp, c, v, y, 68, loss, 250 * world, lr, epochs, 0)
    for r in range(world):
        assert within_rel(got[r], w_ref, 1e-9), max_rel_err(got[r], w_ref)
        assert np.array_equal(got[r], got[0])
