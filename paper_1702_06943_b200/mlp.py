"""Network training on TOC-compressed batches (reference training.py:81-98, 224-228, 284-293;
BASELINE.json configs[4]).

The first layer touches the features only through A.W1 (matmat_right, forward) and
(delta^T . A)^T (matmat_left, weight gradient); both run on the compressed batches with the
toc_matmat kernels.  The rest of the network is small and dense (h x k weights) and runs as torch
ops on the same stream (cuBLAS / elementwise kernels): it is not part of the TOC hot path.

* ``train_nn``: the reference's own net (loss_kind="nn_mse"): sigmoid hidden layer, linear scalar
  output, half squared error, no biases, uniform init from default_rng(seed) (training.py:319-333).
* ``train_mlp``: the config-5 classifier (784-200-10, ReLU, softmax cross-entropy, biases, Xavier
  uniform init from seed 0).  The reference has no such model: its parity is against a CPU
  restatement (tests), not against reference outputs.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .matrix import LabeledDataset


@dataclass
class NnModel:
    """One hidden layer with logistic-sigmoid activation, linear output (training.py:81-98)."""

    w1: np.ndarray
    w2: np.ndarray

    def __post_init__(self):
        self.w1 = np.asarray(self.w1, dtype=np.float64)
        self.w2 = np.asarray(self.w2, dtype=np.float64)
        if self.w1.ndim != 2 or self.w2.ndim != 2 or self.w2.shape != (self.w1.shape[1], 1):
            raise ValueError(f"layer shapes do not chain: w1 {self.w1.shape}, w2 {self.w2.shape}")

    @property
    def hidden_units(self) -> int:
        return self.w1.shape[1]


@dataclass
class MlpModel:
    """784-200-10 style classifier: ReLU hidden layer, softmax output, biases."""

    w1: np.ndarray
    b1: np.ndarray
    w2: np.ndarray
    b2: np.ndarray


def init_nn(n_cols: int, hidden: int, seed: int):
    """training.py:327-333: uniform(+-1/sqrt(m)) and uniform(+-1/sqrt(h)) from default_rng(seed)."""
    rng = np.random.default_rng(seed)
    s1 = 1.0 / math.sqrt(max(n_cols, 1))
    s2 = 1.0 / math.sqrt(hidden)
    return rng.uniform(-s1, s1, size=(n_cols, hidden)), rng.uniform(-s2, s2, size=(hidden, 1))


def init_mlp(n_in: int, hidden: int, classes: int, seed: int = 0):
    """Xavier/Glorot uniform weights, zero biases (config 5)."""
    rng = np.random.default_rng(seed)
    l1 = math.sqrt(6.0 / (n_in + hidden))
    l2 = math.sqrt(6.0 / (hidden + classes))
    return (rng.uniform(-l1, l1, size=(n_in, hidden)), np.zeros(hidden),
            rng.uniform(-l2, l2, size=(hidden, classes)), np.zeros(classes))


class _Net:
    """Device-resident batches + per-step first-layer products on them."""

    def __init__(self, dataset: LabeledDataset, batch_size: int, seed: int, step_cache: bool = False):
        from .training import DeviceBatches, shuffle_once

        self.torch = N.require_cuda()
        self.batches = DeviceBatches(shuffle_once(dataset, seed), batch_size)
        self.arena = self.batches.arena
        # once per run: the compact step cache the native epoch decodes from (with the TOC1 codes),
        # else the node records both per-step first-layer products read
        self.step_cache = step_cache and self.arena.build_mlpcache()
        if not self.step_cache:
            self.arena.build_matcache()
        self.rb = self.arena.row_base
        self.nrows = self.arena.meta["n_rows"].astype(np.int64)
        lens = np.diff(np.asarray(dataset.features.row_ptr))
        self.dense_rows = bool(len(lens) and np.all(lens == dataset.n_cols))  # every row has all columns

    def first_layer(self, b, W1, h):  # A_b . W1
        return self.arena.matmat(0, W1, h, batch=b)

    def first_layer_grad(self, b, delta, h):  # (delta^T . A_b)^T  [m x h]
        return self.arena.matmat(1, delta, h, batch=b)[0].t()

    def labels(self, b):
        return self.batches.labels[int(self.rb[b]) : int(self.rb[b]) + int(self.nrows[b])]


def train_nn(dataset: LabeledDataset, config, counter=None):
    """training.train for loss_kind='nn_mse' on the device (training.py:336-361)."""
    from .training import LossTrace

    net = _Net(dataset, config.batch_size, config.seed)
    torch = net.torch
    w1_h, w2_h = init_nn(dataset.n_cols, config.hidden_units, config.seed)
    W1 = torch.from_numpy(w1_h).cuda()
    W2 = torch.from_numpy(w2_h).cuda()
    h = config.hidden_units
    lr = float(config.learning_rate)
    trace = LossTrace()
    y_all = net.batches.labels
    for _ in range(config.epochs):
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        for b in range(net.arena.n_blocks):
            y = net.labels(b)
            h1 = torch.sigmoid(net.first_layer(b, W1, h))
            err = h1 @ W2 - y[:, None]
            g_w2 = h1.t() @ err
            delta = ((err @ W2.t()) * h1 * (1.0 - h1)).contiguous()
            g_w1 = net.first_layer_grad(b, delta, h)
            step = lr / int(net.nrows[b])
            W1 = W1 - step * g_w1
            W2 = W2 - step * g_w2
        end.record()
        end.synchronize()
        trace.seconds.append(start.elapsed_time(end) / 1e3)
        h1 = torch.sigmoid(net.arena.matmat(0, W1, h))
        yhat = (h1 @ W2)[:, 0]
        trace.risks.append(float(torch.mean(0.5 * (y_all - yhat) ** 2).item()))
    if counter is not None:  # matmat_right + matmat_left per step, width h (test_training.py:217-223)
        m = net.arena.meta
        per = (m["n_pairs"].astype(np.int64) + m["n_derived"] + m["n_codes"]).sum()
        counter.multiply_adds += int(2 * per * h * config.epochs)
    return NnModel(w1=W1.cpu().numpy(), w2=W2.cpu().numpy()), trace


def _native_epoch(net, hidden: int, classes: int):
    """toc_mlp_epoch's and toc_mlp_risk's closures over the run's fixed buffers, or None where they do
    not apply (no step cache; the tail kernel is built for 10 classes and keeps W2 plus 8 rows in
    shared memory)."""
    import ctypes

    if not net.step_cache or classes != 10 or 8 * (hidden * classes + 9 * classes + 16 * hidden) > 200 * 1024:
        return None
    torch = net.torch
    L = N.lib()
    a = net.arena
    nrows = np.ascontiguousarray(net.nrows, np.int32)
    nb = ctypes.c_int64(0)
    N.check(L.toc_mlp_scratch(int(nrows.max(initial=0)), a.n_cols, hidden, classes, ctypes.byref(nb)),
            "toc_mlp_scratch")
    scratch = torch.empty(max(int(nb.value), 8), dtype=torch.uint8, device=a.data.device)
    cache_off = np.ascontiguousarray(a.mlpcache_off[:-1], np.int64)
    block_off = np.ascontiguousarray(a.block_off, np.int64)
    row_base = np.ascontiguousarray(net.rb, np.int64)
    labels = net.batches.labels.to(torch.float64).contiguous()
    loss = torch.empty(max(int(nrows.sum()), 1), dtype=torch.float64, device=a.data.device)

    def run(w1, b1, w2, b2, lr):
        N.check(L.toc_mlp_epoch(a.data.data_ptr(), block_off.ctypes.data, a.mlpcache.data_ptr(), cache_off.ctypes.data,
                                row_base.ctypes.data, nrows.ctypes.data, a.n_blocks, a.n_cols, hidden, classes,
                                labels.data_ptr(), w1.data_ptr(), b1.data_ptr(), w2.data_ptr(), b2.data_ptr(), lr,
                                int(net.dense_rows), scratch.data_ptr(), scratch.numel(), N.stream_handle()),
                "toc_mlp_epoch")

    def risk(w1, b1, w2, b2):  # mean cross-entropy over every row (forward pass only)
        N.check(L.toc_mlp_risk(a.data.data_ptr(), block_off.ctypes.data, a.mlpcache.data_ptr(), cache_off.ctypes.data,
                               row_base.ctypes.data, nrows.ctypes.data, a.n_blocks, a.n_cols, hidden, classes,
                               labels.data_ptr(), w1.data_ptr(), b1.data_ptr(), w2.data_ptr(), b2.data_ptr(),
                               int(net.dense_rows), loss.data_ptr(), scratch.data_ptr(), scratch.numel(),
                               N.stream_handle()), "toc_mlp_risk")
        return float(loss[: int(nrows.sum())].mean().item())

    run.risk = risk
    return run


def train_mlp(dataset: LabeledDataset, hidden: int = 200, classes: int = 10, batch_size: int = 250,
              learning_rate: float = 0.05, epochs: int = 5, seed: int = 0, native: bool = True):
    """Config-5 MLP on compressed batches: labels are class ids 0..classes-1 (as floats).
    Returns (MlpModel, LossTrace) with the mean cross-entropy over all rows after each epoch.
    native: each epoch is one toc_mlp_epoch call (four kernels per step, first layer on the fp64
    tensor cores); False, or a shape it does not cover: the per-step path (matmat kernels plus
    torch ops for the dense tail).  Both compute the same step; results agree to fp64 rounding."""
    from .training import LossTrace

    net = _Net(dataset, batch_size, seed, step_cache=native)
    torch = net.torch
    trace = LossTrace()
    w1, b1, w2, b2 = (torch.from_numpy(x).cuda() for x in init_mlp(dataset.n_cols, hidden, classes, seed))
    lr = float(learning_rate)
    labels_all = net.batches.labels.long()
    epoch_fn = _native_epoch(net, hidden, classes) if native else None
    a = net.arena
    if epoch_fn is not None:  # what the run keeps in HBM and what each step reads of it
        meta = a.meta
        codes = (meta["n_codes"].astype(np.int64) * meta["w_codes"].astype(np.int64)).sum()
        entries = int(a.mlpcache_off[-1])
        trace.memory = {"toc1_bytes": int(a.block_bytes), "step_cache_bytes": entries,
                        "step_cache_over_toc1": entries / max(int(a.block_bytes), 1),
                        "dense_bytes": 8 * int(meta["n_rows"].sum()) * a.n_cols,
                        "decode_reads_per_step": float((codes + entries) / max(a.n_blocks, 1)),
                        "note": "per step the decode reads the batch's TOC1 code stream and its step-cache entry "
                                "(4-byte node records, pair records, value index)"}
    if native and epoch_fn is None and net.step_cache:  # a shape the native step does not cover
        net.arena.build_matcache()

    def forward(z1):
        a1 = torch.relu(z1 + b1)
        return a1, a1 @ w2 + b2

    for _ in range(epochs):
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        if epoch_fn is not None:
            epoch_fn(w1, b1, w2, b2, lr)
        for b in range(net.arena.n_blocks if epoch_fn is None else 0):
            y = net.labels(b).long()
            a1, logits = forward(net.first_layer(b, w1, hidden))
            p = torch.softmax(logits, dim=1)
            p[torch.arange(len(y), device=p.device), y] -= 1.0  # d(sum CE)/d logits
            g_w2 = a1.t() @ p
            g_b2 = p.sum(0)
            delta = ((p @ w2.t()) * (a1 > 0)).contiguous()
            g_b1 = delta.sum(0)
            g_w1 = net.first_layer_grad(b, delta, hidden)
            step = lr / len(y)
            w1 = w1 - step * g_w1
            b1 = b1 - step * g_b1
            w2 = w2 - step * g_w2
            b2 = b2 - step * g_b2
        end.record()
        end.synchronize()
        trace.seconds.append(start.elapsed_time(end) / 1e3)
        if epoch_fn is not None:
            trace.risks.append(epoch_fn.risk(w1, b1, w2, b2))
        else:
            _, logits = forward(net.arena.matmat(0, w1, hidden))
            trace.risks.append(float(torch.nn.functional.cross_entropy(logits, labels_all).item()))
    model = MlpModel(*(x.cpu().numpy() for x in (w1, b1, w2, b2)))
    return model, trace
