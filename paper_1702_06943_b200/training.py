"""Mini-batch gradient descent over TOC-compressed batches on the device (reference
training.py:1-361).

``train`` keeps the reference's contract: shuffle once with the stdlib RNG (training.py:131-142),
carve contiguous batches (the last may be short, :145-167), start GLM weights at zero (:319-326),
run the configured epochs with ``w <- w - (lr / |B|) * g`` per batch (:296-316), and record the
full-dataset empirical risk after every epoch plus the epoch's batch-loop time (:336-361).
Compression happens once, on the GPU (codec.compress_csr); each epoch is ONE cooperative kernel
launch (toc_glm_epoch) whose CTAs relay the weights step to step through L2.
"""

from __future__ import annotations

import ctypes
import math
import random
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .codec import compress_csr
from . import kernels
from .kernels import CompressedMatrix, OpCounter
from .matrix import (DenseMatrix, LabeledDataset, SparseRowMatrix, as_vector, csr_matmat_left, csr_matmat_right,
                     csr_matvec, csr_vecmat, dense_matmat, dense_matvec, dense_vecmat, sparse_to_dense)
from .mlp import NnModel, init_nn

LOSS_KINDS = ("squared", "logistic", "hinge", "nn_mse")
EXECUTION_MODES = ("compressed", "dense", "csr")
LOSS_CODE = {"squared": 0, "logistic": 1, "hinge": 2}


@dataclass
class TrainConfig:
    """Training hyper-parameters (reference training.py:46-68)."""

    loss_kind: str
    batch_size: int
    learning_rate: float
    epochs: int
    seed: int = 0
    hidden_units: int = 16
    execution: str = "compressed"

    def __post_init__(self) -> None:
        if self.loss_kind not in LOSS_KINDS:
            raise ValueError(f"loss_kind must be one of {LOSS_KINDS}, got {self.loss_kind!r}")
        if self.execution not in EXECUTION_MODES:
            raise ValueError(f"execution must be one of {EXECUTION_MODES}, got {self.execution!r}")
        if self.batch_size < 1:
            raise ValueError(f"batch_size must be at least 1, got {self.batch_size}")
        if self.epochs < 1:
            raise ValueError(f"epochs must be at least 1, got {self.epochs}")
        if not (math.isfinite(self.learning_rate) and self.learning_rate > 0):
            raise ValueError(f"learning_rate must be positive and finite, got {self.learning_rate}")
        if self.loss_kind == "nn_mse" and self.hidden_units < 1:
            raise ValueError(f"hidden_units must be at least 1, got {self.hidden_units}")


@dataclass
class GlmModel:
    """Linear model x . weights (training.py:71-78)."""

    weights: np.ndarray

    def __post_init__(self) -> None:
        self.weights = as_vector(self.weights, len(self.weights), "weights")


@dataclass
class LossTrace:
    """Per-epoch full-dataset risk plus the batch-loop time (training.py:123-128)."""

    risks: list = field(default_factory=list)
    seconds: list = field(default_factory=list)


def shuffle_order(n_rows: int, seed: int) -> np.ndarray:
    """The permutation of shuffle_once (training.py:138-139): stdlib Fisher-Yates, once."""
    order = list(range(n_rows))
    random.Random(seed).shuffle(order)
    return np.asarray(order, dtype=np.int64)


def shuffle_once(dataset: LabeledDataset, seed: int) -> LabeledDataset:
    order = shuffle_order(dataset.n_rows, seed)
    return LabeledDataset(features=dataset.features.take_rows(order), labels=dataset.labels[order])


class DeviceBatches:
    """The epoch's mini-batches as TOC1 blocks in HBM, labels per row (make_batches with
    execution='compressed', training.py:145-167, but one arena instead of one object per batch)."""

    def __init__(self, dataset: LabeledDataset, batch_size: int):
        torch = N.require_cuda()
        s = dataset.features
        n = s.n_rows
        if n == 0:
            raise ValueError("cannot batch an empty dataset")
        if batch_size < 1:
            raise ValueError(f"batch_size must be at least 1, got {batch_size}")
        batch_row = np.concatenate([np.arange(0, n, batch_size), [n]]).astype(np.int64)
        self.arena = compress_csr(s.n_cols, s.row_ptr, s.cols, s.vals, batch_row)
        self.labels = torch.from_numpy(np.ascontiguousarray(dataset.labels, np.float64)).cuda()
        self.n_cols = s.n_cols
        self.n_rows = n
        self.batch_sizes = np.diff(batch_row)

    def kernel_cost_per_step(self) -> np.ndarray:
        m = self.arena.meta
        return (m["n_pairs"].astype(np.int64) + m["n_derived"] + m["n_codes"]).astype(np.int64)


def _bind():
    L = N.lib()
    if not getattr(L, "_mgd_bound", False):
        P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        L.toc_mgd_workspace.argtypes = [P, I64, I32, I32, ctypes.POINTER(ctypes.c_int64)]
        L.toc_glm_epoch.argtypes = [P, P, P, P, P, I64, I32, I32, D, P, P, P, P, P]
        L.toc_glm_grad.argtypes = [P, P, P, P, P, I64, I32, I32, P, P, P, P, P]
        L.toc_glm_risk.argtypes = [P, P, I64, I32, P, I32, P]
        L.toc_mgd_image_plan.argtypes = [P, I64, I32, I32, ctypes.POINTER(ctypes.c_int32), P]
        L.toc_mgd_build_images.argtypes = [P, P, P, P, P, I64, I32, I32, P, P, P, P]
        L.toc_glm_epoch_images.argtypes = [P, P, P, P, I64, I32, I32, I32, D, P, P]
        L.toc_mgd_parts_scratch.argtypes = [P, I64, I32, ctypes.POINTER(ctypes.c_int64)]
        L.toc_mgd_parts_count.argtypes = [P, P, P, P, P, I64, I32, I32, P, P, P, P]
        L.toc_mgd_parts_offsets.argtypes = [P, P, I64, I32, P, ctypes.POINTER(ctypes.c_int64)]
        L.toc_mgd_parts_build.argtypes = [P, P, P, P, P, I64, I32, I32, P, P, P, P, P, P]
        L.toc_mgd_parts_fit.argtypes = [P, P, I64, I32, I64, ctypes.POINTER(ctypes.c_int32)]
        L.toc_glm_epoch_parts.argtypes = [P, P, P, P, I64, I32, I32, I32, D, P, P, I64, P]
        L.toc_glm_grad_parts.argtypes = [P, P, P, P, I64, I32, I32, I32, I64, P, P, P, I64, P]
        L.toc_mgd_parts_cluster_max.argtypes = [ctypes.c_void_p]
        L.toc_glm_epoch_images_dp.argtypes = [P, P, P, P, I64, I32, I32, I32, D, P, I32, I32, P, P, P,
                                               ctypes.c_uint32, P]
        L.toc_glm_epoch_images_dp_emulated.argtypes = [P, P, I64, I32, I32, I32, D, I32, P, P, P, ctypes.c_uint32, P]
        L._mgd_bound = True
    return L


_PARTS_CLUSTER = 0


def parts_cluster() -> int:
    """Cluster size for the part-image epoch: the largest power of two (<= 16) the device
    co-schedules at a full shared-memory carve-out (toc_mgd_parts_cluster_max); 16 CTAs measured
    8.0 us/step at config 4 vs 10.9 at 8."""
    global _PARTS_CLUSTER
    if not _PARTS_CLUSTER:
        c = ctypes.c_int32()
        N.check(_bind().toc_mgd_parts_cluster_max(ctypes.byref(c)), "toc_mgd_parts_cluster_max")
        _PARTS_CLUSTER = c.value
    return _PARTS_CLUSTER


class GlmTrainer:
    """Device-resident GLM training state over DeviceBatches.

    mode "images" (the default when it fits shared memory): each batch's step image -- its decode
    tree, value index, unpacked first-layer pairs and labels -- is built once here, the device form
    of the reference's once-only per-batch tree cache (kernels.py:68-77), and every epoch is one
    launch of a thread-block cluster over them (toc_glm_epoch_images; cluster=0 picks its size).
    mode "relay": no cache, each step rebuilds its tables from the TOC1 block (toc_glm_epoch).
    Both give the same results up to fp64 summation order."""

    def __init__(self, batches: DeviceBatches, loss_kind: str, learning_rate: float, mode: str = "auto",
                 cluster: int = 0):
        if mode not in ("auto", "images", "parts", "relay"):
            raise ValueError(f"mode must be auto, images, parts or relay, got {mode!r}")
        self.torch = N.require_cuda()
        self.b = batches
        self.loss = LOSS_CODE[loss_kind]
        self.lr = float(learning_rate)
        torch = self.torch
        self.w = torch.zeros(max(batches.n_cols, 1), dtype=torch.float64, device="cuda")
        self.sync = torch.zeros(64, dtype=torch.int32, device="cuda")  # counter @0, abort flag @32
        self.partial = torch.zeros(148, dtype=torch.float64, device="cuda")
        L = _bind()
        a = batches.arena
        nbytes = ctypes.c_int64()
        N.check(L.toc_mgd_workspace(a.meta.ctypes.data_as(ctypes.c_void_p), a.n_blocks, batches.n_cols, 0,
                                    ctypes.byref(nbytes)), "toc_mgd_workspace")
        self.scratch = torch.empty(max(nbytes.value, 16), dtype=torch.uint8, device="cuda")
        self.mode = "relay"
        self.image_build_seconds = 0.0
        self.cluster = 0
        if mode in ("auto", "images"):
            self._build_images(mode == "images", cluster)
        if self.mode == "relay" and mode in ("auto", "parts"):
            self._build_parts(mode == "parts", cluster or parts_cluster())

    def _build_images(self, required: bool, cluster_req: int) -> None:
        torch = self.torch
        a = self.b.arena
        a.raise_corrupt()
        L = _bind()
        meta = a.meta.ctypes.data_as(ctypes.c_void_p)
        off = np.zeros(a.n_blocks + 1, dtype=np.int64)
        ok = ctypes.c_int32()
        N.check(L.toc_mgd_image_plan(meta, a.n_blocks, self.b.n_cols, int(cluster_req), ctypes.byref(ok),
                                     off.ctypes.data_as(ctypes.c_void_p)), "toc_mgd_image_plan")
        if not ok.value:
            if required:
                raise ValueError("step images do not fit the single-CTA epoch (shared memory); use mode='relay'")
            return
        self.image_off = off
        self.image_off_d = torch.from_numpy(off).cuda()
        self.images = torch.empty(max(int(off[-1]), 16), dtype=torch.uint8, device="cuda")
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        N.check(L.toc_mgd_build_images(a.data.data_ptr(), a.block_off_d.data_ptr(), a.meta_d.data_ptr(), meta,
                                       a.row_base_d.data_ptr(), a.n_blocks, self.b.n_cols, ok.value,
                                       self.b.labels.data_ptr(),
                                       self.images.data_ptr(), self.image_off_d.data_ptr(), N.stream_handle()),
                "toc_mgd_build_images")
        end.record()
        end.synchronize()
        self.image_build_seconds = start.elapsed_time(end) / 1e3
        self.mode = "images"
        self.cluster = ok.value

    def _build_parts(self, required: bool, cluster: int) -> None:
        """Per-CTA part images for models too wide for shared memory (toc_images_large.cu)."""
        torch = self.torch
        a = self.b.arena
        if self.loss not in (LOSS_CODE["logistic"], LOSS_CODE["hinge"]):
            if required:
                raise ValueError("mode='parts' trains logistic / hinge losses (squared: use the relay)")
            return
        a.raise_corrupt()
        L = _bind()
        meta = a.meta.ctypes.data_as(ctypes.c_void_p)
        nb = ctypes.c_int64()
        N.check(L.toc_mgd_parts_scratch(meta, a.n_blocks, self.b.n_cols, ctypes.byref(nb)), "toc_mgd_parts_scratch")
        scratch = torch.empty(max(nb.value, 16), dtype=torch.uint8, device="cuda")
        counts = torch.zeros(a.n_blocks * cluster * 4, dtype=torch.int32, device="cuda")
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        N.check(L.toc_mgd_parts_count(a.data.data_ptr(), a.block_off_d.data_ptr(), a.meta_d.data_ptr(), meta,
                                      a.row_base_d.data_ptr(), a.n_blocks, self.b.n_cols, cluster,
                                      self.b.labels.data_ptr(), counts.data_ptr(), scratch.data_ptr(),
                                      N.stream_handle()), "toc_mgd_parts_count")
        counts_h = counts.cpu().numpy()
        off = np.zeros(a.n_blocks * cluster + 1, dtype=np.int64)
        mx = ctypes.c_int64()
        N.check(L.toc_mgd_parts_offsets(meta, counts_h.ctypes.data_as(ctypes.c_void_p), a.n_blocks, cluster,
                                        off.ctypes.data_as(ctypes.c_void_p), ctypes.byref(mx)), "toc_mgd_parts_offsets")
        fits = ctypes.c_int32()
        N.check(L.toc_mgd_parts_fit(meta, counts_h.ctypes.data_as(ctypes.c_void_p), a.n_blocks, cluster, mx.value,
                                    ctypes.byref(fits)), "toc_mgd_parts_fit")
        if not fits.value:
            if required:
                raise ValueError("part images do not fit shared memory; use mode='relay'")
            return
        self.part_off_d = torch.from_numpy(off).cuda()
        self.images = torch.empty(max(int(off[-1]), 16), dtype=torch.uint8, device="cuda")
        N.check(L.toc_mgd_parts_build(a.data.data_ptr(), a.block_off_d.data_ptr(), a.meta_d.data_ptr(), meta,
                                      a.row_base_d.data_ptr(), a.n_blocks, self.b.n_cols, cluster,
                                      self.b.labels.data_ptr(), counts.data_ptr(), self.part_off_d.data_ptr(),
                                      self.images.data_ptr(), scratch.data_ptr(), N.stream_handle()),
                "toc_mgd_parts_build")
        end.record()
        end.synchronize()
        self.image_build_seconds = start.elapsed_time(end) / 1e3
        self.parts_counts = counts_h
        self.parts_max = mx.value
        self.image_off = off
        self.gacc = torch.zeros(max(self.b.n_cols, 1), dtype=torch.int64, device="cuda")
        self.mode = "parts"
        self.cluster = cluster

    def epoch(self) -> float:
        """One epoch; returns its device time in seconds (CUDA events on the launch stream)."""
        torch = self.torch
        a = self.b.arena
        a.raise_corrupt()
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if self.mode == "parts":
            start.record()
            N.check(_bind().toc_glm_epoch_parts(self.images.data_ptr(), self.part_off_d.data_ptr(),
                                                a.meta.ctypes.data_as(ctypes.c_void_p),
                                                self.parts_counts.ctypes.data_as(ctypes.c_void_p), a.n_blocks,
                                                self.b.n_cols, self.cluster, self.loss, self.lr, self.w.data_ptr(),
                                                self.gacc.data_ptr(), self.parts_max, N.stream_handle()),
                    "toc_glm_epoch_parts")
            end.record()
            end.synchronize()
            return start.elapsed_time(end) / 1e3
        if self.mode == "images":
            start.record()
            N.check(_bind().toc_glm_epoch_images(self.images.data_ptr(), self.image_off_d.data_ptr(),
                                                 a.meta_d.data_ptr(), a.meta.ctypes.data_as(ctypes.c_void_p),
                                                 a.n_blocks, self.b.n_cols, self.cluster, self.loss, self.lr,
                                                 self.w.data_ptr(), N.stream_handle()),
                    "toc_glm_epoch_images")
            end.record()
            end.synchronize()
            return start.elapsed_time(end) / 1e3
        start.record()
        N.check(_bind().toc_glm_epoch(a.data.data_ptr(), a.block_off_d.data_ptr(), a.meta_d.data_ptr(),
                                      a.meta.ctypes.data_as(ctypes.c_void_p), a.row_base_d.data_ptr(), a.n_blocks,
                                      self.b.n_cols, self.loss, self.lr, self.b.labels.data_ptr(), self.w.data_ptr(),
                                      self.sync.data_ptr(), self.scratch.data_ptr(), N.stream_handle()),
                "toc_glm_epoch")
        end.record()
        end.synchronize()
        if int(self.sync[32].item()):
            raise RuntimeError("toc_glm_epoch aborted (step hand-off timed out)")
        return start.elapsed_time(end) / 1e3

    def risk(self) -> float:
        """Mean loss over every row (empirical_risk, training.py:231-258), on the device."""
        a = self.b.arena
        z = a.matvec(self.w[: self.b.n_cols])
        N.check(_bind().toc_glm_risk(z.data_ptr(), self.b.labels.data_ptr(), self.b.n_rows, self.loss,
                                     self.partial.data_ptr(), self.partial.numel(), N.stream_handle()), "toc_glm_risk")
        return float(self.partial.sum().item()) / self.b.n_rows

    def weights(self) -> np.ndarray:
        return self.w[: self.b.n_cols].cpu().numpy().copy()


def init_model(config: TrainConfig, n_cols: int):
    """Zero weights for GLMs; the network's seeded uniform weights (training.py:319-333)."""
    if config.loss_kind != "nn_mse":
        return GlmModel(weights=np.zeros(n_cols, dtype=np.float64))
    w1, w2 = init_nn(n_cols, config.hidden_units, config.seed)
    return NnModel(w1=w1, w2=w2)


# ---- the reference's per-batch API (training.py:103-316) ------------------------------------------
# Layout-generic building blocks: a Batch carries a CompressedMatrix, DenseMatrix or
# SparseRowMatrix, and every touch of the features runs on the device -- the TOC kernels for
# compressed batches, the bit-exact uncompressed baselines (csrc/toc_dense.cu) otherwise.  The loss
# scalars between the two touches are torch ops on the device.  ``train`` uses these only for the
# dense / csr layouts; compressed GLM training runs the fused epoch kernels (GlmTrainer).

@dataclass
class Batch:
    """One mini-batch: features in some layout plus its labels (training.py:103-111)."""

    features: object
    labels: np.ndarray

    @property
    def size(self) -> int:
        return len(self.labels)


@dataclass
class BatchStore:
    """Batches in shuffle order, all in one layout (training.py:114-120)."""

    batches: list
    n_cols: int
    execution: str


def make_batches(dataset: LabeledDataset, batch_size: int, execution: str) -> BatchStore:
    """Consecutive batches, the last possibly short (training.py:145-167); compressed batches are
    encoded on the device, each with a fresh dictionary."""
    if execution not in EXECUTION_MODES:
        raise ValueError(f"execution must be one of {EXECUTION_MODES}, got {execution!r}")
    if batch_size < 1:
        raise ValueError(f"batch_size must be at least 1, got {batch_size}")
    if dataset.n_rows == 0:
        raise ValueError("cannot batch an empty dataset")
    out = []
    for lo in range(0, dataset.n_rows, batch_size):
        hi = min(lo + batch_size, dataset.n_rows)
        piece = dataset.features.take_rows(np.arange(lo, hi))
        if execution == "compressed":
            feats = CompressedMatrix.from_sparse(piece)
        elif execution == "dense":
            feats = sparse_to_dense(piece)
        else:
            feats = piece
        out.append(Batch(features=feats, labels=dataset.labels[lo:hi]))
    return BatchStore(batches=out, n_cols=dataset.features.n_cols, execution=execution)


def _matvec(features, w, counter):
    if isinstance(features, CompressedMatrix):
        return kernels.matvec(features, w, counter)
    if isinstance(features, DenseMatrix):
        return dense_matvec(features, w)
    return csr_matvec(features, w)


def _vecmat(v, features, counter):
    if isinstance(features, CompressedMatrix):
        return kernels.vecmat(v, features, counter)
    if isinstance(features, DenseMatrix):
        return dense_vecmat(v, features)
    return csr_vecmat(v, features)


def _matmat_right(features, m: DenseMatrix, counter):
    if isinstance(features, CompressedMatrix):
        return kernels.matmat_right(features, m, counter)
    if isinstance(features, DenseMatrix):
        return dense_matmat(features, m)
    return csr_matmat_right(features, m)


def _matmat_left(m: DenseMatrix, features, counter):
    if isinstance(features, CompressedMatrix):
        return kernels.matmat_left(m, features, counter)
    if isinstance(features, DenseMatrix):
        return dense_matmat(m, features)
    return csr_matmat_left(m, features)


def _cuda(x):
    torch = N.require_cuda()
    return torch.from_numpy(np.array(x, dtype=np.float64)).cuda()


def _sigmoid(z):
    """training.py:215-221 on the device: 1/(1+e^-z) for z >= 0, e^z/(1+e^z) below (no overflow)."""
    torch = N.require_cuda()
    ez = torch.exp(-torch.abs(z))
    return torch.where(z >= 0, 1.0 / (1.0 + ez), ez / (1.0 + ez))


def _nn_forward(features, model: NnModel, counter):
    """(h1, yhat) on the device; the first layer through the features' own layout."""
    h1 = _sigmoid(_cuda(_matmat_right(features, DenseMatrix(model.w1), counter).values))
    return h1, h1 @ _cuda(model.w2)


def empirical_risk(model, dataset: LabeledDataset, loss_kind: str) -> float:
    """Mean loss over the whole (unshuffled) dataset on its plain sparse features
    (training.py:231-258): the scores by the device CSR kernel, the losses on the device."""
    if loss_kind not in LOSS_KINDS:
        raise ValueError(f"loss_kind must be one of {LOSS_KINDS}, got {loss_kind!r}")
    if dataset.n_rows == 0:
        raise ValueError("empirical risk of an empty dataset is undefined")
    y = _cuda(dataset.labels)
    if loss_kind == "nn_mse":
        if not isinstance(model, NnModel):
            raise TypeError("nn_mse risk needs an NnModel")
        _, yhat = _nn_forward(dataset.features, model, None)
        return float((0.5 * (y - yhat[:, 0]) ** 2).mean().item())
    if not isinstance(model, GlmModel):
        raise TypeError(f"{loss_kind} risk needs a GlmModel")
    import torch

    z = _cuda(csr_matvec(dataset.features, model.weights))
    if loss_kind == "squared":
        losses = 0.5 * (y - z) ** 2
    elif loss_kind == "logistic":
        t = -y * z  # softplus(t) = log(1 + e^t), written overflow-free like training.py:206-212
        losses = torch.clamp(t, min=0.0) + torch.log1p(torch.exp(-torch.abs(t)))
    else:
        losses = torch.clamp(1.0 - y * z, min=0.0)
    return float(losses.mean().item())


def glm_gradient(batch: Batch, model: GlmModel, loss_kind: str, counter: OpCounter | None = None) -> np.ndarray:
    """Summed gradient of the batch loss (training.py:261-281): one matvec scores the batch, the
    per-row loss derivative is formed on the device, one vecmat folds it back."""
    if loss_kind not in LOSS_CODE:
        raise ValueError(f"glm_gradient cannot handle loss_kind {loss_kind!r}")
    import torch

    z = _cuda(_matvec(batch.features, model.weights, counter))
    y = _cuda(batch.labels)
    if loss_kind == "squared":
        s = z - y
    elif loss_kind == "logistic":
        s = -y / (1.0 + torch.exp(y * z))
    else:  # hinge subgradient: the flat side of the kink contributes zero
        s = torch.where(y * z < 1.0, -y, torch.zeros_like(y))
    return _vecmat(s.cpu().numpy(), batch.features, counter)


def nn_gradient(batch: Batch, model: NnModel, counter: OpCounter | None = None):
    """Summed (dW1, dW2) of the half squared error (training.py:284-293): the first layer's two
    products through the batch's layout, the rest on the device."""
    h1, yhat = _nn_forward(batch.features, model, counter)
    err = yhat - _cuda(batch.labels)[:, None]
    g_w2 = h1.t() @ err
    delta = (err @ _cuda(model.w2).t()) * h1 * (1.0 - h1)
    g_w1_t = _matmat_left(DenseMatrix(delta.t().cpu().numpy()), batch.features, counter)
    return np.ascontiguousarray(g_w1_t.values.T), g_w2.cpu().numpy()


def apply_update(weights: np.ndarray, gradient: np.ndarray, learning_rate: float, batch_size: int) -> np.ndarray:
    """weights - (learning_rate / batch_size) * gradient (training.py:296-300)."""
    return weights - (learning_rate / batch_size) * gradient


def mgd_step(model, batch: Batch, config: TrainConfig, counter: OpCounter | None = None):
    """One descent step on one batch, returning a new model (training.py:303-316)."""
    if config.loss_kind == "nn_mse":
        g_w1, g_w2 = nn_gradient(batch, model, counter)
        return NnModel(w1=apply_update(model.w1, g_w1, config.learning_rate, batch.size),
                       w2=apply_update(model.w2, g_w2, config.learning_rate, batch.size))
    g = glm_gradient(batch, model, config.loss_kind, counter)
    return GlmModel(weights=apply_update(model.weights, g, config.learning_rate, batch.size))


def _train_batches(dataset: LabeledDataset, config: TrainConfig, counter):
    """The reference's own epoch loop over a BatchStore (training.py:349-361), step by step."""
    store = make_batches(shuffle_once(dataset, config.seed), config.batch_size, config.execution)
    model = init_model(config, dataset.n_cols)
    trace = LossTrace()
    for _ in range(config.epochs):
        t0 = time.perf_counter()
        for batch in store.batches:
            model = mgd_step(model, batch, config, counter)
        trace.seconds.append(time.perf_counter() - t0)
        trace.risks.append(empirical_risk(model, dataset, config.loss_kind))
    return model, trace


def train(dataset: LabeledDataset, config: TrainConfig, counter: OpCounter | None = None):
    """Shuffle once, batch once, then run the configured epochs (training.py:336-361)."""
    if dataset.n_rows == 0:
        raise ValueError("cannot train on an empty dataset")
    if config.loss_kind in ("logistic", "hinge"):
        bad = [float(v) for v in np.unique(dataset.labels) if v not in (-1.0, 1.0)]
        if bad:
            raise ValueError(f"{config.loss_kind} loss needs labels in {{-1, +1}}, found {bad}")
    if config.execution != "compressed":  # dense / csr layouts: the reference's per-batch loop
        return _train_batches(dataset, config, counter)
    if config.loss_kind == "nn_mse":
        from .mlp import train_nn

        return train_nn(dataset, config, counter)
    shuffled = shuffle_once(dataset, config.seed)
    batches = DeviceBatches(shuffled, config.batch_size)
    trainer = GlmTrainer(batches, config.loss_kind, config.learning_rate)
    trace = LossTrace()
    per_step = batches.kernel_cost_per_step()
    for _ in range(config.epochs):
        trace.seconds.append(trainer.epoch())
        trace.risks.append(trainer.risk())
        if counter is not None:  # one matvec + one vecmat per step (test_training.py:217-223)
            counter.multiply_adds += int(2 * per_step.sum())
            nodes = int((batches.arena.meta["n_pairs"].astype(np.int64) + batches.arena.meta["n_derived"]).sum())
            counter.tree_nodes_visited += 2 * nodes
            counter.codes_visited += 2 * int(batches.arena.meta["n_codes"].astype(np.int64).sum())
    return GlmModel(weights=trainer.weights()), trace


class _ChunkBatches:
    """DeviceBatches-shaped view of one streamed store chunk."""

    def __init__(self, arena, labels, n_cols: int):
        self.arena = arena
        self.labels = labels
        self.n_cols = n_cols
        self.n_rows = arena.n_rows_total


def train_store(path, config: TrainConfig, chunk: int = 4096):
    """MGD over the batches of a TOCS store, streamed from disk chunk by chunk (SURVEY.md 8(f) #2:
    datasets larger than HBM).  The store's batches are the mini-batches, in store order (the
    reference's compress step writes them from the dataset in order, cli.py:152-174); each epoch
    runs the same epoch kernels as ``train`` over every chunk with the weights carried across
    chunks, then the risk (empirical_risk, training.py:231-258) over the store's rows, also
    streamed.  GLM losses only.  Returns (GlmModel, LossTrace)."""
    from .store import BatchStoreStream

    torch = N.require_cuda()
    if config.loss_kind not in LOSS_CODE:
        raise ValueError(f"train_store trains GLMs; got loss_kind={config.loss_kind!r}")
    with BatchStoreStream(path, chunk) as probe:
        n_cols, n_rows = probe.n_cols, probe.index.total_rows
    if n_rows == 0:
        raise ValueError("cannot train on an empty dataset")
    w = torch.zeros(max(n_cols, 1), dtype=torch.float64, device="cuda")
    trace = LossTrace()
    loss = LOSS_CODE[config.loss_kind]
    partial = torch.zeros(148, dtype=torch.float64, device="cuda")
    L = _bind()
    for _ in range(config.epochs):
        secs = 0.0
        with BatchStoreStream(path, chunk) as st:
            for ch in st:
                tr = GlmTrainer(_ChunkBatches(ch.arena, ch.labels, n_cols), config.loss_kind, config.learning_rate)
                tr.w = w
                secs += tr.epoch()
        trace.seconds.append(secs)
        total = 0.0
        with BatchStoreStream(path, chunk) as st:
            for ch in st:
                z = ch.arena.matvec(w[:n_cols])
                N.check(L.toc_glm_risk(z.data_ptr(), ch.labels.data_ptr(), ch.arena.n_rows_total, loss,
                                       partial.data_ptr(), partial.numel(), N.stream_handle()), "toc_glm_risk")
                total += float(partial.sum().item())
        trace.risks.append(total / n_rows)
    return GlmModel(weights=w[:n_cols].cpu().numpy().copy()), trace
