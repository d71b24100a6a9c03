"""Multi-GPU execution.

* Matrix-op sweep: mini-batches are independent, so rank r of G simply owns a contiguous shard
  of the batches -- no collective on the data path (weak scaling).
* Synchronous data-parallel MGD: at step t the global batch is rows [t*B*G, (t+1)*B*G) of the
  once-shuffled order (training.py:131-167 with batch_size = B*G); rank r compresses and holds the
  rows [t*B*G + r*B, t*B*G + (r+1)*B) as its local mini-batch.  Each step every rank computes the
  summed gradient of its local batch on the device (toc_glm_grad), the gradients are all-reduced
  (sum), and every rank applies w <- w - (lr / |B_t|) * g with |B_t| the global batch size
  (training.py:296-300).  The union of the local batches is exactly the reference's batch at
  batch_size = B*G, so the parity oracle is the reference trainer at that batch size.

The per-step gradient function and the all-reduce are injectable so the host logic runs (and is
tested) on CPU with the gloo backend; on the device path they are toc_glm_grad and NCCL.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Callable

import numpy as np

from . import _native as N


def shard_range(n_items: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous near-equal shard [lo, hi) of n_items for rank (sweep: batches per GPU)."""
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


@dataclass
class StepPlan:
    """Rows of the shuffled order this rank holds at each step, and the global batch sizes."""

    local_rows: list  # per step: (lo, hi) in shuffled-row space (hi == lo: empty local batch)
    global_sizes: np.ndarray  # per step: |B_t|


def dp_step_plan(n_rows: int, local_batch: int, world: int, rank: int) -> StepPlan:
    gb = local_batch * world
    steps = (n_rows + gb - 1) // gb
    rows, sizes = [], np.zeros(steps, np.int64)
    for t in range(steps):
        g0 = t * gb
        sizes[t] = min(gb, n_rows - g0)
        lo = min(n_rows, g0 + rank * local_batch)
        hi = min(n_rows, lo + local_batch, g0 + gb)
        rows.append((lo, max(lo, hi)))
    return StepPlan(rows, sizes)


def apply_update(w, g, lr: float, batch_size: int):
    """w - (lr / batch_size) * g (training.py:296-300), in place on a torch tensor."""
    step = lr / batch_size
    w.sub_(g * step)
    return w


class DataParallelGLM:
    """Synchronous DP-MGD over local mini-batches.

    grad_fn(t, w) -> summed gradient of this rank's local batch of step t (zeros if empty);
    allreduce(g) sums g across ranks in place."""

    def __init__(self, n_cols: int, plan: StepPlan, lr: float, grad_fn: Callable, allreduce: Callable, w0):
        self.n_cols = n_cols
        self.plan = plan
        self.lr = float(lr)
        self.grad_fn = grad_fn
        self.allreduce = allreduce
        self.w = w0

    def epoch(self):
        for t, gsize in enumerate(self.plan.global_sizes):
            g = self.grad_fn(t, self.w)
            self.allreduce(g)
            apply_update(self.w, g, self.lr, int(gsize))
        return self.w


# ---- device pieces -------------------------------------------------------------------------
def batch_gradients(batches, loss_kind: str, w, out=None):
    """Summed gradient of every batch of a DeviceBatches at weights w (device tensor), on the GPU
    (toc_glm_grad).  Returns a [n_batches, n_cols] float64 device tensor."""
    from .training import LOSS_CODE, _bind

    torch = N.require_cuda()
    a = batches.arena
    L = _bind()
    m = batches.n_cols
    if out is None:
        out = torch.empty((a.n_blocks, m), dtype=torch.float64, device="cuda")
    nbytes = ctypes.c_int64()
    N.check(L.toc_mgd_workspace(a.meta.ctypes.data_as(ctypes.c_void_p), a.n_blocks, m, 1, ctypes.byref(nbytes)),
            "toc_mgd_workspace")
    scratch = torch.empty(max(nbytes.value, 16), dtype=torch.uint8, device="cuda")
    N.check(L.toc_glm_grad(a.data.data_ptr(), a.block_off_d.data_ptr(), a.meta_d.data_ptr(),
                           a.meta.ctypes.data_as(ctypes.c_void_p), a.row_base_d.data_ptr(), a.n_blocks, m,
                           LOSS_CODE[loss_kind], batches.labels.data_ptr(), w.data_ptr(), out.data_ptr(),
                           scratch.data_ptr(), N.stream_handle()), "toc_glm_grad")
    return out


def capture_epoch(steps, probe, group=None):
    """Record `steps()` (an epoch's launches and NCCL collectives) as one CUDA graph.  The
    communicator is warmed with one all-reduce of `probe` on a side stream first (a collective's
    first call sets up state that cannot be captured).  Capture executes nothing."""
    import torch
    import torch.distributed as dist

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        dist.all_reduce(probe, op=dist.ReduceOp.SUM, group=group)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    probe.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        steps()
    return g


class DeviceDPEpoch:
    """One DP-MGD epoch on this rank's GPU, recorded once as a CUDA graph and replayed:
    per step t the summed gradient of the local batch, the NCCL all-reduce (sum) of the gradient,
    and w <- w - (lr / |B_t|) * g (training.py:296-300).  The gradient comes from the thread-block
    cluster kernel over per-CTA part images built once (toc_glm_grad_parts, logistic / hinge),
    else from toc_glm_grad on the batch's slice of the local arena (offset pointers, no per-step
    host work).  A step whose local batch is empty contributes a zero gradient.  `graph=False`
    (or a capture failure) runs the same sequence eagerly."""

    def __init__(self, batches, plan: StepPlan, steps_with_rows, loss_kind: str, lr: float, w, group=None,
                 graph: bool = True):
        import torch

        from .training import LOSS_CODE, _bind

        self.torch, self.group = torch, group
        self.batches, self.plan, self.w, self.lr = batches, plan, w, float(lr)
        self.loss = LOSS_CODE[loss_kind]
        self.local_of = {t: i for i, t in enumerate(steps_with_rows)}
        m = w.numel()
        self.g = torch.zeros(m, dtype=torch.float64, device="cuda")
        self.L = _bind()
        if batches is not None:
            a = batches.arena
            nbytes = ctypes.c_int64()
            N.check(self.L.toc_mgd_workspace(a.meta.ctypes.data_as(ctypes.c_void_p), a.n_blocks, m, 1,
                                             ctypes.byref(nbytes)), "toc_mgd_workspace")
            self.scratch = torch.empty(max(nbytes.value, 16), dtype=torch.uint8, device="cuda")
        self.parts = None
        if batches is not None and loss_kind in ("logistic", "hinge"):
            from .training import GlmTrainer

            try:
                self.parts = GlmTrainer(batches, loss_kind, lr, mode="parts")
            except ValueError:  # part images do not fit shared memory
                self.parts = None
        self.mode = "parts" if self.parts is not None else "grad"
        self.graph = None
        if graph:
            try:
                self._capture()
            except Exception:  # capture unsupported here: keep the eager sequence
                self.graph = None
                torch.cuda.synchronize()

    def _steps(self):
        import torch.distributed as dist

        a = self.batches.arena if self.batches is not None else None
        m = self.w.numel()
        for t, gsize in enumerate(self.plan.global_sizes):
            i = self.local_of.get(t)
            if i is None:
                self.g.zero_()
            elif self.parts is not None:  # touched columns of g; g stays zero elsewhere
                tr = self.parts
                N.check(self.L.toc_glm_grad_parts(
                    tr.images.data_ptr(), tr.part_off_d.data_ptr(), a.meta.ctypes.data_as(ctypes.c_void_p),
                    tr.parts_counts.ctypes.data_as(ctypes.c_void_p), a.n_blocks, m, tr.cluster, self.loss, i,
                    self.w.data_ptr(), tr.gacc.data_ptr(), self.g.data_ptr(), tr.parts_max, N.stream_handle()),
                    "toc_glm_grad_parts")
            else:
                N.check(self.L.toc_glm_grad(
                    a.data.data_ptr(), a.block_off_d.data_ptr() + 8 * i, a.meta_d.data_ptr() + 68 * i,
                    a.meta[i:].ctypes.data_as(ctypes.c_void_p), a.row_base_d.data_ptr() + 8 * i, 1, m, self.loss,
                    self.batches.labels.data_ptr(), self.w.data_ptr(), self.g.data_ptr(), self.scratch.data_ptr(),
                    N.stream_handle()), "toc_glm_grad")
            dist.all_reduce(self.g, op=dist.ReduceOp.SUM, group=self.group)
            self.w.add_(self.g, alpha=-self.lr / int(gsize))
            if self.parts is not None:
                self.g.zero_()

    def _capture(self):
        self.graph = capture_epoch(self._steps, self.g, self.group)

    def epoch(self):
        if self.graph is not None:
            self.graph.replay()
        else:
            self._steps()
        return self.w


class FusedDPEpoch:
    """DP-MGD epoch with the gradient all-reduce fused into the cluster epoch kernel
    (toc_glm_epoch_images_dp): one launch per epoch per GPU; every step CTA 0 stores the rank's
    dense gradient into every rank's receive buffer over NVLink (torch symmetric memory maps the
    peer buffers; each holds the receive slots and the flags), raises its flag there, and each rank
    applies the update
    once all ranks' gradients of the step have landed (sum in rank order, so every rank holds the
    same weights).  Requires the step images to fit (GlmTrainer mode "images") and a local batch at
    every global step; raises ValueError otherwise."""

    def __init__(self, batches, plan: StepPlan, loss_kind: str, lr: float, group=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm

        from .training import GlmTrainer, _bind

        if batches is None or batches.arena.n_blocks != len(plan.global_sizes):
            raise ValueError("the fused exchange needs a local batch at every step")
        self.tr = GlmTrainer(batches, loss_kind, lr, mode="images")
        if batches.n_cols > int(batches.arena.meta["n_pairs"].max()) + 1:
            raise ValueError("the gradient scratch (the P1 table) is smaller than n_cols")
        self.torch, self.L, self.symm = torch, _bind(), symm
        self.group = group or dist.group.WORLD
        self.world, self.rank = dist.get_world_size(self.group), dist.get_rank(self.group)
        self.handle = None
        self.gsize = torch.tensor(np.asarray(plan.global_sizes, np.int32), device="cuda")
        self.n_steps = len(plan.global_sizes)
        self.epochs = 0
        self.w = self.tr.w

    def connect(self):
        """Collective: map every rank's receive buffer (call on all ranks once all can run).  Each
        rank's symmetric buffer holds its receive slots [2][world][n_cols] f64 followed by its
        flags [world] u32 (zeroed here; the barrier keeps peers from signalling earlier)."""
        import torch.distributed as dist

        torch = self.torch
        m = max(self.tr.b.n_cols, 1)
        n_dbl = 2 * self.world * m
        self.recv = self.symm.empty(n_dbl + (self.world + 1) // 2, dtype=torch.float64, device="cuda")
        self.recv.zero_()
        self.handle = self.symm.rendezvous(self.recv, self.group)
        ptrs = [int(x) for x in self.handle.buffer_ptrs]
        self.buf_ptrs = torch.tensor(ptrs, dtype=torch.int64, device="cuda")
        self.flag_ptrs = torch.tensor([x + 8 * n_dbl for x in ptrs], dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        dist.barrier(group=self.group)
        return self

    def epoch(self):
        tr, a = self.tr, self.tr.b.arena
        N.check(self.L.toc_glm_epoch_images_dp(
            tr.images.data_ptr(), tr.image_off_d.data_ptr(), a.meta_d.data_ptr(), a.meta.ctypes.data_as(ctypes.c_void_p),
            a.n_blocks, tr.b.n_cols, tr.cluster, tr.loss, tr.lr, tr.w.data_ptr(), self.world, self.rank,
            self.buf_ptrs.data_ptr(), self.flag_ptrs.data_ptr(), self.gsize.data_ptr(),
            (self.epochs * self.n_steps) & 0xFFFFFFFF, N.stream_handle()), "toc_glm_epoch_images_dp")
        self.epochs += 1
        return self.w


class EmulatedDPEpochs:
    """The fused data-parallel epoch (toc_glm_epoch_images_dp) for `world` ranks on ONE GPU, in one
    cooperative launch (toc_glm_epoch_images_dp_emulated): cluster r runs rank r's local batches
    of dp_step_plan with its own weights, and the clusters exchange gradients through the same
    receive-slot / flag protocol as the NVLink path (plain device memory here).  Separate launches
    spinning on each other are never guaranteed co-resident on one GPU, so this is how the
    multi-rank protocol runs with fewer GPUs than ranks.  Every rank's weights must equal the
    reference trainer's at batch_size = local_batch * world."""

    def __init__(self, dataset, local_batch: int, world: int, loss_kind: str, lr: float, seed: int = 0):
        import torch

        from .matrix import LabeledDataset
        from .training import DeviceBatches, GlmTrainer, _bind, shuffle_order

        order = shuffle_order(dataset.n_rows, seed)
        self.torch, self.L, self.world = torch, _bind(), world
        self.trainers, metas = [], []
        plans = [dp_step_plan(dataset.n_rows, local_batch, world, r) for r in range(world)]
        self.n_steps = len(plans[0].global_sizes)
        cluster = 0
        for r, plan in enumerate(plans):
            if any(hi <= lo for lo, hi in plan.local_rows):
                raise ValueError("every rank needs a local batch at every step")
            local = np.concatenate([order[lo:hi] for lo, hi in plan.local_rows])
            sub = LabeledDataset(features=dataset.features.take_rows(local), labels=dataset.labels[local])
            tr = GlmTrainer(DeviceBatches(sub, local_batch), loss_kind, lr, mode="images", cluster=cluster)
            if tr.mode != "images":
                raise ValueError("the step images do not fit shared memory")
            cluster = tr.cluster
            self.trainers.append(tr)
            metas.append(tr.b.arena.meta)
        self.cluster = cluster
        self.h_meta = np.ascontiguousarray(np.concatenate(metas))
        m = max(dataset.n_cols, 1)
        n_dbl = 2 * world * m
        self.recv = [torch.zeros(n_dbl + (world + 1) // 2, dtype=torch.float64, device="cuda") for _ in range(world)]
        ptrs = [t.data_ptr() for t in self.recv]
        self.buf_ptrs = torch.tensor(ptrs, dtype=torch.int64, device="cuda")
        self.flag_ptrs = torch.tensor([x + 8 * n_dbl for x in ptrs], dtype=torch.int64, device="cuda")
        self.ranks = torch.tensor([[t.images.data_ptr(), t.image_off_d.data_ptr(), t.b.arena.meta_d.data_ptr(),
                                    t.w.data_ptr()] for t in self.trainers], dtype=torch.int64, device="cuda")
        self.gsize = torch.tensor(np.asarray(plans[0].global_sizes, np.int32), device="cuda")
        self.n_cols, self.loss, self.lr = dataset.n_cols, self.trainers[0].loss, float(lr)
        self.epochs = 0

    def epoch(self):
        """One epoch on every rank (one launch); returns the ranks' weight tensors."""
        N.check(self.L.toc_glm_epoch_images_dp_emulated(
            self.ranks.data_ptr(), self.h_meta.ctypes.data_as(ctypes.c_void_p), self.trainers[0].b.arena.n_blocks,
            self.n_cols, self.cluster, self.loss, self.lr, self.world, self.buf_ptrs.data_ptr(),
            self.flag_ptrs.data_ptr(), self.gsize.data_ptr(), (self.epochs * self.n_steps) & 0xFFFFFFFF,
            N.stream_handle()), "toc_glm_epoch_images_dp_emulated")
        self.epochs += 1
        return [t.w for t in self.trainers]


def train_data_parallel(dataset, config, world: int, rank: int, group=None, graph: bool = True,
                        fused: bool = True):
    """DP-MGD on this rank's GPU; every rank returns the same weights and the risk trace (the
    risk is all-reduced).  Launch one process per GPU (torchrun); NCCL all-reduces the gradient,
    and each epoch is one CUDA-graph replay (DeviceDPEpoch)."""
    import torch
    import torch.distributed as dist

    from .matrix import LabeledDataset
    from .training import DeviceBatches, LossTrace, GlmModel, shuffle_order

    order = shuffle_order(dataset.n_rows, config.seed)
    plan = dp_step_plan(dataset.n_rows, config.batch_size, world, rank)
    # this rank's local batches, in step order, as one arena (empty local batches are skipped)
    idx = [order[lo:hi] for lo, hi in plan.local_rows if hi > lo]
    steps_with_rows = [t for t, (lo, hi) in enumerate(plan.local_rows) if hi > lo]
    local = np.concatenate(idx) if idx else np.zeros(0, np.int64)
    sub = LabeledDataset(features=dataset.features.take_rows(local), labels=dataset.labels[local])
    batches = DeviceBatches(sub, config.batch_size) if len(local) else None
    runner = None
    if fused and os.environ.get("TOC_DP_FUSED", "1") != "0":
        # the fused NVLink exchange where every rank can run it (decided collectively, twice: the
        # step images, then the symmetric-memory rendezvous; any failure -> NCCL on every rank)
        try:
            runner = FusedDPEpoch(batches, plan, config.loss_kind, config.learning_rate, group)
            ok = 1
        except Exception:  # images do not fit, a rank lacks some step
            runner, ok = None, 0
        flag = torch.tensor([ok], dtype=torch.int32, device="cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        if not int(flag.item()):
            runner = None
        else:
            try:
                runner.connect()
                ok = 1
            except Exception:  # no symmetric memory / peer access on this node
                ok = 0
            flag = torch.tensor([ok], dtype=torch.int32, device="cuda")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
            if not int(flag.item()):
                runner = None
    if runner is not None:
        w = runner.w
        trace = LossTrace()
        trace.graph, trace.mode = False, "fused"
    else:
        w = torch.zeros(dataset.n_cols, dtype=torch.float64, device="cuda")
        runner = DeviceDPEpoch(batches, plan, steps_with_rows, config.loss_kind, config.learning_rate, w, group, graph)
        trace = LossTrace()
        trace.graph = runner.graph is not None
        trace.mode = runner.mode
    for _ in range(config.epochs):
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        runner.epoch()
        end.record()
        end.synchronize()
        t = torch.tensor([start.elapsed_time(end) / 1e3], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        trace.seconds.append(float(t.item()))
        trace.risks.append(_dp_risk(batches, w, config.loss_kind, dataset.n_rows, group))
    return GlmModel(weights=w.cpu().numpy()), trace


def _dp_risk(batches, w, loss_kind, n_total, group):
    import torch
    import torch.distributed as dist

    from .training import LOSS_CODE, _bind

    s = torch.zeros(1, dtype=torch.float64, device="cuda")
    if batches is not None:
        z = batches.arena.matvec(w)
        part = torch.zeros(148, dtype=torch.float64, device="cuda")
        N.check(_bind().toc_glm_risk(z.data_ptr(), batches.labels.data_ptr(), batches.n_rows, LOSS_CODE[loss_kind],
                                     part.data_ptr(), 148, N.stream_handle()), "toc_glm_risk")
        s += part.sum()
    dist.all_reduce(s, op=dist.ReduceOp.SUM, group=group)
    return float(s.item()) / n_total


def train_mlp_data_parallel(dataset, world: int, rank: int, hidden: int = 200, classes: int = 10,
                            batch_size: int = 250, learning_rate: float = 0.05, epochs: int = 5, seed: int = 0,
                            group=None, graph: bool = True):
    """Config 5 (784-h-10 ReLU softmax-CE MLP) with synchronous data parallelism: the per-rank
    batches as in train_data_parallel; per step the rank's summed gradient of all parameters from
    the native step kernels in gradient-only mode (toc_mlp_step_grad: decode, A.W1 and A^T.delta on
    the fp64 tensor cores, softmax-CE tail), one NCCL all-reduce of the flat gradient
    [W1 | W2 | b1 | b2], and params -= (lr / |B_t|) * g; each epoch one CUDA-graph replay.
    At world 1 this is train_mlp (mlp.py) step for step.  Returns (MlpModel, LossTrace)."""
    import torch
    import torch.distributed as dist

    from .matrix import LabeledDataset
    from .mlp import MlpModel, init_mlp
    from .training import DeviceBatches, LossTrace, shuffle_order

    L = N.lib()
    n, m, h, k = dataset.n_rows, dataset.n_cols, hidden, classes
    order = shuffle_order(n, seed)
    plan = dp_step_plan(n, batch_size, world, rank)
    idx = [order[lo:hi] for lo, hi in plan.local_rows if hi > lo]
    steps_with_rows = [t for t, (lo, hi) in enumerate(plan.local_rows) if hi > lo]
    local_of = {t: i for i, t in enumerate(steps_with_rows)}
    local = np.concatenate(idx) if idx else np.zeros(0, np.int64)
    sub = LabeledDataset(features=dataset.features.take_rows(local), labels=dataset.labels[local])
    batches = DeviceBatches(sub, batch_size) if len(local) else None
    sizes = (m * h, h * k, h, k)
    P = torch.zeros(sum(sizes), dtype=torch.float64, device="cuda")
    w1, w2, b1, b2 = torch.split(P, sizes)
    w1, w2 = w1.view(m, h), w2.view(h, k)
    iw1, ib1, iw2, ib2 = init_mlp(m, h, k, seed)
    w1.copy_(torch.from_numpy(iw1))
    w2.copy_(torch.from_numpy(iw2))
    b1.copy_(torch.from_numpy(ib1))
    b2.copy_(torch.from_numpy(ib2))
    G = torch.zeros_like(P)
    lr = float(learning_rate)
    if batches is not None:
        a = batches.arena
        if not a.build_mlpcache():
            raise ValueError("a batch's decode-tree ids do not fit the MLP step cache")
        nrows = np.ascontiguousarray(a.meta["n_rows"], np.int32)
        cache_off = np.ascontiguousarray(a.mlpcache_off[:-1], np.int64)
        block_off = np.ascontiguousarray(a.block_off, np.int64)
        row_base = np.ascontiguousarray(a.row_base, np.int64)
        labels = batches.labels.to(torch.float64).contiguous()
        lens = np.diff(np.asarray(sub.features.row_ptr))
        dense = int(bool(len(lens) and np.all(lens == m)))
        nb = ctypes.c_int64(0)
        N.check(L.toc_mlp_scratch(int(nrows.max(initial=0)), m, h, k, ctypes.byref(nb)), "toc_mlp_scratch")
        scratch = torch.empty(max(int(nb.value), 8), dtype=torch.uint8, device="cuda")

    def steps():
        for t, gsize in enumerate(plan.global_sizes):
            i = local_of.get(t)
            if i is None:
                G.zero_()
            else:
                N.check(L.toc_mlp_step_grad(
                    a.data.data_ptr(), block_off.ctypes.data, a.mlpcache.data_ptr(), cache_off.ctypes.data,
                    row_base.ctypes.data, nrows.ctypes.data,
                    a.n_blocks, i, m, h, k, labels.data_ptr(), w1.data_ptr(), b1.data_ptr(), w2.data_ptr(),
                    b2.data_ptr(), dense, G.data_ptr(), scratch.data_ptr(), scratch.numel(), N.stream_handle()),
                    "toc_mlp_step_grad")
            dist.all_reduce(G, op=dist.ReduceOp.SUM, group=group)
            P.add_(G, alpha=-lr / int(gsize))

    g = None
    if graph:
        try:
            g = capture_epoch(steps, G, group)
        except Exception:  # capture unsupported here: eager sequence
            g = None
            torch.cuda.synchronize()
    trace = LossTrace()
    trace.graph = g is not None
    for _ in range(epochs):
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        if g is not None:
            g.replay()
        else:
            steps()
        end.record()
        end.synchronize()
        t = torch.tensor([start.elapsed_time(end) / 1e3], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        trace.seconds.append(float(t.item()))
        ce = torch.zeros(1, dtype=torch.float64, device="cuda")
        if batches is not None:  # mean cross-entropy over all rows (local sums, all-reduced)
            logits = torch.relu(batches.arena.matmat(0, w1, h) + b1) @ w2 + b2
            ce += torch.nn.functional.cross_entropy(logits, batches.labels.long(), reduction="sum")
        dist.all_reduce(ce, op=dist.ReduceOp.SUM, group=group)
        trace.risks.append(float(ce.item()) / n)
    model = MlpModel(*(x.cpu().numpy() for x in (w1, b1, w2, b2)))
    return model, trace
