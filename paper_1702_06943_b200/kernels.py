"""Linear algebra on compressed matrices (reference kernels.py:1-285), on the device.

Reference-API mirror: ``CompressedMatrix``, ``matvec``, ``vecmat``, ``matmat_right``,
``matmat_left``, ``kernel_cost``, ``OpCounter``.  Each call runs the sm_100a kernels of
libtoc_b200.so on the matrix's device-resident TOC1 block; the operation counters are charged
from the block metadata with the reference's closed form (kernels.py:250-266), which its kernels
report exactly.

``BatchSweep`` is the batched public entry point: many mini-batches' TOC1 bytes on the host,
one call = upload + validate + A.v and v^T.A for every batch + download.
"""

from __future__ import annotations

import ctypes
import math
import threading
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .arena import BlockArena
from .codec import LogicalEncoding, compress_csr
from .matrix import DenseMatrix, SparseRowMatrix, as_vector

KERNEL_KINDS = ("matvec", "vecmat", "matmat_right", "matmat_left")


@dataclass
class OpCounter:
    """Tally of work done by compressed kernels (kernels.py:32-38)."""

    multiply_adds: int = 0
    tree_nodes_visited: int = 0
    codes_visited: int = 0


class CompressedMatrix:
    """A TOC1 block resident on the device plus its logical encoding (kernels.py:41-84).

    The device "tree" (the par/key tables the kernels rebuild in shared memory) costs nothing to
    keep, so there is no lazy host tree build; ``tree`` materialises the reference's DecodeTree
    on demand, once, under a lock (kernels.py:68-77)."""

    __slots__ = ("_enc", "_arena", "_lock", "_tree", "_block", "_exact")

    def __init__(self, encoding: LogicalEncoding | None = None, *, _arena: BlockArena | None = None):
        self._enc = encoding
        self._arena = _arena
        self._lock = threading.Lock()
        self._tree = None
        self._block = None
        self._exact = None

    @classmethod
    def from_sparse(cls, s: SparseRowMatrix) -> "CompressedMatrix":
        arena, logical = compress_csr(s.n_cols, s.row_ptr, s.cols, s.vals, np.array([0, s.n_rows], np.int64),
                                      keep_logical=True)
        ic, iv, cd, of = logical[0]
        cdl = cd.tolist()
        enc = LogicalEncoding(n_rows=s.n_rows, n_cols=s.n_cols,
                              pairs=[(int(c), float(v)) for c, v in zip(ic.tolist(), iv.tolist())],
                              rows=[cdl[of[i] : of[i + 1]] for i in range(s.n_rows)])
        return cls(enc, _arena=arena)

    @property
    def encoding(self) -> LogicalEncoding:
        return self._enc

    @property
    def arena(self) -> BlockArena:
        if self._arena is None:
            from .physical import serialize_block

            with self._lock:
                if self._arena is None:
                    self._arena = BlockArena.from_bytes([serialize_block(self._enc)])
        return self._arena

    @property
    def n_rows(self) -> int:
        return self._enc.n_rows

    @property
    def n_cols(self) -> int:
        return self._enc.n_cols

    @property
    def tree(self):
        """The reference's DecodeTree, built on the device once, under a lock (kernels.py:68-77)."""
        if self._tree is None:
            arena = self.arena  # takes the lock itself when it has to serialize
            with self._lock:
                if self._tree is None:
                    self._tree = arena.decode_trees()[0]
        return self._tree

    def exact_plan(self) -> "_ExactPlan":
        """The device schedule of the reference-order products (toc_exact.cu), built once."""
        if self._exact is None:
            tree = self.tree
            with self._lock:
                if self._exact is None:
                    self._exact = _ExactPlan(tree, self.encoding.rows, self.n_cols)
        return self._exact

    def decode(self) -> SparseRowMatrix:
        """Rows back bit for bit (kernels.py:79-80 -> codec.decode), decoded on the device."""
        rp, c, v = self.arena.decode()
        return SparseRowMatrix.from_csr(self.n_cols, rp.cpu().numpy(), c.cpu().numpy(), v.cpu().numpy(), check=False)

    def _charge(self, counter: OpCounter | None, width: int) -> None:
        if counter is not None:
            m = self.arena.meta[0]
            nodes = int(m["n_pairs"]) + int(m["n_derived"])
            codes = int(m["n_codes"])
            counter.multiply_adds += (nodes + codes) * width
            counter.tree_nodes_visited += nodes
            counter.codes_visited += codes

    def __repr__(self):
        e = self._enc
        return f"CompressedMatrix({e.n_rows}x{e.n_cols}, I={len(e.pairs)}, codes={e.total_codes})"


def scalar_multiply(a: CompressedMatrix, c: float) -> CompressedMatrix:
    """Scale every stored value; code rows are shared, not copied (kernels.py:87-102).  The new
    block is rebuilt on the device (value index + repack, physical.rewrite_arena); no tree is
    built.  Scaling by zero keeps the entries as explicit zeros."""
    c = float(c)
    if not math.isfinite(c):
        raise ValueError("scale factor must be finite")
    e = a.encoding
    enc = LogicalEncoding(n_rows=e.n_rows, n_cols=e.n_cols, pairs=[(col, c * val) for col, val in e.pairs],
                          rows=e.rows)
    from .physical import rewrite_arena

    return CompressedMatrix(enc, _arena=rewrite_arena(a.arena, fn=lambda x: x * c))


def elementwise_power(a: CompressedMatrix, p: float) -> CompressedMatrix:
    """Raise every stored value to the power p (kernels.py:105-112).  The values are math.pow's,
    exactly the reference's; the block is rebuilt on the device."""
    p = float(p)
    e = a.encoding
    enc = LogicalEncoding(n_rows=e.n_rows, n_cols=e.n_cols, pairs=[(col, math.pow(val, p)) for col, val in e.pairs],
                          rows=e.rows)
    from .physical import rewrite_arena

    return CompressedMatrix(enc, _arena=rewrite_arena(a.arena, values=[v for _, v in enc.pairs]))


def scalar_add(a: CompressedMatrix, c: float) -> DenseMatrix:
    """A + c as a dense matrix (kernels.py:237-247): adding to the implicit zeros densifies, so this
    decodes -- on the device -- and adds there."""
    c = float(c)
    if not math.isfinite(c):
        raise ValueError("addend must be finite")
    import torch

    rp, cols, vals = a.arena.decode()
    out = torch.zeros((a.n_rows, a.n_cols), dtype=torch.float64, device=vals.device)
    r = torch.repeat_interleave(torch.arange(a.n_rows, device=vals.device), rp[1:] - rp[:-1])
    out[r, cols.long()] = vals
    return DenseMatrix((out + c).cpu().numpy())


def _dev(x: np.ndarray):
    import torch

    return torch.from_numpy(np.array(x, dtype=np.float64, order="C")).cuda()


class _ExactPlan:
    """Device schedule of the reference-order products over one DecodeTree (toc_exact.cu): nodes by
    depth, each row's codes, each node's occurrence rows in row order, its children in descending id
    order, each column's nodes in descending id order."""

    def __init__(self, tree, rows, n_cols: int):
        torch = N.require_cuda()
        par = np.asarray(tree.parent, np.int64)
        T = len(par)
        self.T, self.n_cols, self.n_rows = T, n_cols, len(rows)
        depth = np.zeros(T, np.int64)
        ids = np.arange(1, T)
        if T > 1:  # parents precede children: settle depth one level per pass
            pp = np.maximum(par[1:], 0)
            while True:
                nd = depth[pp] + 1
                if np.array_equal(nd, depth[1:]):
                    break
                depth[1:] = nd
        nodes = ids[np.argsort(depth[1:], kind="stable")]
        maxd = int(depth.max()) if T > 1 else 0
        self.level_off = np.searchsorted(depth[nodes], np.arange(1, maxd + 2)).astype(np.int64)
        col = np.asarray(tree.column, np.int64)
        o = np.lexsort((-ids, par[1:])) if T > 1 else np.zeros(0, np.int64)
        child_off = np.r_[0, np.cumsum(np.bincount(par[1:], minlength=T))] if T > 1 else np.zeros(T + 1, np.int64)
        o2 = np.lexsort((-ids, col[1:])) if T > 1 else np.zeros(0, np.int64)
        col_off = np.r_[0, np.cumsum(np.bincount(col[1:], minlength=n_cols))] if T > 1 else np.zeros(n_cols + 1)
        lens = np.array([len(r) for r in rows], np.int64)
        codes = np.concatenate([np.asarray(r, np.int64) for r in rows]) if len(rows) else np.zeros(0, np.int64)
        rowid = np.repeat(np.arange(len(rows)), lens)
        o3 = np.argsort(codes, kind="stable")
        occ_off = np.r_[0, np.cumsum(np.bincount(codes, minlength=T))]

        def d(x, dt):
            x = np.ascontiguousarray(x, dt)
            return torch.from_numpy(x if x.size else np.zeros(1, dt)).cuda()

        self.parent = d(np.where(par < 0, 0, par), np.int32)
        self.column = d(col, np.int32)
        self.value = d(np.asarray(tree.value, np.float64), np.float64)
        self.level_nodes = d(nodes, np.int32)
        self.rowoff = d(np.r_[0, np.cumsum(lens)], np.int64)
        self.codes = d(codes, np.int32)
        self.occ_off = d(occ_off, np.int64)
        self.occ_row = d(rowid[o3], np.int32)
        self.child_off = d(child_off, np.int64)
        self.child = d(ids[o], np.int32)
        self.col_off = d(col_off, np.int64)
        self.col_node = d(ids[o2], np.int32)
        self.scratch = torch.empty(max(T, 1), dtype=torch.float64, device="cuda")


def matvec(a: CompressedMatrix, v, counter: OpCounter | None = None) -> np.ndarray:
    """A @ v without decompressing A (kernels.py:115-142, Algorithm 5), in the reference's own
    operation order: H node by node, each row summed left to right -- equal to the reference bit
    for bit (toc_exact_matvec).  The batched paths (BlockArena.linalg) reorder sums for speed."""
    vec = as_vector(v, a.n_cols, "vector")
    arena = a.arena
    arena.raise_corrupt()
    out = np.zeros(a.n_rows)
    if a.n_rows and a.n_cols:
        p = a.exact_plan()
        torch = N.require_cuda()
        R = torch.empty(a.n_rows, dtype=torch.float64, device="cuda")
        N.check(N.lib().toc_exact_matvec(p.parent.data_ptr(), p.column.data_ptr(), p.value.data_ptr(),
                                         p.level_nodes.data_ptr(), p.level_off.ctypes.data, len(p.level_off) - 1,
                                         p.rowoff.data_ptr(), p.codes.data_ptr(), a.n_rows, _dev(vec).data_ptr(),
                                         R.data_ptr(), p.scratch.data_ptr(), N.stream_handle()), "toc_exact_matvec")
        out = R.cpu().numpy()
    a._charge(counter, 1)
    return np.asarray(out, dtype=np.float64)


def vecmat(v, a: CompressedMatrix, counter: OpCounter | None = None) -> np.ndarray:
    """v @ A without decompressing A (kernels.py:145-174, Algorithm 6), in the reference's own
    operation order -- equal to the reference bit for bit (toc_exact_vecmat)."""
    vec = as_vector(v, a.n_rows, "vector")
    arena = a.arena
    arena.raise_corrupt()
    out = np.zeros(a.n_cols)
    if a.n_cols:
        p = a.exact_plan()
        torch = N.require_cuda()
        O = torch.empty(a.n_cols, dtype=torch.float64, device="cuda")
        u = _dev(vec) if a.n_rows else torch.zeros(1, dtype=torch.float64, device="cuda")
        N.check(N.lib().toc_exact_vecmat(p.column.data_ptr(), p.value.data_ptr(), p.T, p.level_nodes.data_ptr(),
                                         p.level_off.ctypes.data, len(p.level_off) - 1, p.occ_off.data_ptr(),
                                         p.occ_row.data_ptr(), p.child_off.data_ptr(), p.child.data_ptr(),
                                         p.col_off.data_ptr(), p.col_node.data_ptr(), a.n_cols, u.data_ptr(),
                                         O.data_ptr(), p.scratch.data_ptr(), N.stream_handle()), "toc_exact_vecmat")
        out = O.cpu().numpy()
    a._charge(counter, 1)
    return np.asarray(out, dtype=np.float64)


def matmat_right(a: CompressedMatrix, m: DenseMatrix, counter: OpCounter | None = None) -> DenseMatrix:
    """A @ M without decompressing A (kernels.py:177-203, Algorithm 8)."""
    if a.n_cols != m.n_rows:
        raise ValueError(f"inner dimensions differ: left has {a.n_cols} columns, right has {m.n_rows} rows")
    p = m.n_cols
    if a.n_rows == 0 or p == 0:
        out = np.zeros((a.n_rows, p))
    else:
        arena = a.arena
        out = arena.matmat(0, _dev(m.values), p).cpu().numpy()
    a._charge(counter, p)
    return DenseMatrix(out)


def matmat_left(m: DenseMatrix, a: CompressedMatrix, counter: OpCounter | None = None) -> DenseMatrix:
    """M @ A without decompressing A (kernels.py:206-234, Algorithm 9)."""
    if m.n_cols != a.n_rows:
        raise ValueError(f"inner dimensions differ: left has {m.n_cols} columns, right has {a.n_rows} rows")
    p = m.n_rows
    if a.n_rows == 0 or p == 0 or a.n_cols == 0:
        out = np.zeros((p, a.n_cols))
    else:
        arena = a.arena
        out = arena.matmat(1, _dev(np.ascontiguousarray(m.values.T)), p)[0].cpu().numpy()
    a._charge(counter, p)
    return DenseMatrix(out)


def kernel_cost(a: CompressedMatrix, kind: str, width: int = 1) -> int:
    """Predicted multiply-add count (kernels.py:250-266)."""
    if kind not in KERNEL_KINDS:
        raise ValueError(f"unknown kernel kind {kind!r}; expected one of {KERNEL_KINDS}")
    if width < 1:
        raise ValueError(f"width must be positive, got {width}")
    if kind in ("matvec", "vecmat") and width != 1:
        raise ValueError(f"{kind} has a single lane; width {width} is meaningless")
    e = a.encoding
    return (len(e.pairs) + e.derived_node_count() + e.total_codes) * width


def dense_kernel_cost(n_rows: int, n_cols: int, kind: str, width: int = 1) -> int:
    if kind not in KERNEL_KINDS:
        raise ValueError(f"unknown kernel kind {kind!r}; expected one of {KERNEL_KINDS}")
    return 2 * n_rows * n_cols * width


def csr_kernel_cost(nnz: int, kind: str, width: int = 1) -> int:
    if kind not in KERNEL_KINDS:
        raise ValueError(f"unknown kernel kind {kind!r}; expected one of {KERNEL_KINDS}")
    return 2 * nnz * width


class BatchSweep:
    """Public batched API over host-resident TOC1 blocks.

    ``run(v, u)`` uploads the blocks and operands from pinned host memory, validates/indexes the
    blocks on the device, runs A.v and v^T.A for every batch (fused launches), and returns host
    arrays (R: concatenated row results, O: one n_cols row per batch).  The batches are split
    into chunks: the host->device copy of chunk k+1 (copy stream) overlaps validation and compute
    of chunk k (compute stream) and the device->host copy of chunk k-1's results (third stream).  This replaces the reference's per-batch loop over ``matvec`` /
    ``vecmat`` (cli.py:340-356)."""

    def __init__(self, blocks_h: np.ndarray, block_off, block_len, chunks: int = 8):
        torch = N.require_cuda()
        self.torch = torch
        block_off = np.asarray(block_off, np.int64)
        block_len = np.asarray(block_len, np.int64)
        nbytes = int(len(blocks_h))
        self.host = torch.zeros(nbytes + 16, dtype=torch.uint8, pin_memory=True)  # +16 tail padding
        self.host.numpy()[:nbytes] = blocks_h[:nbytes]
        self.nbytes = nbytes
        self.dev = torch.empty_like(self.host, device="cuda")
        self.dev.copy_(self.host)
        nb = len(block_off)
        bounds = np.linspace(0, nb, min(max(chunks, 1), max(nb, 1)) + 1).astype(np.int64)
        self.chunks = []
        row0 = 0
        for b0, b1 in zip(bounds[:-1], bounds[1:]):
            if b1 <= b0:
                continue
            arena = BlockArena(self.dev, block_off[b0:b1], block_len[b0:b1])
            lo = int(block_off[b0])
            hi = int(block_off[b1 - 1] + block_len[b1 - 1]) if b1 < nb else nbytes
            hi = min(nbytes + 16, (hi + 15) & ~15) if b1 < nb else nbytes + 16
            self.chunks.append((arena, int(b0), int(b1), lo, hi, row0))
            row0 += arena.n_rows_total
        self.n_rows = row0
        self.n_cols = self.chunks[0][0].n_cols if self.chunks else 0
        self.n_blocks = nb
        self.v_h = torch.empty(max(self.n_cols, 1), dtype=torch.float64, pin_memory=True)
        self.u_h = torch.empty(max(self.n_rows, 1), dtype=torch.float64, pin_memory=True)
        self.v_d = torch.empty_like(self.v_h, device="cuda")
        self.u_d = torch.empty_like(self.u_h, device="cuda")
        self.R_d = torch.empty(max(self.n_rows, 1), dtype=torch.float64, device="cuda")
        self.O_d = torch.empty((max(nb, 1), max(self.n_cols, 1)), dtype=torch.float64, device="cuda")
        self.R_h = torch.empty_like(self.R_d, device="cpu").pin_memory()
        self.O_h = torch.empty_like(self.O_d, device="cpu").pin_memory()
        # own streams: work on the legacy default stream would wait for every upload enqueued before it
        self.copy_stream = torch.cuda.Stream()
        self.comp_stream = torch.cuda.Stream()
        self.d2h_stream = torch.cuda.Stream()
        # the native pipeline's chunk descriptors (toc_sweep_upload / toc_sweep_compute)
        self.meta_all_h = torch.empty(max(nb, 1) * N.META_DTYPE.itemsize, dtype=torch.uint8, pin_memory=True)
        self.cdesc = (N.TocSweepChunk * max(len(self.chunks), 1))()
        for k, (arena, b0, b1, lo, hi, r0) in enumerate(self.chunks):
            plan = arena.plan(N.TOC_MATVEC | N.TOC_VECMAT)
            scratch = arena._scratch_for(plan)
            d = self.cdesc[k]
            d.byte_lo, d.byte_hi = lo, hi
            d.d_arena = arena.data.data_ptr()
            d.d_block_off, d.d_block_len = arena.block_off_d.data_ptr(), arena.block_len_d.data_ptr()
            d.d_meta, d.d_row_base = arena.meta_d.data_ptr(), arena.row_base_d.data_ptr()
            d.d_scratch = scratch.data_ptr() if scratch is not None else None
            d.n_blocks, d.b0, d.row0, d.n_rows = arena.n_blocks, b0, r0, arena.n_rows_total
            d.plan = plan
        N.check(N.lib().toc_sweep_events(self.cdesc, len(self.chunks)), "toc_sweep_events")  # this sweep's own
        self.h2d_bytes = nbytes + 8 * self.n_cols + 8 * self.n_rows
        self.d2h_bytes = 8 * self.n_rows + 8 * nb * self.n_cols + sum(c[0].meta_d.numel() for c in self.chunks)

    @classmethod
    def from_host_blocks(cls, blocks_h, block_off, block_len, chunks: int = 8) -> "BatchSweep":
        return cls(np.asarray(blocks_h, np.uint8), block_off, block_len, chunks)

    def __del__(self):
        try:
            N.lib().toc_sweep_events_free(self.cdesc, len(self.chunks))
        except Exception:  # interpreter shutdown
            pass

    def run(self, v, u, out=None):
        """``submit`` then ``finish``: one step, results ready on return."""
        self.submit(v, u, out=out)
        return self.finish()

    def submit(self, v, u, out=None):
        """Enqueue one step without waiting for it (``finish`` waits and returns the results).  Two
        BatchSweep objects over the same host blocks, submitted alternately, keep the host link busy
        across steps: while one's last chunks are validated, swept and downloaded, the other's
        uploads are already under way.  At most one step per object may be in flight.

        The first chunk's block bytes are enqueued (two chunks when v / u must be staged into
        pinned buffers first; v and u given as pinned float64 CPU tensors are copied from in place);
        then the operands, the other chunks' bytes (all on one copy stream: host -> device copies
        are served in submission order), every chunk's validation and fused A.v + v^T.A (each as
        soon as its bytes and operands are in) and the result downloads (toc_sweep.cu).
        Returns (R [n_rows], O [n_blocks, n_cols]) as new arrays; with out=(R_h, O_h) -- float64
        CPU tensors of those shapes, pinned for asynchronous copies -- the results are downloaded
        straight into them and they are returned (no extra host copy)."""
        if getattr(self, "_pending", None) is not None:
            raise RuntimeError("BatchSweep.submit(): the previous step has not been finished")
        torch = self.torch
        L = N.lib()
        caller = torch.cuda.current_stream()
        cs, comp, ds = self.copy_stream, self.comp_stream, self.d2h_stream
        for st in (cs, comp, ds):
            st.wait_stream(caller)  # the caller's earlier work on these buffers is done
        n = len(self.chunks)

        def pinned(x, size):  # the caller's own pinned float64 vector: copied from in place
            return (isinstance(x, torch.Tensor) and x.device.type == "cpu" and x.dtype == torch.float64
                    and x.dim() == 1 and x.numel() == size and x.is_contiguous() and x.is_pinned())

        direct = pinned(v, self.n_cols) and pinned(u, self.n_rows)
        # with staged operands the host copies v / u into pinned buffers first: two chunks go ahead
        # so the link stays busy meanwhile; pinned operands follow the first chunk at once
        k_first = min(n, 1 if direct else 2)
        N.check(L.toc_sweep_upload(self.host.data_ptr(), self.dev.data_ptr(), self.cdesc, 0, k_first, cs.cuda_stream),
                "toc_sweep_upload")
        if direct:
            v_src, u_src = v.data_ptr(), u.data_ptr()
        else:
            self.v_h.numpy()[: self.n_cols] = as_vector(v, self.n_cols, "vector")
            self.u_h.numpy()[: self.n_rows] = as_vector(u, self.n_rows, "vector")
            v_src, u_src = self.v_h.data_ptr(), self.u_h.data_ptr()
        N.check(L.toc_sweep_operands(self.cdesc, n, self.n_cols, v_src, self.v_d.data_ptr(), u_src,
                                     self.u_d.data_ptr(), cs.cuda_stream), "toc_sweep_operands")
        N.check(L.toc_sweep_upload(self.host.data_ptr(), self.dev.data_ptr(), self.cdesc, k_first, n, cs.cuda_stream),
                "toc_sweep_upload")
        if out is not None:
            R_o, O_o = out
            if (R_o.dtype != torch.float64 or O_o.dtype != torch.float64 or R_o.device.type != "cpu"
                    or O_o.device.type != "cpu" or R_o.numel() < self.n_rows or O_o.numel() < self.n_blocks * self.n_cols
                    or not R_o.is_contiguous() or not O_o.is_contiguous()):
                raise ValueError("out must be contiguous float64 CPU tensors of n_rows and n_blocks x n_cols")
            R_dst, O_dst = R_o.data_ptr(), O_o.data_ptr()
        else:
            R_dst, O_dst = self.R_h.data_ptr(), self.O_h.data_ptr()
        N.check(L.toc_sweep_compute(self.cdesc, n, self.n_cols, self.v_d.data_ptr(), self.u_d.data_ptr(),
                                    self.R_d.data_ptr(), R_dst, self.O_d.data_ptr(), O_dst,
                                    self.meta_all_h.data_ptr(), comp.cuda_stream, ds.cuda_stream), "toc_sweep_compute")
        self._pending = (caller, out, (v, u))  # operands stay referenced until the copies are done

    def finish(self):
        """Wait for the submitted step: block-format / corrupt-tree errors are raised here (the
        reference's exception classes); returns (R, O) as ``run`` does."""
        pending = getattr(self, "_pending", None)
        if pending is None:
            raise RuntimeError("BatchSweep.finish() without a submitted step")
        caller, out, _operands = pending
        self._pending = None
        ds = self.d2h_stream
        ds.synchronize()
        caller.wait_stream(ds)
        meta = np.frombuffer(self.meta_all_h.numpy().tobytes(), dtype=N.META_DTYPE)[: self.n_blocks]
        if np.any(meta["status"] != N.TOC_OK) or np.any(meta["corrupt"] != 0):
            for arena, b0, b1, *_rest in self.chunks:
                arena.meta = meta[b0:b1].copy()
                arena.raise_format_errors()
                arena.raise_corrupt()
        if out is not None:
            return out
        return self.R_h.numpy()[: self.n_rows].copy(), self.O_h.numpy()[: self.n_blocks, : self.n_cols].copy()
