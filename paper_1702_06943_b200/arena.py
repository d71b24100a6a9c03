"""Device-resident arena of TOC1 blocks: the HBM layout every kernel reads.

Layout:
  * ``data``: one uint8 buffer holding the exact TOC1 bytes of every batch (reference
    physical.py:1-21), batch b at ``block_off[b]``, each block 16-byte aligned;
  * ``meta``: one 68-byte TocBlockMeta per batch, written on the device by toc_index_blocks;
  * 16 bytes of tail padding after the last block (the sequential unpackers may read one
    aligned word past a section);
  * ``row_base``: the first row of each batch in the concatenated row space (outputs of A.v and
    the u operand of v^T.A are indexed by it).

The arena replaces a list of reference ``CompressedMatrix`` objects (kernels.py:41-84) and the
per-batch Python loops of cli.py:299-383 / training.py:355-358 with one launch per operation.
"""

from __future__ import annotations

import ctypes
from typing import Sequence

import numpy as np

from . import _native as N
from .errors import raise_for_meta


def _ptr(t):
    """Device pointer of a tensor; a 1-element dummy stands in for empty operands."""
    if t is None:
        return None
    if t.numel() == 0:
        return _EMPTY.setdefault((t.device, t.dtype), t.new_zeros(1)).data_ptr()
    return t.data_ptr()


_EMPTY: dict = {}


def _align16(x: int) -> int:
    return (x + 15) & ~15


class BlockArena:
    def __init__(self, data, block_off: np.ndarray, block_len: np.ndarray, meta_d=None, *,
                 check: bool = True):
        torch = N.require_cuda()
        self.torch = torch
        self.data = data
        self.block_off = np.ascontiguousarray(block_off, np.int64)
        self.block_len = np.ascontiguousarray(block_len, np.int64)
        self.n_blocks = len(self.block_off)
        dev = data.device
        self.block_off_d = torch.from_numpy(self.block_off).to(dev)
        self.block_len_d = torch.from_numpy(self.block_len).to(dev)
        if meta_d is None:
            meta_d = torch.empty(max(self.n_blocks, 1) * N.META_DTYPE.itemsize, dtype=torch.uint8, device=dev)
            rc = N.lib().toc_index_blocks(data.data_ptr(), self.block_off_d.data_ptr(),
                                          self.block_len_d.data_ptr(), self.n_blocks, meta_d.data_ptr(),
                                          N.stream_handle())
            N.check(rc, "toc_index_blocks")
        self.meta_d = meta_d
        self.meta = np.frombuffer(meta_d.cpu().numpy().tobytes(), dtype=N.META_DTYPE)[: self.n_blocks].copy()
        if check:
            self.raise_format_errors()
        rows = self.meta["n_rows"].astype(np.int64)
        self.row_base = np.zeros(self.n_blocks, np.int64)
        if self.n_blocks:
            np.cumsum(rows[:-1], out=self.row_base[1:])
        self.n_rows_total = int(rows.sum())
        self.row_base_d = torch.from_numpy(self.row_base).to(dev)
        self.n_cols = int(self.meta["n_cols"][0]) if self.n_blocks else 0
        self._plans: dict[int, N.TocPlan] = {}
        self._scratch = None
        self.trees = None  # device tree cache (build_trees)
        self.levels = None  # level cache (build_levels)

    # ---- construction ------------------------------------------------------------------------
    @classmethod
    def from_bytes(cls, blocks: Sequence[bytes], device: str = "cuda", check: bool = True) -> "BlockArena":
        """Upload serialized TOC1 blocks (reference physical.serialize_block output)."""
        torch = N.require_cuda()
        lens = np.fromiter((len(b) for b in blocks), dtype=np.int64, count=len(blocks))
        offs = np.zeros(len(blocks), np.int64)
        pos = 0
        for i, n in enumerate(lens):
            offs[i] = pos
            pos = _align16(pos + int(n))
        host = torch.zeros(pos + 16, dtype=torch.uint8, pin_memory=True)  # +16: tail padding (unpackers)
        hv = host.numpy()
        for i, b in enumerate(blocks):
            hv[offs[i] : offs[i] + lens[i]] = np.frombuffer(b, dtype=np.uint8)
        data = host.to(device, non_blocking=True)
        return cls(data, offs, lens, check=check)

    def raise_format_errors(self) -> None:
        bad = np.flatnonzero(self.meta["status"] != N.TOC_OK)
        if len(bad):
            b = int(bad[0])
            head = bytes(self.data[int(self.block_off[b]) : int(self.block_off[b]) + 4].cpu().numpy())
            raise_for_meta(self.meta[b], head)

    def raise_corrupt(self) -> None:
        bad = np.flatnonzero(self.meta["corrupt"] != 0)
        if len(bad):
            raise_for_meta(self.meta[int(bad[0])], lazy=True)

    # ---- accounting --------------------------------------------------------------------------
    @property
    def block_bytes(self) -> int:
        """Sum of the TOC1 block sizes (the algorithmic bytes of one pass)."""
        return int(self.block_len.sum())

    def tree_lengths(self) -> np.ndarray:
        return 1 + self.meta["n_pairs"].astype(np.int64) + self.meta["n_derived"].astype(np.int64)

    # ---- kernels -----------------------------------------------------------------------------
    def plan(self, kind: int) -> N.TocPlan:
        p = self._plans.get(kind)
        if p is None:
            p = N.TocPlan()
            rc = N.lib().toc_plan(self.meta.ctypes.data_as(ctypes.c_void_p), self.n_blocks, kind, ctypes.byref(p))
            N.check(rc, "toc_plan")
            self._plans[kind] = p
        return p

    def _scratch_for(self, plan: N.TocPlan):
        if plan.scratch_bytes == 0:
            return None
        if self._scratch is None or self._scratch.numel() < plan.scratch_bytes:
            self._scratch = self.torch.empty(plan.scratch_bytes, dtype=self.torch.uint8, device=self.data.device)
        return self._scratch

    def decode(self):
        """All rows back as CSR on the device: (row_ptr int64 [n_rows_total + 1], cols int32, vals
        float64), batch b's rows at row_base[b] (codec.py:274-292, bit for bit)."""
        self.raise_format_errors()
        self.raise_corrupt()
        torch = self.torch
        dev = self.data.device
        plan = self.plan(N.TOC_MATVEC)
        scratch = self._scratch_for(plan)
        sp = scratch.data_ptr() if scratch is not None else None
        L = N.lib()
        nnz = torch.zeros(max(self.n_rows_total, 1), dtype=torch.int64, device=dev)
        N.check(L.toc_decode_counts(self.data.data_ptr(), self.block_off_d.data_ptr(), self.meta_d.data_ptr(),
                                    self.row_base_d.data_ptr(), self.n_blocks, ctypes.byref(plan), nnz.data_ptr(), sp,
                                    N.stream_handle()), "toc_decode_counts")
        row_ptr = torch.zeros(self.n_rows_total + 1, dtype=torch.int64, device=dev)
        torch.cumsum(nnz[: self.n_rows_total], 0, out=row_ptr[1:])
        total = int(row_ptr[-1].item())
        cols = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
        vals = torch.empty(max(total, 1), dtype=torch.float64, device=dev)
        N.check(L.toc_decode_rows(self.data.data_ptr(), self.block_off_d.data_ptr(), self.meta_d.data_ptr(),
                                  self.row_base_d.data_ptr(), self.n_blocks, ctypes.byref(plan), row_ptr.data_ptr(),
                                  cols.data_ptr(), vals.data_ptr(), sp, N.stream_handle()), "toc_decode_rows")
        return row_ptr, cols[:total], vals[:total]

    def scalar_multiply(self, c: float) -> "BlockArena":
        """Every block's values scaled by c, rebuilt on the device (kernels.py:87-102 per block)."""
        import math

        from .physical import rewrite_arena

        c = float(c)
        if not math.isfinite(c):
            raise ValueError("scale factor must be finite")
        return rewrite_arena(self, fn=lambda x: x * c)

    def elementwise_power(self, p: float) -> "BlockArena":
        """Every block's values raised to p on the device (kernels.py:105-112 per block).  torch.pow:
        exact for p = 1, 2 and 0.5 (square, sqrt); otherwise within CUDA pow's 2 ulp of math.pow."""
        from .physical import rewrite_arena

        p = float(p)
        return rewrite_arena(self, fn=lambda x: self.torch.pow(x, p))

    def decode_trees(self) -> list:
        """Every block's DecodeTree (reference codec.py:194-259) built on the device."""
        from .codec import DecodeTree

        self.raise_format_errors()
        self.raise_corrupt()
        torch = self.torch
        dev = self.data.device
        plan = self.plan(N.TOC_MATVEC)
        scratch = self._scratch_for(plan)
        T = self.tree_lengths()
        base = np.concatenate([[0], np.cumsum(T)]).astype(np.int64)
        total = int(base[-1])
        base_d = torch.from_numpy(base[:-1].copy()).to(dev)
        par = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
        col = torch.empty_like(par)
        fcol = torch.empty_like(par)
        val = torch.empty(max(total, 1), dtype=torch.float64, device=dev)
        fval = torch.empty_like(val)
        N.check(N.lib().toc_tree_arrays(self.data.data_ptr(), self.block_off_d.data_ptr(), self.meta_d.data_ptr(),
                                        self.n_blocks, ctypes.byref(plan), base_d.data_ptr(), par.data_ptr(),
                                        col.data_ptr(), val.data_ptr(), fcol.data_ptr(), fval.data_ptr(),
                                        scratch.data_ptr() if scratch is not None else None, N.stream_handle()),
                "toc_tree_arrays")
        h = [x.cpu().numpy() for x in (par, col, val, fcol, fval)]
        out = []
        for b in range(self.n_blocks):
            lo, hi = int(base[b]), int(base[b + 1])
            out.append(DecodeTree(n_cols=int(self.meta["n_cols"][b]), parent=h[0][lo:hi].tolist(),
                                  column=h[1][lo:hi].tolist(), value=h[2][lo:hi].tolist(),
                                  first_col=h[3][lo:hi].tolist(), first_val=h[4][lo:hi].tolist()))
        return out

    def build_trees(self):
        """Build the device tree cache: each batch's tree prefix (row offsets, derived-node bases,
        final codes, node table), once -- the device counterpart of the reference's lazily built,
        reused CompressedMatrix.tree (kernels.py:68-77).  Later linalg calls pull it into shared
        memory with one bulk copy per batch instead of rebuilding it from the codes."""
        torch = self.torch
        self.raise_corrupt()
        plan = self.plan(N.TOC_MATVEC | N.TOC_VECMAT)
        off = np.zeros(self.n_blocks + 1, np.int64)
        N.check(N.lib().toc_tree_offsets(self.meta.ctypes.data_as(ctypes.c_void_p), self.n_blocks, plan.wide,
                                         off.ctypes.data_as(ctypes.c_void_p)), "toc_tree_offsets")
        trees = torch.empty(int(off[-1]) + 16, dtype=torch.uint8, device=self.data.device)
        tree_off_d = torch.from_numpy(off[:-1].copy()).to(self.data.device)
        scratch = self._scratch_for(plan)
        N.check(N.lib().toc_build_trees(self.data.data_ptr(), self.block_off_d.data_ptr(), self.meta_d.data_ptr(),
                                        self.n_blocks, ctypes.byref(plan), tree_off_d.data_ptr(), trees.data_ptr(),
                                        scratch.data_ptr() if scratch is not None else None, N.stream_handle()),
                "toc_build_trees")
        self.trees, self.tree_off_d, self.tree_bytes = trees, tree_off_d, int(off[-1])
        return self

    def build_levels(self, n_threads: int = 0) -> bool:
        """Build the slot cache (toc_levels_build, csrc/toc_levels.cu): per batch the pairs in
        column order, the inner nodes of C' (those a used derived node hangs off) with their
        (parent, key) records, and the code stream as slot references cut into equal per-thread
        ranges -- built once on the host from a copy of the arena, the counterpart of the
        reference's cached CompressedMatrix.tree (kernels.py:68-77).  Returns False (and keeps no
        cache) when some batch needs slots wider than 16 bits or the tables do not fit shared
        memory; linalg then uses the tree cache / block-only paths."""
        torch = self.torch
        self.raise_corrupt()
        L = N.lib()
        host = self.data.cpu().numpy()
        h = L.toc_levels_build(host.ctypes.data_as(ctypes.c_void_p), self.block_off.ctypes.data_as(ctypes.c_void_p),
                               self.meta.ctypes.data_as(ctypes.c_void_p), self.n_blocks, n_threads)
        if not h:
            raise N.NativeError("toc_levels_build failed")
        try:
            total, max_slots, max_stage, max_rows = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
            rc = L.toc_levels_info(h, ctypes.byref(total), ctypes.byref(max_slots), ctypes.byref(max_stage),
                                   ctypes.byref(max_rows))
            if rc == N.TOC_E_ARG:
                self.levels = None
                return False
            N.check(rc, "toc_levels_build")
            buf = np.zeros(int(total.value) + 16, np.uint8)
            off = np.zeros(self.n_blocks + 1, np.int64)
            N.check(L.toc_levels_copy(h, buf.ctypes.data_as(ctypes.c_void_p), off.ctypes.data_as(ctypes.c_void_p)),
                    "toc_levels_copy")
        finally:
            L.toc_levels_free(h)
        _, optin, _ = N.device_info()
        need = L.toc_levels_smem(N.TOC_MATVEC | N.TOC_VECMAT, self.n_cols, max_slots.value, max_stage.value,
                                 max_rows.value)
        if need < 0 or need > optin or self.n_cols > 65536:
            self.levels = None
            return False
        dev = self.data.device
        self.levels = torch.from_numpy(buf).to(dev)
        self.levels_off_d = torch.from_numpy(off).to(dev)
        self.levels_bytes = int(total.value)
        self.levels_dims = (max_slots.value, max_stage.value, max_rows.value)
        return True

    def _launch_levels(self, kind: int, v, R, u, O, b0: int, b1: int, stream) -> None:
        """toc_linalg_levels over batches [b0, b1) of the slot cache (pointers are device
        addresses; O points at batch b0's row)."""
        slots, stage, rows = self.levels_dims
        rc = N.lib().toc_linalg_levels(
            self.row_base_d.data_ptr() + 8 * b0, int(b1 - b0), kind, self.n_cols, slots, stage, rows,
            v if kind & N.TOC_MATVEC else None, R if kind & N.TOC_MATVEC else None,
            u if kind & N.TOC_VECMAT else None, O if kind & N.TOC_VECMAT else None,
            self.levels.data_ptr(), self.levels_off_d.data_ptr() + 8 * b0, stream)
        N.check(rc, "toc_linalg_levels")

    def linalg(self, kind: int, v=None, u=None, R=None, O=None, use_trees: bool = True, use_levels=None):
        """kind = TOC_MATVEC | TOC_VECMAT.  v: device float64 [n_cols]; u: device float64
        [n_rows_total].  Returns (R [n_rows_total], O [n_blocks, n_cols]) device tensors.  Uses
        the slot cache when it has been built (use_levels None or True; False skips it), else the
        tree cache when it has been built (and use_trees), else rebuilds trees per call."""
        torch = self.torch
        self.raise_corrupt()
        dev = self.data.device
        if kind & N.TOC_MATVEC:
            if R is None:  # never a NULL pointer, even for zero rows
                R = torch.empty(max(self.n_rows_total, 1), dtype=torch.float64, device=dev)[: self.n_rows_total]
        if kind & N.TOC_VECMAT:
            if O is None:
                O = torch.empty(max(self.n_blocks * self.n_cols, 1), dtype=torch.float64,
                                device=dev)[: self.n_blocks * self.n_cols].view(self.n_blocks, self.n_cols)
        if use_levels is not False and getattr(self, "levels", None) is not None:
            self._launch_levels(kind, _ptr(v), _ptr(R), _ptr(u), _ptr(O), 0, self.n_blocks, N.stream_handle())
            return R, O
        plan = self.plan(kind)
        scratch = self._scratch_for(plan)
        trees = self.trees is not None and use_trees
        rc = N.lib().toc_linalg_trees(
            self.data.data_ptr(), self.block_off_d.data_ptr(), self.meta_d.data_ptr(), self.row_base_d.data_ptr(),
            self.n_blocks, ctypes.byref(plan), kind,
            _ptr(v), _ptr(R), _ptr(u), _ptr(O),
            scratch.data_ptr() if scratch is not None else None,
            self.trees.data_ptr() if trees else None, self.tree_off_d.data_ptr() if trees else None,
            N.stream_handle())
        N.check(rc, "toc_linalg")
        return R, O

    def linalg_pipelined(self, kind: int, v_h, u_h, R_h, O_h, chunks: int = 4, slot: int = 0, wait: bool = True):
        """A.v and / or v^T.A with the operands and results in pinned host tensors and the arena
        (with its slot cache, else its tree cache) resident: the batches go in `chunks` slices so that the upload of
        slice k's u, its launch, and the read-back of slice k-1's R / O overlap on three streams.
        v_h [n_cols], u_h [n_rows_total], R_h [n_rows_total], O_h [n_blocks, n_cols]: float64, pinned.
        The step's stream work is captured into a CUDA graph the second time it is called with the
        same host tensors and replayed from then on (one launch call per step instead of dozens).
        Returns when R_h / O_h hold the results; with wait=False it returns once the step is
        enqueued (``pipelined_wait(slot)`` waits) -- `slot` selects one of several sets of device
        buffers, so steps submitted alternately on slots 0 and 1 overlap one step's read-back with
        the next step's upload and launches."""
        torch = self.torch
        self.raise_corrupt()
        slots = getattr(self, "levels", None) is not None
        if self.trees is None and not slots:
            self.build_trees()
        dev = self.data.device
        pipes = getattr(self, "_pipes", None)
        if pipes is None:
            pipes = self._pipes = {}
        st = pipes.get(slot)
        if st is None:
            st = pipes[slot] = {"up": torch.cuda.Stream(), "run": torch.cuda.Stream(), "down": torch.cuda.Stream(),
                                "main": torch.cuda.Stream(), "graphs": {}, "seen": set(),
                                "v": torch.empty(max(self.n_cols, 1), dtype=torch.float64, device=dev),
                                "u": torch.empty(max(self.n_rows_total, 1), dtype=torch.float64, device=dev),
                                "R": torch.empty(max(self.n_rows_total, 1), dtype=torch.float64, device=dev),
                                "O": torch.empty((max(self.n_blocks, 1), max(self.n_cols, 1)), dtype=torch.float64,
                                                 device=dev)}
        key = (kind, v_h.data_ptr(), u_h.data_ptr(), R_h.data_ptr(), O_h.data_ptr(), chunks, slots)
        main = st["main"]
        main.wait_stream(torch.cuda.current_stream())
        g = st["graphs"].get(key)
        if g is not None:
            with torch.cuda.stream(main):
                g.replay()
        elif key in st["seen"] and len(st["graphs"]) < 8:
            main.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=main):
                self._pipeline_enqueue(st, kind, v_h, u_h, R_h, O_h, chunks, slots)
            st["graphs"][key] = g
            st["keep"] = (v_h, u_h, R_h, O_h)  # the graph holds their addresses
            with torch.cuda.stream(main):
                g.replay()
        else:
            st["seen"].add(key)
            with torch.cuda.stream(main):
                self._pipeline_enqueue(st, kind, v_h, u_h, R_h, O_h, chunks, slots)
        if wait:
            main.synchronize()
        return R_h, O_h

    def pipelined_wait(self, slot: int = 0) -> None:
        """Wait for the step submitted on `slot` with linalg_pipelined(..., wait=False)."""
        st = getattr(self, "_pipes", {}).get(slot)
        if st is not None:
            st["main"].synchronize()

    def _pipeline_enqueue(self, st, kind, v_h, u_h, R_h, O_h, chunks, slots) -> None:
        """One pipelined step on the current stream (eager, or under CUDA graph capture): fork to the
        upload / launch / read-back streams, slice by slice, and join them back."""
        torch = self.torch
        mv, vm = bool(kind & N.TOC_MATVEC), bool(kind & N.TOC_VECMAT)
        plan = None if slots else self.plan(kind)
        scratch = None if slots else self._scratch_for(plan)
        L = N.lib()
        bounds = np.linspace(0, self.n_blocks, min(max(chunks, 1), max(self.n_blocks, 1)) + 1).astype(np.int64)
        rb = np.concatenate([self.row_base, [self.n_rows_total]])
        cur = torch.cuda.current_stream()
        for s in (st["up"], st["run"], st["down"]):
            s.wait_stream(cur)
        with torch.cuda.stream(st["up"]):
            if mv:
                st["v"].copy_(v_h, non_blocking=True)
        for b0, b1 in zip(bounds[:-1].tolist(), bounds[1:].tolist()):
            if b1 <= b0:
                continue
            r0, r1 = int(rb[b0]), int(rb[b1])
            up = torch.cuda.Event()
            with torch.cuda.stream(st["up"]):
                if vm:
                    st["u"][r0:r1].copy_(u_h[r0:r1], non_blocking=True)
                up.record()
            done = torch.cuda.Event()
            with torch.cuda.stream(st["run"]):
                st["run"].wait_event(up)
                if slots:
                    self._launch_levels(kind, st["v"].data_ptr() if mv else None, st["R"].data_ptr() if mv else None,
                                        st["u"].data_ptr() if vm else None,
                                        st["O"].data_ptr() + 8 * int(b0) * self.n_cols if vm else None, b0, b1,
                                        ctypes.c_void_p(st["run"].cuda_stream))
                else:
                    rc = L.toc_linalg_trees(
                        self.data.data_ptr(), self.block_off_d.data_ptr() + 8 * b0, self.meta_d.data_ptr() + 68 * b0,
                        self.row_base_d.data_ptr() + 8 * b0, int(b1 - b0), ctypes.byref(plan), kind,
                        st["v"].data_ptr() if mv else None, st["R"].data_ptr() if mv else None,
                        st["u"].data_ptr() if vm else None,
                        st["O"].data_ptr() + 8 * int(b0) * self.n_cols if vm else None,
                        scratch.data_ptr() if scratch is not None else None, self.trees.data_ptr(),
                        self.tree_off_d.data_ptr() + 8 * b0, ctypes.c_void_p(st["run"].cuda_stream))
                    N.check(rc, "toc_linalg_trees")
                done.record()
            with torch.cuda.stream(st["down"]):
                st["down"].wait_event(done)
                if mv:
                    R_h[r0:r1].copy_(st["R"][r0:r1], non_blocking=True)
                if vm:
                    O_h[b0:b1].copy_(st["O"][b0:b1], non_blocking=True)
        for s in (st["up"], st["run"], st["down"]):
            cur.wait_stream(s)

    def linalg32(self, kind: int, v=None, u=None, R=None, O=None, use_levels=None):
        """The fp32 variant: v [n_cols], u [n_rows_total] float32 device tensors -> (R [n_rows_total],
        O [n_blocks, n_cols]) float32.  Over the slot cache when it has been built
        (toc_linalg_levels32; use_levels False skips it), else over the tree cache (toc_linalg32,
        built on first use)."""
        torch = self.torch
        dev = self.data.device
        if kind & N.TOC_MATVEC and R is None:
            R = torch.empty(max(self.n_rows_total, 1), dtype=torch.float32, device=dev)[: self.n_rows_total]
        if kind & N.TOC_VECMAT and O is None:
            O = torch.empty((max(self.n_blocks, 1), max(self.n_cols, 1)), dtype=torch.float32,
                            device=dev)[: self.n_blocks, : self.n_cols]
        if use_levels is not False and getattr(self, "levels", None) is not None and self.n_blocks:
            self.raise_corrupt()
            slots, stage, rows = self.levels_dims
            N.check(N.lib().toc_linalg_levels32(
                self.row_base_d.data_ptr(), self.n_blocks, kind, self.n_cols, slots, stage, rows,
                _ptr(v) if kind & N.TOC_MATVEC else None, _ptr(R) if kind & N.TOC_MATVEC else None,
                _ptr(u) if kind & N.TOC_VECMAT else None, _ptr(O) if kind & N.TOC_VECMAT else None,
                self.levels.data_ptr(), self.levels_off_d.data_ptr(), N.stream_handle()), "toc_linalg_levels32")
            return R, O
        if getattr(self, "trees", None) is None:
            self.build_trees()
        plan = self.plan(N.TOC_MATVEC | N.TOC_VECMAT)
        N.check(N.lib().toc_linalg32(self.data.data_ptr(), self.block_off_d.data_ptr(), self.meta_d.data_ptr(),
                                     self.row_base_d.data_ptr(), self.n_blocks, ctypes.byref(plan), kind,
                                     _ptr(v) if kind & N.TOC_MATVEC else None, _ptr(R) if kind & N.TOC_MATVEC else None,
                                     _ptr(u) if kind & N.TOC_VECMAT else None, _ptr(O) if kind & N.TOC_VECMAT else None,
                                     self.trees.data_ptr(), self.tree_off_d.data_ptr(), N.stream_handle()),
                "toc_linalg32")
        return R, O

    def build_matcache(self):
        """Per-batch node-record cache for the matmat kernels (toc_matcache_*): built once, after
        which matmat reads it instead of rebuilding each batch's tree per call -- the path for
        batches whose trees exceed shared memory (config 5)."""
        torch = self.torch
        self.raise_corrupt()
        L = N.lib()
        off = np.zeros(self.n_blocks + 1, np.int64)
        N.check(L.toc_matcache_offsets(self.meta.ctypes.data_as(ctypes.c_void_p), self.n_blocks,
                                       off.ctypes.data_as(ctypes.c_void_p)), "toc_matcache_offsets")
        plan = self.plan(N.TOC_MATVEC)
        scratch = self._scratch_for(plan)
        cache = torch.empty(int(off[-1]) + 16, dtype=torch.uint8, device=self.data.device)
        off_d = torch.from_numpy(off[:-1].copy()).to(self.data.device)
        N.check(L.toc_matcache_build(self.data.data_ptr(), self.block_off_d.data_ptr(), self.meta_d.data_ptr(),
                                     self.n_blocks, ctypes.byref(plan), off_d.data_ptr(), cache.data_ptr(),
                                     scratch.data_ptr() if scratch is not None else None, N.stream_handle()),
                "toc_matcache_build")
        self.matcache, self.matcache_off, self.matcache_off_d = cache, off, off_d
        return self

    def build_mlpcache(self) -> bool:
        """The MLP step cache (toc_mlpcache_build): per batch the decode tree in 4 bytes per node,
        pair records and the value index; each step decodes its batch from it and the TOC1 block's
        own code stream.  Returns False (no cache) when some batch's ids do not fit its fields."""
        torch = self.torch
        self.raise_corrupt()
        L = N.lib()
        off = np.zeros(self.n_blocks + 1, np.int64)
        rc = L.toc_mlpcache_offsets(self.meta.ctypes.data_as(ctypes.c_void_p), self.n_blocks,
                                    off.ctypes.data_as(ctypes.c_void_p))
        if rc == N.TOC_E_ARG:
            self.mlpcache = None
            return False
        N.check(rc, "toc_mlpcache_offsets")
        plan = self.plan(N.TOC_MATVEC)
        scratch = self._scratch_for(plan)
        cache = torch.empty(int(off[-1]) + 16, dtype=torch.uint8, device=self.data.device)
        off_d = torch.from_numpy(off[:-1].copy()).to(self.data.device)
        N.check(L.toc_mlpcache_build(self.data.data_ptr(), self.block_off_d.data_ptr(), self.meta_d.data_ptr(),
                                     self.n_blocks, ctypes.byref(plan), off_d.data_ptr(), cache.data_ptr(),
                                     scratch.data_ptr() if scratch is not None else None, N.stream_handle()),
                "toc_mlpcache_build")
        self.mlpcache, self.mlpcache_off = cache, off
        return True

    def _matmat_cached(self, side: int, M, p: int, batch, out):
        torch = self.torch
        L = N.lib()
        dev = self.data.device
        b0, nb = (0, self.n_blocks) if batch is None else (int(batch), 1)
        rows = self.n_rows_total if batch is None else int(self.meta["n_rows"][batch])
        if side == 0:
            if out is None:
                out = torch.empty((max(rows, 1), p), dtype=torch.float64, device=dev)[:rows]
            if batch is None:
                rb = self.row_base_d.data_ptr()
            else:
                if getattr(self, "_zero_rb", None) is None:
                    self._zero_rb = torch.zeros(1, dtype=torch.int64, device=dev)
                rb = self._zero_rb.data_ptr()
            N.check(L.toc_matcache_right(self.matcache.data_ptr(), self.matcache_off_d.data_ptr() + 8 * b0, rb, nb,
                                         rows, self.n_cols, p, _ptr(M), _ptr(out), N.stream_handle()),
                    "toc_matcache_right")
            return out
        if out is None:
            out = torch.empty((max(nb, 1), p, max(self.n_cols, 1)), dtype=torch.float64, device=dev)[:nb, :, : self.n_cols]
        key = ("mcl", p)
        need = self._mm_scratch.get(key) if hasattr(self, "_mm_scratch") else None
        if need is None:
            c = ctypes.c_int64()
            need = 0
            for b in range(self.n_blocks):
                N.check(L.toc_matcache_left_scratch(self.meta[b : b + 1].ctypes.data_as(ctypes.c_void_p), p,
                                                    self.n_cols, ctypes.byref(c)), "toc_matcache_left_scratch")
                need = max(need, c.value)
            if not hasattr(self, "_mm_scratch"):
                self._mm_scratch = {}
            self._mm_scratch[key] = need
        if self._scratch is None or self._scratch.numel() < need:
            self._scratch = torch.empty(need, dtype=torch.uint8, device=dev)
        for k in range(nb):
            b = b0 + k
            r0 = 0 if batch is not None else int(self.row_base[b])
            n = int(self.meta["n_rows"][b])
            hm = np.ascontiguousarray(self.meta[b : b + 1])
            N.check(L.toc_matcache_left(self.matcache.data_ptr() + int(self.matcache_off[b]),
                                        hm.ctypes.data_as(ctypes.c_void_p), p, self.n_cols,
                                        _ptr(M) + 8 * r0 * p, _ptr(out[k]), self._scratch.data_ptr(),
                                        self._scratch.numel(), N.stream_handle()), "toc_matcache_left")
            del n
        return out

    def matmat(self, side: int, M, p: int, batch: int | None = None, out=None):
        """side 0: A.M (M: device [n_cols x p]) -> [rows x p];  side 1: M_b.A_b (M: device M^T
        [rows x p]) -> [blocks, p, n_cols].  batch=None: every batch of the arena; batch=b: only
        batch b (rows indexed from 0).  Uses the node-record cache when build_matcache() ran."""
        torch = self.torch
        self.raise_corrupt()
        if getattr(self, "matcache", None) is not None and 268 * self.n_cols <= 227 * 1024:
            return self._matmat_cached(side, M, p, batch, out)
        L = N.lib()
        if batch is None:
            b0, nb, rows = 0, self.n_blocks, self.n_rows_total
            row_base = self.row_base_d.data_ptr()
        else:
            b0, nb, rows = int(batch), 1, int(self.meta["n_rows"][batch])
            if getattr(self, "_zero_rb", None) is None:
                self._zero_rb = torch.zeros(1, dtype=torch.int64, device=self.data.device)
            row_base = self._zero_rb.data_ptr()
        hmeta = self.meta[b0 : b0 + nb]
        key = (side, p, batch is None)
        nbytes = self._mm_scratch.get(key) if hasattr(self, "_mm_scratch") else None
        if nbytes is None:
            c = ctypes.c_int64()
            meta_all = np.ascontiguousarray(self.meta)
            if batch is None:
                N.check(L.toc_matmat_scratch(meta_all.ctypes.data_as(ctypes.c_void_p), self.n_blocks, self.n_cols, side,
                                             p, ctypes.byref(c)), "toc_matmat_scratch")
                nbytes = c.value
            else:  # one batch per call: the worst case over the batches
                nbytes = 0
                for b in range(self.n_blocks):
                    N.check(L.toc_matmat_scratch(meta_all[b : b + 1].ctypes.data_as(ctypes.c_void_p), 1, self.n_cols,
                                                 side, p, ctypes.byref(c)), "toc_matmat_scratch")
                    nbytes = max(nbytes, c.value)
            if not hasattr(self, "_mm_scratch"):
                self._mm_scratch = {}
            self._mm_scratch[key] = nbytes
        dev = self.data.device
        if out is None:
            if side == 0:
                out = torch.empty((max(rows, 1), p), dtype=torch.float64, device=dev)[:rows]
            else:
                out = torch.empty((max(nb, 1), p, max(self.n_cols, 1)), dtype=torch.float64,
                                  device=dev)[:nb, :, : self.n_cols]
        if nbytes > 0 and (self._scratch is None or self._scratch.numel() < nbytes):
            self._scratch = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        scratch = self._scratch
        hm = np.ascontiguousarray(hmeta)
        N.check(L.toc_matmat(self.data.data_ptr(), self.block_off_d.data_ptr() + 8 * b0,
                             self.meta_d.data_ptr() + N.META_DTYPE.itemsize * b0, hm.ctypes.data_as(ctypes.c_void_p),
                             row_base, nb, self.n_cols, side, p, _ptr(M), _ptr(out),
                             scratch.data_ptr() if scratch is not None else None,
                             scratch.numel() if scratch is not None else 0, N.stream_handle()), "toc_matmat")
        return out

    def matvec(self, v):
        return self.linalg(N.TOC_MATVEC, v=v)[0]

    def vecmat(self, u):
        return self.linalg(N.TOC_VECMAT, u=u)[1]
