"""TOCS batch stores (reference store.py:1-129) and streaming them into device arenas.

Same on-disk layout as the reference, byte for byte:

    magic "TOCS" | version u8 (= 1) | batch_count u32 | batch_size u32 | total_rows u32 |
    n_cols u32 | seed i64 | per batch: block_len u32 | TOC1 block | label_count u32 | f64 labels

``load_batch_store`` parses with the reference's checks, in its order, and decodes every block on
the device.  ``BatchStoreStream`` is the out-of-core path: the file is
memory-mapped, batches are gathered chunk by chunk into pinned host buffers, copied to the device
on a side stream while the previous chunk is being used, and indexed / validated on the device.
``verify_store`` is the reference's `toc verify` check (cli.py:194-221) on the device: decode must
reproduce the dataset's rows and labels bit for bit and re-encoding must reproduce every block.
"""

from __future__ import annotations

import mmap
import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _native as N
from .codec import LogicalEncoding
from .errors import (BadMagicError, BlockFormatError, TruncatedBlockError, UnsupportedVersionError,
                     raise_for_meta)

STORE_MAGIC = b"TOCS"
STORE_VERSION = 1
_HEADER = struct.Struct("<BIIIIq")  # after the magic: 25 bytes


class VerificationError(Exception):
    """A store does not reproduce its dataset (reference cli.py:83)."""


@dataclass
class BatchStoreData:
    """A parsed batch store: header fields plus (encoding, labels) pairs (store.py:44-56)."""

    batch_size: int
    n_cols: int
    seed: int
    batches: list

    @property
    def total_rows(self) -> int:
        return sum(enc.n_rows for enc, _ in self.batches)


def save_batch_store(path, blocks, labels, batch_size: int, n_cols: int, seed: int) -> None:
    """store.py:59-78."""
    if len(blocks) != len(labels):
        raise ValueError(f"{len(blocks)} blocks but {len(labels)} label groups")
    total_rows = sum(len(ls) for ls in labels)
    with open(path, "wb") as fh:
        fh.write(STORE_MAGIC)
        fh.write(_HEADER.pack(STORE_VERSION, len(blocks), batch_size, total_rows, n_cols, seed))
        for block, batch_labels in zip(blocks, labels):
            fh.write(struct.pack("<I", len(block)))
            fh.write(bytes(block))
            arr = np.ascontiguousarray(batch_labels, dtype="<f8")
            fh.write(struct.pack("<I", len(arr)))
            fh.write(arr.tobytes())


def save_arena_store(path, arena, labels, batch_size: int, seed: int) -> None:
    """A device arena (e.g. from codec.compress_csr) and its per-row labels written as a store."""
    data = arena.data.cpu().numpy()
    lab = np.asarray(labels.cpu().numpy() if hasattr(labels, "cpu") else labels, np.float64)
    rb = arena.row_base
    n = arena.meta["n_rows"].astype(np.int64)
    blocks = [data[int(o) : int(o) + int(ln)] for o, ln in zip(arena.block_off, arena.block_len)]
    save_batch_store(path, blocks, [lab[int(r) : int(r) + int(k)] for r, k in zip(rb, n)], batch_size,
                     int(arena.meta["n_cols"][0]) if arena.n_blocks else 0, seed)


@dataclass
class StoreIndex:
    """Structure of a store without decoding a block: file offsets of every block and label run."""

    batch_size: int
    n_cols: int
    seed: int
    total_rows: int
    block_off: np.ndarray
    block_len: np.ndarray
    label_off: np.ndarray
    label_count: np.ndarray


def _take(size: int, offset: int, n: int, what: str) -> int:
    if offset + n > size:
        raise TruncatedBlockError(f"store {what} truncated at offset {offset}")
    return offset + n


def _index(data) -> tuple:
    """Walk the store in the reference's order (store.py:87-129).  Returns (index, pending): pending
    is (batch, exception) for the first error that the reference would raise *after* decoding that
    batch's block (label count, column count, trailing bytes, row total), or None.  Errors the
    reference raises before decoding the block are raised here."""
    size = len(data)
    _take(size, 0, 4, "magic")
    if bytes(data[:4]) != STORE_MAGIC:
        raise BadMagicError(f"bad store magic {bytes(data[:4])!r}")
    offset = _take(size, 4, 25, "header")
    version, batch_count, batch_size, total_rows, n_cols, seed = _HEADER.unpack_from(data, 4)
    if version != STORE_VERSION:
        raise UnsupportedVersionError(f"unsupported store version {version}")
    boff, blen, loff, lcnt = [], [], [], []
    rows_seen = 0
    for b in range(batch_count):
        try:  # every error here waits until the blocks before it have been decoded (and may fail)
            end = _take(size, offset, 4, f"batch {b} block length")
            (block_len,) = struct.unpack_from("<I", data, offset)
            offset = end
            end = _take(size, offset, block_len, f"batch {b} block")
            boff.append(offset)
            blen.append(block_len)
            # the reference decodes the block here; its header gives n_rows / n_cols for the checks below
            blk_rows = blk_cols = None
            if block_len >= 13 and bytes(data[offset : offset + 4]) == b"TOC1":
                _, blk_rows, blk_cols = struct.unpack_from("<BII", data, offset + 4)
            offset = end
            end = _take(size, offset, 4, f"batch {b} label count")
            (label_count,) = struct.unpack_from("<I", data, offset)
            offset = end
            if blk_rows is not None and label_count != blk_rows:
                raise BlockFormatError(f"batch {b}: {label_count} labels for {blk_rows} rows")
            end = _take(size, offset, 8 * label_count, f"batch {b} labels")
            loff.append(offset)
            lcnt.append(label_count)
            offset = end
            if blk_cols is not None and blk_cols != n_cols:
                raise BlockFormatError(f"batch {b}: block has {blk_cols} columns, store header says {n_cols}")
        except (TruncatedBlockError, BlockFormatError) as e:
            return _mk(batch_size, n_cols, seed, total_rows, boff, blen, loff, lcnt), (b, e)
        rows_seen += label_count
    pending = None
    if offset != size:
        pending = (batch_count, BlockFormatError(f"{size - offset} trailing bytes after store"))
    elif rows_seen != total_rows:
        pending = (batch_count, BlockFormatError(f"store header says {total_rows} rows, batches hold {rows_seen}"))
    return _mk(batch_size, n_cols, seed, total_rows, boff, blen, loff, lcnt), pending


def _mk(batch_size, n_cols, seed, total_rows, boff, blen, loff, lcnt) -> StoreIndex:
    pad = len(blen) - len(lcnt)  # a batch whose block was read but whose labels were not
    a = lambda x: np.asarray(x, np.int64)  # noqa: E731
    return StoreIndex(batch_size, n_cols, seed, total_rows, a(boff), a(blen), a(list(loff) + [0] * pad),
                      a(list(lcnt) + [0] * pad))


def _raise_block(arena, b: int) -> None:
    o = int(arena.block_off[b])
    raise_for_meta(arena.meta[b], bytes(arena.data[o : o + 4].cpu().numpy()))


def _device_arena(data, idx: StoreIndex, lo: int, hi: int, pinned=None, stream=None):
    """Blocks [lo, hi) gathered 16-byte aligned (host, optionally into a pinned buffer) and copied to
    the device (on `stream` if given).  Returns (device bytes, block offsets, block lengths, labels)."""
    import torch

    blen = idx.block_len[lo:hi]
    padded = (blen + 15) & ~15
    boff = np.concatenate([[0], np.cumsum(padded)[:-1]]).astype(np.int64)
    total = int(padded.sum()) + 16
    nlab = int(idx.label_count[lo:hi].sum())
    host = pinned if pinned is not None and pinned.numel() >= total + 8 * nlab else \
        torch.empty(total + 8 * nlab, dtype=torch.uint8, pin_memory=True)
    h = host.numpy()
    h[:total] = 0
    src = np.frombuffer(data, np.uint8)
    for k, b in enumerate(range(lo, hi)):
        h[boff[k] : boff[k] + blen[k]] = src[idx.block_off[b] : idx.block_off[b] + blen[k]]
    pos = total
    for b in range(lo, hi):
        n8 = 8 * int(idx.label_count[b])
        h[pos : pos + n8] = src[idx.label_off[b] : idx.label_off[b] + n8]
        pos += n8
    dev = torch.empty(total + 8 * nlab, dtype=torch.uint8, device="cuda")
    if stream is not None:
        with torch.cuda.stream(stream):
            dev.copy_(host[: total + 8 * nlab], non_blocking=True)
    else:
        dev.copy_(host[: total + 8 * nlab], non_blocking=True)
    return dev, boff, blen, host


def load_batch_store(path) -> BatchStoreData:
    """store.py:87-129, with every block validated and decoded on the device."""
    from .arena import BlockArena
    from .physical import unpack_arena

    N.require_cuda()
    data = Path(path).read_bytes()
    idx, pending = _index(data)
    nb = len(idx.block_len)
    batches = []
    if nb:
        dev, boff, blen, _ = _device_arena(data, idx, 0, nb)
        total = int(((blen + 15) & ~15).sum()) + 16
        arena = BlockArena(dev[:total], boff, blen)
        bad = np.flatnonzero(arena.meta["status"] != 0)
        if len(bad) and (pending is None or int(bad[0]) <= pending[0]):
            _raise_block(arena, int(bad[0]))
        if pending is not None:
            raise pending[1]
        lab = np.frombuffer(dev[total:].cpu().numpy().tobytes(), "<f8").astype(np.float64)
        pos = 0
        for b, (ic, iv, cd, of) in enumerate(unpack_arena(arena)):
            rec = arena.meta[b]
            n = int(rec["n_rows"])
            cdl = cd.tolist()
            enc = LogicalEncoding(n_rows=n, n_cols=int(rec["n_cols"]),
                                  pairs=[(int(c), float(v)) for c, v in zip(ic.tolist(), iv.tolist())],
                                  rows=[cdl[of[i] : of[i + 1]] for i in range(n)])
            k = int(idx.label_count[b])
            batches.append((enc, lab[pos : pos + k].copy()))
            pos += k
    elif pending is not None:
        raise pending[1]
    return BatchStoreData(batch_size=idx.batch_size, n_cols=idx.n_cols, seed=idx.seed, batches=batches)


@dataclass
class StoreChunk:
    """Batches [first, first + n) of a store, resident on the device."""

    first: int
    arena: object  # BlockArena
    labels: object  # float64 device tensor, batch order


class BatchStoreStream:
    """Stream a TOCS store through the device `chunk` batches at a time (out-of-core, section
    8(f) #2): memory-mapped file -> pinned host buffer (two, alternating) -> H2D on a side stream,
    overlapped with the consumer's work on the previous chunk -> device index / validation.  The
    store's structure is checked up front (same checks and order as load_batch_store); each
    chunk's blocks raise the reference's exception classes on the device."""

    def __init__(self, path, chunk: int = 1024):
        import torch

        N.require_cuda()
        if chunk < 1:
            raise ValueError(f"chunk must be positive, got {chunk}")
        self._fh = open(path, "rb")
        size = Path(path).stat().st_size
        self._data = mmap.mmap(self._fh.fileno(), 0, access=mmap.ACCESS_READ) if size else b""
        self.index, pending = _index(self._data)
        self._pending = pending
        self.chunk = chunk
        self.n_batches = len(self.index.block_len)
        self._stream = torch.cuda.Stream()
        self._pinned = [None, None]

    @property
    def n_cols(self) -> int:
        return self.index.n_cols

    def close(self) -> None:
        if isinstance(self._data, mmap.mmap):
            self._data.close()
        self._fh.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _issue(self, k: int):
        import torch

        lo, hi = k * self.chunk, min((k + 1) * self.chunk, self.n_batches)
        slot = k & 1
        dev, boff, blen, host = _device_arena(self._data, self.index, lo, hi, self._pinned[slot], self._stream)
        self._pinned[slot] = host
        ev = torch.cuda.Event()
        ev.record(self._stream)
        return lo, hi, dev, boff, blen, ev

    def __iter__(self):
        import torch

        from .arena import BlockArena

        n_chunks = -(-self.n_batches // self.chunk)
        nxt = self._issue(0) if n_chunks else None
        for k in range(n_chunks):
            lo, hi, dev, boff, blen, ev = nxt
            if k + 1 < n_chunks:
                if k >= 1:  # the pinned buffer about to be refilled fed chunk k-1's copy
                    self._prev_ev.synchronize()
                self._prev_ev = ev
                nxt = self._issue(k + 1)
            torch.cuda.current_stream().wait_event(ev)
            total = int(((blen + 15) & ~15).sum()) + 16
            arena = BlockArena(dev[:total], boff, blen)
            bad = np.flatnonzero(arena.meta["status"] != 0)
            if len(bad) and (self._pending is None or lo + int(bad[0]) <= self._pending[0]):
                _raise_block(arena, int(bad[0]))
            if self._pending is not None and hi > self._pending[0]:
                raise self._pending[1]
            yield StoreChunk(first=lo, arena=arena, labels=dev[total:].view(torch.float64))
        if self._pending is not None and self._pending[0] >= self.n_batches:
            raise self._pending[1]


def decompress_store(path):
    """Every row and label of a store, decoded on the device (reference cli.py:177-191):
    returns (row_ptr int64, cols int32, vals float64, labels float64) as host arrays."""
    rps, cs, vs, ls = [np.zeros(1, np.int64)], [], [], []
    base = 0
    with BatchStoreStream(path) as st:
        for ch in st:
            rp, c, v = ch.arena.decode()
            rps.append(rp[1:].cpu().numpy() + base)
            base += int(rp[-1].item())
            cs.append(c.cpu().numpy())
            vs.append(v.cpu().numpy())
            ls.append(ch.labels.cpu().numpy())
    cat = lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(0, dt)  # noqa: E731
    return cat(rps, np.int64), cat(cs, np.int32), cat(vs, np.float64), cat(ls, np.float64)


def verify_store(path, dataset) -> int:
    """cli.py:194-221 on the device: the store must decode to the dataset's rows (bit for bit) and
    labels, and re-encoding the decoded rows must reproduce every stored block byte for byte.
    Returns the number of rows verified; raises VerificationError naming the first mismatch."""
    import torch

    from .codec import compress_csr

    s = dataset.features
    with BatchStoreStream(path) as st:
        if st.n_cols != s.n_cols:
            raise VerificationError(f"store has {st.n_cols} columns, dataset has {s.n_cols}")
        if st.index.total_rows != s.n_rows:
            raise VerificationError(f"store holds {st.index.total_rows} rows, dataset has {s.n_rows}")
        rp_all = torch.from_numpy(np.asarray(s.row_ptr, np.int64)).cuda()
        c_all = torch.from_numpy(np.asarray(s.cols, np.int32)).cuda()
        v_all = torch.from_numpy(np.ascontiguousarray(s.vals, np.float64)).cuda()
        y_all = torch.from_numpy(np.ascontiguousarray(dataset.labels, np.float64)).cuda()
        row = 0
        for ch in st:
            a = ch.arena
            n = a.n_rows_total
            rp, c, v = a.decode()
            want_rp = rp_all[row : row + n + 1] - rp_all[row]
            lo, hi = int(rp_all[row].item()), int(rp_all[row + n].item())
            ok_rows = torch.zeros(n, dtype=torch.bool, device=rp.device)
            if torch.equal(rp, want_rp):
                same = (c == c_all[lo:hi]) & (v.view(torch.int64) == v_all[lo:hi].view(torch.int64))
                r_of = torch.repeat_interleave(torch.arange(n, device=rp.device), rp[1:] - rp[:-1])
                bad_rows = torch.zeros(n, dtype=torch.int32, device=rp.device)
                bad_rows.index_add_(0, r_of, (~same).to(torch.int32))
                ok_rows = bad_rows == 0
            else:
                lens_ok = (rp[1:] - rp[:-1]) == (want_rp[1:] - want_rp[:-1])
                ok_rows = lens_ok  # a length mismatch is a differing row; report the first
                first_len = int(torch.nonzero(~lens_ok)[0, 0].item())
                ok_rows[first_len:] = False
            if not bool(ok_rows.all()):
                r = int(torch.nonzero(~ok_rows)[0, 0].item())
                b = int(np.searchsorted(a.row_base, r, side="right") - 1)
                raise VerificationError(f"batch {ch.first + b}, dataset row {row + r}: decoded row differs")
            lab_ok = ch.labels.view(torch.int64) == y_all[row : row + n].view(torch.int64)
            if not bool(lab_ok.all()):
                r = int(torch.nonzero(~lab_ok)[0, 0].item())
                b = int(np.searchsorted(a.row_base, r, side="right") - 1)
                raise VerificationError(f"batch {ch.first + b}, dataset row {row + r}: label differs")
            # determinism: re-encoding the decoded rows reproduces every block byte for byte
            br = np.concatenate([a.row_base, [n]]).astype(np.int64)
            re = compress_csr(s.n_cols, rp.cpu().numpy(), c.cpu().numpy(), v.cpu().numpy(), br)
            for b in range(a.n_blocks):
                if int(re.block_len[b]) != int(a.block_len[b]) or not torch.equal(
                        re.data[int(re.block_off[b]) : int(re.block_off[b]) + int(re.block_len[b])],
                        a.data[int(a.block_off[b]) : int(a.block_off[b]) + int(a.block_len[b])]):
                    raise VerificationError(f"batch {ch.first + b}: re-encoding does not reproduce the stored block")
            row += n
    return row


# ---- TOCM model container (reference store.py:131-172) ------------------------------------------
#     magic "TOCM" | version u8 (= 1) | loss code u8 | n_cols u32 | hidden u32 | f64 weights
# hidden = 0 marks a linear model; a network stores W1 row-major, then W2.  Labels for the loss
# code: the position of the loss kind in training.LOSS_KINDS.

MODEL_MAGIC = b"TOCM"
MODEL_VERSION = 1
_MODEL_HEADER = struct.Struct("<BBII")  # after the magic: 10 bytes


def save_model(path, model, loss_kind: str) -> None:
    from .training import LOSS_KINDS, GlmModel

    if loss_kind not in LOSS_KINDS:
        raise ValueError(f"loss_kind must be one of {LOSS_KINDS}, got {loss_kind!r}")
    code = LOSS_KINDS.index(loss_kind)
    if isinstance(model, GlmModel):
        head = _MODEL_HEADER.pack(MODEL_VERSION, code, len(model.weights), 0)
        body = np.ascontiguousarray(model.weights, "<f8").tobytes()
    else:
        n_cols, hidden = model.w1.shape
        head = _MODEL_HEADER.pack(MODEL_VERSION, code, n_cols, hidden)
        body = (np.ascontiguousarray(model.w1, "<f8").tobytes() + np.ascontiguousarray(model.w2, "<f8").tobytes())
    Path(path).write_bytes(MODEL_MAGIC + head + body)


def load_model(path):
    """(model, loss_kind) with the reference's checks in its order: magic, header, version, loss
    code, weight bytes, trailing bytes."""
    from .training import LOSS_KINDS, GlmModel, NnModel

    data = Path(path).read_bytes()
    if len(data) < 4:
        raise TruncatedBlockError("model magic truncated at offset 0")
    if data[:4] != MODEL_MAGIC:
        raise BadMagicError(f"bad model magic {data[:4]!r}")
    if len(data) < 4 + _MODEL_HEADER.size:
        raise TruncatedBlockError("model header truncated at offset 4")
    version, code, n_cols, hidden = _MODEL_HEADER.unpack_from(data, 4)
    if version != MODEL_VERSION:
        raise UnsupportedVersionError(f"unsupported model version {version}")
    if code >= len(LOSS_KINDS):
        raise BlockFormatError(f"unknown loss code {code}")
    count = n_cols if hidden == 0 else (n_cols + 1) * hidden
    start = 4 + _MODEL_HEADER.size
    end = start + 8 * count
    if end > len(data):
        raise TruncatedBlockError(f"model weights truncated at offset {start}")
    if end != len(data):
        raise BlockFormatError(f"{len(data) - end} trailing bytes after model")
    flat = np.frombuffer(data, "<f8", count, start).astype(np.float64)
    if hidden == 0:
        return GlmModel(weights=flat), LOSS_KINDS[code]
    return NnModel(w1=flat[: n_cols * hidden].reshape(n_cols, hidden),
                   w2=flat[n_cols * hidden :].reshape(hidden, 1)), LOSS_KINDS[code]
