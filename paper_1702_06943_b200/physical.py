"""TOC1 block serialization (reference physical.py:1-186), executed on the device.

``serialize_block`` uploads a LogicalEncoding, builds the value index and packs the bytes with
the same kernels the batch compressor uses (toc_serialize_sizes + toc_pack_blocks);
``deserialize_block`` uploads the bytes, validates them with toc_index_blocks (raising the
reference's exception for the first failing check) and unpacks them with toc_unpack_blocks.
``pack_ints`` / ``unpack_ints`` are the format's host-side helpers (physical.py:54-85).
"""

from __future__ import annotations

import ctypes
import struct

import numpy as np

from . import _native as N
from .codec import INFO_DTYPE, LogicalEncoding, TocEncodeSizes, _bind
from .errors import (BadMagicError, BlockFormatError, TruncatedBlockError,  # noqa: F401
                     UnsupportedVersionError)

MAGIC = b"TOC1"
VERSION = 1


def _int_width(largest: int) -> int:
    return max(1, -(-largest.bit_length() // 8))


def pack_ints(values) -> bytes:
    """Pack non-negative ints at the smallest fixed byte width (physical.py:54-68)."""
    vals = [int(v) for v in values]
    largest = 0
    for v in vals:
        if v < 0:
            raise ValueError(f"cannot pack negative value {v}")
        largest = max(largest, v)
    if largest >= 1 << 32:
        raise ValueError(f"value {largest} does not fit in four bytes")
    w = _int_width(largest)
    arr = np.asarray(vals, dtype=np.uint64)
    payload = np.zeros((len(vals), 8), np.uint8)
    if len(vals):
        payload = arr.astype("<u8").view(np.uint8).reshape(len(vals), 8)
    return struct.pack("<IB", len(vals), w) + payload[:, :w].tobytes()


def unpack_ints(data: bytes, offset: int = 0):
    """Inverse of pack_ints; returns (values, offset past the array) (physical.py:71-85)."""
    if offset + 5 > len(data):
        raise TruncatedBlockError(f"packed array header truncated at offset {offset}")
    count, width = struct.unpack_from("<IB", data, offset)
    offset += 5
    if width not in (1, 2, 3, 4):
        raise BlockFormatError(f"bytes_per_int must be 1..4, got {width} at offset {offset - 1}")
    end = offset + count * width
    if end > len(data):
        raise TruncatedBlockError(f"packed array payload truncated: need {end - len(data)} more bytes at offset {offset}")
    raw = np.frombuffer(data, np.uint8, count * width, offset).reshape(count, width).astype(np.uint64)
    vals = np.zeros(count, np.uint64)
    for k in range(width):
        vals |= raw[:, k] << np.uint64(8 * k)
    return [int(v) for v in vals], end


def build_value_index(values) -> tuple:
    """(uniques, refs): the distinct values by bit pattern in first-occurrence order and each
    value's index into them (reference physical.py:88-101; the device serializer,
    toc_serialize_sizes, builds the same index for every block)."""
    bits = np.asarray(values, dtype=np.float64).view(np.uint64)
    if bits.size == 0:
        return [], []
    _, first, inverse = np.unique(bits, return_index=True, return_inverse=True)
    rank = np.empty(len(first), np.int64)  # unique slot -> position in first-occurrence order
    rank[np.argsort(first, kind="stable")] = np.arange(len(first))
    order = np.sort(first)
    return bits[order].view(np.float64).tolist(), rank[inverse.reshape(-1)].tolist()


def value_index_lookup(uniques, ref: int) -> float:
    """uniques[ref] with the format's range check (reference physical.py:104-107)."""
    if not 0 <= ref < len(uniques):
        raise BlockFormatError(f"value ref {ref} out of range for {len(uniques)} unique values")
    return uniques[ref]


def serialize_block(enc: LogicalEncoding) -> bytes:
    """TOC1 bytes of one logical encoding, produced on the device (physical.py:110-130)."""
    torch = N.require_cuda()
    L = _bind()
    dev = torch.device("cuda")
    nI, C, n = len(enc.pairs), enc.total_codes, enc.n_rows
    cap = max(nI, C, 1)
    eb = np.array([0, cap], np.int64)
    sizes = TocEncodeSizes()
    N.check(L.toc_encode_sizes(1, eb.ctypes.data_as(ctypes.c_void_p), ctypes.byref(sizes)), "toc_encode_sizes")
    I_cols = np.zeros(cap, np.int32)
    I_vals = np.zeros(cap, np.float64)
    codes = np.zeros(cap, np.int32)
    if nI:
        I_cols[:nI] = [c for c, _ in enc.pairs]
        I_vals[:nI] = [v for _, v in enc.pairs]
    flat = [c for r in enc.rows for c in r]
    if any(c >= 1 << 32 for c in flat):
        raise ValueError("code does not fit in four bytes")
    if C:
        codes[:C] = np.asarray(flat, np.uint32).view(np.int32)
    offsets = np.zeros(n + 1, np.int64)
    np.cumsum([len(r) for r in enc.rows], out=offsets[1:])
    info = np.zeros(1, INFO_DTYPE)
    info["n_rows"], info["n_cols"], info["n_pairs"], info["n_codes"] = n, enc.n_cols, nI, C
    t = {k: torch.from_numpy(v).to(dev) for k, v in dict(
        I_cols=I_cols, I_vals=I_vals, codes=codes, offsets=offsets.astype(np.uint32).view(np.int32),
        eb=eb, br=np.array([0, n], np.int64), info=info.view(np.uint8)).items()}
    work = torch.empty(sizes.work_bytes, dtype=torch.uint8, device=dev)
    refs = torch.empty(cap, dtype=torch.int32, device=dev)
    uniques = torch.empty(cap, dtype=torch.float64, device=dev)
    s = N.stream_handle()
    N.check(L.toc_serialize_sizes(1, t["br"].data_ptr(), t["eb"].data_ptr(), t["I_cols"].data_ptr(),
                                  t["I_vals"].data_ptr(), t["codes"].data_ptr(), t["offsets"].data_ptr(),
                                  ctypes.byref(sizes), work.data_ptr(), refs.data_ptr(), uniques.data_ptr(),
                                  t["info"].data_ptr(), s), "toc_serialize_sizes")
    info_h = np.frombuffer(t["info"].cpu().numpy().tobytes(), INFO_DTYPE)
    size = int(info_h["block_bytes"][0])
    arena = torch.zeros(max(size, 16), dtype=torch.uint8, device=dev)
    boff = torch.zeros(1, dtype=torch.int64, device=dev)
    N.check(L.toc_pack_blocks(1, t["br"].data_ptr(), t["eb"].data_ptr(), t["I_cols"].data_ptr(), refs.data_ptr(),
                              uniques.data_ptr(), t["codes"].data_ptr(), t["offsets"].data_ptr(),
                              t["info"].data_ptr(), boff.data_ptr(), arena.data_ptr(), s), "toc_pack_blocks")
    return bytes(arena[:size].cpu().numpy())


def unpack_arena(arena):
    """Logical arrays of every block of an indexed BlockArena (toc_unpack_blocks)."""
    torch = arena.torch
    L = _bind()
    m = arena.meta
    nI = m["n_pairs"].astype(np.int64)
    C = m["n_codes"].astype(np.int64)
    nR = m["n_rows"].astype(np.int64) + 1
    pb, cb, ob = (np.concatenate([[0], np.cumsum(x)[:-1]]).astype(np.int64) for x in (nI, C, nR))
    dev = arena.data.device
    d = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in dict(pb=pb, cb=cb, ob=ob).items()}
    I_cols = torch.empty(max(int(nI.sum()), 1), dtype=torch.int32, device=dev)
    I_vals = torch.empty(max(int(nI.sum()), 1), dtype=torch.float64, device=dev)
    codes = torch.empty(max(int(C.sum()), 1), dtype=torch.int32, device=dev)
    offsets = torch.empty(max(int(nR.sum()), 1), dtype=torch.int32, device=dev)
    N.check(L.toc_unpack_blocks(arena.data.data_ptr(), arena.block_off_d.data_ptr(), arena.meta_d.data_ptr(),
                                arena.n_blocks, d["pb"].data_ptr(), d["cb"].data_ptr(), d["ob"].data_ptr(),
                                I_cols.data_ptr(), I_vals.data_ptr(), codes.data_ptr(), offsets.data_ptr(),
                                N.stream_handle()), "toc_unpack_blocks")
    ic, iv = I_cols.cpu().numpy(), I_vals.cpu().numpy()
    cd, of = codes.cpu().numpy().view(np.uint32), offsets.cpu().numpy().view(np.uint32)
    out = []
    for b in range(arena.n_blocks):
        out.append((ic[pb[b] : pb[b] + nI[b]], iv[pb[b] : pb[b] + nI[b]], cd[cb[b] : cb[b] + C[b]],
                    of[ob[b] : ob[b] + nR[b]]))
    return out


def deserialize_block(data: bytes) -> LogicalEncoding:
    """Parse one block; the entire buffer must belong to it (physical.py:138-186)."""
    from .arena import BlockArena

    arena = BlockArena.from_bytes([bytes(data)])
    ic, iv, cd, of = unpack_arena(arena)[0]
    rec = arena.meta[0]
    pairs = [(int(c), float(v)) for c, v in zip(ic.tolist(), iv.tolist())]
    cdl = cd.tolist()
    rows = [cdl[of[i] : of[i + 1]] for i in range(int(rec["n_rows"]))]
    return LogicalEncoding(n_rows=int(rec["n_rows"]), n_cols=int(rec["n_cols"]), pairs=pairs, rows=rows)


def rewrite_arena(arena, fn=None, values=None):
    """Every block with its pair values replaced, the value index rebuilt (physical.py:88-101) and
    the blocks repacked (physical.py:110-130) -- all on the device; codes, columns and row
    offsets are carried over unchanged.  The sparse-safe rewrites (kernels.py:87-112) over a whole
    arena.  ``fn`` maps the float64 tensor of all pair values (pair order, block by block) on the
    device; or ``values`` gives them directly.  Raises ValueError like LogicalEncoding
    (codec.py:151-162) when a new value is not finite."""
    from .arena import BlockArena

    torch = arena.torch
    L = _bind()
    arena.raise_format_errors()
    m = arena.meta
    B = arena.n_blocks
    nI = m["n_pairs"].astype(np.int64)
    C = m["n_codes"].astype(np.int64)
    n = m["n_rows"].astype(np.int64)
    cap = np.maximum(np.maximum(nI, C), 1)
    eb = np.concatenate([[0], np.cumsum(cap)]).astype(np.int64)
    br = np.concatenate([[0], np.cumsum(n)]).astype(np.int64)
    ob = (br[:-1] + np.arange(B)).astype(np.int64)
    dev = arena.data.device
    d = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in dict(eb=eb, br=br, ob=ob).items()}
    E = int(eb[-1])
    I_cols = torch.zeros(E, dtype=torch.int32, device=dev)
    I_vals = torch.zeros(E, dtype=torch.float64, device=dev)
    codes = torch.zeros(E, dtype=torch.int32, device=dev)
    offsets = torch.zeros(int(br[-1]) + B, dtype=torch.int32, device=dev)
    s = N.stream_handle()
    N.check(L.toc_unpack_blocks(arena.data.data_ptr(), arena.block_off_d.data_ptr(), arena.meta_d.data_ptr(), B,
                                d["eb"].data_ptr(), d["eb"].data_ptr(), d["ob"].data_ptr(), I_cols.data_ptr(),
                                I_vals.data_ptr(), codes.data_ptr(), offsets.data_ptr(), s), "toc_unpack_blocks")
    # pair slots of every block, in pair order
    slot = (torch.arange(int(nI.sum()), device=dev, dtype=torch.int64)
            - torch.from_numpy(np.repeat(np.concatenate([[0], np.cumsum(nI)[:-1]]) - eb[:-1], nI)).to(dev))
    old = I_vals[slot]
    new = fn(old) if fn is not None else torch.as_tensor(values, dtype=torch.float64, device=dev)
    if new.shape != old.shape:
        raise ValueError(f"{new.numel()} new values for {old.numel()} pairs")
    bad = torch.nonzero(~torch.isfinite(new))
    if bad.numel():
        col = int(I_cols[slot[int(bad[0, 0])]].item())
        raise ValueError(f"pair value for column {col} is not finite")
    I_vals[slot] = new
    sizes = TocEncodeSizes()
    N.check(L.toc_encode_sizes(B, eb.ctypes.data_as(ctypes.c_void_p), ctypes.byref(sizes)), "toc_encode_sizes")
    info = np.zeros(B, INFO_DTYPE)
    info["n_rows"], info["n_cols"], info["n_pairs"], info["n_codes"] = n, m["n_cols"], nI, C
    info_d = torch.from_numpy(info.view(np.uint8)).to(dev)
    work = torch.empty(max(sizes.work_bytes, 16), dtype=torch.uint8, device=dev)
    refs = torch.empty(E, dtype=torch.int32, device=dev)
    uniques = torch.empty(E, dtype=torch.float64, device=dev)
    N.check(L.toc_serialize_sizes(B, d["br"].data_ptr(), d["eb"].data_ptr(), I_cols.data_ptr(), I_vals.data_ptr(),
                                  codes.data_ptr(), offsets.data_ptr(), ctypes.byref(sizes), work.data_ptr(),
                                  refs.data_ptr(), uniques.data_ptr(), info_d.data_ptr(), s), "toc_serialize_sizes")
    info_h = np.frombuffer(info_d.cpu().numpy().tobytes(), INFO_DTYPE)
    blen = info_h["block_bytes"].astype(np.int64)
    padded = (blen + 15) & ~15
    boff = np.concatenate([[0], np.cumsum(padded)[:-1]]).astype(np.int64)
    total = int(padded.sum())
    data = torch.zeros(total + 16, dtype=torch.uint8, device=dev)  # +16: tail padding (arena.py)
    boff_d = torch.from_numpy(boff).to(dev)
    N.check(L.toc_pack_blocks(B, d["br"].data_ptr(), d["eb"].data_ptr(), I_cols.data_ptr(), refs.data_ptr(),
                              uniques.data_ptr(), codes.data_ptr(), offsets.data_ptr(), info_d.data_ptr(),
                              boff_d.data_ptr(), data.data_ptr(), s), "toc_pack_blocks")
    return BlockArena(data, boff, blen)
