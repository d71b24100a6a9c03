"""CPU checks of the slot-cache builder (toc_levels_build, csrc/toc_levels.cu; host code, no GPU).

The entries the library builds are decoded here and evaluated with a numpy restatement of the
slot kernel's arithmetic (P1 for the pair slots, inner-node H by chain, per-thread code ranges
with head / tail partials; T scatter, push along inner chains, column sums), then compared with
the oracle's matvec / vecmat (kernels.py:115-174) at the 1e-9 bar.  The structural invariants the
kernel relies on are asserted too: column-sorted pair slots, inner nodes after their parents,
keys are pairs, every stream reference a valid slot, column starts monotone.  This pins the
builder before any GPU run; tests/test_gpu_linalg.py runs the kernel itself ("levels" mode).
"""

from __future__ import annotations

import ctypes
import struct

import numpy as np
import pytest

from conftest import max_rel_err, within_rel
from helpers import TOY_ROWS, TREE_ROWS, random_alphabet_rows

REL = 1e-9
HDR = ["nP", "nQ", "S", "C", "K", "T", "n_rows", "n_cols", "nU", "off_uniq", "off_rowoff", "off_prs", "off_inner",
       "off_colst", "off_stream", "off_trow"]


def host_meta(block: bytes, N):
    """TocBlockMeta of a well-formed TOC1 block, parsed on the host (physical.py:1-21 layout)."""
    m = np.zeros(1, N.META_DTYPE)[0]
    n_rows, n_cols = struct.unpack_from("<II", block, 5)
    nU = struct.unpack_from("<I", block, 13)[0]
    m["n_rows"], m["n_cols"], m["n_uniques"], m["off_uniques"] = n_rows, n_cols, nU, 17
    o = 17 + 8 * nU
    nI = struct.unpack_from("<I", block, o)[0]
    o += 4

    def packed(o):
        cnt, w = struct.unpack_from("<IB", block, o)
        return cnt, w, o + 5, o + 5 + cnt * w

    _, m["w_cols"], m["off_cols"], o = packed(o)
    _, m["w_refs"], m["off_refs"], o = packed(o)
    C = struct.unpack_from("<I", block, o)[0]
    _, m["w_codes"], m["off_codes"], o = packed(o + 4)
    _, m["w_offsets"], m["off_offsets"], o = packed(o)
    w = int(m["w_offsets"])
    offs = [int.from_bytes(block[m["off_offsets"] + i * w: m["off_offsets"] + (i + 1) * w], "little")
            for i in range(n_rows + 1)]
    m["n_pairs"], m["n_codes"] = nI, C
    m["n_derived"] = sum(max(offs[i + 1] - offs[i] - 1, 0) for i in range(n_rows))
    return m


def build(blocks):
    from paper_1702_06943_b200 import _native as N

    offs, pos, parts = [], 0, []
    for b in blocks:
        offs.append(pos)
        pad = (-len(b)) % 16
        parts.append(b + b"\0" * pad)
        pos += len(b) + pad
    arena = np.frombuffer(b"".join(parts) + b"\0" * 16, np.uint8).copy()
    off = np.asarray(offs, np.int64)
    meta = np.array([host_meta(b, N) for b in blocks], N.META_DTYPE)
    L = N.lib()
    h = L.toc_levels_build(arena.ctypes.data_as(ctypes.c_void_p), off.ctypes.data_as(ctypes.c_void_p),
                           meta.ctypes.data_as(ctypes.c_void_p), len(blocks), 2)
    assert h
    try:
        total, slots, stage, rows = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        rc = L.toc_levels_info(h, ctypes.byref(total), ctypes.byref(slots), ctypes.byref(stage), ctypes.byref(rows))
        if rc:
            return rc, None, None
        buf = np.zeros(total.value + 16, np.uint8)
        eo = np.zeros(len(blocks) + 1, np.int64)
        assert L.toc_levels_copy(h, buf.ctypes.data_as(ctypes.c_void_p), eo.ctypes.data_as(ctypes.c_void_p)) == 0
    finally:
        L.toc_levels_free(h)
    return 0, buf, eo


def entry(buf, o):
    h = dict(zip(HDR, struct.unpack_from("<16I", buf, o)))
    h["vmax"] = struct.unpack_from("<d", buf, o + 64)[0]
    u32 = lambda off, n: np.frombuffer(buf, np.uint32, n, o + off).astype(np.int64)  # noqa: E731
    h["prs"] = u32(h["off_prs"], h["nP"])
    inner = u32(h["off_inner"], h["nQ"])  # references -> slot numbers: par | key << 16
    h["inner"] = slot_of(inner & 0xFFFF) | (slot_of(inner >> 16) << 16)
    T, K = h["T"], h["K"]
    st = np.frombuffer(buf, np.uint16, T * K, o + h["off_stream"]).astype(np.int64)
    # record k of thread t is the u16 at (k // 8) * 8T + 8t + k % 8  ->  row order j = t*K + k
    k = np.arange(K)
    pos = (k[None, :] // 8) * 8 * T + 8 * np.arange(T)[:, None] + (k[None, :] % 8)
    st = st[pos.reshape(-1)][: h["C"]]
    h["stream"] = slot_of(st & 0x7FFF) | (st & 0x8000)  # one slot per record | row-end flag
    h["colst"] = np.frombuffer(buf, np.uint16, h["n_cols"] + 1, o + h["off_colst"]).astype(np.int64)
    h["uniq"] = np.frombuffer(buf, np.float64, h["nU"], o + h["off_uniq"]).copy()
    h["rowoff"] = u32(h["off_rowoff"], h["n_rows"] + 1)
    h["trow"] = np.frombuffer(buf, np.uint16, T, o + h["off_trow"]).astype(np.int64)
    return h


def slot_of(ref):
    """Slot number of a reference (toc_levels.cu slot_ref: 2p + bit 4 of p)."""
    ref = np.asarray(ref, np.int64)
    p = ref >> 1
    assert np.all((ref & 1) == ((p >> 4) & 1)), "reference parity"
    return p


def value_index(block):
    """The block's own value index: uniques in first-occurrence order and each pair's ref."""
    nU = struct.unpack_from("<I", block, 13)[0]
    uniq = np.frombuffer(block, np.float64, nU, 17).copy()
    o = 17 + 8 * nU + 4
    cnt, w = struct.unpack_from("<IB", block, o)
    o += 5 + cnt * w
    cnt, w = struct.unpack_from("<IB", block, o)
    refs = np.array([int.from_bytes(block[o + 5 + i * w: o + 5 + (i + 1) * w], "little") for i in range(cnt)],
                    np.int64)
    return uniq, refs


def emulate(h, enc, uniq, refs, v, u):
    """The slot kernel's arithmetic in numpy, in the kernel's operation order (per-thread ranges,
    head / tail partials combined in thread order)."""
    nP, nQ, S, C, K, T = h["nP"], h["nQ"], h["S"], h["C"], h["K"], h["T"]
    prs, inner, st = h["prs"], h["inner"], h["stream"]
    # pairs numbered by column (any order within a column: the builder picks it for the value
    # gather's banks): the same (column, ref) records as the block
    cols_b, refs_b = np.asarray(enc.I_cols, np.int64), np.asarray(refs, np.int64)
    assert np.all(np.diff(prs & 0xFFFF) >= 0)
    assert np.array_equal(np.sort((prs & 0xFFFF) << 16 | ((prs >> 16) & 0x7FFF)), np.sort(cols_b << 16 | refs_b))
    last = np.r_[(prs[1:] & 0xFFFF) != (prs[:-1] & 0xFFFF), True] if nP else np.zeros(0, bool)
    assert np.array_equal((prs >> 31) == 1, last), "column-end flags"
    prs = prs & 0x7FFFFFFF
    H = np.zeros(S)
    H[1:nP + 1] = uniq[prs >> 16] * v[prs & 0xFFFF]

    def chain(y):  # slots visited from inner slot y: keys, then the root pair
        rec = inner[y - nP - 1]
        out, p = [rec >> 16], rec & 0xFFFF
        while p > nP:
            rec = inner[p - nP - 1]
            out.append(rec >> 16)
            p = rec & 0xFFFF
        return out + [p]

    for y in range(nP + 1, S):
        hv = 0.0
        for i, x in enumerate(chain(y)):
            hv = H[x] if i == 0 else hv + H[x]
        H[y] = hv
    off = h["rowoff"]  # row offsets into the record stream
    n = h["n_rows"]
    row_of = np.repeat(np.arange(n), np.diff(off))
    R = np.zeros(n)
    head, tail = np.zeros(T), np.zeros(T)
    for t in range(T):
        s0, e0 = t * K, min(t * K + K, C)
        if s0 >= e0:
            continue
        acc = 0.0
        for j in range(s0, e0):
            acc += H[st[j] & 0x7FFF]
            r = row_of[j]
            if j + 1 == off[r + 1]:
                if off[r] >= s0:
                    R[r] = acc
                else:
                    head[t] = acc
                acc = 0.0
        tail[t] = acc
    for r in range(n):
        lo, hi = off[r], off[r + 1]
        if lo < hi and lo // K != (hi - 1) // K:
            t0, t1 = lo // K, (hi - 1) // K
            x = tail[t0]
            for t in range(t0 + 1, t1):
                x += tail[t]
            R[r] = x + head[t1]
    # v^T.A: T[slot] += u[r] (the kernel's fixed point is exact; fp64 here), push, columns
    Tv = np.zeros(S)
    for j in range(C):
        Tv[st[j] & 0x7FFF] += u[row_of[j]]
    Tv[0] = 0.0  # slot 0 collects the empty rows' records; nothing reads it
    own = Tv.copy()
    for y in range(nP + 1, S):
        for x in chain(y):
            Tv[x] += own[y]
    O = np.zeros(enc.n_cols)
    cs = h["colst"]
    for c in range(enc.n_cols):
        p = np.arange(cs[c], cs[c + 1])
        O[c] = np.sum(uniq[prs[p - 1] >> 16] * Tv[p]) if len(p) else 0.0
    return R, O


def structure(h, enc):
    nP, nQ, S = h["nP"], h["nQ"], h["S"]
    assert nP == len(enc.I_cols) and S == 1 + nP + nQ
    assert h["K"] % 8 == 0 and h["K"] * h["T"] >= h["C"]
    # records: one per code with a slot, two per leaf, one (slot 0) per empty row
    codes_per_row = np.diff(np.asarray(enc.offsets, np.int64))
    recs_per_row = np.diff(h["rowoff"])
    assert h["rowoff"][0] == 0 and h["rowoff"][-1] == h["C"]
    assert np.all(recs_per_row >= np.maximum(codes_per_row, 1)) and np.all(recs_per_row <= np.maximum(2 * codes_per_row, 1))
    assert np.all(np.diff(h["prs"] & 0xFFFF) >= 0), "pairs not column-sorted"
    par, key = h["inner"] & 0xFFFF, h["inner"] >> 16
    assert np.all((key >= 1) & (key <= nP)), "inner keys must be pairs"
    assert np.all((par >= 1) & (par < S) & (par != nP + 1 + np.arange(nQ))), "inner parents"
    for y in range(nQ):  # parent chains end at a pair (inner slots are numbered for banks, not by depth)
        p, steps = par[y], 0
        while p > nP:
            p, steps = par[p - nP - 1], steps + 1
            assert steps <= nQ, "inner parent cycle"
    a_ = h["stream"] & 0x7FFF
    assert np.all(a_ < S), "stream references"
    off = h["rowoff"]
    empty = np.repeat(codes_per_row == 0, recs_per_row)
    assert np.array_equal(a_ == 0, empty), "slot 0 marks exactly the empty rows"
    ends = np.zeros(h["C"], bool)
    ends[off[1:] - 1] = True
    assert np.array_equal((h["stream"] & 0x8000) != 0, ends), "row-end flags"
    cs = h["colst"]
    assert cs[0] == 1 and cs[-1] == nP + 1 and np.all(np.diff(cs) >= 0)
    starts = np.arange(0, h["C"], h["K"])  # each thread's first code: its row, and whether it starts it
    rows = np.searchsorted(off, starts, side="right") - 1
    assert np.array_equal(h["trow"][: len(starts)] & 0x7FFF, rows)
    assert np.array_equal(h["trow"][: len(starts)] >> 15, (off[rows] == starts).astype(np.int64))
    cols = h["prs"] & 0xFFFF
    for c in np.unique(cols):
        assert np.all(cols[cs[c] - 1:cs[c + 1] - 1] == c)


def cases():
    rng = np.random.default_rng(11)
    out = [("toy", TOY_ROWS, 5), ("tree", TREE_ROWS, 5)]
    for k, (n, m, dens) in enumerate([(40, 30, 0.3), (300, 20, 0.9), (64, 200, 0.05), (5, 8, 1.0)]):
        out.append((f"rand{k}", random_alphabet_rows(rng, n, m, dens, alphabet_size=4 + k), m))
    out.append(("empty_rows", [[], [(1, 2.0)], [], [(0, 1.0), (1, 2.0)], []], 3))
    out.append(("long_rows", [[(c, 1.0) for c in range(400)]] * 6, 400))
    return out


@pytest.mark.parametrize("name,rows,m", cases(), ids=[c[0] for c in cases()])
def test_level_cache_matches_oracle(oracle, name, rows, m):
    encs = [oracle.encode_rows(m, rows)]
    blocks = [oracle.serialize(e) for e in encs]
    rc, buf, eo = build(blocks)
    assert rc == 0
    rng = np.random.default_rng(3)
    for b, e in enumerate(encs):
        h = entry(buf, int(eo[b]))
        structure(h, e)
        uniq, refs = value_index(blocks[b])
        assert np.array_equal(h["uniq"], uniq) and h["vmax"] == (np.abs(uniq).max() if len(uniq) else 0.0)
        v = rng.standard_normal(m)
        u = rng.standard_normal(e.n_rows)
        R, O = emulate(h, e, uniq, refs, v, u)
        t = oracle.Tree.from_encoding(e)
        assert within_rel(R, t.matvec(v), REL), max_rel_err(R, t.matvec(v))
        assert within_rel(O, t.vecmat(u), REL), max_rel_err(O, t.vecmat(u))


def test_level_cache_config2_batches(oracle):
    from paper_1702_06943_b200 import synth

    encs, blocks = [], []
    for b in range(3):
        rp, c, v = synth.dense_to_csr(synth.cfg2_batch_dense(0, b))
        e = oracle.encode_csr(784, rp, c, v)
        encs.append(e)
        blocks.append(oracle.serialize(e))
    rc, buf, eo = build(blocks)
    assert rc == 0
    rng = np.random.default_rng(5)
    for b, e in enumerate(encs):
        h = entry(buf, int(eo[b]))
        structure(h, e)
        assert h["S"] <= 16384 and h["nQ"] < h["C"] // 4
        uniq, refs = value_index(blocks[b])
        assert np.array_equal(h["uniq"], uniq) and h["vmax"] == (np.abs(uniq).max() if len(uniq) else 0.0)
        v, u = rng.standard_normal(784), rng.standard_normal(e.n_rows)
        R, O = emulate(h, e, uniq, refs, v, u)
        t = oracle.Tree.from_encoding(e)
        assert within_rel(R, t.matvec(v), REL)
        assert within_rel(O, t.vecmat(u), REL)


def test_level_cache_rejects_corrupt_codes(oracle):
    e = oracle.encode_rows(5, TOY_ROWS)
    blk = bytearray(oracle.serialize(e))
    from paper_1702_06943_b200 import _native as N

    m = host_meta(bytes(blk), N)
    # first code of row 0 -> a node id that does not exist yet (codec.py:235-244)
    w = int(m["w_codes"])
    blk[m["off_codes"]: m["off_codes"] + w] = (200).to_bytes(w, "little")
    rc, _, _ = build([bytes(blk)])
    assert rc == N.TOC_E_CORRUPT
