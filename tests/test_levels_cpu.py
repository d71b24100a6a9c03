"""CPU checks of the level-cache builder (toc_levels_build, csrc/toc_levels.cu; host code, no GPU).

The entries the library builds are decoded here and evaluated with a numpy restatement of the
level kernel's arithmetic (P1, top-down H by depth, row sums; occurrence sums, bottom-up sibling
runs, column-sorted sums), then compared with the oracle's matvec / vecmat (kernels.py:115-174)
at the 1e-9 bar.  The structural invariants the kernel relies on are asserted too: breadth-first
ids, parents one level up, siblings contiguous, every code's id valid.  This pins the builder
before any GPU run; tests/test_gpu_linalg.py runs the kernel itself ("levels" mode).
"""

from __future__ import annotations

import ctypes
import struct

import numpy as np
import pytest

from conftest import max_rel_err, within_rel
from helpers import TOY_ROWS, TREE_ROWS, random_alphabet_rows

REL = 1e-9
HDR = ["nP", "nD", "N", "C", "n_rows", "maxd", "n_multi", "n_segs", "off_lvl", "off_prs", "off_nrec", "off_codes",
       "off_occ", "off_multi", "off_slnode", "off_kl", "off_wsplit", "off_segs"]
W = 32  # slices (one per warp)


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
        total, nodes = ctypes.c_int64(), ctypes.c_int32()
        rc = L.toc_levels_info(h, ctypes.byref(total), ctypes.byref(nodes))
        if rc:
            return rc, None, None
        buf = np.zeros(total.value + 16, np.uint8)
        eo = np.zeros(len(blocks) + 1, np.int64)
        assert L.toc_levels_copy(h, buf.ctypes.data_as(ctypes.c_void_p), eo.ctypes.data_as(ctypes.c_void_p)) == 0
    finally:
        L.toc_levels_free(h)
    return 0, buf, eo


def entry(buf, o, occ_w=1):
    h = dict(zip(HDR, struct.unpack_from("<18I", buf, o)))
    u32 = lambda off, n: np.frombuffer(buf, np.uint32, n, o + off).astype(np.int64)  # noqa: E731
    u16 = lambda off, n: np.frombuffer(buf, np.uint16, n, o + off).astype(np.int64)  # noqa: E731
    nl = h["maxd"] + 1 if h["maxd"] else 1
    h["lvl"] = u32(h["off_lvl"], nl)
    h["prs"] = u32(h["off_prs"], h["nP"])
    h["nrec"] = u32(h["off_nrec"], h["nD"])
    h["codes"] = u16(h["off_codes"], h["C"])
    h["occ"] = np.frombuffer(buf, np.uint8 if occ_w == 1 else np.uint16, h["N"], o + h["off_occ"]).astype(np.int64)
    h["occ_w"] = occ_w
    h["multi"] = u32(h["off_multi"], h["n_multi"])
    h["slnode"] = u16(h["off_slnode"], (h["maxd"] + 1) * (W + 1)).reshape(-1, W + 1)
    h["kl"] = u16(h["off_kl"], h["nD"])
    h["wsplit"] = u16(h["off_wsplit"], 2 * (W + 1)).reshape(2, W + 1)
    h["segs"] = u32(h["off_segs"], h["n_segs"] + 1)
    return h


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
    """The level kernel's arithmetic in numpy (same operation order per node), walking the
    per-warp slices the way the kernel does."""
    nP, N = h["nP"], h["N"]
    par, key = h["nrec"] & 0xFFFF, h["nrec"] >> 16
    prs = h["prs"]
    # pairs renumbered by (column, old id): the same (column, ref) records as the block
    old = sorted(range(nP), key=lambda i: (enc.I_cols[i], i))
    assert np.array_equal(prs & 0xFFFF, np.asarray(enc.I_cols, np.int64)[old])
    assert np.array_equal(prs >> 16, refs[old])
    tab = np.zeros(N)
    tab[:nP] = uniq[prs >> 16] * v[prs & 0xFFFF]
    for w in range(W):
        for d in range(1, h["maxd"]):
            for x in range(h["slnode"][d, w], h["slnode"][d, w + 1]):
                tab[x] = tab[key[x - nP]] + tab[par[x - nP]]
    off = np.asarray(enc.offsets, np.int64)
    R = np.array([tab[h["codes"][off[r]:off[r + 1]]].sum() for r in range(h["n_rows"])])
    none, multi = (0xFF, 0xFE) if h["occ_w"] == 1 else (0xFFFF, 0xFFFE)
    S = np.where(h["occ"] < multi, u[np.minimum(h["occ"], len(u) - 1)], 0.0)
    mrec = h["multi"]
    ws = h["wsplit"]
    assert ws[1][0] == 0 and ws[1][-1] == h["n_multi"] and ws[0][0] == 0 and ws[0][-1] == h["nD"]
    for w in range(W):  # multi records: a warp's range never splits a node
        a, b = ws[1][w], ws[1][w + 1]
        if 0 < a < h["n_multi"]:
            assert (mrec[a] & 0xFFFF) != (mrec[a - 1] & 0xFFFF)
    mx = mrec & 0xFFFF
    for x in np.unique(mx):
        S[x] = u[mrec[mx == x] >> 16].sum()
    for w in range(W):
        for d in range(h["maxd"] - 1, 0, -1):
            for x in range(h["slnode"][d, w], h["slnode"][d, w + 1]):
                S[par[x - nP]] += S[x]
    kl = h["kl"]
    assert np.all(np.diff(key[kl - nP]) >= 0), "kl not sorted by key"
    for x in kl:
        S[key[x - nP]] += S[x]
    O = np.zeros(enc.n_cols)
    for s in range(h["n_segs"]):
        a, b = h["segs"][s] & 0xFFFF, h["segs"][s + 1] & 0xFFFF
        assert np.all((prs[a:b] & 0xFFFF) == h["segs"][s] >> 16)
        O[h["segs"][s] >> 16] = np.sum(uniq[prs[a:b] >> 16] * S[a:b])
    return R, O


def structure(h, enc):
    nP, N, lvl = h["nP"], h["N"], h["lvl"]
    par = h["nrec"] & 0xFFFF
    assert nP == len(enc.I_cols) and lvl[0] == 0 and lvl[-1] == N
    if h["maxd"] >= 1:
        assert lvl[1] == nP
    assert np.all(np.diff(lvl) >= 0) and np.all(np.diff(h["prs"] & 0xFFFF) >= 0), "pairs not column-sorted"
    for d in range(1, h["maxd"]):
        p = par[lvl[d] - nP:lvl[d + 1] - nP]
        assert np.all((p >= lvl[d - 1]) & (p < lvl[d])), "parent not one level up"
        assert np.all(np.diff(p) >= 0), "siblings not contiguous"
    assert np.all(h["codes"] < N) and np.all((h["nrec"] >> 16) < nP)
    used = np.zeros(N, bool)
    used[h["codes"]] = True
    assert used[nP:].all(), "every derived node in the cache is a code"
    for d in range(1, h["maxd"]):  # the slices tile each level; a slice's parents are in the slice
        sl = h["slnode"][d]
        assert sl[0] == lvl[d] and sl[-1] == lvl[d + 1] and np.all(np.diff(sl) >= 0)
        if d >= 2:
            for w in range(W):
                p = par[sl[w] - nP:sl[w + 1] - nP]
                assert np.all((p >= h["slnode"][d - 1][w]) & (p < h["slnode"][d - 1][w + 1]))


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
        h = entry(buf, int(eo[b]), 1 if e.n_rows <= 253 else 2)
        structure(h, e)
        uniq, refs = value_index(blocks[b])
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
        h = entry(buf, int(eo[b]), 1 if e.n_rows <= 253 else 2)
        structure(h, e)
        assert h["N"] < 32768 and h["maxd"] <= 16
        uniq, refs = value_index(blocks[b])
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
