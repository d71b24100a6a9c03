"""Compression on the device (reference codec.py:112-191 + physical.py:88-130).

``compress_csr`` is the batch pipeline: upload CSR rows once, encode every mini-batch on the GPU
(toc_encode), build the value index and sizes (toc_serialize_sizes), and pack bit-exact TOC1
blocks straight into a device arena (toc_pack_blocks).  ``encode`` mirrors the reference's
single-matrix entry point and returns a host-side LogicalEncoding.
"""

from __future__ import annotations

import ctypes
import warnings
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import CorruptEncodingError  # noqa: F401  (re-exported, reference codec.py:33)
from .matrix import SparseRowMatrix

INFO_DTYPE = np.dtype([
    ("n_rows", "<u4"), ("n_cols", "<u4"), ("n_pairs", "<u4"), ("n_codes", "<u4"), ("n_uniques", "<u4"),
    ("w_cols", "u1"), ("w_refs", "u1"), ("w_codes", "u1"), ("w_offsets", "u1"),
    ("status", "<i4"), ("detail_a", "<u4"), ("detail_b", "<u4"), ("pad_", "<u4"), ("block_bytes", "<i8"),
])
assert INFO_DTYPE.itemsize == 48


class TocEncodeSizes(ctypes.Structure):
    _fields_ = [("hash_slots", ctypes.c_int64), ("n_elems", ctypes.c_int64), ("work_bytes", ctypes.c_int64)]


def _bind():
    L = N.lib()
    if not getattr(L, "_enc_bound", False):
        P, I64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        S = ctypes.POINTER(TocEncodeSizes)
        L.toc_encode_sizes.argtypes = [I64, P, S]
        L.toc_encode.argtypes = [I64, I32, P, P, P, P, P, S, P, P, P, P, P, P, P]
        L.toc_serialize_sizes.argtypes = [I64, P, P, P, P, P, P, S, P, P, P, P, P]
        L.toc_pack_blocks.argtypes = [I64, P, P, P, P, P, P, P, P, P, P, P]
        L.toc_unpack_blocks.argtypes = [P, P, P, I64, P, P, P, P, P, P, P, P]
        L._enc_bound = True
    return L


@dataclass
class LogicalEncoding:
    """First-layer pairs I and per-row codes D (reference codec.py:142-174)."""

    n_rows: int
    n_cols: int
    pairs: list
    rows: list

    def __post_init__(self):
        if self.n_rows != len(self.rows):
            raise ValueError(f"n_rows={self.n_rows} but {len(self.rows)} code rows")
        for col, val in self.pairs:
            if not 0 <= col < self.n_cols:
                raise ValueError(f"pair column {col} out of range for n_cols={self.n_cols}")
            if not np.isfinite(val):
                raise ValueError(f"pair value for column {col} is not finite")
        for i, row in enumerate(self.rows):
            for code in row:
                if code < 1:
                    raise ValueError(f"row {i}: code {code} is not a valid node")

    @property
    def total_codes(self) -> int:
        return sum(len(r) for r in self.rows)

    def derived_node_count(self) -> int:
        return sum(len(r) - 1 for r in self.rows if r)

    def tree_length(self) -> int:
        return 1 + len(self.pairs) + self.derived_node_count()


def _input_error(info_rec, row_ptr_h, batch_row_h, b, cols_h=None) -> ValueError:
    r = int(batch_row_h[b]) + int(info_rec["detail_a"])
    return ValueError(f"row {r}: invalid entry at position {int(info_rec['detail_b'])} "
                      "(columns must be strictly increasing in [0, n_cols), values finite and non-zero)")


def _align16(x):
    return (x + 15) & ~15


def compress_csr(n_cols: int, row_ptr, cols, vals, batch_row, *, max_work_bytes: int = 2 << 30,
                 keep_logical: bool = False):
    """Encode mini-batches (rows [batch_row[b], batch_row[b+1]) of the CSR matrix) into a device
    BlockArena of bit-exact TOC1 blocks.  Inputs are host numpy arrays.  With keep_logical the
    per-batch logical arrays are also returned (host numpy)."""
    torch = N.require_cuda()
    from .arena import BlockArena

    L = _bind()
    row_ptr = np.ascontiguousarray(row_ptr, np.int64)
    cols = np.ascontiguousarray(cols, np.int32)
    vals = np.ascontiguousarray(vals, np.float64)
    batch_row = np.ascontiguousarray(batch_row, np.int64)
    n_batches = len(batch_row) - 1
    elem_base_all = row_ptr[batch_row]
    dev = torch.device("cuda")
    stream = N.stream_handle()
    # chunk the batches so the hash workspace stays bounded (the workspace grows with the chunk:
    # binary search for the longest chunk that fits, at least one batch)
    def work(b0, b1):
        s = TocEncodeSizes()
        eb = np.ascontiguousarray(elem_base_all[b0 : b1 + 1] - elem_base_all[b0])
        N.check(L.toc_encode_sizes(b1 - b0, eb.ctypes.data_as(ctypes.c_void_p), ctypes.byref(s)), "sizes")
        return s.work_bytes

    chunks, start = [], 0
    while start < n_batches:
        if work(start, n_batches) <= max_work_bytes:
            end = n_batches
        else:
            lo, hi = start + 1, n_batches  # work(start, lo) may exceed: one batch is still a chunk
            while hi - lo > 1:
                mid = (lo + hi) // 2
                if work(start, mid) <= max_work_bytes:
                    lo = mid
                else:
                    hi = mid
            end = lo
        chunks.append((start, end))
        start = end
    pieces, logical = [], []
    for (b0, b1) in chunks:
        nb = b1 - b0
        r0, r1 = int(batch_row[b0]), int(batch_row[b1])
        e0, e1 = int(row_ptr[r0]), int(row_ptr[r1])
        rp = row_ptr[r0 : r1 + 1] - e0
        br = batch_row[b0 : b1 + 1] - r0
        eb = np.ascontiguousarray(rp[br])
        sizes = TocEncodeSizes()
        N.check(L.toc_encode_sizes(nb, eb.ctypes.data_as(ctypes.c_void_p), ctypes.byref(sizes)), "toc_encode_sizes")
        d_rp = torch.from_numpy(np.ascontiguousarray(rp)).to(dev)
        with warnings.catch_warnings():  # read-only views (matrix.py freezes its arrays): uploaded, never written
            warnings.simplefilter("ignore", UserWarning)
            d_cols = torch.from_numpy(cols[e0:e1] if e1 > e0 else np.zeros(1, np.int32)).to(dev)
            d_vals = torch.from_numpy(vals[e0:e1] if e1 > e0 else np.zeros(1)).to(dev)
        d_br = torch.from_numpy(np.ascontiguousarray(br)).to(dev)
        d_eb = torch.from_numpy(eb).to(dev)
        n_el = max(int(sizes.n_elems), 1)
        n_rows = int(br[-1])
        work = torch.empty(max(sizes.work_bytes, 1), dtype=torch.uint8, device=dev)
        I_cols = torch.empty(n_el, dtype=torch.int32, device=dev)
        I_vals = torch.empty(n_el, dtype=torch.float64, device=dev)
        codes = torch.empty(n_el, dtype=torch.int32, device=dev)
        offsets = torch.empty(n_rows + nb, dtype=torch.int32, device=dev)
        refs = torch.empty(n_el, dtype=torch.int32, device=dev)
        uniques = torch.empty(n_el, dtype=torch.float64, device=dev)
        info = torch.zeros(nb * INFO_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        N.check(L.toc_encode(nb, n_cols, d_rp.data_ptr(), d_cols.data_ptr(), d_vals.data_ptr(), d_br.data_ptr(),
                             d_eb.data_ptr(), ctypes.byref(sizes), work.data_ptr(), I_cols.data_ptr(),
                             I_vals.data_ptr(), codes.data_ptr(), offsets.data_ptr(), info.data_ptr(), stream),
                "toc_encode")
        N.check(L.toc_serialize_sizes(nb, d_br.data_ptr(), d_eb.data_ptr(), I_cols.data_ptr(), I_vals.data_ptr(),
                                      codes.data_ptr(), offsets.data_ptr(), ctypes.byref(sizes), work.data_ptr(),
                                      refs.data_ptr(), uniques.data_ptr(), info.data_ptr(), stream),
                "toc_serialize_sizes")
        info_h = np.frombuffer(info.cpu().numpy().tobytes(), dtype=INFO_DTYPE)
        bad = np.flatnonzero(info_h["status"] != N.TOC_OK)
        if len(bad):
            raise _input_error(info_h[bad[0]], row_ptr, batch_row, b0 + int(bad[0]))
        blen = info_h["block_bytes"].astype(np.int64)
        boff = np.zeros(nb, np.int64)
        pos = 0
        for i in range(nb):
            boff[i] = pos
            pos = _align16(pos + int(blen[i]))
        arena = torch.zeros(pos + 16, dtype=torch.uint8, device=dev)  # +16: tail padding read by the unpackers
        d_boff = torch.from_numpy(boff).to(dev)
        N.check(L.toc_pack_blocks(nb, d_br.data_ptr(), d_eb.data_ptr(), I_cols.data_ptr(), refs.data_ptr(),
                                  uniques.data_ptr(), codes.data_ptr(), offsets.data_ptr(), info.data_ptr(),
                                  d_boff.data_ptr(), arena.data_ptr(), stream), "toc_pack_blocks")
        pieces.append((arena, boff, blen, pos))
        if keep_logical:
            ic, iv, cd, of = I_cols.cpu().numpy(), I_vals.cpu().numpy(), codes.cpu().numpy(), offsets.cpu().numpy()
            for i in range(nb):
                a = int(eb[i])
                ob = int(br[i]) + i
                logical.append((ic[a : a + info_h["n_pairs"][i]].astype(np.int64).copy(),
                                iv[a : a + info_h["n_pairs"][i]].copy(),
                                cd[a : a + info_h["n_codes"][i]].astype(np.int64).copy(),
                                of[ob : ob + info_h["n_rows"][i] + 1].astype(np.int64).copy()))
        del work
    if len(pieces) == 1:
        arena, boff, blen, _ = pieces[0]
    else:
        total = sum(p[3] for p in pieces)
        arena = torch.zeros(total + 16, dtype=torch.uint8, device=dev)
        boffs, blens, pos = [], [], 0
        for a, bo, bl, size in pieces:
            arena[pos : pos + size].copy_(a[:size])
            boffs.append(bo + pos)
            blens.append(bl)
            pos += size
        boff, blen = np.concatenate(boffs), np.concatenate(blens)
    out = BlockArena(arena, boff, blen)
    return (out, logical) if keep_logical else out


def encode(s: SparseRowMatrix) -> LogicalEncoding:
    """Compress a sparse row matrix losslessly (reference codec.encode, codec.py:177-191)."""
    _, logical = compress_csr(s.n_cols, s.row_ptr, s.cols, s.vals, np.array([0, s.n_rows], np.int64),
                              keep_logical=True)
    ic, iv, cd, of = logical[0]
    pairs = [(int(c), float(v)) for c, v in zip(ic.tolist(), iv.tolist())]
    cdl = cd.tolist()
    rows = [cdl[of[i] : of[i + 1]] for i in range(s.n_rows)]
    return LogicalEncoding(n_rows=s.n_rows, n_cols=s.n_cols, pairs=pairs, rows=rows)


NOT_FOUND = -1  # reference codec.py:30


@dataclass
class DecodeTree:
    """Prefix tree rebuilt from a logical encoding (reference codec.py:194-212): node 0 is the root,
    nodes 1..len(pairs) mirror I, later nodes are derived one per non-final code in scan order;
    first_col / first_val hold each node's first pair.  Built on the device (toc_tree_arrays)."""

    n_cols: int
    parent: list
    column: list
    value: list
    first_col: list
    first_val: list

    def __len__(self) -> int:
        return len(self.parent)


def build_prefix_tree(enc: LogicalEncoding) -> DecodeTree:
    """Rebuild C' (reference codec.py:215-259) on the device.  Raises CorruptEncodingError when a
    code references a node that does not exist yet at its point of use."""
    from .arena import BlockArena
    from .physical import serialize_block

    return BlockArena.from_bytes([serialize_block(enc)]).decode_trees()[0]


def node_sequence(tree: DecodeTree, code: int) -> list:
    """The (column, value) pairs a tree node stands for, in row order (reference codec.py:262-271)."""
    if not 1 <= code < len(tree):
        raise ValueError(f"code {code} out of range for tree of length {len(tree)}")
    pairs = []
    while code != 0:
        pairs.append((tree.column[code], tree.value[code]))
        code = tree.parent[code]
    pairs.reverse()
    return pairs


def decode(enc: LogicalEncoding) -> SparseRowMatrix:
    """Invert encode exactly, values bit for bit (reference codec.py:274-292), on the device."""
    from .arena import BlockArena
    from .physical import serialize_block

    rp, c, v = BlockArena.from_bytes([serialize_block(enc)]).decode()
    return SparseRowMatrix.from_csr(enc.n_cols, rp.cpu().numpy(), c.cpu().numpy(), v.cpu().numpy(), check=False)


class EncoderDictionary:
    """The encoder's prefix-tree dictionary (reference codec.py:37-87) as a host data structure.

    Codes 0..n_cols-1 are per-column start markers; every later code extends its parent's pair
    sequence by one (column, value) pair, looked up by the key (parent, column, value).  Value
    equality is Python float equality, as in the reference.  The device encoder (toc_encode) keeps
    its own hash tables in HBM; this class is the reference-API view of the same dictionary
    (``encode_rows`` rebuilds it from the device's output)."""

    __slots__ = ("n_cols", "_entries", "_child")

    def __init__(self, n_cols: int):
        if n_cols < 0:
            raise ValueError(f"n_cols must be non-negative, got {n_cols}")
        self.n_cols = n_cols
        # entry = (parent code or NOT_FOUND, column, value, start column)
        self._entries = [(NOT_FOUND, c, 0.0, c) for c in range(n_cols)]
        self._child = {}

    def __len__(self) -> int:
        return len(self._entries)

    def add(self, parent_code: int, column: int, value: float) -> int:
        """Append the child of parent_code that extends it by (column, value); returns its code."""
        code = len(self._entries)
        start = column if parent_code == NOT_FOUND else self._entries[parent_code][3]
        self._entries.append((parent_code, column, value, start))
        self._child[(parent_code, column, value)] = code
        return code

    def get(self, parent_code: int, column: int, value: float) -> int:
        return self._child.get((parent_code, column, value), NOT_FOUND)

    def sequence(self, code: int) -> list:
        """The (column, value) pairs code stands for, in row order."""
        if not 0 <= code < len(self._entries):
            raise ValueError(f"code {code} out of range")
        out = []
        while code >= self.n_cols:
            parent, column, value, _ = self._entries[code]
            out.append((column, value))
            code = parent
        return out[::-1]

    def start_index(self, code: int) -> int:
        return self._entries[code][3]

    @property
    def parent(self) -> list:
        return [e[0] for e in self._entries]

    @property
    def column(self) -> list:
        return [e[1] for e in self._entries]

    @property
    def value(self) -> list:
        return [e[2] for e in self._entries]

    @property
    def start(self) -> list:
        return [e[3] for e in self._entries]


def get_longest_match(dictionary: EncoderDictionary, row, pos: int) -> tuple:
    """Greedy longest match of row[pos:] (reference codec.py:90-109): (code, end) with the matched
    pairs row[pos:end]; never crosses the row's end.  The first pair must be a seeded entry."""
    col, val = row[pos]
    code = dictionary.get(col, col, val)
    if code == NOT_FOUND:
        raise ValueError(f"pair ({col}, {val}) not present in dictionary")
    end = pos + 1
    while end < len(row):
        nxt = dictionary.get(code, row[end][0], row[end][1])
        if nxt == NOT_FOUND:
            break
        code, end = nxt, end + 1
    return code, end


def encode_rows(s: SparseRowMatrix):
    """The encoder's dictionary and per-row codes in its working numbering, start markers at
    0..n_cols-1 (reference codec.py:112-139).  The encoding runs on the device (toc_encode);
    the dictionary is then rebuilt from the decode tree, whose nodes are exactly the encoder's
    entries in creation order (seeds = the pairs I, then one entry per non-final code in scan
    order, codec.py:227-251): stored code k is working code k + n_cols - 1."""
    enc = encode(s)
    m = s.n_cols
    shift = m - 1
    d = EncoderDictionary(m)
    if enc.pairs:
        tree = build_prefix_tree(enc)
        for k in range(1, len(tree)):
            par = tree.parent[k]
            d.add(tree.column[k] if par == 0 else par + shift, tree.column[k], tree.value[k])
    return d, [[c + shift for c in row] for row in enc.rows]
