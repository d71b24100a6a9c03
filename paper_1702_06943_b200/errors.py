"""Exception classes of the reference API and the mapping from native status codes to them.

The classes mirror the reference's: CorruptEncodingError (reference codec.py:33), and the
BlockFormatError family (physical.py:33-42).  Device kernels report a status code plus a detail
code and two integers (include/toc_b200.h); ``raise_for_meta`` rebuilds the reference's message
for the first failing check.
"""

from __future__ import annotations

from . import _native as N


class CorruptEncodingError(ValueError):
    """A stored encoding violates the invariants the decoder relies on (codec.py:33-34)."""


class BlockFormatError(ValueError):
    """A serialized block cannot be parsed (physical.py:33-34)."""


class BadMagicError(BlockFormatError):
    pass


class UnsupportedVersionError(BlockFormatError):
    pass


class TruncatedBlockError(BlockFormatError):
    pass


def format_error(status: int, detail: int, a: int, b: int, n_uniques: int = 0, n_cols: int = 0,
                 n_rows: int = 0, head: bytes = b"") -> Exception:
    """Exception for a failed TocBlockMeta check; messages follow physical.py:71-186 and
    codec.py:151-162, 235-244."""
    if status == N.TOC_E_BAD_MAGIC:
        return BadMagicError(f"bad magic {head[:4]!r}")
    if status == N.TOC_E_BAD_VERSION:
        return UnsupportedVersionError(f"unsupported block version {a}")
    if status == N.TOC_E_TRUNCATED:
        return TruncatedBlockError(f"block truncated at offset {a}")
    if status == N.TOC_E_CORRUPT or detail == N.D_UNDEF:
        return CorruptEncodingError(f"row {a}: code {b} references an undefined node")
    msg = {
        N.D_WIDTH: lambda: f"bytes_per_int must be 1..4, got {b} at offset {a}",
        N.D_PAIR_COUNT: lambda: f"pair count {a} does not match packed arrays ({b} columns)",
        N.D_CODE_COUNT: lambda: f"code count {a} does not match packed array ({b})",
        N.D_TRAILING: lambda: f"{a} trailing bytes after block",
        N.D_OFFS_COUNT: lambda: f"expected {a} row offsets, got {b}",
        N.D_OFFS_SPAN: lambda: "row offsets do not span the code array",
        N.D_OFFS_MONO: lambda: f"row offsets not monotone at row {a}",
        N.D_REF_RANGE: lambda: f"value ref {b} out of range for {n_uniques} unique values",
        N.D_PAIR_COL: lambda: f"pair column {b} out of range for n_cols={n_cols}",
        N.D_PAIR_VAL: lambda: f"pair value for column {b} is not finite",
        N.D_CODE_LT1: lambda: f"row {a}: code 0 is not a valid node",
    }.get(detail, lambda: f"block format error (detail {detail})")()
    return BlockFormatError(msg)


def raise_for_meta(rec, head: bytes = b"", lazy: bool = False) -> None:
    """Raise the reference exception for one metadata record (numpy record of META_DTYPE).
    ``lazy`` also raises the CorruptEncodingError that the reference defers to tree build."""
    st = int(rec["status"])
    if st != N.TOC_OK:
        raise format_error(st, int(rec["detail"]), int(rec["detail_a"]), int(rec["detail_b"]),
                           int(rec["n_uniques"]), int(rec["n_cols"]), int(rec["n_rows"]), head)
    if lazy and int(rec["corrupt"]):
        raise CorruptEncodingError(
            f"row {int(rec['detail_a'])}: code {int(rec['detail_b'])} references an undefined node")
