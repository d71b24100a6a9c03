"""Golden TOCS batch store from the reference (store.py:59-129), plus the reference's verdict on a
set of damaged copies.  Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_store_golden.py

Outputs tests/golden/store.tocs (the reference's save_batch_store bytes) and store.json (the input
rows and labels, header fields, and for each damaged variant the exception class the reference's
load_batch_store raises).  The reference is not needed at test time.
"""

from __future__ import annotations

import json
import os
import struct
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(HERE))

from toc import codec, physical, store  # noqa: E402  (the reference)
from toc.matrix import SparseRowMatrix  # noqa: E402

from helpers import random_alphabet_rows  # noqa: E402


def fhex(a):
    return [struct.pack("<d", float(x)).hex() for x in np.asarray(a, dtype=np.float64).ravel()]


def verdict(data: bytes, path: str) -> str:
    with open(path, "wb") as f:
        f.write(data)
    try:
        store.load_batch_store(path)
        return "OK"
    except Exception as e:  # noqa: BLE001 -- the class name is the fixture
        return type(e).__name__


def main():
    rng = np.random.default_rng(2024)
    n_cols, batch_size, seed = 9, 7, -5
    rows = random_alphabet_rows(rng, 24, n_cols, 0.6)  # 3 full batches + a short one of 3 rows
    labels = rng.standard_normal(len(rows))
    blocks, labs = [], []
    for lo in range(0, len(rows), batch_size):
        piece = SparseRowMatrix(n_cols, rows[lo : lo + batch_size])
        blocks.append(physical.serialize_block(codec.encode(piece)))
        labs.append(labels[lo : lo + batch_size])
    path = os.path.join(HERE, "store.tocs")
    store.save_batch_store(path, blocks, labs, batch_size, n_cols, seed)
    data = open(path, "rb").read()
    tmp = os.path.join(HERE, "_tmp.tocs")
    first = 29 + 4  # header, then batch 0's length
    variants = {
        "bad_magic": b"TOCX" + data[4:],
        "bad_version": data[:4] + b"\x02" + data[5:],
        "truncated_header": data[:20],
        "truncated_block": data[: first + 10],
        "truncated_labels": data[: len(data) - 5],
        "trailing_bytes": data + b"\x00",
        "inner_block_magic": data[:first] + b"\xff" + data[first + 1 :],
        "row_total": data[:13] + struct.pack("<I", 99) + data[17:],  # header: total_rows at 13..16
        "column_header": data[:17] + struct.pack("<I", n_cols + 1) + data[21:],  # n_cols at 17..20
    }
    # label count of batch 0 off by one (its length field sits right after block 0)
    blen0 = struct.unpack_from("<I", data, 29)[0]
    lc_off = 29 + 4 + blen0
    variants["label_count"] = data[:lc_off] + struct.pack("<I", 6) + data[lc_off + 4 :]
    # batch 2's block damaged (after a good batch 0 and 1), and batch 3 truncated: the inner error first
    pos = 29
    offs = []
    for _ in range(len(blocks)):
        bl = struct.unpack_from("<I", data, pos)[0]
        offs.append(pos + 4)
        lc = struct.unpack_from("<I", data, pos + 4 + bl)[0]
        pos += 4 + bl + 4 + 8 * lc
    d2 = bytearray(data)
    d2[offs[2] + 4] = 9  # TOC1 version byte of batch 2
    variants["inner_version_then_truncated"] = bytes(d2[: offs[3] + 3])
    out = {"n_cols": n_cols, "batch_size": batch_size, "seed": seed,
           "rows": [[[c, fhex([v])[0]] for c, v in r] for r in rows], "labels": fhex(labels),
           "blocks": [b.hex() for b in blocks],
           "variants": {k: {"data": v.hex(), "raises": verdict(v, tmp)} for k, v in variants.items()}}
    os.remove(tmp)
    with open(os.path.join(HERE, "store.json"), "w") as f:
        json.dump(out, f, indent=0)
    print({k: v["raises"] for k, v in out["variants"].items()})


if __name__ == "__main__":
    main()
