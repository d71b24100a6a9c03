"""GPU parity for compression: device encoder + TOC1 packer bit-exact with the reference
(golden fixtures from make_golden.py) and with the oracle on the configs' batches; device
deserialization raises the reference's exception classes on corrupt blocks."""

from __future__ import annotations

import json
import os
import struct

import numpy as np
import pytest

from helpers import random_alphabet_rows

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "golden.json")))


def rows_of(case):
    return [[(c, struct.unpack("<d", bytes.fromhex(x))[0]) for c, x in r] for r in case["rows"]]


@pytest.mark.parametrize("i", range(len(GOLD["cases"])))
def test_encode_matches_reference(i):
    from paper_1702_06943_b200.codec import encode
    from paper_1702_06943_b200.matrix import SparseRowMatrix
    from paper_1702_06943_b200.physical import deserialize_block, serialize_block

    case = GOLD["cases"][i]
    s = SparseRowMatrix(case["n_cols"], rows_of(case))
    enc = encode(s)
    assert [[c, struct.pack("<d", x).hex()] for c, x in enc.pairs] == case["pairs"]
    assert enc.rows == case["codes"]
    blk = serialize_block(enc)
    assert blk.hex() == case["block"]
    back = deserialize_block(blk)
    assert back.rows == enc.rows and back.pairs == enc.pairs


def test_batch_compressor_cfg1():
    from paper_1702_06943_b200 import synth
    from paper_1702_06943_b200.codec import compress_csr

    g = np.load(os.path.join(HERE, "golden", "cfg1.npz"))
    rp, c, v = synth.dense_to_csr(synth.cfg1_dense(0))
    arena = compress_csr(128, rp, c, v, np.array([0, 256]))
    got = arena.data[: int(arena.block_len[0])].cpu().numpy().tobytes()
    assert got == g["block"].tobytes()


def test_batch_compressor_cfg2_many(oracle):
    from paper_1702_06943_b200 import synth
    from paper_1702_06943_b200.codec import compress_csr

    nb = 24
    rp, c, v, counts = synth.cfg2_batches_csr(11, range(nb))
    br = np.concatenate([[0], np.cumsum(counts)])
    arena = compress_csr(784, rp, c, v, br)
    data = arena.data.cpu().numpy()
    for b in range(nb):
        lo, hi = rp[br[b]], rp[br[b + 1]]
        brp = rp[br[b] : br[b + 1] + 1] - lo
        want = oracle.serialize(oracle.encode_csr(784, brp, c[lo:hi], v[lo:hi]))
        off, n = int(arena.block_off[b]), int(arena.block_len[b])
        assert off % 16 == 0
        assert data[off : off + n].tobytes() == want, b


def test_long_rows_and_ragged_batches(oracle):
    """Rows longer than the shared-memory row scratch (1024) and batches of uneven size."""
    from paper_1702_06943_b200.codec import compress_csr

    rng = np.random.default_rng(3)
    n_cols = 1500
    rows = random_alphabet_rows(rng, 40, n_cols, 0.9, 4)
    rows += [rows[i % 7] for i in range(20)] + [[] for _ in range(3)]
    rp, c, v = oracle.rows_to_csr(rows)
    br = np.array([0, 1, 2, 30, 30, 50, 63])
    arena = compress_csr(n_cols, rp, c, v, br)
    data = arena.data.cpu().numpy()
    for b in range(len(br) - 1):
        lo, hi = rp[br[b]], rp[br[b + 1]]
        want = oracle.serialize(oracle.encode_csr(n_cols, rp[br[b] : br[b + 1] + 1] - lo, c[lo:hi], v[lo:hi]))
        off, n = int(arena.block_off[b]), int(arena.block_len[b])
        assert data[off : off + n].tobytes() == want, b


def test_invalid_rows_rejected():
    from paper_1702_06943_b200.codec import compress_csr

    rp = np.array([0, 2, 4])
    with pytest.raises(ValueError):
        compress_csr(5, rp, np.array([0, 3, 2, 2]), np.array([1.0, 2.0, 3.0, 4.0]), np.array([0, 2]))
    with pytest.raises(ValueError):
        compress_csr(5, rp, np.array([0, 3, 1, 2]), np.array([1.0, 0.0, 3.0, 4.0]), np.array([0, 2]))


@pytest.mark.parametrize("i", range(len(GOLD["corrupt"])))
def test_corrupt_blocks(i):
    from paper_1702_06943_b200 import errors
    from paper_1702_06943_b200.arena import BlockArena

    c = GOLD["corrupt"][i]
    data = bytes.fromhex(c["block"])
    kind = "OK"
    try:
        arena = BlockArena.from_bytes([data])
        arena.raise_corrupt()
    except errors.CorruptEncodingError:
        kind = "CorruptEncodingError"
    except errors.BlockFormatError as e:
        kind = type(e).__name__
    assert kind == c["kind"], (c["label"], c["message"])
