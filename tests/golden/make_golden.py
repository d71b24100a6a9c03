"""Generate the golden fixtures that pin the oracle (and through it the GPU path) to the
reference implementation.  Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the reference package `toc` (read-only, /root/reference/pkg/src) and records its
outputs on seeded inputs.  The fixtures are small and committed; the reference itself is not
needed at test time (it does not exist on the GPU box).

Outputs: tests/golden/golden.json (+ cfg1.npz for the config-1 batch).
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
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from toc import codec, kernels, physical, training  # noqa: E402  (the reference)
from toc.matrix import DenseMatrix, LabeledDataset, SparseRowMatrix  # noqa: E402

from helpers import TOY_ROWS, TREE_ROWS, random_alphabet_rows  # noqa: E402
from paper_1702_06943_b200 import synth  # noqa: E402


def fhex(a) -> list[str]:
    """float64 values as exact hex strings (bit-level pins)."""
    return [struct.pack("<d", float(x)).hex() for x in np.asarray(a, dtype=np.float64).ravel()]


def case_record(n_cols, rows, rng):
    s = SparseRowMatrix(n_cols, rows)
    enc = codec.encode(s)
    cm = kernels.CompressedMatrix(enc)
    tree = cm.tree
    blk = physical.serialize_block(enc)
    v = rng.standard_normal(n_cols)
    u = rng.standard_normal(s.n_rows)
    Mr = rng.standard_normal((n_cols, 3))
    Ml = rng.standard_normal((2, s.n_rows))
    counter = kernels.OpCounter()
    mv = kernels.matvec(cm, v, counter)
    return {
        "n_cols": n_cols,
        "rows": [[[c, struct.pack("<d", x).hex()] for c, x in r] for r in rows],
        "pairs": [[c, struct.pack("<d", x).hex()] for c, x in enc.pairs],
        "codes": enc.rows,
        "block": blk.hex(),
        "parent": tree.parent,
        "column": tree.column,
        "value": fhex(tree.value),
        "v": fhex(v),
        "u": fhex(u),
        "Mr": fhex(Mr),
        "Ml": fhex(Ml),
        "matvec": fhex(mv),
        "vecmat": fhex(kernels.vecmat(u, cm)),
        "matmat_right": fhex(kernels.matmat_right(cm, DenseMatrix(Mr)).values),
        "matmat_left": fhex(kernels.matmat_left(DenseMatrix(Ml), cm).values),
        "kernel_cost": kernels.kernel_cost(cm, "matvec"),
        "counter": [counter.multiply_adds, counter.tree_nodes_visited, counter.codes_visited],
    }


def corrupt_cases(toy_block: bytes):
    """Byte corruptions of the worked-example block and the reference's verdict on each."""
    out = []

    def verdict(data: bytes):
        try:
            physical.deserialize_block(data)
        except physical.BlockFormatError as e:
            return type(e).__name__, str(e)
        try:
            codec.build_prefix_tree(physical.deserialize_block(data))
        except codec.CorruptEncodingError as e:
            return type(e).__name__, str(e)
        return "OK", ""

    rng = np.random.default_rng(1234)
    muts = [(b"XOC1" + toy_block[4:], "bad magic")]
    for keep in (0, 3, 7, 12, 20, 50, 80, 100, len(toy_block) - 1):
        muts.append((toy_block[:keep], f"truncate {keep}"))
    muts.append((toy_block + b"\x00", "trailing"))
    for i in range(60):  # random single-byte corruptions
        pos = int(rng.integers(4, len(toy_block)))
        val = int(rng.integers(0, 256))
        b = bytearray(toy_block)
        b[pos] = val
        muts.append((bytes(b), f"byte {pos} := {val}"))
    for data, label in muts:
        kind, msg = verdict(data)
        out.append({"label": label, "block": data.hex(), "kind": kind, "message": msg})
    # logically corrupt encodings (valid bytes, undefined node references): codec.py:233-244
    for pairs, rows in [([(0, 1.0)], [[2]]), ([(0, 1.0), (1, 2.0)], [[1, 9]]), ([(0, 1.0), (1, 2.0)], [[3, 1]]),
                        ([(0, 1.0), (1, 2.0)], [[1, 2], [3]]), ([(0, 1.0), (1, 2.0)], [[1, 2, 3]])]:
        enc = codec.LogicalEncoding(n_rows=len(rows), n_cols=2, pairs=pairs, rows=rows)
        data = physical.serialize_block(enc)
        kind, msg = verdict(data)
        out.append({"label": f"logical {rows}", "block": data.hex(), "kind": kind, "message": msg})
    return out


def training_cases():
    out = []
    rng = np.random.default_rng(17)
    rows = random_alphabet_rows(rng, 120, 6, 0.7)
    w = rng.standard_normal(6)
    z = np.array([sum(val * w[c] for c, val in r) for r in rows])
    for loss, labels, lr in [("squared", z, 1e-3), ("logistic", np.where(z >= 0, 1.0, -1.0), 5e-2),
                             ("hinge", np.where(z >= 0, 1.0, -1.0), 5e-2)]:
        ds = LabeledDataset(features=SparseRowMatrix(6, rows), labels=labels)
        cfg = training.TrainConfig(loss_kind=loss, batch_size=16, learning_rate=lr, epochs=4, seed=3)
        model, trace = training.train(ds, cfg)
        out.append({"loss": loss, "n_cols": 6, "rows": [[[c, struct.pack("<d", x).hex()] for c, x in r] for r in rows],
                    "labels": fhex(labels), "batch_size": 16, "lr": lr, "epochs": 4, "seed": 3,
                    "risks": fhex(trace.risks), "weights": fhex(model.weights)})
    # the reference's one-hidden-layer network (training.py:81-98, 224-228, 284-293)
    ds = LabeledDataset(features=SparseRowMatrix(6, rows), labels=z)
    cfg = training.TrainConfig(loss_kind="nn_mse", batch_size=16, learning_rate=2e-2, epochs=3, seed=5,
                               hidden_units=4)
    model, trace = training.train(ds, cfg)
    out.append({"loss": "nn_mse", "n_cols": 6, "rows": [[[c, struct.pack("<d", x).hex()] for c, x in r] for r in rows],
                "labels": fhex(z), "batch_size": 16, "lr": 2e-2, "epochs": 3, "seed": 5, "hidden_units": 4,
                "risks": fhex(trace.risks), "w1": fhex(model.w1), "w2": fhex(model.w2)})
    return out


def main():
    rng = np.random.default_rng(20261020)
    cases = [case_record(5, TOY_ROWS, rng), case_record(5, TREE_ROWS, rng)]
    edge = [(4, []), (3, [[(0, 1.0)], [], [(2, 2.0)]]), (1, [[(0, -2.5)]]),
            (8, [[(0, 1.0), (5, 2.0)], [(0, 1.0), (7, 2.0)]]), (3, [[(0, 1.0), (1, 2.0), (2, 3.0)]] * 6)]
    for n_cols, rows in edge:
        cases.append(case_record(n_cols, rows, rng))
    for i in range(40):
        n_rows = int(rng.integers(1, 30))
        n_cols = int(rng.integers(1, 12))
        rows = random_alphabet_rows(rng, n_rows, n_cols, float(rng.uniform(0.1, 1.0)), 16, bool(i % 2))
        cases.append(case_record(n_cols, rows, rng))
    # wider packed widths: columns >= 256 (2-byte cols) and many codes (2-byte codes)
    rows = random_alphabet_rows(rng, 200, 300, 0.3, 40)
    cases.append(case_record(300, rows, rng))

    toy_block = bytes.fromhex(cases[0]["block"])
    golden = {
        "generated_by": "tests/golden/make_golden.py (reference toc imported from /root/reference/pkg/src)",
        "cases": cases,
        "corrupt": corrupt_cases(toy_block),
        "training": training_cases(),
    }
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(golden, f, separators=(",", ":"))

    # config-1 batch (BASELINE.json configs[0])
    A = synth.cfg1_dense(0)
    v, u = synth.cfg1_operands(0)
    s = SparseRowMatrix.from_rows_unchecked(128, synth.csr_rows(*synth.dense_to_csr(A)))
    enc = codec.encode(s)
    cm = kernels.CompressedMatrix(enc)
    blk = physical.serialize_block(enc)
    np.savez_compressed(os.path.join(HERE, "cfg1.npz"), block=np.frombuffer(blk, np.uint8), v=v, u=u,
                        matvec=kernels.matvec(cm, v), vecmat=kernels.vecmat(u, cm),
                        kernel_cost=kernels.kernel_cost(cm, "matvec"), tree_len=len(cm.tree))
    print(f"cases={len(cases)} corrupt={len(golden['corrupt'])} training={len(golden['training'])} "
          f"cfg1 block={len(blk)}B T={len(cm.tree)}")


if __name__ == "__main__":
    main()
