"""Host-side parts of the reference API mirror (no GPU): the export list, the encoder dictionary's
data structure, the value index helper and the TOCM model container."""

from __future__ import annotations

import ast
import os
import struct

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# reference toc/__init__.py:63-110, restated: the 43 public names
REFERENCE_ALL = {
    "BadMagicError", "BlockFormatError", "CompressedMatrix", "CorruptEncodingError", "DecodeTree", "DenseMatrix",
    "EncoderDictionary", "GlmModel", "LabeledDataset", "LogicalEncoding", "LossTrace", "NnModel", "OpCounter",
    "SparseRowMatrix", "TrainConfig", "TruncatedBlockError", "UnsupportedVersionError", "build_prefix_tree",
    "csr_matvec", "csr_vecmat", "decode", "dense_matmat", "dense_matvec", "dense_to_sparse", "dense_vecmat",
    "deserialize_block", "elementwise_power", "empirical_risk", "encode", "get_longest_match", "kernel_cost",
    "matmat_left", "matmat_right", "matvec", "node_sequence", "pack_ints", "scalar_add", "scalar_multiply",
    "serialize_block", "sparse_to_dense", "train", "unpack_ints", "vecmat",
}


def test_public_names_match_reference():
    import paper_1702_06943_b200 as P

    assert set(P.__all__) == REFERENCE_ALL
    for name in P.__all__:
        assert getattr(P, name) is not None


def test_encoder_dictionary_host_structure():
    from paper_1702_06943_b200.codec import NOT_FOUND, EncoderDictionary, get_longest_match

    d = EncoderDictionary(3)
    assert len(d) == 3 and d.sequence(1) == [] and [d.start_index(i) for i in range(3)] == [0, 1, 2]
    s0 = d.add(0, 0, 1.0)
    d.add(1, 1, 2.0)
    pair = d.add(s0, 1, 2.0)
    assert (s0, pair) == (3, 5)
    assert d.get(s0, 1, 2.0) == 5 and d.get(s0, 1, 3.0) == NOT_FOUND
    assert d.sequence(pair) == [(0, 1.0), (1, 2.0)] and d.start_index(pair) == 0
    assert get_longest_match(d, [(0, 1.0), (1, 2.0)], 0) == (5, 2)
    assert get_longest_match(d, [(0, 1.0)], 0) == (3, 1)  # never crosses the row end
    with pytest.raises(ValueError):
        get_longest_match(d, [(2, 9.0)], 0)
    with pytest.raises(ValueError):
        EncoderDictionary(-1)


def test_value_index_first_occurrence_by_bits():
    from paper_1702_06943_b200.physical import build_value_index, value_index_lookup
    from paper_1702_06943_b200.errors import BlockFormatError

    vals = [3.0, 1.0, 3.0, -0.0, 0.0, 2.0, 1.0, float("nan")]
    u, refs = build_value_index(vals)
    assert [struct.pack("<d", x) for x in u] == [struct.pack("<d", x) for x in (3.0, 1.0, -0.0, 0.0, 2.0,
                                                                               float("nan"))]
    assert refs == [0, 1, 0, 2, 3, 4, 1, 5]
    assert build_value_index([]) == ([], [])
    assert value_index_lookup(u, 4) == 2.0
    with pytest.raises(BlockFormatError):
        value_index_lookup(u, 6)


def test_model_container_roundtrip_and_errors(tmp_path):
    from paper_1702_06943_b200.errors import BadMagicError, BlockFormatError, TruncatedBlockError
    from paper_1702_06943_b200.store import MODEL_MAGIC, load_model, save_model
    from paper_1702_06943_b200.training import GlmModel, NnModel

    rng = np.random.default_rng(3)
    g = GlmModel(weights=rng.standard_normal(11))
    save_model(tmp_path / "g.tocm", g, "hinge")
    back, kind = load_model(tmp_path / "g.tocm")
    assert kind == "hinge" and back.weights.tobytes() == g.weights.tobytes()
    n = NnModel(w1=rng.standard_normal((5, 3)), w2=rng.standard_normal((3, 1)))
    save_model(tmp_path / "n.tocm", n, "nn_mse")
    back, kind = load_model(tmp_path / "n.tocm")
    assert kind == "nn_mse" and back.w1.tobytes() == n.w1.tobytes() and back.w2.tobytes() == n.w2.tobytes()
    with pytest.raises(ValueError, match="loss_kind"):
        save_model(tmp_path / "x.tocm", g, "absolute")
    (tmp_path / "c.tocm").write_bytes(MODEL_MAGIC + struct.pack("<BBII", 1, 200, 1, 0) + struct.pack("<d", 0.5))
    with pytest.raises(BlockFormatError, match="loss code 200"):
        load_model(tmp_path / "c.tocm")
    data = (tmp_path / "g.tocm").read_bytes()
    (tmp_path / "t.tocm").write_bytes(data[:-3])
    with pytest.raises(TruncatedBlockError, match="weights"):
        load_model(tmp_path / "t.tocm")
    (tmp_path / "t.tocm").write_bytes(data + b"\x01")
    with pytest.raises(BlockFormatError, match="trailing"):
        load_model(tmp_path / "t.tocm")
    (tmp_path / "t.tocm").write_bytes(b"TOCS" + data[4:])
    with pytest.raises(BadMagicError, match="model magic"):
        load_model(tmp_path / "t.tocm")


def test_training_api_validations_without_device():
    from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix
    from paper_1702_06943_b200.training import GlmModel, TrainConfig, apply_update, empirical_risk, make_batches

    ds = LabeledDataset(features=SparseRowMatrix(1, [[(0, 1.0)], [(0, 2.0)]]), labels=np.array([1.0, 3.0]))
    with pytest.raises(ValueError, match="execution"):
        make_batches(ds, 2, "gpu")
    with pytest.raises(ValueError, match="batch_size"):
        make_batches(ds, 0, "csr")
    with pytest.raises(ValueError, match="loss_kind"):
        empirical_risk(GlmModel(np.zeros(1)), ds, "absolute")
    assert apply_update(np.array([0.0, 0.0]), np.array([-1.0, -2.0]), 0.1, 1).tolist() == [0.1, 0.2]
    assert TrainConfig("squared", 4, 0.1, 2, execution="dense").execution == "dense"


def test_reference_suite_stager_is_test_infrastructure():
    """The stager only writes under oracle/_ref (git-ignored) and the product never imports it."""
    src = open(os.path.join(ROOT, "oracle", "stage_reference_tests.py")).read()
    assert "_ref" in src and "TEST INFRASTRUCTURE" in src
    gi = open(os.path.join(ROOT, ".gitignore")).read().split()
    assert "oracle/_ref/" in gi
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_1702_06943_b200")):
        for f in files:
            if f.endswith(".py"):
                tree = ast.parse(open(os.path.join(dirpath, f)).read())
                mods = [n.module for n in ast.walk(tree) if isinstance(n, ast.ImportFrom) and n.module]
                assert not any(m.startswith("oracle") for m in mods), f
