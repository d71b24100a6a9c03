"""GPU parity at the BASELINE.json sizes (configs 3, 4 and 5), against the oracle port.

The smaller-subset tests elsewhere pin the kernels; these pin the full runs the bench times:
* config 3: 2,000,000 x 68 logistic MGD, batch 250, lr 0.1, 10 epochs;
* config 4: 800,000 x 47,236 hinge MGD, batch 250, lr 0.01, 5 epochs;
* config 5: the 784-200-10 MLP over 40 steps (10,000 rows) at hidden = 200.
Bar (north_star): loss curves within 1e-6 relative per epoch; weights within 1e-6 relative to
each weight itself (a 1e-12 x max|w| floor for exact zeros), not the max(1, |w|) form that would
make config 4's ~1e-5 weights vacuous.  Each test takes tens of seconds (the oracle's epochs and
the data generation on the host).
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REL = 1e-6


def _pure_rel_err(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    floor = 1e-12 * np.max(np.abs(want), initial=0.0)
    return float(np.max(np.abs(got - want) / (np.abs(want) + floor + 1e-300), initial=0.0))


def _glm_full(oracle, cfg):
    from paper_1702_06943_b200 import synth
    from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix
    from paper_1702_06943_b200.training import TrainConfig, train

    if cfg == 3:
        rp, c, v, y = synth.cfg3_dataset()
        m, loss, lr, epochs = 68, "logistic", 0.1, 10
    else:
        rp, c, v, y = synth.cfg4_dataset()
        m, loss, lr, epochs = 47_236, "hinge", 0.01, 5
    ds = LabeledDataset(features=SparseRowMatrix.from_csr(m, rp, c, v, check=False), labels=y)
    model, trace = train(ds, TrainConfig(loss, 250, lr, epochs))
    w_ref, risks_ref = oracle.train_glm(rp, c, v, y, m, loss, 250, lr, epochs, 0)
    risk_err = _pure_rel_err(trace.risks, risks_ref)
    w_err = _pure_rel_err(model.weights, w_ref)
    assert risk_err <= REL, (trace.risks, risks_ref)
    assert w_err <= REL, w_err
    assert np.count_nonzero(w_ref) > m // 10  # the run moved the weights (not a vacuous check)


def test_cfg3_full_size_vs_oracle(oracle):
    _glm_full(oracle, 3)


def test_cfg4_full_size_vs_oracle(oracle):
    _glm_full(oracle, 4)


def test_cfg5_hidden200_40_steps_vs_oracle(oracle):
    from paper_1702_06943_b200 import synth
    from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix
    from paper_1702_06943_b200.mlp import train_mlp

    rp, c, v, y = synth.cfg5_dataset(10_000)
    ds = LabeledDataset(features=SparseRowMatrix.from_csr(784, rp, c, v), labels=y)
    model, trace = train_mlp(ds, hidden=200, classes=10, batch_size=250, learning_rate=0.05, epochs=1, seed=0)
    (w1, b1, w2, b2), risks = oracle.train_mlp(rp, c, v, y, 784, 200, 10, 250, 0.05, 1, 0)
    assert _pure_rel_err(trace.risks, risks) <= REL, (trace.risks, risks)
    for got, want in ((model.w1, w1), (model.b1, b1), (model.w2, w2), (model.b2, b2)):
        assert _pure_rel_err(got, want) <= REL, _pure_rel_err(got, want)
