"""The kernel families under the bounds-checked build (libtoc_b200_checked.so, `make checked`,
-DTOC_CHECKED): index and size invariants of the hot kernels are asserted in the kernels (slot and
row indices of the slot cache, node ids of the chain walks, image and part sizes against the
shared-memory plan), each case also checked against the oracle (tools/sanitize_cases.py).  This
stands in for compute-sanitizer memcheck, which is closed on this GPU pool
(profiles/r02/sanitize_refused_r02.txt).  And every kernel family is deterministic: repeated runs
are bit-identical (every sum has a fixed order; a shared-memory race would show up here)."""

from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_1702_06943_b200", "libtoc_b200_checked.so")


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["linalg", "slots", "encode", "mgd3", "mgd4", "mlp", "dp"])
def test_checked_build(case):
    assert os.path.exists(CHECKED), "build it: make -C paper_1702_06943_b200/csrc checked"
    env = dict(os.environ, TOC_LIB=CHECKED)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py"), case], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-2000:])
    assert f"case {case} ok libtoc_b200_checked.so" in r.stdout


@pytest.mark.gpu
def test_repeated_runs_bit_identical():
    import torch

    from paper_1702_06943_b200 import codec, synth

    rp, c, v, counts = synth.cfg2_batches_csr(3, range(24), 250, 784)
    br = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    arena = codec.compress_csr(784, rp, c, v, br)
    vd = torch.randn(784, dtype=torch.float64, device="cuda")
    ud = torch.randn(int(br[-1]), dtype=torch.float64, device="cuda")
    modes = {"block": dict(use_trees=False, use_levels=False)}
    first = {k: [x.clone() for x in arena.linalg(3, v=vd, u=ud, **kw)] for k, kw in modes.items()}
    arena.build_trees()
    modes["trees"] = dict(use_levels=False)
    first["trees"] = [x.clone() for x in arena.linalg(3, v=vd, u=ud, use_levels=False)]
    assert arena.build_levels()
    modes["slots"] = {}
    first["slots"] = [x.clone() for x in arena.linalg(3, v=vd, u=ud)]
    for _ in range(4):
        for k, kw in modes.items():
            R, O = arena.linalg(3, v=vd, u=ud, **kw)
            assert torch.equal(R, first[k][0]) and torch.equal(O, first[k][1]), k
    again = codec.compress_csr(784, rp, c, v, br)
    assert torch.equal(again.data, arena.data)
