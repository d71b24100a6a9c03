"""The reference's own test suite run against this package (SURVEY.md section 7's shim).

oracle/stage_reference_tests.py packs the reference's test files into oracle/_ref/reftests.tar.gz
(git-ignored test infrastructure that travels to the GPU box).  Here they are unpacked into a
scratch directory next to a ``toc`` package that aliases ``toc.codec``, ``toc.kernels``,
``toc.matrix``, ``toc.physical``, ``toc.store`` and ``toc.training`` to this package's modules, so
every ``from toc.X import Y`` in the reference's tests binds to the device implementation.  Two
out-of-scope reference modules the acceptance tests import as fixtures are provided too:
``toc.datasets`` (the reference's own synthetic generator, staged as a fixture) and
``toc.reports`` (its three byte-accounting formulas, reports.py:38-55, restated below; the
physical size is this package's serialize_block).  The suites for the CLI, reports and dataset IO
are not run (out of scope).
"""

from __future__ import annotations

import os
import re
import subprocess
import sys
import tarfile

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TARBALL = os.path.join(ROOT, "oracle", "_ref", "reftests.tar.gz")

TOC_INIT = '''"""Alias package: the reference's module paths bound to paper_1702_06943_b200."""
import importlib
import sys

for _m in ("codec", "kernels", "matrix", "physical", "store", "training"):
    sys.modules[__name__ + "." + _m] = importlib.import_module("paper_1702_06943_b200." + _m)
from paper_1702_06943_b200 import *  # noqa: E402,F401,F403
from paper_1702_06943_b200 import __all__, __version__  # noqa: E402,F401
'''

TOC_REPORTS = '''"""Byte accounting of the reference's reports module (reports.py:38-55), for test_acceptance."""
from paper_1702_06943_b200.physical import serialize_block


def dense_bytes(n_rows, n_cols):
    return 8 * n_rows * n_cols


def csr_bytes(s):
    return 12 * s.nnz + 4 * (s.n_rows + 1)


def physical_bytes(enc):
    return len(serialize_block(enc))
'''


@pytest.fixture(scope="module")
def suite_dir(tmp_path_factory):
    if not os.path.exists(TARBALL):
        pytest.skip("oracle/_ref/reftests.tar.gz not staged (run oracle/stage_reference_tests.py where the "
                    "reference is present)")
    d = tmp_path_factory.mktemp("reference_suite")
    with tarfile.open(TARBALL) as tar:
        tar.extractall(d, filter="data")
    pkg = d / "shim" / "toc"
    pkg.mkdir(parents=True)
    (pkg / "__init__.py").write_text(TOC_INIT)
    (pkg / "reports.py").write_text(TOC_REPORTS)
    (pkg / "datasets.py").write_text((d / "fixtures" / "datasets.py").read_text())
    return d


def test_reference_suite_passes_on_device(suite_dir):
    """Every collected reference test passes through the device implementation."""
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(suite_dir / "shim"), ROOT, env.get("PYTHONPATH", "")])
    log = os.path.join(ROOT, "gpurun_out", "reference_suite.log")
    os.makedirs(os.path.dirname(log), exist_ok=True)
    proc = subprocess.run([sys.executable, "-m", "pytest", str(suite_dir / "tests"), "-q", "-p", "no:cacheprovider",
                           "-o", "addopts=", "--rootdir", str(suite_dir / "tests"), "-rf"],
                          capture_output=True, text=True, env=env, cwd=str(suite_dir), timeout=3000)
    with open(log, "w") as f:
        f.write(proc.stdout + proc.stderr)
    tail = "\n".join(proc.stdout.strip().splitlines()[-40:])
    m = re.search(r"(\d+) passed", proc.stdout)
    passed = int(m.group(1)) if m else 0
    assert proc.returncode == 0, tail
    assert passed >= 190, tail
