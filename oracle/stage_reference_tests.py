"""TEST INFRASTRUCTURE (not product code): stage the reference's own test suite for the GPU box.

Run here, where /root/reference exists (``__graft_entry__.build()`` calls it): packs the
reference's test files (pkg/tests/*.py) and its dataset generator (toc/datasets.py, which
test_acceptance uses only as a fixture source) into oracle/_ref/reftests.tar.gz.  oracle/_ref/ is
git-ignored and travels to the GPU box with the snapshot, where tests/test_reference_suite.py
unpacks it and runs the reference's tests against this package (``toc`` aliased to it).  Nothing
on the GPU box reads /root/reference.
"""

from __future__ import annotations

import io
import os
import sys
import tarfile

REF = "/root/reference/pkg"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref", "reftests.tar.gz")
# the suites on the hot path's API; test_cli / test_reports / test_datasets cover out-of-scope modules
SUITES = ("conftest.py", "test_codec.py", "test_kernels.py", "test_matrix.py", "test_physical.py", "test_store.py",
          "test_training.py", "test_acceptance.py")


def stage() -> str | None:
    if not os.path.isdir(REF):
        return None
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with tarfile.open(OUT, "w:gz") as tar:
        for name in SUITES:
            tar.add(os.path.join(REF, "tests", name), arcname=f"tests/{name}")
        tar.add(os.path.join(REF, "src", "toc", "datasets.py"), arcname="fixtures/datasets.py")
        info = tarfile.TarInfo("SOURCE")
        note = f"staged from {REF} by oracle/stage_reference_tests.py\n".encode()
        info.size = len(note)
        tar.addfile(info, io.BytesIO(note))
    return OUT


if __name__ == "__main__":
    out = stage()
    print(out or "reference absent: nothing staged")
    sys.exit(0)
