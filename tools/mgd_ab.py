"""A/B of MGD epoch times between library builds: python tools/mgd_ab.py CONFIG ROWS lib.so [lib.so ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

cfg, rows, libs = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3:]
from paper_1702_06943_b200 import _native as N, synth  # noqa: E402
from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix  # noqa: E402

if cfg == 3:
    m, loss, lr = 68, "logistic", 0.1
    rp, c, v, y = synth.cfg3_dataset(rows)
else:
    m, loss, lr = 47_236, "hinge", 0.01
    rp, c, v, y = synth.cfg4_dataset(rows)
ds = LabeledDataset(features=SparseRowMatrix.from_csr(m, rp, c, v, check=False), labels=y)
for rep in range(2):
    for lib in libs:
        N.LIB_PATH = os.path.abspath(lib)
        N._lib = None
        from paper_1702_06943_b200 import training as T

        tr = T.GlmTrainer(T.DeviceBatches(T.shuffle_once(ds, 0), 250), loss, lr)
        secs = [tr.epoch() for _ in range(4)]
        w = tr.w.cpu().numpy()
        print(os.path.basename(lib), tr.mode, "epoch s", [round(x, 5) for x in secs], "us/step",
              round(min(secs) / tr.b.arena.n_blocks * 1e6, 3), "w sum", float(np.sum(w)), flush=True)
