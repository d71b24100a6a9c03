"""Config-5 MLP (784-200-10, ReLU, softmax-CE, f64) epoch seconds at a given size."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
p = argparse.ArgumentParser()
p.add_argument("--rows", type=int, default=1_000_000)
p.add_argument("--epochs", type=int, default=2)
a = p.parse_args()

from paper_1702_06943_b200 import synth  # noqa: E402
from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix  # noqa: E402
from paper_1702_06943_b200.mlp import train_mlp  # noqa: E402

t = time.time()
rp, c, v, y = synth.cfg5_dataset(a.rows)
tg = time.time() - t
ds = LabeledDataset(features=SparseRowMatrix.from_csr(784, rp, c, v, check=False), labels=y)
t = time.time()
model, trace = train_mlp(ds, epochs=a.epochs)
tt = time.time() - t
print(json.dumps({"rows": a.rows, "nnz": int(rp[-1]), "gen_s": tg, "train_wall_s": tt, "epoch_seconds": trace.seconds,
                  "risks": trace.risks, "memory": getattr(trace, "memory", None)}))
