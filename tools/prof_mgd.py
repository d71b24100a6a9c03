"""One config-3 MGD epoch over step images (for ncu: kernel epoch_solo_kernel)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
p = argparse.ArgumentParser()
p.add_argument("--rows", type=int, default=200_000)
p.add_argument("--mode", default="images")
p.add_argument("--cluster", type=int, default=0)
a = p.parse_args()

import torch  # noqa: E402

from paper_1702_06943_b200 import synth  # noqa: E402
from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix  # noqa: E402
from paper_1702_06943_b200.training import DeviceBatches, GlmTrainer, shuffle_once  # noqa: E402

rp, c, v, y = synth.cfg3_dataset(a.rows)
ds = LabeledDataset(features=SparseRowMatrix.from_csr(68, rp, c, v, check=False), labels=y)
tr = GlmTrainer(DeviceBatches(shuffle_once(ds, 0), 250), "logistic", 0.1, mode=a.mode, cluster=a.cluster)
print("epoch s", tr.epoch(), "mode", tr.mode)
torch.cuda.synchronize()
