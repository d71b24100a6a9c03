"""Profiling driver: compress N config-2 batches on the GPU, then launch the compressed
linear-algebra kernel a few times (kind: 1 matvec, 2 vecmat, 3 both).  Used under ncu."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

p = argparse.ArgumentParser()
p.add_argument("--batches", type=int, default=1024)
p.add_argument("--kind", type=int, default=3)
p.add_argument("--reps", type=int, default=3)
p.add_argument("--trees", type=int, default=1)
p.add_argument("--levels", type=int, default=0)
p.add_argument("--prefetch", type=int, default=-1)
p.add_argument("--splits", type=int, default=-1)
p.add_argument("--depth", type=int, default=-1)
a = p.parse_args()

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1702_06943_b200.codec import compress_csr  # noqa: E402

rp, c, v, br = bench.make_shard(0, a.batches)
arena = compress_csr(bench.COLS, rp, c, v, br)
if a.depth >= 0:
    from paper_1702_06943_b200 import _native as N
    N.lib().toc_tree_set_depth_order(a.depth)
if a.trees:
    arena.build_trees()
if a.levels:
    assert arena.build_levels()
if a.splits >= 0:
    from paper_1702_06943_b200 import _native as N
    N.lib().toc_linalg_set_splits(a.splits)
if a.prefetch >= 0:
    from paper_1702_06943_b200 import _native as N
    N.lib().toc_levels_set_prefetch(a.prefetch)
vd = torch.randn(bench.COLS, dtype=torch.float64, device="cuda")
ud = torch.randn(arena.n_rows_total, dtype=torch.float64, device="cuda")
for _ in range(a.reps):
    arena.linalg(a.kind, v=vd, u=ud, use_levels=bool(a.levels))
torch.cuda.synchronize()
print("ok", arena.n_blocks, arena.block_bytes, "levels_bytes", getattr(arena, "levels_bytes", None),
      "tree_bytes", getattr(arena, "tree_bytes", None))
