"""One config-2 sweep launch of a given kind in tree-cache mode (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1702_06943_b200.codec import compress_csr  # noqa: E402

kind = int(sys.argv[1]) if len(sys.argv) > 1 else 3
rp, c, v, br = bench.make_shard(0, 1024)
arena = compress_csr(bench.COLS, rp, c, v, br).build_trees()
vd = torch.randn(bench.COLS, dtype=torch.float64, device="cuda")
ud = torch.randn(arena.n_rows_total, dtype=torch.float64, device="cuda")
for _ in range(2):
    arena.linalg(kind, v=vd, u=ud)
torch.cuda.synchronize()
print("ok")
