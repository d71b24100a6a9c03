import sys, time; sys.path.insert(0, '.')
import numpy as np, torch, bench
from paper_1702_06943_b200 import _native as N
from paper_1702_06943_b200.codec import compress_csr
rp, c, v, br = bench.make_shard(0, 1024)
a = compress_csr(bench.COLS, rp, c, v, br); a.build_trees()
vh = torch.randn(784, dtype=torch.float64).pin_memory(); uh = torch.randn(a.n_rows_total, dtype=torch.float64).pin_memory()
Rh = torch.empty(a.n_rows_total, dtype=torch.float64).pin_memory(); Oh = torch.empty((a.n_blocks, 784), dtype=torch.float64).pin_memory()
for ch in (1, 2, 3, 4, 8):
    for _ in range(3): a.linalg_pipelined(3, vh, uh, Rh, Oh, chunks=ch)
    t = time.perf_counter()
    for _ in range(20): a.linalg_pipelined(3, vh, uh, Rh, Oh, chunks=ch)
    dt = (time.perf_counter() - t) / 20
    print(ch, "chunks: ms", dt * 1e3, "M rows/s", a.n_rows_total / dt / 1e6)
