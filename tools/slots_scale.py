"""Fixed cost of the slot-cache sweep launch: device time of the fused launch over 148 k config-2
batches (k batches per SM) for k = 1, 2, 4, 7, L2 flushed -- the intercept is launch + prologue +
tail, the slope the steady-state batch time."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1702_06943_b200 import codec  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
x0 = torch.zeros(1 << 26, device="cuda")
pts = []
for k in (1, 2, 4, 7):
    nb = 148 * k
    rp, c, v, br = bench.make_shard(0, nb)
    arena = codec.compress_csr(bench.COLS, rp, c, v, br)
    assert arena.build_levels()
    vd = torch.randn(bench.COLS, dtype=torch.float64, device="cuda")
    ud = torch.randn(arena.n_rows_total, dtype=torch.float64, device="cuda")
    for kind in (3,):
        for _ in range(3):
            arena.linalg(kind, v=vd, u=ud, use_levels=True)
        ts = []
        for _ in range(30):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            arena.linalg(kind, v=vd, u=ud, use_levels=True)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1000)
        ts.sort()
        pts.append((k, ts[len(ts) // 2]))
        warm = []
        for _ in range(30):  # L2 warm (no flush; a long memset first so the CPU runs ahead of the GPU)
            flush[: 64 << 20].fill_(1) if k > 1 else x0.add_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            arena.linalg(kind, v=vd, u=ud, use_levels=True)
            e1.record()
            torch.cuda.synchronize()
            warm.append(e0.elapsed_time(e1) * 1000)
        warm.sort()
        print(f"{nb} batches ({k} per SM): {ts[len(ts) // 2]:.1f} us (min {ts[0]:.1f}); without the L2 flush {warm[len(warm) // 2]:.1f} us", flush=True)
ks = np.array([p[0] for p in pts], float)
tt = np.array([p[1] for p in pts])
b, a = np.polyfit(ks, tt, 1)
print(f"fit: {a:.1f} us fixed + {b:.2f} us per batch per SM")
# an empty launch on the same stream, for the launch + event cost alone
ts = []
x = torch.zeros(1, device="cuda")
for _ in range(30):
    flush.fill_(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x.add_(1)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1000)
ts.sort()
print(f"one trivial kernel between the same events: {ts[len(ts) // 2]:.1f} us")
