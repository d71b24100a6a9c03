"""Timeline of one BatchSweep.run (native pipeline diagnostic)."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1702_06943_b200 import _native as N  # noqa: E402
from paper_1702_06943_b200.codec import compress_csr  # noqa: E402
from paper_1702_06943_b200.kernels import BatchSweep  # noqa: E402

rp, c, v, br = bench.make_shard(0, 1024)
arena = compress_csr(bench.COLS, rp, c, v, br)
bh = arena.data[: int(arena.block_off[-1] + arena.block_len[-1])].cpu().numpy()
L = N.lib()
L.toc_sweep_set_timing.argtypes = [ctypes.c_int32]
L.toc_sweep_timeline.argtypes = [ctypes.c_int64, ctypes.c_void_p]
import time  # noqa: E402

import torch  # noqa: E402

for chunks, pin in ((8, False), (8, True), (4, True), (16, True)):
    sw = BatchSweep.from_host_blocks(bh, arena.block_off, arena.block_len, chunks=chunks)
    vh = np.random.default_rng(0).standard_normal(784)
    uh = np.random.default_rng(1).standard_normal(sw.n_rows)
    if pin:
        vh, uh = torch.from_numpy(vh).pin_memory(), torch.from_numpy(uh).pin_memory()
    out = (torch.empty(sw.n_rows, dtype=torch.float64).pin_memory(),
           torch.empty((sw.n_blocks, sw.n_cols), dtype=torch.float64).pin_memory())
    for _ in range(3):
        sw.run(vh, uh, out=out)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        sw.run(vh, uh, out=out)
    print(f"chunks {chunks} pinned operands {pin}: {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms per run (wall)")
    for _ in range(3):
        sw.run(vh, uh)
    L.toc_sweep_set_timing(1)
    sw.run(vh, uh, out=out)
    L.toc_sweep_set_timing(0)
    out = np.zeros(5 * len(sw.chunks), np.float32)
    N.check(L.toc_sweep_timeline(len(sw.chunks), out.ctypes.data), "timeline")
    print(f"  per chunk (upload end, index start, index end, compute end, d2h end) ms")
    for k in range(len(sw.chunks)):
        print("  ", np.round(out[5 * k : 5 * k + 5], 3))
