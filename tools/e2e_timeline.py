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
for chunks in (4, 8, 16):
    sw = BatchSweep.from_host_blocks(bh, arena.block_off, arena.block_len, chunks=chunks)
    vh = np.random.default_rng(0).standard_normal(784)
    uh = np.random.default_rng(1).standard_normal(sw.n_rows)
    for _ in range(3):
        sw.run(vh, uh)
    L.toc_sweep_set_timing(1)
    sw.run(vh, uh)
    L.toc_sweep_set_timing(0)
    out = np.zeros(5 * len(sw.chunks), np.float32)
    N.check(L.toc_sweep_timeline(len(sw.chunks), out.ctypes.data), "timeline")
    print(f"chunks {chunks}: per chunk (upload end, index start, index end, compute end, d2h end) ms")
    for k in range(len(sw.chunks)):
        print("  ", np.round(out[5 * k : 5 * k + 5], 3))
