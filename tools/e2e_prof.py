"""Where the e2e sweep step goes: host prep, H2D of the blocks alone, device work alone."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1702_06943_b200 import _native as N  # noqa: E402
from paper_1702_06943_b200.codec import compress_csr  # noqa: E402
from paper_1702_06943_b200.kernels import BatchSweep  # noqa: E402
from paper_1702_06943_b200.matrix import as_vector  # noqa: E402

rp, c, v, br = bench.make_shard(0, 1024)
arena = compress_csr(bench.COLS, rp, c, v, br)
blocks_h = arena.data[: int(arena.block_off[-1] + arena.block_len[-1])].cpu().numpy()
sw = BatchSweep.from_host_blocks(blocks_h, arena.block_off, arena.block_len)
vh = np.random.default_rng(0).standard_normal(784)
uh = np.random.default_rng(1).standard_normal(sw.n_rows)
for _ in range(3):
    sw.run(vh, uh)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    sw.run(vh, uh)
print("run() ms", (time.perf_counter() - t0) / 10 * 1e3)
t0 = time.perf_counter()
for _ in range(10):
    sw.u_h.numpy()[: sw.n_rows] = as_vector(uh, sw.n_rows, "vector")
print("host prep of u ms", (time.perf_counter() - t0) / 10 * 1e3)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    sw.dev[: sw.nbytes].copy_(sw.host[: sw.nbytes], non_blocking=True)
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / 10
print("H2D blocks ms", ms, "GB/s", sw.nbytes / ms / 1e6)
e0.record()
for _ in range(10):
    for arena_c, b0, b1, lo, hi, r0 in sw.chunks:
        N.check(N.lib().toc_index_blocks(arena_c.data.data_ptr(), arena_c.block_off_d.data_ptr(),
                                         arena_c.block_len_d.data_ptr(), arena_c.n_blocks, arena_c.meta_d.data_ptr(),
                                         N.stream_handle()), "idx")
e1.record()
e1.synchronize()
print("index ms", e0.elapsed_time(e1) / 10)
e0.record()
for _ in range(10):
    for arena_c, b0, b1, lo, hi, r0 in sw.chunks:
        nr = arena_c.n_rows_total
        arena_c.linalg(3, v=sw.v_d[:784], u=sw.u_d[r0 : r0 + nr], R=sw.R_d[r0 : r0 + nr], O=sw.O_d[b0:b1])
e1.record()
e1.synchronize()
print("linalg (block-only) ms", e0.elapsed_time(e1) / 10)
