"""e2e rows/s of BatchSweep.run (host TOC1 bytes -> device -> fused sweep -> host) per chunk count."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1702_06943_b200.codec import compress_csr  # noqa: E402
from paper_1702_06943_b200.kernels import BatchSweep  # noqa: E402

rp, c, v, br = bench.make_shard(0, 1024)
arena = compress_csr(bench.COLS, rp, c, v, br)
bh = arena.data[: int(arena.block_off[-1] + arena.block_len[-1])].cpu().numpy()
rng = np.random.default_rng(0)
v_h, u_h = rng.standard_normal(bench.COLS), rng.standard_normal(arena.n_rows_total)
for chunks in [int(x) for x in (sys.argv[1:] or ["6", "8", "10", "12", "8"])]:
    sw = BatchSweep.from_host_blocks(bh, arena.block_off, arena.block_len, chunks=chunks)
    out = (torch.empty(sw.n_rows, dtype=torch.float64).pin_memory(),
           torch.empty((sw.n_blocks, sw.n_cols), dtype=torch.float64).pin_memory())
    for _ in range(3):
        sw.run(v_h, u_h, out=out)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(30):
        sw.run(v_h, u_h, out=out)
    dt = (time.perf_counter() - t) / 30
    print(f"chunks {chunks}: {dt * 1e3:.3f} ms/step  {sw.n_rows / dt / 1e6:.1f} M rows/s", flush=True)
