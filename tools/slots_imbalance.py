"""How much of the fused sweep's launch time is imbalance between SMs: 1036 different config-2
batches (7 per SM) against 1036 copies of one batch (every SM does identical work)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1702_06943_b200 import codec, synth  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(arena):
    vd = torch.randn(bench.COLS, dtype=torch.float64, device="cuda")
    ud = torch.randn(arena.n_rows_total, dtype=torch.float64, device="cuda")
    for _ in range(3):
        arena.linalg(3, v=vd, u=ud, use_levels=True)
    ts = []
    for _ in range(40):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        arena.linalg(3, v=vd, u=ud, use_levels=True)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1000)
    ts.sort()
    return sum(ts[3:-3]) / (len(ts) - 6)


nb = 1036
rp, c, v, br = bench.make_shard(0, nb)
arena = codec.compress_csr(bench.COLS, rp, c, v, br)
assert arena.build_levels()
print(f"{nb} different batches: {timed(arena):.1f} us", flush=True)
for pick in (0, 1, 5):
    r1, c1, v1 = synth.dense_to_csr(synth.cfg2_batch_dense(0, pick))
    rp2 = np.concatenate([[0], np.cumsum(np.tile(np.diff(r1), nb))]).astype(np.int64)
    arena2 = codec.compress_csr(bench.COLS, rp2, np.tile(c1, nb), np.tile(v1, nb), np.arange(nb + 1) * 250)
    assert arena2.build_levels()
    print(f"{nb} copies of batch {pick}: {timed(arena2):.1f} us", flush=True)
