"""Per-batch floor of the fused slot-cache sweep: 1036 nearly empty 250 x 784 batches (a few
non-zeros per row) -- what a batch costs in barriers, copies and latencies before any real work."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1702_06943_b200 import codec, synth  # noqa: E402

flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for p_zero in (0.995, 0.95, 0.8):
    for nb in (148, 1036):
        ptr, cols, vals, base = [np.zeros(1, np.int64)], [], [], 0
        for b in range(nb):
            rp, c, v = synth.dense_to_csr(synth.cfg2_batch_dense(0, b, p_zero=p_zero))
            ptr.append(rp[1:] + base)
            base += int(rp[-1])
            cols.append(c)
            vals.append(v)
        arena = codec.compress_csr(784, np.concatenate(ptr), np.concatenate(cols), np.concatenate(vals),
                                   np.arange(nb + 1) * 250)
        assert arena.build_levels()
        vd = torch.randn(784, dtype=torch.float64, device="cuda")
        ud = torch.randn(arena.n_rows_total, dtype=torch.float64, device="cuda")
        for _ in range(3):
            arena.linalg(3, v=vd, u=ud, use_levels=True)
        ts = []
        for _ in range(30):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            arena.linalg(3, v=vd, u=ud, use_levels=True)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1000)
        ts.sort()
        print(f"p_zero {p_zero}: {nb} batches, dims {arena.levels_dims}: {sum(ts[2:-2]) / (len(ts) - 4):.1f} us", flush=True)
