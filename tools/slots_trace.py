"""Per-phase cycle breakdown of the slot-cache sweep (toc_levels.cu): CTA 0 stamps clock64 after
every barrier of its first 64 batches (toc_levels_set_trace).  usage: python tools/slots_trace.py [kind]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1702_06943_b200 import _native as N, codec  # noqa: E402

kind = int(sys.argv[1]) if len(sys.argv) > 1 else 3
p_zero = float(sys.argv[2]) if len(sys.argv) > 2 else None  # e.g. 0.995: nearly empty batches (the per-batch floor)
if p_zero is None:
    rp, c, v, br = bench.make_shard(0, 1024)
else:
    from paper_1702_06943_b200 import synth  # noqa: E402

    ptr, cols, vals, base = [np.zeros(1, np.int64)], [], [], 0
    for b_ in range(1024):
        r_, c_, v_ = synth.dense_to_csr(synth.cfg2_batch_dense(0, b_, p_zero=p_zero))
        ptr.append(r_[1:] + base)
        base += int(r_[-1])
        cols.append(c_)
        vals.append(v_)
    rp, c, v, br = np.concatenate(ptr), np.concatenate(cols), np.concatenate(vals), np.arange(1025) * 250
arena = codec.compress_csr(bench.COLS, rp, c, v, br)
assert arena.build_levels()
vd = torch.randn(bench.COLS, dtype=torch.float64, device="cuda")
ud = torch.randn(arena.n_rows_total, dtype=torch.float64, device="cuda")
tr = torch.zeros(64 * 10, dtype=torch.int64, device="cuda")
L = N.lib()
L.toc_levels_set_trace.argtypes = [ctypes.c_void_p]
for _ in range(3):
    arena.linalg(kind, v=vd, u=ud, use_levels=True)
N.check(L.toc_levels_set_trace(tr.data_ptr()), "trace")
arena.linalg(kind, v=vd, u=ud, use_levels=True)
torch.cuda.synchronize()
N.check(L.toc_levels_set_trace(None), "trace")
t = tr.cpu().numpy().reshape(64, 10)
nb = (arena.n_blocks + 147) // 148
print(f"prologue: kernel entry to the first batch's staged region landed {t[0, 0] - t[0, 9]} cycles; "
      f"first batch {t[0, 7] - t[0, 0]} cycles; CTA 0 entry to its last batch's end {t[nb - 1, 7] - t[0, 9]} cycles")
t = t[: nb - 1]
names = ["scatterT", "push", "colparts", "coltot+P1", "innerH", "rowsAv", "rowtot+zeroT"]
d = np.diff(t[:, :8], axis=1)
tot = t[:, 7] - t[:, 0]
print(f"kind {kind}: batches traced {len(t)}, cycles per batch mean {tot.mean():.0f}")
for i, nm in enumerate(names):
    col = d[:, i]
    if col.any():
        print(f"  {nm:16s} {col.mean():8.0f}  ({100 * col.mean() / tot.mean():4.1f}%)")
gap = t[1:, 0] - t[:-1, 7]
print(f"  between batches  {gap.mean():8.0f}  (includes the stamps' own 64-bit divisions)")
