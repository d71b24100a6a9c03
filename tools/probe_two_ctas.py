"""Timing side of tools/probe_two_ctas.sh: the fused slot-cache sweep over column-halved config-2
batches (2048 batches of 250 x 392: the non-zeros of 1024 full batches) with each library given."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1702_06943_b200 import _native as N, codec, synth  # noqa: E402

HALF = 392
nb = 1024
ptr, cols, vals = [np.zeros(1, np.int64)], [], []
base = 0
for half in (0, 1):
    for b in range(nb):
        A = synth.cfg2_batch_dense(0, b)[:, half * HALF:(half + 1) * HALF]
        rp, c, v = synth.dense_to_csr(A)
        ptr.append(rp[1:] + base)
        base += int(rp[-1])
        cols.append(c)
        vals.append(v)
rp = np.concatenate(ptr)
br = np.arange(2 * nb + 1) * 250
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ref = None
for lib in sys.argv[1:]:
    N.LIB_PATH = os.path.abspath(lib)
    N._lib = None
    arena = codec.compress_csr(HALF, rp, np.concatenate(cols), np.concatenate(vals), br)
    assert arena.build_levels()
    g = torch.Generator("cuda").manual_seed(1)
    vd = torch.randn(HALF, dtype=torch.float64, device="cuda", generator=g)
    ud = torch.randn(arena.n_rows_total, dtype=torch.float64, device="cuda", generator=g)
    out = {}
    for kind in (1, 2, 3):
        for _ in range(3):
            R, O = arena.linalg(kind, v=vd, u=ud, use_levels=True)
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
        out[kind] = round(sum(ts[2:-2]) / (len(ts) - 4), 1)
    R, O = arena.linalg(3, v=vd, u=ud, use_levels=True)
    if ref is None:
        ref = (R.clone(), O.clone())
    same = bool(torch.equal(R, ref[0]) and torch.equal(O, ref[1]))
    print(os.path.basename(lib), "slot cache", arena.levels_bytes, "dims", arena.levels_dims, out,
          "us (A.v / v^T.A / fused); equal to the first library's results:", same, flush=True)
