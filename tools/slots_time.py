"""Device time of the config-2 sweep over 1024 batches: slot cache (toc_levels.cu) per kind
(1 = A.v, 2 = v^T.A, 3 = both) beside the tree-cache chain walk, L2 flushed between reps, and the
slot-cache results checked against the chain walk.
usage: python tools/slots_time.py [lib.so ...]   (each library timed in turn; default: the in-tree one)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1702_06943_b200 import _native as N, codec  # noqa: E402


def timeit(fn, flush, reps=30):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return sum(ts[2:-2]) / (len(ts) - 4) * 1000.0  # trimmed mean: the event clock ticks at ~1 us


libs = [x for x in sys.argv[1:] if x.endswith(".so")]
rp, c, v, br = bench.make_shard(0, 1024)
if libs:
    N.LIB_PATH = os.path.abspath(libs[0])
    N._lib = None
arena = codec.compress_csr(bench.COLS, rp, c, v, br)
arena.build_trees()
import time  # noqa: E402

t0 = time.perf_counter()
ok = arena.build_levels()
print("slot cache built", ok, "in", round(time.perf_counter() - t0, 3), "s;", arena.levels_bytes, "bytes; dims",
      arena.levels_dims, "tree cache", arena.tree_bytes, flush=True)
vd = torch.randn(bench.COLS, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
ud = torch.randn(arena.n_rows_total, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(2))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
Rt, Ot = arena.linalg(3, v=vd, u=ud, use_levels=False)
Rt, Ot = Rt.clone(), Ot.clone()
Rl, Ol = arena.linalg(3, v=vd, u=ud, use_levels=True)
torch.cuda.synchronize()


def rel(a, b):
    return ((a - b).abs() / b.abs().clamp_min(1.0)).max().item()


print("parity vs chain walk: R", rel(Rl, Rt), "O", rel(Ol, Ot), flush=True)
R1, _ = arena.linalg(1, v=vd, use_levels=True)
_, O2 = arena.linalg(2, u=ud, use_levels=True)
print("parity single kinds: R", rel(R1, Rt), "O", rel(O2, Ot), flush=True)
for rep in range(2):
    for lib in libs or [N.LIB_PATH]:
        if libs:  # rebuild this library's cache (the entry format may differ between builds)
            N.LIB_PATH = os.path.abspath(lib)
            N._lib = None
            arena.levels = None
            assert arena.build_levels()
        out = {}
        for k in (1, 2, 3):
            out[f"slots{k}"] = timeit(lambda: arena.linalg(k, v=vd, u=ud, use_levels=True), flush)
        if rep == 0 and lib == (libs or [N.LIB_PATH])[0]:
            out["trees3"] = timeit(lambda: arena.linalg(3, v=vd, u=ud, use_levels=False), flush)
        print(os.path.basename(lib), {k: round(t, 1) for k, t in out.items()}, "us", flush=True)
