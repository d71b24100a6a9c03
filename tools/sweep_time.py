"""Device time of the config-2 tree-cache sweep per kind (1 = A.v, 2 = v^T.A, 3 = both), L2 flushed
between reps.  usage: python tools/sweep_time.py [lib.so ...] -- each library timed in turn."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1702_06943_b200 import _native as N  # noqa: E402

libs = sys.argv[1:] or [N.LIB_PATH]
rp, c, v, br = bench.make_shard(0, 1024)
res = {}
for lib in libs:
    N.LIB_PATH = os.path.abspath(lib)
    N._lib = None
    import importlib

    from paper_1702_06943_b200 import codec
    importlib.reload(codec)
    arena = codec.compress_csr(bench.COLS, rp, c, v, br)
    block = codec.compress_csr(bench.COLS, rp, c, v, br)
    arena.build_trees()
    vd = torch.randn(bench.COLS, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
    ud = torch.randn(arena.n_rows_total, dtype=torch.float64, device="cuda",
                     generator=torch.Generator("cuda").manual_seed(2))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = {}
    vf, uf = vd.float(), ud.float()
    runs = {1: lambda: arena.linalg(1, v=vd, u=ud), 2: lambda: arena.linalg(2, v=vd, u=ud),
            3: lambda: arena.linalg(3, v=vd, u=ud), "blk3": lambda: block.linalg(3, v=vd, u=ud),
            "blk2": lambda: block.linalg(2, v=vd, u=ud), "f32": lambda: arena.linalg32(3, v=vf, u=uf)}
    for kind, fn in runs.items():
        for _ in range(3):
            fn()
        ts = []
        for _ in range(30):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        out[kind] = ts[len(ts) // 2]
    R, O = arena.linalg(3, v=vd, u=ud)
    res[lib] = (out, R.double().sum().item(), O.double().sum().item())
    print(os.path.basename(lib), {k: round(t * 1000, 1) for k, t in out.items()}, "us  checks", res[lib][1:], flush=True)
