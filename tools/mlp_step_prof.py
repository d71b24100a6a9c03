"""Time the pieces of one config-5 MLP step (CUDA events, averaged over many batches)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1702_06943_b200 import synth  # noqa: E402
from paper_1702_06943_b200.codec import compress_csr  # noqa: E402

rp, c, v, y = synth.cfg5_dataset(50_000)
arena = compress_csr(784, rp, c, v, np.concatenate([np.arange(0, 50_000, 250), [50_000]])).build_matcache()
W1 = torch.randn(784, 200, dtype=torch.float64, device="cuda") * 0.03
d = torch.randn(250, 200, dtype=torch.float64, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for name, fn in [("right A.W1", lambda b: arena.matmat(0, W1, 200, batch=b)),
                 ("left (d^T.A)", lambda b: arena.matmat(1, d, 200, batch=b))]:
    for b in range(5):
        fn(b)
    torch.cuda.synchronize()
    ev[0].record()
    for b in range(200):
        fn(b)
    ev[1].record()
    ev[1].synchronize()
    print(name, "us/call", ev[0].elapsed_time(ev[1]) / 200 * 1e3)
m = arena.matcache_off
print("cache bytes per batch", int(m[1] - m[0]), "T", int(arena.tree_lengths()[0]), "codes", int(arena.meta["n_codes"][0]))
