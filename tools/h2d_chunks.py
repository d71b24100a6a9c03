"""Host->device copy rate of the e2e sweep's pinned TOC1 bytes: one copy, the 8 chunk copies back
to back, and the chunk copies with the sweep's concurrent device->host result copies -- to see what
holds the streamed e2e below the link's single-copy rate."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1702_06943_b200.codec import compress_csr  # noqa: E402
from paper_1702_06943_b200.kernels import BatchSweep  # noqa: E402

rp, c, v, br = bench.make_shard(0, 1024)
arena = compress_csr(bench.COLS, rp, c, v, br)
sw = BatchSweep.from_host_blocks(arena.data[: int(arena.block_off[-1] + arena.block_len[-1])].cpu().numpy(),
                                 arena.block_off, arena.block_len)
host, dev = sw.host, sw.dev
nb = host.numel()
print("pinned host buffer:", host.is_pinned(), nb, "bytes")
cs = torch.cuda.Stream()
ds = torch.cuda.Stream()
rh = torch.empty(8_500_000 // 8, dtype=torch.float64).pin_memory()
rd = torch.empty_like(rh, device="cuda")


def timed(fn, reps=10):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cs)
        fn()
        e1.record(cs)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return best


def one():
    with torch.cuda.stream(cs):
        dev[:nb].copy_(host, non_blocking=True)


def chunks(k, with_d2h=False):
    def f():
        step = (nb + k - 1) // k
        for i in range(k):
            with torch.cuda.stream(cs):
                dev[i * step: min(nb, (i + 1) * step)].copy_(host[i * step: min(nb, (i + 1) * step)], non_blocking=True)
            if with_d2h:
                with torch.cuda.stream(ds):
                    rh[: rh.numel() // k].copy_(rd[: rh.numel() // k], non_blocking=True)
    return f


for name, fn in (("one copy", one), ("8 chunks", chunks(8)), ("16 chunks", chunks(16)), ("4 chunks", chunks(4)),
                 ("8 chunks + d2h", chunks(8, True))):
    t = timed(fn)
    print(f"{name:16s} {t * 1e3:.3f} ms  {nb / t / 1e9:.1f} GB/s")
