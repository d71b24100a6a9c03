"""Time toc_index_blocks on resident config-2 blocks (validation cost of the e2e sweep)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1702_06943_b200 import _native as N  # noqa: E402
from paper_1702_06943_b200.codec import compress_csr  # noqa: E402

rp, c, v, br = bench.make_shard(0, 1024)
arena = compress_csr(bench.COLS, rp, c, v, br)
L = N.lib()
meta = torch.empty(1024 * 64, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
print("block bytes mean", float(arena.block_len.mean()))
for nb in (64, 128, 296, 1024):
    for _ in range(3):
        N.check(L.toc_index_blocks(arena.data.data_ptr(), arena.block_off_d.data_ptr(), arena.block_len_d.data_ptr(), nb,
                                   meta.data_ptr(), s.cuda_stream), "index")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        N.check(L.toc_index_blocks(arena.data.data_ptr(), arena.block_off_d.data_ptr(), arena.block_len_d.data_ptr(), nb,
                                   meta.data_ptr(), s.cuda_stream), "index")
    e1.record()
    torch.cuda.synchronize()
    print(f"blocks {nb}: {e0.elapsed_time(e1) / 20 * 1000:.1f} us")
