"""e2e with the arena resident (BlockArena.linalg_pipelined): one step at a time vs two in flight."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1702_06943_b200 import codec, synth  # noqa: E402

rp, c, v, br = bench.make_shard(0, 1024)
arena = codec.compress_csr(bench.COLS, rp, c, v, br)
assert arena.build_levels()
v_h, u_h = synth.cfg2_operands(0, 1024)
for steps in (20, 60):
    r = bench.run_e2e_resident(torch, arena, v_h, u_h, steps, 1)
    print(steps, "steps: two in flight", round(r["value"] / 1e6, 1), "M rows/s; one at a time",
          round(r["serial_value"] / 1e6, 1), "M rows/s; identical", r["both_slots_bit_identical"], flush=True)
