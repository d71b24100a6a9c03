"""e2e of the sweep through BatchSweep: one step at a time (run) vs two steps in flight (two
sweeps over the same host blocks, submit / finish alternately).  Prints M rows/s for both."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1702_06943_b200 import codec, synth  # noqa: E402

rp, c, v, br = bench.make_shard(0, 1024)
arena = codec.compress_csr(bench.COLS, rp, c, v, br)
v_h, u_h = synth.cfg2_operands(0, 1024)
for steps in (20, 40):
    r = bench.run_e2e(torch, arena, v_h, u_h, steps, 1)
    print(steps, "steps: two in flight", round(r["value"] / 1e6, 1), "M rows/s; one at a time",
          round(r["serial_value"] / 1e6, 1), "M rows/s; link", round(r["h2d_link_gbs"], 1), "GB/s, used",
          round(r["link_frac"], 3), "identical", r["both_sweeps_bit_identical"], flush=True)
