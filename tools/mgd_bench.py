"""Epoch seconds of device MGD at a config's full size (BASELINE.json configs[2] / [3])."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

p = argparse.ArgumentParser()
p.add_argument("--config", type=int, default=3)
p.add_argument("--rows", type=int, default=0)
p.add_argument("--epochs", type=int, default=0)
p.add_argument("--max-ctas", type=int, default=0)
p.add_argument("--cluster", type=int, default=0)
p.add_argument("--threads", type=int, default=0)
a = p.parse_args()

from paper_1702_06943_b200 import synth  # noqa: E402
from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix  # noqa: E402
from paper_1702_06943_b200.training import DeviceBatches, GlmTrainer, shuffle_once  # noqa: E402

if a.config == 3:
    n, m, loss, lr, epochs = a.rows or 2_000_000, 68, "logistic", 0.1, a.epochs or 10
    t = time.time(); rp, c, v, y = synth.cfg3_dataset(n); tg = time.time() - t
else:
    n, m, loss, lr, epochs = a.rows or 800_000, 47_236, "hinge", 0.01, a.epochs or 5
    t = time.time(); rp, c, v, y = synth.cfg4_dataset(n); tg = time.time() - t
ds = LabeledDataset(features=SparseRowMatrix.from_csr(m, rp, c, v, check=False), labels=y)
t = time.time(); sh = shuffle_once(ds, 0); ts = time.time() - t
t = time.time(); batches = DeviceBatches(sh, 250); import torch; torch.cuda.synchronize(); te = time.time() - t
if a.threads:
    from paper_1702_06943_b200 import _native as _N0
    _N0.lib().toc_mgd_set_image_threads(a.threads)
tr = GlmTrainer(batches, loss, lr, cluster=a.cluster)
if a.max_ctas:
    from paper_1702_06943_b200 import _native as _N
    _N.lib().toc_mgd_set_max_ctas(a.max_ctas)
secs, risks = [], []
for _ in range(epochs):
    secs.append(tr.epoch())
    risks.append(tr.risk())
print("untraced epoch s:", [round(x, 5) for x in secs], "us/step:", round(min(secs) / batches.arena.n_blocks * 1e6, 3),
      "mode", tr.mode, "cluster", tr.cluster)
print(json.dumps({"config": a.config, "rows": n, "steps_per_epoch": batches.arena.n_blocks, "epoch_seconds": secs,
                  "risks": risks, "gen_s": tg, "shuffle_s": ts, "compress_s": te,
                  "block_bytes": batches.arena.block_bytes}))

# phase trace of the epoch kernel (clock64 stamps, cycles at the SM clock)
import ctypes  # noqa: E402
from paper_1702_06943_b200 import _native as N  # noqa: E402
from paper_1702_06943_b200.training import _bind  # noqa: E402

L = _bind()
P = ctypes.c_void_p
L.toc_glm_epoch_traced.argtypes = [P, P, P, P, P, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
                                   P, P, P, P, P, P]
ar = batches.arena
trace = torch.zeros(ar.n_blocks * 8, dtype=torch.int64, device="cuda")
N.check(L.toc_glm_epoch_traced(ar.data.data_ptr(), ar.block_off_d.data_ptr(), ar.meta_d.data_ptr(),
                               ar.meta.ctypes.data_as(P), ar.row_base_d.data_ptr(), ar.n_blocks, batches.n_cols,
                               tr.loss, tr.lr, batches.labels.data_ptr(), tr.w.data_ptr(), tr.sync.data_ptr(),
                               tr.scratch.data_ptr(), trace.data_ptr(), N.stream_handle()), "traced")
torch.cuda.synchronize()
info = np.zeros(8, np.int64)
L.toc_mgd_plan_info.argtypes = [P, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, P]
L.toc_mgd_plan_info(ar.meta.ctypes.data_as(P), ar.n_blocks, batches.n_cols, 0, info.ctypes.data_as(P))
print("plan (smem, budget, small_m, -, max_pairs, ctas, slab, wide):", info.tolist())
T = trace.view(-1, 8).cpu().numpy().astype(np.int64)
d = np.diff(T, axis=1)
names = ["wait", "p1", "matvec+loss", "bound", "vecmat", "update", "fence"]
print("phase cycles (median per step):", {n: int(np.median(d[:, i])) for i, n in enumerate(names)})
print("step critical path (median cycles, acquire->release):", int(np.median(T[:, 7] - T[:, 1])))

if tr.mode == "images":
    L.toc_glm_epoch_images_traced.argtypes = [P, P, P, P, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                              ctypes.c_int32, ctypes.c_double, P, P, P]
    trace.zero_()
    N.check(L.toc_glm_epoch_images_traced(tr.images.data_ptr(), tr.image_off_d.data_ptr(), ar.meta_d.data_ptr(),
                                          ar.meta.ctypes.data_as(P), ar.n_blocks, batches.n_cols, tr.cluster, tr.loss,
                                          tr.lr, tr.w.data_ptr(), trace.data_ptr(), N.stream_handle()),
            "images traced")
    torch.cuda.synchronize()
    T = trace.view(-1, 8).cpu().numpy().astype(np.int64)
    d = np.diff(T, axis=1)
    names = ["image wait", "p1", "matvec+loss", "bound", "vecmat", "col partials+cluster sync", "update"]
    print("cluster", tr.cluster, "phase cycles (median per step):",
          {n: int(np.median(d[:, i])) for i, n in enumerate(names)})
    print("step (median cycles):", int(np.median(np.diff(T[:, 0]))), "image build s", tr.image_build_seconds)
    m = ar.meta
    print("batch shape (median): rows", int(np.median(m["n_rows"])), "pairs", int(np.median(m["n_pairs"])),
          "codes", int(np.median(m["n_codes"])), "derived", int(np.median(m["n_derived"])))

if tr.mode == "parts":
    L.toc_mgd_parts_set_trace.argtypes = [P]
    trace = torch.zeros(ar.n_blocks * 8, dtype=torch.int64, device="cuda")
    N.check(L.toc_mgd_parts_set_trace(trace.data_ptr()), "parts trace")
    tr.epoch()
    torch.cuda.synchronize()
    N.check(L.toc_mgd_parts_set_trace(None), "parts trace off")
    T = trace.view(-1, 8).cpu().numpy().astype(np.int64)[:, :7]
    d = np.diff(T, axis=1)
    names = ["part wait", "p1", "matvec+loss", "vecmat", "gradient REDs+cluster barrier", "update+cluster barrier"]
    print("cluster", tr.cluster, "phase cycles (median per step):",
          {n: int(np.median(d[:, i])) for i, n in enumerate(names)})
    print("step (median cycles):", int(np.median(np.diff(T[:, 0]))))
