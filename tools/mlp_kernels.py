"""In-stream time per step of each config-5 step kernel (toc_mlp_set_kernels masks), 200k rows."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1702_06943_b200 import _native as N  # noqa: E402
from paper_1702_06943_b200 import mlp, synth  # noqa: E402
from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
rp, c, v, y = synth.cfg5_dataset(rows)
ds = LabeledDataset(features=SparseRowMatrix.from_csr(784, rp, c, v, check=False), labels=y)
net = mlp._Net(ds, 250, 0, step_cache=True)
w1, b1, w2, b2 = (torch.from_numpy(x).cuda() for x in mlp.init_mlp(784, 200, 10, 0))
run = mlp._native_epoch(net, 200, 10)
L = N.lib()
L.toc_mlp_set_kernels.argtypes = [ctypes.c_int32]
L.toc_mlp_set_graph.argtypes = [ctypes.c_int32]
steps = net.arena.n_blocks
L.toc_mlp_set_decode_ctas.argtypes = [ctypes.c_int32]
L.toc_mlp_set_fused.argtypes = [ctypes.c_int32]
for fz in (0, 1):
    L.toc_mlp_set_fused(fz)
    L.toc_mlp_set_kernels(15)
    run(w1, b1, w2, b2, 0.0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run(w1, b1, w2, b2, 0.0)
    e1.record()
    torch.cuda.synchronize()
    print(f"fused {fz}: all {e0.elapsed_time(e1) * 1000 / steps:7.2f} us/step", flush=True)
for dc in [int(x) for x in os.environ.get("DECODE_CTAS", "").split(",") if x]:
    N.check(L.toc_mlp_set_decode_ctas(dc), "decode ctas")
    L.toc_mlp_set_kernels(15)
    run(w1, b1, w2, b2, 0.0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run(w1, b1, w2, b2, 0.0)
    e1.record()
    torch.cuda.synchronize()
    print(f"decode ctas/SM {dc:2d}: all {e0.elapsed_time(e1) * 1000 / steps:7.2f} us/step", flush=True)
for graph in (0, 1):
    L.toc_mlp_set_graph(graph)
    for name, mask in [("all", 15), ("decode", 1), ("right", 2), ("tail", 4), ("left", 8), ("none", 0)]:
        L.toc_mlp_set_kernels(mask)
        run(w1, b1, w2, b2, 0.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run(w1, b1, w2, b2, 0.0)
        e1.record()
        torch.cuda.synchronize()
        print(f"graph {graph} {name:7s} {e0.elapsed_time(e1) * 1000 / steps:7.2f} us/step", flush=True)
L.toc_mlp_set_kernels(15)
L.toc_mlp_set_graph(1)
