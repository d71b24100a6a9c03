"""Device time of the fp32 variant over 1024 config-2 batches: slot cache (toc_linalg_levels32) per kind
beside the tree-cache kernel (toc_linalg32), L2 flushed, and the results against the fp64 chain walk."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
from paper_1702_06943_b200 import codec
rp, c, v, br = bench.make_shard(0, 1024)
arena = codec.compress_csr(bench.COLS, rp, c, v, br)
vd = torch.randn(bench.COLS, dtype=torch.float64, device="cuda"); ud = torch.randn(arena.n_rows_total, dtype=torch.float64, device="cuda")
R64, O64 = arena.linalg(3, v=vd, u=ud, use_levels=False)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def timeit(fn):
    for _ in range(3): fn()
    ts=[]
    for _ in range(30):
        flush.fill_(1); e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1)*1000)
    ts.sort(); return sum(ts[2:-2])/(len(ts)-4)
v32,u32=vd.float(),ud.float()
t_tree=timeit(lambda: arena.linalg32(3,v=v32,u=u32))
assert arena.build_levels()
for k in (1,2,3):
    t=timeit(lambda: arena.linalg32(k,v=v32,u=u32))
    R,O=arena.linalg32(k,v=v32,u=u32)
    er = ((R.double()-R64).abs()/R64.abs().clamp_min(1)).max().item() if k&1 else 0
    eo = ((O.double()-O64).abs()/O64.abs().clamp_min(1)).max().item() if k&2 else 0
    print('slots32 kind',k,round(t,1),'us  max rel R',er,'O',eo)
print('tree32 fused',round(t_tree,1),'us')
