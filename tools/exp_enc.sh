timeout 600 python -m pytest tests/test_gpu_codec.py -x -q > gpurun_out/t_enc.log 2>&1; echo rc=$? >> gpurun_out/t_enc.log
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:encode_kernel -c 1 python tools/prof_sweep.py --reps 1 --kind 1 --trees 0 > gpurun_out/exp_enc.log 2>&1
python - > gpurun_out/exp_enc2.log 2>&1 <<'PY'
import sys, time; sys.path.insert(0, '.')
import torch, bench
from paper_1702_06943_b200.codec import compress_csr
rp, c, v, br = bench.make_shard(0, 1024)
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); a = compress_csr(bench.COLS, rp, c, v, br); torch.cuda.synchronize()
    print("compress_csr 1024 cfg2 batches s", time.perf_counter() - t)
PY
