timeout 600 python -m pytest tests/test_gpu_codec.py tests/test_gpu_training.py -x -q > gpurun_out/t_enc.log 2>&1; echo rc=$? >> gpurun_out/t_enc.log
python - > gpurun_out/exp_enc2.log 2>&1 <<'PY'
import sys, time; sys.path.insert(0, '.')
import numpy as np, torch, bench
from paper_1702_06943_b200 import synth
from paper_1702_06943_b200.codec import compress_csr
rp, c, v, br = bench.make_shard(0, 1024)
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); a = compress_csr(bench.COLS, rp, c, v, br); torch.cuda.synchronize()
    print("cfg2 1024 batches s", time.perf_counter() - t)
rp, c, v, y = synth.cfg3_dataset()
br = np.arange(0, len(y) + 1, 250)
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); a = compress_csr(68, rp, c, v, br); torch.cuda.synchronize()
    print("cfg3 8000 batches s", time.perf_counter() - t)
PY
