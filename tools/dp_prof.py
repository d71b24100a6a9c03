"""One DP epoch of config 4 (or 3) at world 1, for ncu: which kernels make up a step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1702_06943_b200 import synth  # noqa: E402
from paper_1702_06943_b200.distributed import train_data_parallel  # noqa: E402
from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix  # noqa: E402
from paper_1702_06943_b200.training import TrainConfig  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
n = 25_000
if cfg == 3:
    rp, c, v, y = synth.cfg3_dataset(n)
    m, loss, lr = 68, "logistic", 0.1
else:
    rp, c, v, y = synth.cfg4_dataset(n)
    m, loss, lr = 47_236, "hinge", 0.01
ds = LabeledDataset(features=SparseRowMatrix.from_csr(m, rp, c, v, check=False), labels=y)
train_data_parallel(ds, TrainConfig(loss, 250, lr, 1), 1, 0, graph=False)
dist.destroy_process_group()
