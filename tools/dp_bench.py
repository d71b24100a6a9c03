"""DP-MGD epoch seconds (configs 3 / 4) through distributed.train_data_parallel, one rank per GPU
(torchrun).  Prints one JSON line per config from rank 0."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1702_06943_b200 import synth  # noqa: E402
from paper_1702_06943_b200.distributed import train_data_parallel  # noqa: E402
from paper_1702_06943_b200.matrix import LabeledDataset, SparseRowMatrix  # noqa: E402
from paper_1702_06943_b200.training import TrainConfig  # noqa: E402

rank, world, local = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
graph = os.environ.get("DP_GRAPH", "1") == "1"
cfgs = [int(x) for x in os.environ.get("DP_CFGS", "3,4").split(",")]
for cfg in cfgs:
    if cfg == 5:
        from paper_1702_06943_b200.distributed import train_mlp_data_parallel

        rp, c, v, y = synth.cfg5_dataset(int(os.environ.get("DP_ROWS5", "1000000")))
        ds = LabeledDataset(features=SparseRowMatrix.from_csr(784, rp, c, v, check=False), labels=y)
        _, tr = train_mlp_data_parallel(ds, world, rank, epochs=2, graph=graph)
        if rank == 0:
            print(json.dumps({"config": 5, "world": world, "graph": tr.graph, "epoch_seconds": tr.seconds,
                              "risks": tr.risks}), flush=True)
        continue
    if cfg == 3:
        rp, c, v, y = synth.cfg3_dataset()
        m, loss, lr, epochs = 68, "logistic", 0.1, 3
    else:
        rp, c, v, y = synth.cfg4_dataset()
        m, loss, lr, epochs = 47_236, "hinge", 0.01, 2
    ds = LabeledDataset(features=SparseRowMatrix.from_csr(m, rp, c, v, check=False), labels=y)
    _, tr = train_data_parallel(ds, TrainConfig(loss, 250, lr, epochs), world, rank, graph=graph)
    if rank == 0:
        print(json.dumps({"config": cfg, "world": world, "graph": tr.graph, "epoch_seconds": tr.seconds,
                          "risks": tr.risks}), flush=True)
dist.destroy_process_group()
