"""Probe: torch symmetric memory on a one-rank NCCL group (peer pointers + signal pads)."""
import os
import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29541")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
try:
    print("backend", symm_mem.get_backend(torch.device("cuda", 0)))
except Exception as e:
    print("get_backend failed", e)
t = symm_mem.empty(1024, dtype=torch.float64, device="cuda")
h = symm_mem.rendezvous(t, dist.group.WORLD)
print("world", h.world_size, "rank", h.rank, "ptrs", h.buffer_ptrs, "signal pad size", h.signal_pad_size,
      "sig ptrs", h.signal_pad_ptrs, "multicast", h.has_multicast_support, "ptrs_dev", h.buffer_ptrs_dev)
dist.destroy_process_group()
