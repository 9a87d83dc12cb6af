"""Probe: torch symmetric memory on a 1-rank NCCL group (peer pointers)."""
import os

import torch
import torch.distributed as dist

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
import torch.distributed._symmetric_memory as symm  # noqa: E402

t = symm.empty(1024, dtype=torch.float32, device="cuda:0")
h = symm.rendezvous(t, dist.group.WORLD)
print("ok", h.world_size, h.rank, [hex(p) for p in h.buffer_ptrs], hex(h.signal_pad_ptrs[0]))
dist.destroy_process_group()
