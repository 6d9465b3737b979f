"""Probe: torch symmetric memory on this box (world size 1, NCCL)."""
import os
import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
try:
    symm_mem.set_backend("CUDA")
except Exception as e:
    print("set_backend:", e)
t = symm_mem.empty(4096, dtype=torch.int64, device="cuda")
h = symm_mem.rendezvous(t, group=dist.group.WORLD)
print("world", h.world_size, "rank", h.rank, "buffer_ptrs", h.buffer_ptrs, "t.ptr", t.data_ptr())
print("signal_pad_ptrs", getattr(h, "signal_pad_ptrs", None))
print([n for n in dir(h) if not n.startswith("_")])
dist.destroy_process_group()
