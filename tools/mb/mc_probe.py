"""Does this box give a multicast (NVLS) mapping for torch symmetric memory at world size 1?"""
import os
import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
print("has_multicast_support", symm_mem._SymmetricMemory.has_multicast_support(symm_mem.DeviceType.CUDA, 0) if hasattr(symm_mem, "DeviceType") else "?")
t = symm_mem.empty(1024, dtype=torch.int32, device="cuda")
h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
print("multicast_ptr", hex(h.multicast_ptr), "world", h.world_size, "buffer_ptrs", [hex(x) for x in h.buffer_ptrs])
dist.destroy_process_group()
