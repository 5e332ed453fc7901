"""Probe: does torch symmetric memory get an NVLS multicast address on this box?  (Run with
MASTER_ADDR/MASTER_PORT set; world size 1.)  Round 1, one B200: multicast_ptr = 0 ("Gracefully
skipping multicast initialization"), so the multimem.st variant of the fused gather is untestable here."""
import os, torch, torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
buf = symm_mem.empty((1024, 1024), dtype=torch.bfloat16, device="cuda")
h = symm_mem.rendezvous(buf, dist.group.WORLD)
print("attrs:", [x for x in dir(h) if not x.startswith("_")])
print("multicast_ptr:", getattr(h, "multicast_ptr", None), "buffer_ptrs:", h.buffer_ptrs)
dist.destroy_process_group()
