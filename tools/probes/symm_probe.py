"""Probe torch symmetric memory on the box: allocation, peer pointers, signal pads, graph capture."""
import os, torch, torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem

local = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
rank, P = dist.get_rank(), dist.get_world_size()
print(rank, "backend", symm_mem.get_backend(dev) if hasattr(symm_mem, "get_backend") else None, flush=True)
t = symm_mem.empty(1024, dtype=torch.float32, device=dev)
t.fill_(rank)
hdl = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
print(rank, "buffer_ptrs", [hex(p) for p in hdl.buffer_ptrs], "pad", [hex(p) for p in hdl.signal_pad_ptrs],
      "pad size", hdl.signal_pad_size, "mc", hdl.has_multicast_support if hasattr(hdl, "has_multicast_support") else None, flush=True)
hdl.barrier()
peer = (rank + 1) % P
pt = hdl.get_buffer(peer, (1024,), torch.float32)
print(rank, "peer view", pt[:4].tolist(), flush=True)
pt.add_(100)   # write into the peer's buffer through NVLink
torch.cuda.synchronize(); hdl.barrier(); torch.cuda.synchronize()
print(rank, "mine after peer write", t[:4].tolist(), flush=True)
t2 = symm_mem.empty(1 << 20, dtype=torch.bfloat16, device=dev)
h2 = symm_mem.rendezvous(t2, dist.group.WORLD.group_name)
print(rank, "second buffer ptrs", [hex(p) for p in h2.buffer_ptrs], flush=True)
dist.barrier(); dist.destroy_process_group()
