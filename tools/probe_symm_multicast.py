"""Probe: does torch's CUDA symmetric memory hand out an NVLS multicast pointer on this box
(world size 1, NCCL process group)?  Prints has_multicast_support and multicast_ptr."""
import json
import os

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29531")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1)
out = {}
try:
    from torch._C._distributed_c10d import _SymmetricMemory
    out["has_multicast_support"] = bool(_SymmetricMemory.has_multicast_support(torch._C._autograd.DeviceType.CUDA, 0))
except Exception as e:  # noqa: BLE001
    out["has_multicast_support_error"] = repr(e)
for backend in (None, "CUDA", "NVSHMEM"):
    try:
        if backend:
            symm_mem.set_backend(backend)
        t = symm_mem.empty(1 << 20, dtype=torch.uint8, device="cuda:0")
        h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
        out[f"{backend}_multicast_ptr"] = int(h.multicast_ptr)
        out[f"{backend}_backend"] = str(symm_mem.get_backend(torch.device("cuda:0")))
    except Exception as e:  # noqa: BLE001
        out[f"{backend}_error"] = repr(e)[:300]
print(json.dumps(out))
dist.destroy_process_group()
