"""One-process-per-GPU TP groups (torchrun): plumbing only.

torch.distributed is used to agree on the shared-memory name of the library's control plane and
for barriers / max-over-ranks timing; all swap and forward work runs in libmpsw.so.
"""
import os

import torch.distributed as dist


def agree_shm_name(prefix="/mpsw"):
    """Rank 0 picks a unique POSIX shm name and broadcasts it (works on gloo and nccl)."""
    obj = [f"{prefix}_{os.getpid()}_{os.urandom(4).hex()}" if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def open_group_ctx(local_device, **kw):
    """Create this process's rank of a TP group spanning all torch.distributed ranks."""
    from . import mpsw as M
    world, rank = dist.get_world_size(), dist.get_rank()
    name = agree_shm_name()
    return M.Ctx(device_ids=(local_device,), world_size=world, world_rank=rank, shm_name=name, **kw)


def max_over_ranks(values, device=None):
    """Element-wise max of a list of floats across ranks (timing: max over ranks)."""
    import torch
    t = torch.tensor(values, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()
