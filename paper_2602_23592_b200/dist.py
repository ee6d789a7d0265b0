"""KV-head sharding over torch.distributed.

torch.distributed is plumbing here: it launches one process per GPU and
carries the 128-byte NCCL unique id from rank 0 to the others.  The
per-layer collectives run inside the library on its own NCCL communicator
(comm.cu); every rank then drives the same C-ABI calls.
"""
from __future__ import annotations

from typing import Optional

import paper_2602_23592_b200 as kb


def share_nccl_id(group=None) -> bytes:
    """Rank 0 creates the NCCL unique id; every rank of `group` receives it."""
    import torch.distributed as dist
    obj = [kb.comm_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return obj[0]


def sharded_context(L: int, H: int, d: int, mlp: int, V: int, seed: int, numerics: int = kb.FAST,
                    device: Optional[int] = None, group=None) -> kb.Context:
    """One context per rank of `group` (default: the world), each owning
    H / world heads; a single-process world gives the plain 1-GPU context."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if device is None:
        import os
        device = int(os.environ.get("LOCAL_RANK", 0))
    if world == 1:
        return kb.Context(L, H, d, mlp, V, seed, numerics, device=device)
    nid = share_nccl_id(group)
    return kb.Context(L, H, d, mlp, V, seed, numerics, device=device, world=world, rank=rank, nccl_id=nid)
