"""Process-group plumbing for the multi-GPU exchange.

One process per GPU (torchrun).  torch.distributed is used only to hand the
128-byte NCCL unique id from rank 0 to every rank and for barriers / the
max-over-ranks timing reduction; the exchange itself runs on the library's
own NCCL communicator (lmscale_init).
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env_rank_world():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def broadcast_bytes(payload: bytes | None, src: int = 0, group=None) -> bytes:
    """Broadcast a bytes object from ``src`` to all ranks (any backend)."""
    obj = [payload if dist.get_rank(group) == src else None]
    dist.broadcast_object_list(obj, src=src, group=group)
    return obj[0]


def share_nccl_id(make_id=None, group=None) -> bytes:
    """Rank 0 creates the NCCL id (lmscale_get_nccl_id); everyone receives it."""
    if make_id is None:
        from .lmscale import get_nccl_id as make_id
    rank = dist.get_rank(group)
    nid = make_id() if rank == 0 else None
    nid = broadcast_bytes(nid, 0, group)
    assert isinstance(nid, (bytes, bytearray)) and len(nid) == 128
    return bytes(nid)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (timing: the slowest rank defines the step)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def make_context(vocab, max_tokens, dim, flags=0, group=None):
    """Create this rank's lmscale Context inside an initialised process group."""
    from .lmscale import Context
    rank, world, local = dist.get_rank(group), dist.get_world_size(group), \
        int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    nid = share_nccl_id(group=group) if world > 1 else None
    return Context(vocab, max_tokens, dim, world=world, rank=rank, device=local, flags=flags,
                   nccl_id=nid)
