"""Host-side plumbing of the data-parallel path.

One process per GPU.  Training points and test points are sharded across ranks; every
per-step exchange of the Lanczos loop (the m-length all-reduce of u = W_X q, the alpha,
reorthogonalisation-dot and beta^2 all-reduces) is issued by liblove.so itself over NCCL.
What lives here is only the host side around it: rank discovery, shard bounds, the
broadcast of the 128-byte NCCL unique id through the caller's process group, and the
max-over-ranks reduction of timings.  Everything takes the torch process group it runs in
(NCCL on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

import os
from typing import Optional, Tuple

import torch
import torch.distributed as dist


def env_rank_world() -> Tuple[int, int, int]:
    """(rank, local_rank, world) from the torchrun environment (defaults: one process)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def shard_bounds(n_global: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous, balanced [lo, hi) slice of n_global points owned by `rank` (the first
    n_global % world ranks get one extra point)."""
    if world < 1 or not 0 <= rank < world or n_global < 0:
        raise ValueError(f"bad shard request n={n_global} rank={rank} world={world}")
    base, extra = divmod(n_global, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def broadcast_bytes(payload: Optional[bytes], src: int = 0, group=None) -> bytes:
    """Broadcast a byte string from `src` to every rank of the group."""
    obj = [payload if dist.get_rank(group) == src else None]
    dist.broadcast_object_list(obj, src=src, group=group)
    out = obj[0]
    if not isinstance(out, (bytes, bytearray)):
        raise RuntimeError("broadcast_bytes: nothing received from the source rank")
    return bytes(out)


def nccl_id_for_group(group=None, make_id=None) -> bytes:
    """The NCCL unique id of liblove's communicator: rank 0 creates it
    (love_nccl_unique_id, or `make_id` in tests), every rank receives the same 128 bytes."""
    if dist.get_rank(group) == 0:
        if make_id is None:
            from .love import nccl_unique_id as make_id
        payload = make_id()
        if len(payload) != 128:
            raise RuntimeError("a NCCL unique id is 128 bytes")
    else:
        payload = None
    return broadcast_bytes(payload, 0, group)


def max_over_ranks(value: float, device: Optional[torch.device] = None, group=None) -> float:
    """Max of a per-rank scalar (the bench's step time is the slowest rank's)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sum_over_ranks(value: float, device: Optional[torch.device] = None, group=None) -> float:
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return float(t.item())
