"""Host-side plumbing of the b'-sharded multi-GPU path: the partition, the
NCCL unique-id broadcast through torch.distributed, and max-over-ranks timing.

The matvec and the collectives themselves run inside libheff (order B per shard, NCCL
all-gather of psi, all-reduce of the Lanczos scalars); this module only decides who owns
what and moves the 128-byte id.  Backend-agnostic so the CPU tests drive it with gloo.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(mR: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous equal b' block of rank `rank` (libheff's communicating shards require
    world | mR)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank}/{world}")
    if mR % world:
        raise ValueError(f"mR = {mR} is not divisible by world = {world}")
    nb = mR // world
    return rank * nb, (rank + 1) * nb


def broadcast_uid(uid: bytes | None, device=None, src: int = 0) -> bytes:
    """Broadcast rank `src`'s 128-byte ncclUniqueId to every rank (uid ignored elsewhere)."""
    t = torch.zeros(128, dtype=torch.uint8, device=device)
    if dist.get_rank() == src:
        if uid is None or len(uid) != 128:
            raise ValueError("rank src must pass a 128-byte uid")
        t.copy_(torch.frombuffer(bytearray(uid), dtype=torch.uint8))
    dist.broadcast(t, src)
    return bytes(t.cpu().tolist())


def max_over_ranks(x: float, device=None) -> float:
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def blocked_to_natural(blocked: torch.Tensor, P: int) -> torch.Tensor:
    """Layout map of the all-gather: [P][rows][nb] -> [rows][P*nb] (what libheff's
    relayout kernel computes on the device; used by tests as the reference)."""
    rows, nb = blocked.shape[1], blocked.shape[2]
    assert blocked.shape[0] == P
    return blocked.permute(1, 0, 2).reshape(rows, P * nb)
