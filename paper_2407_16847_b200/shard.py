"""(batch x head) sharding of the hot path over ranks.

(b, h) pairs are independent units (Eq. 1 is per head; sequences of a
batch are independent): a rank owns a contiguous block of them and there
is no exchange on the data path.  The only collectives are outside the timed
region: the max-over-ranks time and the gather of O for validation
(:func:`gather_and_check`), which bench.py and the world-size-2 gloo test share.
"""
from __future__ import annotations

from typing import Callable, Sequence


def bh_range(BH: int, rank: int, world: int, scaling: str = "strong") -> range:
    """(b*H+h) indices rank ``rank`` processes.

    strong : the BH units of one batch are split into contiguous blocks of
             BH / world (BH must be divisible by world) -- SURVEY §8(e);
    weak   : every rank runs its own full batch of BH units, indices
             [rank*BH, (rank+1)*BH) of a world*BH virtual batch.
    """
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if scaling == "weak":
        return range(rank * BH, (rank + 1) * BH)
    if scaling == "strong":
        if BH % world:
            raise ValueError(f"B*H={BH} not divisible by world={world}")
        per = BH // world
        return range(rank * per, (rank + 1) * per)
    raise ValueError(scaling)


def check_slices(world: int, per_rank: int, k: int = 2) -> list[int]:
    """Indices (into the gathered [world*per_rank] stack) re-checked against a one-device run:
    the first and last ``k // 2`` slices of every rank's block (at least ``k`` per rank)."""
    out = []
    for r in range(world):
        lo, hi = r * per_rank, (r + 1) * per_rank
        idx = list(range(lo, min(hi, lo + (k + 1) // 2))) + list(range(max(lo, hi - k // 2), hi))
        for i in idx:
            if i not in out:
                out.append(i)
    return out


def gather_and_check(O_local, recompute: Callable[[Sequence[int]], "object"], k: int = 2) -> dict:
    """Gather every rank's O shard ([per_rank, N, d], equal sizes) and compare slices of every
    rank's block BITWISE with ``recompute(indices)`` -- the same computation run by this rank
    alone on those global slice indices (SURVEY C-4: sharded == one device, no atomics, same
    per-(b, h) work).  Collective: every rank calls it; all ranks get the same verdict."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size()
    parts = [torch.empty_like(O_local) for _ in range(world)]
    dist.all_gather(parts, O_local.contiguous())
    full = torch.cat(parts)
    idx = check_slices(world, O_local.shape[0], k)
    ref = recompute(idx)
    ok = bool(torch.equal(full[idx].cpu(), ref.cpu()))
    flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=O_local.device)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    return {"bitwise_equal_to_one_device": bool(flag.item()), "slices_checked": idx,
            "gathered_slices": int(full.shape[0])}
