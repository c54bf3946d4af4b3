"""(batch x head) sharding of the hot path over ranks.

(b, h) pairs are independent units (Eq. 1 is per head); a rank owns a
contiguous block of them.  There is no exchange on the data path.
"""
from __future__ import annotations


def bh_range(BH: int, rank: int, world: int, scaling: str = "weak") -> range:
    """(b*H+h) indices rank ``rank`` processes.

    weak   : every rank runs its own full batch of BH units, indices
             [rank*BH, (rank+1)*BH) of a world*BH virtual batch;
    strong : the BH units of one batch are split into contiguous blocks
             (BH must be divisible by world).
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
