"""Element sharding across ranks (sharded mode) and the
device-time reduction the bench reports.

Rank r of W owns the global element range [r n, (r+1) n) (weak scaling: n per
rank).  Every PRG draw is addressed by global index (elem_base), so the shards'
outputs are bit-identical to one call over the concatenated batch; no data
moves between ranks.  The timed region is bracketed by barriers and the
reported time is the maximum over ranks."""
from __future__ import annotations

import torch
import torch.distributed as dist


def elem_base(rank: int, n_per_rank: int) -> int:
    """Global index of the first element of `rank`'s shard (a multiple of 8 when
    n_per_rank is, as the C ABI requires)."""
    if n_per_rank % 8:
        raise ValueError("n per rank must be a multiple of 8 (elem_base alignment)")
    return rank * n_per_rank


def max_over_ranks(v: float, device="cpu") -> float:
    """The largest value of v over all ranks (1 rank: v itself)."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return v
    t = torch.tensor([v], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier() -> None:
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()
