"""Multi-GPU plumbing for the query path (torch.distributed).

The COBS query path shards without a data-path collective:
every GPU holds a replica of an index that fits one GPU and answers its own
queries.  Two modes:
  * weak scaling (bench.py): rank r answers its own batch, query ids
    [r*n, (r+1)*n);
  * one batch split over ranks (``shard_range``): contiguous query ranges,
    results merged on rank 0 in query order by ``gather_results`` -- the only
    exchange, a small hit-list gather.
Timing is the max over ranks (``reduce_max``).
"""
from __future__ import annotations

from typing import List, Optional, Tuple

import numpy as np


def shard_range(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [lo, hi) share of n items for `rank` (sizes differ by <= 1)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def weak_query_ids(n_per_rank: int, rank: int) -> np.ndarray:
    return np.arange(rank * n_per_rank, (rank + 1) * n_per_rank, dtype=np.uint64)


def _t(x, device):
    import torch
    return torch.tensor(x, device=device, dtype=torch.float64)


def reduce_max(value: float, device="cpu") -> float:
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return value
    t = _t([float(value)], device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(value: float, device="cpu") -> float:
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return value
    t = _t([float(value)], device)
    dist.all_reduce(t)
    return float(t.item())


def gather_results(ell: np.ndarray, hit_n: np.ndarray, docs: np.ndarray, scores: np.ndarray,
                   doc_offset: int = 0) -> Optional[dict]:
    """Gather per-query (ell, hits) of contiguous query shards to rank 0, in
    rank (= query) order.  `docs` are this rank's hit columns, concatenated
    per query (hit_n[i] each); `doc_offset` shifts them to global columns
    (block sharding).  Returns the merged arrays on rank 0, None elsewhere."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return {"ell": ell, "hit_n": hit_n, "docs": docs + doc_offset, "scores": scores}
    payload = {"ell": np.asarray(ell), "hit_n": np.asarray(hit_n),
               "docs": np.asarray(docs, np.int64) + doc_offset, "scores": np.asarray(scores)}
    out: List[Optional[dict]] = [None] * dist.get_world_size()
    dist.gather_object(payload, out if dist.get_rank() == 0 else None, dst=0)
    if dist.get_rank() != 0:
        return None
    return {k: np.concatenate([o[k] for o in out]) for k in payload}
