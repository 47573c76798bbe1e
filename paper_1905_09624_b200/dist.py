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

Block sharding (an index larger than one GPU): every rank
opens a block range of the compact index (``open_blocks``) and answers the
whole batch; ``gather_block_shards`` brings the per-shard hit lists to rank 0
and ``merge_block_shards`` merges them per query by (score desc, name asc)
and cuts to top_t -- equal to the unsharded query (each shard's own top_t
suffices, the global top_t is a subset of their union).
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


def shard_hits(res, names, column_offset: int) -> dict:
    """One shard's batch result as a picklable payload: per query, hit file
    columns, scores and names (the tie-break key)."""
    n = len(res.hit_n)
    out = {"ell": np.asarray(res.ell), "status": np.asarray(res.status), "hits": []}
    for i in range(n):
        d, sc = res.hits(i)
        out["hits"].append([(int(x) + column_offset, int(y), names[int(x)]) for x, y in zip(d, sc)])
    return out


def merge_block_shards(shards: List[dict], top_t: int = 0) -> List[List[Tuple[int, int, bytes]]]:
    """Per query, the union of the shards' hits ordered by (score desc, name
    asc) (query.cpp:156-160) and truncated to top_t (0 = all); the shards of
    one index see the same l, skipped and status for every query."""
    n = len(shards[0]["hits"])
    for sh in shards[1:]:
        assert len(sh["hits"]) == n and np.array_equal(sh["ell"], shards[0]["ell"])
    merged = []
    for i in range(n):
        hits = [h for sh in shards for h in sh["hits"][i]]
        hits.sort(key=lambda h: (-h[1], h[2]))
        merged.append(hits[:top_t] if top_t else hits)
    return merged


def gather_block_shards(payload: dict, top_t: int = 0) -> Optional[List[List[Tuple[int, int, bytes]]]]:
    """Gather every rank's shard payload to rank 0 and merge there (the one
    exchange step of block sharding).  Returns the merged hits on rank 0,
    None elsewhere; without torch.distributed the payload alone is merged."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return merge_block_shards([payload], top_t)
    out: List[Optional[dict]] = [None] * dist.get_world_size()
    dist.gather_object(payload, out if dist.get_rank() == 0 else None, dst=0)
    if dist.get_rank() != 0:
        return None
    return merge_block_shards(out, top_t)
