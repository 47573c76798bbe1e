"""Multi-GPU plumbing for the query path (torch.distributed).

The COBS query path shards without a data-path collective:
every GPU holds a replica of an index that fits one GPU and answers its own
queries.  Modes:
  * weak scaling (bench.py default): rank r answers its own batch, query ids
    [r*n, (r+1)*n);
  * one batch split over ranks (``shard_range``): contiguous query ranges,
    results merged on rank 0 in query order by ``gather_results``;
  * block sharding (an index larger than one GPU; bench.py ``--shard
    blocks``): every rank holds a block range of the compact index
    (``open_blocks`` / ``synth_c5_blocks``) and answers the whole batch;
    ``gather_block_hits`` brings the per-shard hit lists to rank 0 and
    ``merge_hits`` merges them per query by (score desc, name asc) and cuts
    to top_t -- equal to the unsharded query (each shard applies top_t
    itself; the global top_t is a subset of the union).
The one exchange is a small hit-list gather, done with tensor collectives
(``all_gather`` of padded int64 tensors: NCCL on the GPU, gloo on CPU) --
no pickled objects.  Names never travel: rank 0 holds every document's name
rank (the tie-break key, from the full header).  Timing is the max over
ranks (``reduce_max``).
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import numpy as np


def shard_range(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [lo, hi) share of n items for `rank` (sizes differ by <= 1)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def weak_query_ids(n_per_rank: int, rank: int) -> np.ndarray:
    return np.arange(rank * n_per_rank, (rank + 1) * n_per_rank, dtype=np.uint64)


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def _t(x, device):
    import torch
    return torch.tensor(x, device=device, dtype=torch.float64)


def reduce_max(value: float, device="cpu") -> float:
    dist = _dist()
    if dist is None:
        return value
    t = _t([float(value)], device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(value: float, device="cpu") -> float:
    dist = _dist()
    if dist is None:
        return value
    t = _t([float(value)], device)
    dist.all_reduce(t)
    return float(t.item())


def all_gather_arrays(arrays: Sequence[np.ndarray], device="cpu") -> List[List[np.ndarray]]:
    """Every rank's `arrays` (int64-convertible, 1-D, any lengths): one
    all_gather of the lengths, then one all_gather per array of tensors
    padded to the longest.  Returns out[rank][i]."""
    import torch
    dist = _dist()
    arrays = [np.ascontiguousarray(np.asarray(a).astype(np.int64)) for a in arrays]
    if dist is None:
        return [arrays]
    world = dist.get_world_size()
    lens = torch.tensor([len(a) for a in arrays], dtype=torch.int64, device=device)
    all_lens = [torch.empty_like(lens) for _ in range(world)]
    dist.all_gather(all_lens, lens)
    all_lens = [l.cpu().numpy() for l in all_lens]
    out: List[List[np.ndarray]] = [[None] * len(arrays) for _ in range(world)]
    for i, a in enumerate(arrays):
        m = max(int(l[i]) for l in all_lens)
        buf = torch.zeros(max(m, 1), dtype=torch.int64, device=device)
        if len(a):
            buf[:len(a)] = torch.from_numpy(a).to(device)
        got = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(got, buf)
        for r in range(world):
            out[r][i] = got[r][:int(all_lens[r][i])].cpu().numpy()
    return out


def gather_results(ell: np.ndarray, hit_n: np.ndarray, docs: np.ndarray, scores: np.ndarray,
                   doc_offset: int = 0, device="cpu") -> Optional[dict]:
    """Gather per-query (ell, hits) of contiguous query shards to rank 0, in
    rank (= query) order.  `docs` are this rank's hit columns, concatenated
    per query (hit_n[i] each); `doc_offset` shifts them to global columns.
    Returns the merged arrays on rank 0, None elsewhere."""
    dist = _dist()
    docs = np.asarray(docs, np.int64) + doc_offset
    parts = all_gather_arrays([ell, hit_n, docs, scores], device)
    if dist is not None and dist.get_rank() != 0:
        return None
    keys = ("ell", "hit_n", "docs", "scores")
    return {k: np.concatenate([p[i] for p in parts]) for i, k in enumerate(keys)}


def merge_hits(parts: Sequence[Tuple[np.ndarray, np.ndarray, np.ndarray]], name_rank: np.ndarray,
               top_t: int = 0) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Union of the shards' hits of one batch, per query ordered by (score
    desc, name asc) (query.cpp:156-160; name_rank[col] = the column's rank
    in bytewise name order) and cut to top_t (0 = all).  Each part is
    (hit_n[n], global columns, scores) of one shard.  Returns (hit_n, cols,
    scores) of the merged lists, query-major."""
    n = len(parts[0][0])
    q = np.concatenate([np.repeat(np.arange(n, dtype=np.int64), np.asarray(hn, np.int64))
                        for hn, _, _ in parts]) if parts else np.zeros(0, np.int64)
    cols = np.concatenate([np.asarray(c, np.int64) for _, c, _ in parts])
    sc = np.concatenate([np.asarray(s, np.int64) for _, _, s in parts])
    order = np.lexsort((name_rank[cols], -sc, q))
    q, cols, sc = q[order], cols[order], sc[order]
    hit_n = np.bincount(q, minlength=n).astype(np.int64)
    if top_t:
        start = np.concatenate([[0], np.cumsum(hit_n)[:-1]])
        pos = np.arange(len(q)) - start[q]
        keep = pos < top_t
        q, cols, sc = q[keep], cols[keep], sc[keep]
        hit_n = np.minimum(hit_n, top_t)
    return hit_n, cols, sc


def flat_hits(res) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """A batch result's hit lists as (hit_n, columns, scores), query-major
    (each query's top_t-cut slice [hit_off, hit_off + hit_n) of its arrays)."""
    hn = np.asarray(res.hit_n, np.int64)
    off = np.asarray(res.hit_off, np.int64)
    if hn.sum() == 0:
        return hn, np.zeros(0, np.int64), np.zeros(0, np.int64)
    starts = np.repeat(off - np.concatenate([[0], np.cumsum(hn)[:-1]]), hn)
    idx = np.arange(int(hn.sum()), dtype=np.int64) + starts
    return hn, np.asarray(res.docs, np.int64)[idx], np.asarray(res.scores, np.int64)[idx]


def gather_block_hits(hit_n: np.ndarray, cols: np.ndarray, scores: np.ndarray, name_rank: np.ndarray,
                      top_t: int = 0, device="cpu") -> Optional[Tuple[np.ndarray, np.ndarray, np.ndarray]]:
    """Block sharding's one exchange: this rank's hit lists of the whole
    batch (global columns) to rank 0, merged there (``merge_hits``).
    Returns the merged (hit_n, cols, scores) on rank 0, None elsewhere."""
    dist = _dist()
    parts = all_gather_arrays([hit_n, cols, scores], device)
    if dist is not None and dist.get_rank() != 0:
        return None
    return merge_hits([tuple(p) for p in parts], name_rank, top_t)


def name_ranks(names: Sequence[bytes]) -> np.ndarray:
    """rank[col] of every document in bytewise name order (std::string <)."""
    order = sorted(range(len(names)), key=lambda i: names[i])
    r = np.empty(len(names), np.int64)
    r[np.asarray(order, np.int64)] = np.arange(len(names), dtype=np.int64)
    return r
