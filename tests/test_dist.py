"""Multi-rank host logic on CPU with the gloo backend, world_size 2."""
import os
import random
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1905_09624_b200.dist import shard_range, weak_query_ids


def test_shard_range_partitions():
    for n in (0, 1, 7, 100, 101):
        for world in (1, 2, 3, 8):
            parts = [shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


def test_weak_ids_disjoint():
    a, b = weak_query_ids(5, 0), weak_query_ids(5, 1)
    assert set(a).isdisjoint(b) and len(a) == len(b) == 5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, img, pats, q):
    import torch.distributed as dist
    from oracle import oracle as O
    from paper_1905_09624_b200.dist import gather_results, reduce_max, shard_range
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # this rank's contiguous share of the batch; the CPU oracle stands in for
    # the per-rank engine (no GPU here) -- the merge logic is what is tested
    lo, hi = shard_range(len(pats), rank, world)
    idx = O.OracleIndex.parse(img)
    ell, hn, docs, scores = [], [], [], []
    for p in pats[lo:hi]:
        e, s, h, _ = idx.query(p, 0.5)
        ell.append(e)
        hn.append(len(h))
        docs += [d for d, _ in h]
        scores += [sc for _, sc in h]
    merged = gather_results(np.asarray(ell, np.uint64), np.asarray(hn, np.uint64),
                            np.asarray(docs, np.int64), np.asarray(scores, np.uint64))
    t = reduce_max(float(rank + 1))
    if rank == 0:
        q.put((merged, t))
    dist.destroy_process_group()


def test_two_rank_gather_equals_single_rank():
    from oracle import oracle as O
    rng = random.Random(3)
    docs = [(b"doc%04d" % i, [bytes(rng.choice(b"ACGT") for _ in range(rng.randint(100, 900)))])
            for i in range(15)]
    img = O.build_image(docs, k=2, block_size=4, kind=1)
    pats = [docs[i % 15][1][0][: 80 + i] for i in range(9)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_worker, args=(2, _free_port(), img, pats, q), nprocs=2, join=True,
                       start_method="spawn")
    merged, tmax = q.get(timeout=60)
    assert tmax == 2.0
    idx = O.OracleIndex.parse(img)
    want_docs, want_n = [], []
    for p in pats:
        e, s, h, _ = idx.query(p, 0.5)
        want_n.append(len(h))
        want_docs += [d for d, _ in h]
    assert list(merged["hit_n"]) == want_n
    assert list(merged["docs"]) == want_docs


def _shard_hits(idx, pats, K, top_t, col_lo, col_hi):
    """A block shard's answer (hit_n, global columns, scores), computed from
    the oracle's full-index hits restricted to the shard's columns and cut
    to top_t (what the shard's own engine returns)."""
    names = idx.names()
    hn, cols, scores = [], [], []
    for p in pats:
        e, s, h, _ = idx.query(p, K)
        mine = [(d, sc) for d, sc in h if col_lo <= d < col_hi]
        mine.sort(key=lambda x: (-x[1], names[x[0]]))
        mine = mine[:top_t] if top_t else mine
        hn.append(len(mine))
        cols += [d for d, _ in mine]
        scores += [sc for _, sc in mine]
    return np.asarray(hn, np.int64), np.asarray(cols, np.int64), np.asarray(scores, np.int64)


def _block_worker(rank, world, port, img, pats, top_t, q):
    import torch.distributed as dist
    from oracle import oracle as O
    from paper_1905_09624_b200.dist import gather_block_hits, name_ranks, shard_range
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    idx = O.OracleIndex.parse(img)
    blocks = idx.blocks()
    b_lo, b_hi = shard_range(len(blocks), rank, world)
    col_lo = blocks[b_lo][2]
    col_hi = blocks[b_hi - 1][2] + blocks[b_hi - 1][0]
    hn, cols, sc = _shard_hits(idx, pats, 0.3, top_t, col_lo, col_hi)
    merged = gather_block_hits(hn, cols, sc, name_ranks(idx.names()), top_t)
    if rank == 0:
        q.put(merged)
    dist.destroy_process_group()


def test_two_rank_block_shards_equal_unsharded():
    """Block sharding's one exchange (tensor all_gather, gloo here, NCCL on
    GPUs): rank r holds blocks shard_range(nb, r, 2) of a compact index; the
    rank-0 merge of the shard hit lists by (score desc, name asc), cut to
    top_t, equals querying the whole index."""
    from oracle import oracle as O
    rng = random.Random(8)
    docs = [(b"d%03d" % rng.randrange(1000), [bytes(rng.choice(b"ACGT") for _ in range(rng.randint(60, 700)))])
            for i in range(40)]
    docs = list({n: (n, c) for n, c in docs}.values())
    img = O.build_image(docs, block_size=6, kind=1)
    pats = [docs[i % len(docs)][1][0][:70 + 7 * i] for i in range(10)] + [b"ACGT" * 30]
    idx = O.OracleIndex.parse(img)
    for top_t in (0, 3):
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        mp.start_processes(_block_worker, args=(2, _free_port(), img, pats, top_t, q), nprocs=2, join=True,
                           start_method="spawn")
        hn, cols, sc = q.get(timeout=60)
        o = 0
        for i, p in enumerate(pats):
            _, _, want, _ = idx.query(p, 0.3, top_t)
            got = list(zip(cols[o:o + hn[i]].tolist(), sc[o:o + hn[i]].tolist()))
            o += int(hn[i])
            assert got == want, (top_t, i)
