"""The L2-tiled gather (csrc/tiled.cu: bucket_kernel + tile_kernel) against
the warp-per-(query, slice) gather_kernel and the CPU oracle.  Both compute
the reference's score_range (query.cpp:49-89); the tiled one only reorders
the row reads (row ranges in lockstep, counters in shared memory), so ell,
dense scores and ordered hit lists must be identical, bit for bit."""
import contextlib
import os
import random

import numpy as np
import pytest

import paper_1905_09624_b200 as cb
from oracle import oracle as O
from workloads import synth

pytestmark = pytest.mark.gpu


@contextlib.contextmanager
def env(**kv):
    old = {k: os.environ.get(k) for k in kv}
    os.environ.update({k: str(v) for k, v in kv.items()})
    try:
        yield
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def run(view, pats, K, top=0, scores=True, **kv):
    with env(**kv):
        return cb.query_batch_raw(view, *cb.pack_patterns(pats), K, top, scores=scores)


def same(a, b):
    for f in ("ell", "skipped", "status", "hit_n", "hit_off", "docs", "scores"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert a.messages == b.messages
    if a.dense is not None or b.dense is not None:
        assert a.dense.dtype == b.dense.dtype and np.array_equal(a.dense, b.dense)


def rand(rng, n):
    return bytes(rng.choice(b"ACGT") for _ in range(n))


def c5_patterns(seed, n, rng):
    cfg = synth.replace(synth.CONFIGS["c5"], n_docs=100, n_queries=n, seed=seed)
    qb, qo = synth.queries(cfg)
    pats = [qb[int(qo[i]):int(qo[i + 1])].tobytes() for i in range(n)]
    # ragged edge cases: l = 0 (DataError), repeats (l << windows), short
    pats[3] = b"ACGT" * 5
    pats[11] = b"ACGT" * 250
    pats[17] = pats[17][:31]
    pats[23] = pats[23][:200]
    return pats


def test_tiled_equals_gather_c5_shape(gpu):
    """config-5 generator (procedural bits at density ~0.3), low K so most
    documents are hits: tiled == gather_kernel for dense scores and hit
    lists, across range sizes (many ranges / the 64-range cap), lags, CTA
    shapes and multi-wave batches."""
    view = cb.synth_c5(5, 6000, 1024, 20000.0, 0.5, 0.3, device=gpu)
    rng = random.Random(5)
    pats = c5_patterns(11, 2500, rng)
    ref = run(view, pats, 0.33, COBS_TILED=0)
    assert ref.gather_path == 0
    assert int(ref.hit_n.sum()) > 100000  # a big hit pool (overflow re-run exercised)
    for kv in (dict(), dict(COBS_TILE_SHIFT=10), dict(COBS_TILE_SHIFT=12, COBS_TILE_LAG=1),
               dict(COBS_TILE_LAG=5, COBS_TILE_WARPS=24), dict(COBS_TILE_QS=3),
               dict(COBS_TILE_QS=40, COBS_TILE_SHIFT=11)):
        t = run(view, pats, 0.33, COBS_TILED=1, **kv)
        assert t.gather_path == 1, kv
        same(ref, t)
    # hits only, top_t, another K
    a = run(view, pats, 0.31, top=5, scores=False, COBS_TILED=0)
    b = run(view, pats, 0.31, top=5, scores=False, COBS_TILED=1, COBS_TILE_SHIFT=11)
    assert b.gather_path == 1
    same(a, b)
    view.close()


def test_tiled_nt12_and_multi_slice_vs_oracle(gpu):
    """Built indexes (classic with 2,500 documents = 3 slices per row;
    compact canonical), queries up to 1,024 windows (12 bit planes), some
    drawn from documents: tiled == gather_kernel == the oracle."""
    rng = random.Random(9)
    for kind, canonical, ndocs, bs in ((cb.KIND_CLASSIC, False, 2500, 0), (cb.KIND_COMPACT, True, 1500, 256)):
        docs = [(b"d%05d" % i, [rand(rng, rng.randint(40, 400))]) for i in range(ndocs)]
        params = cb.IndexParams(q=31, k=1, p=0.3, canonical=canonical, block_size=bs or 1024)
        img = cb.build_image(docs, params, kind, device=gpu)
        view = cb.open_image(img, gpu)
        pats = []
        for i in range(300):
            if i % 3 == 0:
                d = docs[rng.randrange(ndocs)][1][0]
                pats.append(d[: rng.randint(31, len(d))])
            elif i % 3 == 1:
                pats.append(rand(rng, 1054))  # 1,024 windows -> 12 planes
            else:
                pats.append(rand(rng, rng.randint(0, 300)))
        a = run(view, pats, 0.2, COBS_TILED=0)
        b = run(view, pats, 0.2, COBS_TILED=1, COBS_TILE_SHIFT=10)
        assert b.gather_path == 1
        same(a, b)
        idx = O.OracleIndex.parse(img)
        for i in range(0, len(pats), 23):
            if b.status[i]:
                continue
            ell, sk, hits, dense = idx.query(pats[i], 0.2, scores=True)
            assert int(b.ell[i]) == ell
            assert np.array_equal(b.dense[i].astype(np.uint32), dense)
            d, s = b.hits(i)
            assert [(int(x), int(y)) for x, y in zip(d, s)] == hits
        view.close()


def test_tiled_not_used_when_ineligible(gpu):
    """k > 1, pruning and > 1,024 windows keep gather_kernel even when forced."""
    rng = random.Random(3)
    docs = [(b"d%03d" % i, [rand(rng, 300)]) for i in range(50)]
    img = cb.build_image(docs, cb.IndexParams(q=31, k=2, p=0.3), cb.KIND_CLASSIC, device=gpu)
    view = cb.open_image(img, gpu)
    assert run(view, [rand(rng, 100)] * 4, 0.5, COBS_TILED=1).gather_path == 0
    view.close()
    img = cb.build_image(docs, cb.IndexParams(q=31, k=1, p=0.3), cb.KIND_CLASSIC, device=gpu)
    view = cb.open_image(img, gpu)
    assert run(view, [rand(rng, 2000)] * 4, 0.5, COBS_TILED=1).gather_path == 0
    assert run(view, [rand(rng, 500)] * 4, 0.5, COBS_TILED=1).gather_path == 1
    with env(COBS_TILED=1):
        b = cb.query_batch_raw(view, *cb.pack_patterns([rand(rng, 500)] * 4), 0.5, prune=True)
    assert b.gather_path == 0
    view.close()
