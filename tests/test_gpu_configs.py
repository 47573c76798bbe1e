"""The five BASELINE.json configs on the GPU.

* scaled instances of C1-C4 (same shapes, oracle-sized): the GPU build is
  byte-identical to the oracle's, and every query's dense scores, l,
  skipped and hit list equal the oracle's;
* full-size C1 against the reference itself (oracle/_ref) when present;
* full-size C5 (100,000 documents, ~100 GB in HBM): generated rows equal the
  host generator's, and a seeded sample of queries scores exactly as the
  oracle over the procedural index.
"""
import os
import random

import numpy as np
import pytest

import paper_1905_09624_b200 as cb
from oracle import oracle as O
from workloads import synth

pytestmark = pytest.mark.gpu


def corpus_docs(cfg):
    buf, off = synth.docs(cfg)
    names = synth.doc_names(cfg)
    return [(names[i], [buf[int(off[i]):int(off[i + 1])].tobytes()]) for i in range(cfg.n_docs)]


def check_config(cfg, n_hit_checks=40):
    docs = corpus_docs(cfg)
    params = cb.IndexParams(q=cfg.q, k=cfg.k, p=cfg.p, canonical=cfg.canonical,
                            block_size=cfg.block_size)
    img = cb.build_image(docs, params, cfg.kind, device=0)
    want = O.build_image(docs, q=cfg.q, k=cfg.k, p=cfg.p, canonical=cfg.canonical,
                         block_size=cfg.block_size, kind=cfg.kind)
    assert img == want, f"{cfg.name}: GPU build differs from the oracle"
    view = cb.open_image(img, 0)
    idx = O.OracleIndex.parse(img)
    qb, qo = synth.queries(cfg)
    # dense scores for every query (threshold-free), then hits at the config K
    got = cb.query_batch_raw(view, qb, qo, 1e-12, scores=True, hits=False)
    ell, sk, st, nh, dense = idx.query_batch(qb, qo, 1e-12, scores=True)
    assert np.array_equal(got.ell.astype(np.uint64), ell)
    assert np.array_equal(got.skipped, sk)
    assert np.array_equal(got.status, st)
    assert np.array_equal(got.dense.astype(np.uint32), dense), cfg.name
    hits = cb.query_batch_raw(view, qb, qo, cfg.K)
    rng = random.Random(cfg.n_docs)
    for i in rng.sample(range(len(qo) - 1), min(n_hit_checks, len(qo) - 1)):
        pat = qb[int(qo[i]):int(qo[i + 1])].tobytes()
        e, s, h, _ = idx.query(pat, cfg.K)
        d, sc = hits.hits(i)
        assert [(int(a), int(b)) for a, b in zip(d, sc)] == h, (cfg.name, i)
    view.close()
    return got, hits


def test_c1_scaled(gpu):
    cfg = synth.scaled(synth.CONFIGS["c1"], 60, len_scale=0.5, n_queries=200)
    check_config(cfg)


def test_c2_scaled(gpu):
    # k = 3, log-uniform lengths
    cfg = synth.scaled(synth.CONFIGS["c2"], 200, len_scale=0.01, n_queries=300)
    check_config(cfg)


def test_c3_scaled(gpu):
    # compact, canonical, B = 1024 (3 blocks), long indel queries (> 4096
    # windows: global-memory dedup sets)
    cfg = synth.scaled(synth.CONFIGS["c3"], 2100, len_scale=0.0005, n_queries=40)
    _, hits = check_config(cfg, n_hit_checks=20)


def test_c3_scaled_small_blocks(gpu):
    cfg = synth.scaled(synth.CONFIGS["c3"], 300, len_scale=0.002, n_queries=60, block_size=64)
    check_config(cfg)


def test_c4_scaled(gpu):
    # 20-letter alphabet, q = 10, k = 2, p = 0.1
    cfg = synth.scaled(synth.CONFIGS["c4"], 500, len_scale=0.01, n_queries=500)
    check_config(cfg)


def test_c1_full_vs_reference(gpu, tmp_path):
    """Full config 1 against the reference itself: the GPU-built file is
    byte-identical to the reference build_classic + write_index output, and
    all 1,000 queries score exactly as the reference query()."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    cfg = synth.CONFIGS["c1"]
    docs = corpus_docs(cfg)
    path = str(tmp_path / "c1.cobs")
    O.ref_build_write(docs, path, q=cfg.q, k=cfg.k, p=cfg.p)
    img = cb.build_classic(docs, cb.IndexParams(q=cfg.q, k=cfg.k, p=cfg.p), device=0)
    assert img == open(path, "rb").read()
    ref = O.RefIndex.open(path)
    view = cb.open_image(img, 0)
    qb, qo = synth.queries(cfg)
    got = cb.query_batch_raw(view, qb, qo, 1e-12, scores=True, hits=False)
    ell, sk, st, nh, dense = ref.query_batch(qb, qo, 0.0, scores=True)
    assert np.array_equal(got.ell.astype(np.uint64), ell)
    assert np.array_equal(got.dense.astype(np.uint32), dense)
    hits = cb.query_batch_raw(view, qb, qo, cfg.K)
    for i in range(0, cfg.n_queries, 25):
        pat = qb[int(qo[i]):int(qo[i + 1])].tobytes()
        e, s, h = ref.query(pat, cfg.K)
        d, sc = hits.hits(i)
        assert [(int(a), int(b)) for a, b in zip(d, sc)] == h
    # drawn queries hit their source document (no false negatives at 1% subst.)
    assert int((got.dense.max(axis=1)[0::2] > 0).sum()) == cfg.n_queries // 2
    view.close()


@pytest.mark.skipif(os.environ.get("COBS_SKIP_C5_FULL") == "1", reason="disabled")
@pytest.mark.parametrize("median", [None, 4.5e6], ids=["c5", "c5_literal_median"])
def test_c5_full_sample(gpu, median):
    """Full-size config 5 (~100 GB in HBM; and the literal 4.5 M median, a
    185 GB index): sampled rows equal the host generator; a seeded sample of
    the batch's queries scores exactly as the oracle over the procedural
    index."""
    cfg = synth.CONFIGS["c5"]
    if median:
        cfg = synth.replace(cfg, c5_median=median)
    view = cb.synth_c5(cfg.seed, cfg.n_docs, cfg.block_size, cfg.c5_median, cfg.c5_sigma, cfg.p)
    assert view.device_bytes() > (180e9 if median else 90e9)
    orc = O.OracleIndex.c5(cfg.seed, cfg.n_docs, cfg.block_size, cfg.c5_median, cfg.c5_sigma, cfg.p)
    blocks = orc.blocks()
    assert [(view.doc_count(b), view.width(b)) for b in range(view.block_count())] == \
        [(dc, w) for dc, w, _ in blocks]
    tcs = np.asarray(orc.term_counts())
    rng = random.Random(55)
    for _ in range(40):
        b = rng.randrange(len(blocks))
        dc, w, base = blocks[b]
        r = rng.randrange(w)
        thr = synth.c5_thr16(w, int(tcs[base:base + dc].max()))
        assert view.row_data(b, r) == synth.c5_row(cfg.seed, b, r, (dc + 7) // 8, thr, dc)
    # the seeded 1 % subsample of the batch (BASELINE.json config 5): dense
    # scores (threshold-free) and hit lists at K = 0.8
    ids = np.asarray(sorted(random.Random(0x1F).sample(range(cfg.n_queries), cfg.n_queries // 100)),
                     dtype=np.uint64)
    qb, qo = synth.queries(cfg, ids)
    got = cb.query_batch_raw(view, qb, qo, 1e-12, scores=True, hits=False)
    ell, sk, st, nh, dense = orc.query_batch(qb, qo, 1e-12, scores=True)
    assert np.array_equal(got.ell.astype(np.uint64), ell)
    assert np.array_equal(got.dense.astype(np.uint32), dense)
    hits = cb.query_batch_raw(view, qb, qo, cfg.K)
    tau = np.ceil(cfg.K * ell.astype(np.float64) - 1e-9).astype(np.int64)
    for i in range(len(ids)):
        want = int((dense[i] >= max(1, tau[i])).sum())
        assert int(hits.hit_n[i]) == want
    view.close()
