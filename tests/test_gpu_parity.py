"""GPU parity: the CUDA path (through the C-ABI) against the reference's golden
fixtures and the CPU oracle.  Bit-exact: hit lists, dense scores, l,
skipped, error messages, built files."""
import json
import os
import random

import numpy as np
import pytest

import paper_1905_09624_b200 as cb
from oracle import oracle as O

pytestmark = pytest.mark.gpu
GDIR = os.path.join(os.path.dirname(__file__), "golden")


def rand(rng, n, alphabet=b"ACGT"):
    return bytes(rng.choice(alphabet) for _ in range(n))


def gpu_hits(view, b, i):
    d, s = b.hits(i)
    return [[int(x), int(y)] for x, y in zip(d, s)]


def test_golden_fixtures(gpu):
    g = json.load(open(os.path.join(GDIR, "golden.json")))
    for name, spec in g["files"].items():
        path = os.path.join(GDIR, name + ".cobs")
        view = cb.open_resident(path, gpu)
        res = g["results"][name]
        # batch every (pattern, K, top_t) group through one call per (K, top_t)
        groups = {}
        for r in res:
            groups.setdefault((r["K"], r["top_t"]), []).append(r)
        for (K, top_t), rs in groups.items():
            b = cb.query_batch(view, [r["pat"].encode() for r in rs], K, top_t)
            for i, r in enumerate(rs):
                if "error" in r:
                    assert b.status[i] == r["error"] and b.messages[i] == r["msg"], (name, r)
                else:
                    assert b.status[i] == 0
                    assert (int(b.ell[i]), int(b.skipped[i])) == (r["ell"], r["skipped"])
                    assert gpu_hits(view, b, i) == r["hits"], (name, r["pat"], K, top_t)
        # the GPU build reproduces the reference's file byte for byte
        docs = [(d[0].encode(), [s.encode() for s in d[1]]) for d in spec["docs"]]
        p = dict(spec["params"])
        kind = p.pop("kind")
        params = cb.IndexParams(**{k: v for k, v in p.items()})
        assert cb.build_image(docs, params, kind, device=gpu) == open(path, "rb").read(), name
        view.close()


def test_query_api_mirror(gpu):
    view = cb.open_resident(os.path.join(GDIR, "classic_k2.cobs"), gpu)
    with pytest.raises(ValueError, match=r"query: K must be in \(0,1\]"):
        cb.query(view, b"A" * 40, cb.QueryOptions(K=0.0))
    with pytest.raises(ValueError):
        cb.query(view, b"A" * 40, cb.QueryOptions(K=1.5))
    with pytest.raises(cb.DataError, match="pattern shorter than q = 31"):
        cb.query(view, b"ACGT")
    r = cb.query(view, b"ACGT" * 20, cb.QueryOptions(K=1e-12))
    assert r.ell > 0
    assert view.params().k == 2 and view.kind() == cb.KIND_CLASSIC


def corpus(rng, n, lo, hi, noisy=False, alphabet=b"ACGT"):
    docs = []
    for i in range(n):
        a = alphabet + b"N" if noisy and i % 4 == 0 else alphabet
        segs = [rand(rng, rng.randint(lo, hi), a) for _ in range(1 + (i % 3 == 0))]
        if i % 7 == 6:
            segs.append(b"")  # empty content string
        docs.append((b"doc%04d" % i, segs))
    return docs


CASES = [
    # (q, k, p, canonical, kind, block_size, alphabet)
    (31, 1, 0.3, False, 0, 1024, b"ACGT"),
    (31, 2, 0.3, True, 1, 4, b"ACGT"),
    (31, 3, 0.3, False, 1, 3, b"ACGT"),
    (10, 2, 0.1, False, 0, 1024, b"ACDEFGHIKLMNPQRSTVWY"),
    (33, 1, 0.25, True, 1, 5, b"ACGT"),     # q >= 32: XXH64 stripe path
    (5, 2, 0.3, False, 1, 2, b"ACGT"),      # tiny q: heavy duplication
    (31, 1, 0.3, False, 1, 1, b"ACGT"),     # one document per block
]


@pytest.mark.parametrize("case", CASES)
def test_random_corpora_scores_and_hits(gpu, case):
    q, k, p, canonical, kind, B, alphabet = case
    rng = random.Random(hash(case) & 0xFFFFFFF)
    docs = corpus(rng, 37, 20, 3000, noisy=canonical, alphabet=alphabet)
    img = O.build_image(docs, q=q, k=k, p=p, canonical=canonical, block_size=B, kind=kind)
    params = cb.IndexParams(q=q, k=k, p=p, canonical=canonical, block_size=B)
    assert cb.build_image(docs, params, kind, device=gpu) == img
    idx = O.OracleIndex.parse(img)
    view = cb.open_image(img, gpu)
    pats = []
    for i in range(40):
        if i % 4 == 0:
            pats.append(rand(rng, rng.randint(0, 400), alphabet))
        else:
            src = docs[i % len(docs)][1][0]
            ln = min(len(src), rng.randint(q, 600))
            st = rng.randrange(len(src) - ln + 1)
            pat = bytearray(src[st:st + ln])
            if i % 5 == 0 and len(pat) > 3:
                pat[len(pat) // 2] = ord("N")
            if i % 9 == 0:
                pat = pat.lower()
            pats.append(bytes(pat))
    for K, top_t in [(1e-12, 0), (0.5, 0), (0.9, 3), (1.0, 0)]:
        b = cb.query_batch(view, pats, K, top_t, scores=True)
        for i, pat in enumerate(pats):
            try:
                ell, sk, hits, dense = idx.query(pat, K, top_t, scores=True)
            except O.OracleError as e:
                assert (b.status[i], b.messages[i]) == (e.code, e.msg)
                continue
            assert b.status[i] == 0
            assert (int(b.ell[i]), int(b.skipped[i])) == (ell, sk)
            assert gpu_hits(view, b, i) == [list(h) for h in hits]
            assert np.array_equal(b.dense[i].astype(np.uint32), dense), (i, K)
    view.close()


def test_long_and_repetitive_patterns(gpu):
    """Global-memory dedup sets (> 4096 windows), heavy duplication, and the
    uint32 counter path at l > 65535 (test_query.cpp:207-234)."""
    rng = random.Random(29)
    big = rand(rng, 70000)
    docs = [(b"big", [big]), (b"small", [rand(rng, 500)]), (b"rep", [b"ACGT" * 3000])]
    img = O.build_image(docs)
    idx = O.OracleIndex.parse(img)
    view = cb.open_image(img, gpu)
    pats = [big, big[1000:41000], b"ACGT" * 5000, b"A" * 9000, rand(rng, 12000),
            (b"ACGTTGCA" * 800)[:6000]]
    b = cb.query_batch(view, pats, 1e-12, scores=True)
    names = view.doc_names()
    for i, pat in enumerate(pats):
        ell, sk, hits, dense = idx.query(pat, 1e-12, scores=True)
        assert int(b.ell[i]) == ell
        assert np.array_equal(b.dense[i].astype(np.uint32), dense)
        assert gpu_hits(view, b, i) == [list(h) for h in hits]
    assert b.dense.dtype == np.uint32  # > 65535 windows in the batch
    r = cb.query(view, big, cb.QueryOptions(K=1.0))
    assert r.hits[0].doc_name == b"big" and r.hits[0].score == r.ell > 65535
    b2 = cb.query_batch(view, [big[1000:41000]], 0.9)
    ell, sk, hits, _ = idx.query(big[1000:41000], 0.9)
    assert gpu_hits(view, b2, 0) == [list(h) for h in hits]
    view.close()


def test_write_index_roundtrip(gpu, tmp_path):
    for name in ("classic_k2", "compact_canon", "compact_k3", "tiny"):
        src = os.path.join(GDIR, name + ".cobs")
        view = cb.open_resident(src, gpu)
        out = str(tmp_path / (name + ".cobs"))
        cb.write_index(view, out)
        assert open(out, "rb").read() == open(src, "rb").read()
        for b in range(view.block_count()):
            idx = O.OracleIndex.parse(open(src, "rb").read())
            rb = view.row_bytes(b)
            blk = idx.blocks()[b]
            assert view.doc_count(b) == blk[0] and view.width(b) == blk[1]
            assert len(view.row_data(b, 0)) == rb
        view.close()


def test_build_errors(gpu):
    with pytest.raises(cb.DataError, match="build: no documents"):
        cb.build_compact([], device=gpu)
    with pytest.raises(cb.DataError, match="duplicate document name: a"):
        cb.build_classic([(b"a", [b"A" * 40]), (b"b", []), (b"a", [])], device=gpu)
    # zero-term documents, forced width, multi-segment documents
    docs = [(b"e", []), (b"s", [b"ACG"]), (b"m", [b"A" * 40, b"C" * 35, b""])]
    for fw in (0, 7, 1):
        assert cb.build_classic(docs, forced_w=fw, device=gpu) == O.build_image(docs, forced_w=fw)
    assert cb.build_compact(docs, cb.IndexParams(block_size=2), device=gpu) == \
        O.build_image(docs, block_size=2, kind=1)


def test_c5_procedural_small(gpu):
    """Config-5 generator: device rows == host rows; header == oracle's
    (and hence the reference writer's, test_oracle_vs_ref.py); scores == the
    oracle over the procedural view."""
    from workloads import synth
    seed, n, B, med, sig, p = 7, 3000, 1024, 4000.0, 0.5, 0.3
    view = cb.synth_c5(seed, n, B, med, sig, p, device=gpu)
    orc = O.OracleIndex.c5(seed, n, B, med, sig, p)
    assert [(view.doc_count(b), view.width(b)) for b in range(view.block_count())] == \
        [(dc, w) for dc, w, _ in orc.blocks()]
    assert view.doc_names() == orc.names()
    tcs = orc.term_counts()
    for b, (dc, w, base) in enumerate(orc.blocks()):
        thr = synth.c5_thr16(w, max(tcs[base:base + dc]))
        for r in (0, 1, w // 2, w - 1):
            assert view.row_data(b, r) == synth.c5_row(seed, b, r, (dc + 7) // 8, thr, dc)
    rng = random.Random(5)
    pats = [rand(rng, 1000) for _ in range(8)]
    bres = cb.query_batch(view, pats, 1e-12, scores=True)
    for i, pat in enumerate(pats):
        ell, sk, hits, dense = orc.query(pat, 1e-12, scores=True)
        assert np.array_equal(bres.dense[i].astype(np.uint32), dense)
        assert gpu_hits(view, bres, i) == [list(h) for h in hits]
    view.close()


def test_build_device_resident(gpu):
    """cobs_gpu_build_ex: device-resident sequences in, queryable index out;
    its image equals the host-input build's and the oracle's."""
    import torch
    from workloads import synth
    cfg = synth.scaled(synth.CONFIGS["c3"], 150, len_scale=0.001, n_queries=20, block_size=32)
    lengths = synth.doc_lengths(cfg)
    dev = torch.empty(int(lengths.sum()), dtype=torch.uint8, device="cuda")
    cb.synth_docs_device(cfg.seed, cfg.alpha, lengths, dev.data_ptr())
    torch.cuda.synchronize()
    host, off = synth.docs(cfg, lengths=lengths)
    assert np.array_equal(dev.cpu().numpy(), host)  # device generator == host generator
    names = synth.doc_names(cfg)
    params = cb.IndexParams(q=cfg.q, k=cfg.k, p=cfg.p, canonical=cfg.canonical,
                            block_size=cfg.block_size)
    view, img = cb.build_device(dev.data_ptr(), off, np.arange(cfg.n_docs + 1), names, params,
                                cfg.kind, seqs_on_device=True, want_image=True)
    docs = [(names[i], [host[int(off[i]):int(off[i + 1])].tobytes()]) for i in range(cfg.n_docs)]
    want = O.build_image(docs, q=cfg.q, k=cfg.k, p=cfg.p, canonical=True, block_size=32, kind=1)
    assert img == want and cb.index_image(view) == want
    qb, qo = synth.queries(cfg, lengths=lengths)
    got = cb.query_batch_raw(view, qb, qo, 1e-12, scores=True)
    idx = O.OracleIndex.parse(want)
    ell, sk, st, nh, dense = idx.query_batch(qb, qo, 1e-12, scores=True)
    assert np.array_equal(got.dense.astype(np.uint32), dense)
    view.close()


@pytest.mark.parametrize("split", [35, 32])
def test_merge_classic(gpu, tmp_path, split):
    """acceptance.cpp criterion 9 on the device: merge of two forced-width
    builds == the single build, byte for byte, == the reference's merge."""
    rng = random.Random(4444 + split)
    docs = [(b"doc%04d" % i, [rand(rng, rng.randint(100, 8000))]) for i in range(60)]
    whole = cb.build_classic(docs, device=gpu)
    w = O.OracleIndex.parse(whole).blocks()[0][1]
    va, _ = cb.build_device(*_packed(docs[:split]), cb.IndexParams(), cb.KIND_CLASSIC, forced_w=w)
    vb, _ = cb.build_device(*_packed(docs[split:]), cb.IndexParams(), cb.KIND_CLASSIC, forced_w=w)
    merged = cb.merge_classic(va, vb)
    img = cb.index_image(merged)
    assert img == whole
    if O.ref_available():
        path = str(tmp_path / "m.cobs")
        O.ref_merge_write(docs, split, path, w)
        assert open(path, "rb").read() == img
    pats = [docs[i][1][0][:200] for i in range(0, 60, 7)]
    x = cb.query_batch(merged, pats, 0.7)
    y = O.OracleIndex.parse(whole)
    for i, p in enumerate(pats):
        ell, sk, hits, _ = y.query(p, 0.7)
        assert gpu_hits(merged, x, i) == [list(h) for h in hits]
    # error taxonomy of classic_index.cpp:96-106
    vc, _ = cb.build_device(*_packed(docs[split:]), cb.IndexParams(), cb.KIND_CLASSIC, forced_w=w + 1)
    with pytest.raises(cb.DataError, match=r"merge: widths differ \(%d vs %d\)" % (w, w + 1)):
        cb.merge_classic(va, vc)
    vd, _ = cb.build_device(*_packed(docs[split:]), cb.IndexParams(k=2), cb.KIND_CLASSIC, forced_w=w)
    with pytest.raises(cb.DataError, match="merge: index parameters differ"):
        cb.merge_classic(va, vd)
    with pytest.raises(cb.DataError, match="duplicate document name: doc0000"):
        cb.merge_classic(va, va)
    for v in (va, vb, vc, vd, merged):
        v.close()


def _packed(docs):
    names = [d[0] for d in docs]
    segs = [s for d in docs for s in d[1]]
    off = np.zeros(len(segs) + 1, np.uint64)
    np.cumsum([len(s) for s in segs], out=off[1:])
    doc_segs = np.zeros(len(docs) + 1, np.uint64)
    np.cumsum([len(d[1]) for d in docs], out=doc_segs[1:])
    buf = np.frombuffer(b"".join(segs), np.uint8) if segs else np.zeros(1, np.uint8)
    return buf, off, doc_segs, names


@pytest.mark.parametrize("from_file", [False, True], ids=["pinned", "file"])
@pytest.mark.parametrize("kind,frac", [(0, 0.9), (0, 0.7), (1, 1.05), (1, 1.5)])
def test_host_resident_streaming(gpu, tmp_path, kind, frac, from_file):
    """Out-of-core mode: with an HBM budget below the pitched payload the index
    stays in pinned host memory (or, from_file, is read from the file every
    batch: pread + repack into pinned group images) and batches stream it
    through two staging
    buffers (slabs of a block's slices, several blocks per group); results are
    identical to the resident index and the oracle; every batch copies the
    whole payload once."""
    from workloads import synth
    cfg = synth.scaled(synth.CONFIGS["c2"], 3000 if kind == 0 else 2600, len_scale=0.001,
                       n_queries=60, kind=kind, block_size=256, k=2)
    docs = [(n, [s]) for n, s in zip(synth.doc_names(cfg), _doc_bytes(cfg))]
    params = cb.IndexParams(q=cfg.q, k=cfg.k, p=cfg.p, block_size=cfg.block_size)
    img = cb.build_image(docs, params, kind, device=gpu)
    path = str(tmp_path / "i.cobs")
    open(path, "wb").write(img)
    res = cb.open_resident(path, gpu)
    pitched = res.device_bytes()
    # classic: a fraction of the payload (slabs split the block's slices);
    # compact: multiples of twice the largest block (several blocks per group)
    biggest = max(res.width(i) * ((res.row_bytes(i) + 31) // 32 * 32) for i in range(res.block_count()))
    budget = int(pitched * frac) if kind == 0 else int(2 * biggest * frac) + 4096
    budget = min(budget, pitched - 256)
    st = cb.open_random_access(path, budget, gpu, from_file=from_file)
    assert st.streaming() and not res.streaming()
    qb, qo = synth.queries(cfg)
    a = cb.query_batch_raw(res, qb, qo, 1e-12, scores=True)
    os.environ["COBS_ZC"] = "0"  # stream the whole payload
    try:
        b = cb.query_batch_raw(st, qb, qo, 1e-12, scores=True)
    finally:
        del os.environ["COBS_ZC"]
    assert np.array_equal(a.dense, b.dense)
    assert np.array_equal(a.ell, b.ell)
    payload = sum(st.width(i) * st.row_bytes(i) for i in range(st.block_count()))
    assert b.h2d_index_bytes == payload and a.h2d_index_bytes == 0
    assert (a.gather_path, b.gather_path) == (0, 2)
    modes = ["0"] if from_file else ["0", "1"]  # zero-copy needs the pinned copy
    for K, top_t in [(0.7, 0), (0.5, 4)]:
        x = cb.query_batch_raw(res, qb, qo, K, top_t)
        for zc in modes:
            os.environ["COBS_ZC"] = zc
            try:
                y = cb.query_batch_raw(st, qb, qo, K, top_t)
            finally:
                del os.environ["COBS_ZC"]
            assert y.gather_path == (1 if zc == "1" else 2)
            for i in range(len(qo) - 1):
                assert gpu_hits(res, x, i) == gpu_hits(st, y, i)
    if not from_file:  # zero-copy: dense scores too, and only the addressed rows cross PCIe
        os.environ["COBS_ZC"] = "1"
        try:
            c = cb.query_batch_raw(st, qb, qo, 1e-12, scores=True)
        finally:
            del os.environ["COBS_ZC"]
        assert np.array_equal(a.dense, c.dense) and c.h2d_index_bytes == c.row_bytes
        # the automatic choice: one query addresses a sliver of the payload
        one = cb.query_batch_raw(st, qb[:int(qo[1])], qo[:2], 0.5)
        assert one.gather_path == 1 and one.h2d_index_bytes == one.row_bytes
    idx = O.OracleIndex.parse(img)
    ell, sk, s_, nh, dense = idx.query_batch(qb, qo, 1e-12, scores=True)
    assert np.array_equal(b.dense.astype(np.uint32), dense)
    assert cb.index_image(st) == img and st.row_data(0, 3) == res.row_data(0, 3)
    res.close()
    st.close()


def _doc_bytes(cfg):
    from workloads import synth
    buf, off = synth.docs(cfg)
    return [buf[int(off[i]):int(off[i + 1])].tobytes() for i in range(cfg.n_docs)]


def test_streaming_budget_too_small(gpu, tmp_path):
    path = os.path.join(GDIR, "classic_k2.cobs")
    with pytest.raises(cb.DataError, match="more than half the budget"):
        cb.open_random_access(path, 1024, gpu)


def test_threshold_pruning_same_hits(gpu):
    """COBS_Q_PRUNE (stop reading a slice's rows once no document can reach
    tau) returns exactly the unpruned hit lists (which equal the oracle's)."""
    from workloads import synth
    for cfg in (synth.scaled(synth.CONFIGS["c1"], 300, len_scale=0.05, n_queries=300),
                synth.scaled(synth.CONFIGS["c2"], 400, len_scale=0.005, n_queries=200)):
        docs = [(n, [s]) for n, s in zip(synth.doc_names(cfg), _doc_bytes(cfg))]
        img = cb.build_image(docs, cb.IndexParams(q=cfg.q, k=cfg.k, p=cfg.p), 0, device=gpu)
        view = cb.open_image(img, gpu)
        qb, qo = synth.queries(cfg)
        idx = O.OracleIndex.parse(img)
        for K, top in [(cfg.K, 0), (0.95, 3), (0.5, 0)]:
            a = cb.query_batch_raw(view, qb, qo, K, top)
            b = cb.query_batch_raw(view, qb, qo, K, top, prune=True)
            assert np.array_equal(a.hit_n, b.hit_n)
            for i in range(len(qo) - 1):
                assert gpu_hits(view, a, i) == gpu_hits(view, b, i)
            for i in range(0, len(qo) - 1, 37):
                ell, sk, hits, _ = idx.query(qb[int(qo[i]):int(qo[i + 1])].tobytes(), K, top)
                assert gpu_hits(view, b, i) == [list(h) for h in hits]
        view.close()
    # config-5 shape: random queries, many slices pruned early
    view = cb.synth_c5(3, 5000, 1024, 30000.0, 0.5, 0.3, device=gpu)
    cfg = synth.replace(synth.CONFIGS["c5"], n_docs=5000, n_queries=500)
    qb, qo = synth.queries(cfg)
    pats = [qb[int(qo[i]):int(qo[i + 1])].tobytes() for i in range(len(qo) - 1)]
    pats[7] = pats[7][:40]  # a short pattern: small l, tau reachable
    a = cb.query_batch(view, pats, 0.8)
    b = cb.query_batch_raw(view, *cb.pack_patterns(pats), 0.8, prune=True)
    assert np.array_equal(a.hit_n, b.hit_n) and np.array_equal(a.docs, b.docs)
    assert np.array_equal(a.scores, b.scores)
    view.close()


def test_build_from_termsets(gpu, tmp_path):
    """build_classic / build_compact over TermSets given directly (the
    reference's own input type): terms hashed as given -- including
    duplicates, unsorted order and non-canonical or non-ACGT terms under
    canonical params -- and term_count = len(terms); files byte-identical to
    the reference's; the reference's term-length error, first failing
    document in its order."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    rng = random.Random(77)
    for q, k, canonical in ((31, 1, False), (31, 3, True), (12, 2, False), (5, 1, True)):
        docs = [(b"d%03d" % i, [rand(rng, rng.randrange(0, 400))]) for i in range(150)]
        ts = []
        for name, content in docs:
            terms, _, _ = O.ref_extract_terms(content, q, canonical)
            ts.append((name, terms))
        # user-made TermSets: duplicates, shuffled, odd bytes, non-canonical
        odd = [rand(rng, q, b"ACGTN") for _ in range(30)] + [rand(rng, q, b"acgt") for _ in range(5)]
        ts.append((b"odd", odd + odd[:7]))
        ts.append((b"empty", []))
        shuffled = list(ts[3][1])
        rng.shuffle(shuffled)
        ts.append((b"shuf", shuffled + shuffled[:3]))
        params = cb.IndexParams(q=q, k=k, canonical=canonical, block_size=32)
        for kind in (cb.KIND_CLASSIC, cb.KIND_COMPACT):
            path = str(tmp_path / f"t{q}{k}{kind}.cobs")
            O.ref_build_terms_write(ts, path, q=q, k=k, canonical=canonical, block_size=32, kind=kind)
            got = cb.build_from_terms(ts, params, kind, device=gpu)
            assert got == open(path, "rb").read(), (q, k, canonical, kind)
    # term length != q: classic reports the first bad document in input
    # order (before the name check); compact in (term_count, name) order
    # after the name check
    bad = [(b"z", [b"A" * 31, b"C" * 30]), (b"a", [b"G" * 31] * 3 + [b"T" * 32]), (b"m", [b"A" * 31])]
    for kind in (cb.KIND_CLASSIC, cb.KIND_COMPACT):
        with pytest.raises(O.OracleError) as want:
            O.ref_build_terms_write(bad, str(tmp_path / "bad.cobs"), kind=kind)
        with pytest.raises(ValueError) as got:
            cb.build_from_terms(bad, cb.IndexParams(), kind, device=gpu)
        assert want.value.code == 1
        assert str(got.value) == want.value.msg, kind
    dup = bad + [(b"z", [b"A" * 31])]
    for kind in (cb.KIND_CLASSIC, cb.KIND_COMPACT):
        with pytest.raises(O.OracleError) as want:
            O.ref_build_terms_write(dup, str(tmp_path / "dup.cobs"), kind=kind)
        with pytest.raises((ValueError, cb.DataError)) as got:
            cb.build_from_terms(dup, cb.IndexParams(), kind, device=gpu)
        assert str(got.value) == want.value.msg, kind


def _build_env(docs, params, kind, **env):
    env.setdefault("COBS_COUNT_PARTITION", 1)  # these corpora are below the size threshold
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        return cb.build_image(docs, params, kind, device=0)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def test_count_partitioned_vs_hashset(gpu):
    """The partitioned distinct count (q <= 32) against the hash-set count and
    the oracle: repetitive documents (one bucket full of duplicates), empty and
    short documents, multi-segment documents, several waves (a small key
    buffer), a document larger than the buffer (hash-set fallback) and
    non-ACGT windows without canonicalisation (wave recounted)."""
    rng = random.Random(404)
    docs = [(b"r%03d" % i, [rand(rng, rng.choice([0, 20, 31, 500, 5000, 60000]))]) for i in range(60)]
    docs += [(b"polyA", [b"A" * 200000]), (b"period7", [b"ACGTTGA" * 40000]),
             (b"multi", [rand(rng, 3000), b"", rand(rng, 40), rand(rng, 9000)]),
             (b"big", [rand(rng, 400000)])]
    with_n = docs + [(b"withN", [rand(rng, 2000) + b"N" + rand(rng, 2000)])]
    for q, canonical in ((31, False), (31, True), (20, False), (32, True)):
        params = cb.IndexParams(q=q, canonical=canonical, block_size=16)
        for corpus in (docs, with_n):
            want = O.build_image(corpus, q=q, canonical=canonical, block_size=16, kind=1)
            assert _build_env(corpus, params, cb.KIND_COMPACT) == want, (q, canonical)
            assert _build_env(corpus, params, cb.KIND_COMPACT, COBS_COUNT_PARTITION=0) == want
            # fingerprint sets capped too small (every wave recounted), and
            # small buckets (many per document, keys staged per bucket)
            assert _build_env(corpus, params, cb.KIND_COMPACT, COBS_PC_SLOTS_CAP=256) == want
            assert _build_env(corpus, params, cb.KIND_COMPACT, COBS_PC_TARGET=512) == want
            assert _build_env(corpus, params, cb.KIND_COMPACT, COBS_PC_DD_NBUF=2, COBS_PC_DEDUP_THREADS=512) == want
            # dedup variants: keys staged in shared memory (one / two buffers), the per-key probe loop
            assert _build_env(corpus, params, cb.KIND_COMPACT, COBS_PC_DD_STAGE=1) == want
            assert _build_env(corpus, params, cb.KIND_COMPACT, COBS_PC_DD_STAGE=1, COBS_PC_DD_NBUF=2,
                              COBS_PC_DEDUP_THREADS=512) == want
            assert _build_env(corpus, params, cb.KIND_COMPACT, COBS_PC_DD_FAST=0) == want
            assert _build_env(corpus, params, cb.KIND_COMPACT, COBS_PC_DD_FAST=0, COBS_PC_DD_STAGE=1) == want
            assert _build_env(corpus, params, cb.KIND_COMPACT, COBS_PC_DD_STAGE=1, COBS_PC_FP_MASK=0x30000) == want
            # 2-bit fingerprints: most probes meet accidental matches and compare whole keys
            assert _build_env(corpus, params, cb.KIND_COMPACT, COBS_PC_FP_MASK=0x30000) == want
            # waves of <= 150,000 keys: many waves, and "big"/"polyA" exceed one
            assert _build_env(corpus, params, cb.KIND_COMPACT, COBS_PC_WAVE_KEYS=150000) == want
            # without the up-front byte scan: the wave holding "withN" is
            # recounted by the hash sets after the partitioned pass flags it
            assert _build_env(corpus, params, cb.KIND_COMPACT, COBS_PC_NO_SCAN=1,
                              COBS_PC_WAVE_KEYS=150000) == want


def test_count_workspace_cache_and_trim(gpu):
    """The partitioned count keeps its workspace between builds (cobs_gpu_trim
    releases it; COBS_BUILD_CACHE=0 never keeps it); the files do not depend
    on whether a build starts from a cached, larger or smaller workspace."""
    rng = random.Random(5)
    small = [(b"s%02d" % i, [rand(rng, 3000)]) for i in range(10)]
    large = [(b"l%02d" % i, [rand(rng, 120000)]) for i in range(10)]
    params = cb.IndexParams(q=31, canonical=True, block_size=8)
    want_s = O.build_image(small, q=31, canonical=True, block_size=8, kind=1)
    want_l = O.build_image(large, q=31, canonical=True, block_size=8, kind=1)
    cb.trim()
    assert cb.trim() == 0
    assert _build_env(small, params, cb.KIND_COMPACT) == want_s
    assert _build_env(large, params, cb.KIND_COMPACT) == want_l   # grows the cached workspace
    assert _build_env(small, params, cb.KIND_COMPACT) == want_s   # reuses a larger one
    kept = cb.trim()
    assert kept >= 16 * sum(len(d[1][0]) - 30 for d in large)     # two 8-byte key buffers
    assert cb.trim() == 0
    assert _build_env(large, params, cb.KIND_COMPACT, COBS_BUILD_CACHE=0) == want_l
    assert cb.trim() == 0


def test_count_partitioned_symbol_codes(gpu):
    """Raw-byte corpora over a small alphabet (<= 32 byte values, q <= 12)
    take the partitioned count with 5-bit symbol codes (SymRoller): the same
    file as the oracle and as the hash-set count, for a protein corpus (the
    config-4 shape), DNA with N at q = 12, several waves; a corpus with more
    than 32 byte values stays on the hash sets."""
    rng = random.Random(77)
    prot = b"ACDEFGHIKLMNPQRSTVWY"
    cases = [
        (10, [(b"p%03d" % i, [rand(rng, rng.choice([0, 5, 10, 300, 4000]), prot)]) for i in range(50)]
         + [(b"rep", [b"MKV" * 3000]), (b"multi", [rand(rng, 500, prot), b"", rand(rng, 9, prot)])]),
        (12, [(b"n%03d" % i, [rand(rng, rng.choice([12, 800, 3000]), b"ACGTN")]) for i in range(40)]),
        (8, [(b"w%03d" % i, [bytes(rng.randrange(40, 120) for _ in range(600))]) for i in range(20)]),
    ]
    for q, docs in cases:
        params = cb.IndexParams(q=q, k=2, p=0.2, block_size=16)
        want = O.build_image(docs, q=q, k=2, p=0.2, block_size=16, kind=1)
        assert _build_env(docs, params, cb.KIND_COMPACT) == want, q
        assert _build_env(docs, params, cb.KIND_COMPACT, COBS_PC_SYMBOLS=0) == want, q
        assert _build_env(docs, params, cb.KIND_COMPACT, COBS_PC_WAVE_KEYS=3000) == want, q


def test_count_partitioned_huge_document(gpu):
    """A document with more buckets than a chunk histogram holds (> 8,192 x
    4,096 windows): buckets above the target size (larger sets)."""
    rng = np.random.default_rng(9)
    big = np.frombuffer(b"ACGT", np.uint8)[rng.integers(0, 4, 36_000_000)].tobytes()
    docs = [(b"huge", [big]), (b"small", [big[:5000]]), (b"mid", [big[1000:800000]])]
    params = cb.IndexParams(canonical=True)
    a = _build_env(docs, params, cb.KIND_CLASSIC)
    b = _build_env(docs, params, cb.KIND_CLASSIC, COBS_COUNT_PARTITION=0)
    assert a == b
    view = cb.open_image(a, 0)
    got = dict(view.doc(0, i) for i in range(view.doc_count(0)))
    view.close()
    if O.ref_available():  # term counts of the two smaller documents vs the reference
        for name, content in docs[1:]:
            terms, _, _ = O.ref_extract_terms(content, 31, True)
            assert got[name] == len(terms)


def test_block_shards(gpu, tmp_path):
    """Block sharding: shards opened with open_blocks answer
    the batch; merged by (score desc, name asc) and cut to top_t they equal
    the unsharded index, their dense scores concatenate to its dense scores,
    and a shard written out is the compact index of its blocks."""
    from paper_1905_09624_b200 import dist as D
    rng = random.Random(31)
    docs = [(b"s%04d" % rng.randrange(10000), [rand(rng, rng.randrange(50, 3000))]) for _ in range(70)]
    docs = list({n: (n, c) for n, c in docs}.values())
    params = cb.IndexParams(block_size=8, canonical=True)
    path = str(tmp_path / "sharded.cobs")
    img = cb.build_compact(docs, params, path=path, device=gpu)
    full = cb.open_resident(path, gpu)
    nb = full.block_count()
    cuts = [0, 2, 5, nb]
    shards = [cb.open_blocks(path, a, b, gpu) for a, b in zip(cuts, cuts[1:])]
    assert [s.column_offset() for s in shards] == [sum(full.doc_count(b) for b in range(c)) for c in cuts[:-1]]
    pats = [d[1][0][10:400] for d in docs[::5]] + [rand(rng, 300), b"ACG"]
    for K, top_t in ((0.3, 0), (0.3, 4), (1e-12, 0), (0.9, 1)):
        want = cb.query_batch(full, pats, K, top_t, scores=(top_t == 0))
        parts = [cb.query_batch(s, pats, K, top_t, scores=(top_t == 0)) for s in shards]
        flat = [D.flat_hits(r) for r in parts]
        hn, cols, sc = D.merge_hits([(h, c + s.column_offset(), x) for (h, c, x), s in zip(flat, shards)],
                                    D.name_ranks(full.doc_names()), top_t)
        w_hn, w_cols, w_sc = D.flat_hits(want)
        assert np.array_equal(hn, w_hn), (K, top_t)
        assert np.array_equal(cols, w_cols) and np.array_equal(sc, w_sc)
        for i in range(len(pats)):
            for r in parts:
                assert r.ell[i] == want.ell[i] and r.status[i] == want.status[i]
        if top_t == 0:
            assert np.array_equal(np.concatenate([r.dense for r in parts], axis=1), want.dense)
    # a shard is itself a compact index of its blocks
    idx = O.OracleIndex.parse(img)
    shard_img = cb.index_image(shards[1])
    sidx = O.OracleIndex.parse(shard_img)
    assert [(dc, w) for dc, w, _ in sidx.blocks()] == [(dc, w) for dc, w, _ in idx.blocks()[2:5]]
    lo = idx.blocks()[2][2]
    assert sidx.names() == idx.names()[lo:lo + len(sidx.names())]
    for b in range(3):
        for r in (0, shards[1].width(b) - 1):
            assert shards[1].row_data(b, r) == full.row_data(b + 2, r)
    # errors: empty / out-of-range block ranges, a classic index split
    for a, b in ((3, 3), (0, nb + 1), (nb, nb + 1)):
        with pytest.raises(ValueError, match="open_blocks"):
            cb.open_blocks(path, a, b, gpu)
    cpath = str(tmp_path / "classic.cobs")
    cb.build_classic(docs[:10], cb.IndexParams(), path=cpath, device=gpu)
    with pytest.raises(ValueError, match="open_blocks"):
        cb.open_blocks(cpath, 0, 2, gpu)
    cb.open_blocks(cpath, 0, 1, gpu).close()  # a classic index is one block: the whole index
    for s in shards:
        s.close()
    full.close()


def test_term_split_equals_warp_per_query(gpu):
    """Small batches split one query's terms over a CTA's 8 warps and add the
    bit-sliced counts (COBS_SPLIT=8); dense scores, l and hit lists are
    identical to the one-warp-per-query kernel (COBS_SPLIT=1), for k = 1..4
    and ℓ around the chunk sizes, and equal the oracle."""
    rng = random.Random(12)
    docs = [(b"t%03d" % i, [rand(rng, rng.randrange(100, 5000))]) for i in range(300)]
    for k, canonical in ((1, False), (2, True), (3, False), (4, False)):
        img = cb.build_compact(docs, cb.IndexParams(q=31, k=k, canonical=canonical, block_size=100), device=gpu)
        view = cb.open_image(img, gpu)
        idx = O.OracleIndex.parse(img)
        pats = [docs[rng.randrange(300)][1][0][:L] for L in (31, 32, 62, 63, 64, 95, 287, 288, 1000)
                if len(docs[0][1][0]) >= 0] + [rand(rng, 2000)]
        pats = [p for p in pats if len(p) >= 31]
        out = {}
        for split in ("1", "8"):
            os.environ["COBS_SPLIT"] = split
            try:
                out[split] = cb.query_batch(view, pats, 0.2, scores=True)
            finally:
                os.environ.pop("COBS_SPLIT", None)
        a, b = out["1"], out["8"]
        assert np.array_equal(a.dense, b.dense) and np.array_equal(a.ell, b.ell)
        assert np.array_equal(a.hit_n, b.hit_n) and np.array_equal(a.docs, b.docs)
        assert np.array_equal(a.scores, b.scores)
        for i, p in enumerate(pats):
            e, s, h, dense = idx.query(p, 0.2, scores=True)
            assert np.array_equal(b.dense[i].astype(np.uint32), dense), (k, i)
        view.close()


def test_sub_batches_equal_one_batch(gpu):
    """A host batch larger than the device budget runs as consecutive
    sub-batches (forced here with COBS_QUERY_BUDGET): hit lists, l, skipped,
    messages and dense scores -- including the 32-bit score width a single
    long pattern forces on the whole batch -- equal the one-batch answer."""
    rng = random.Random(21)
    docs = [(b"u%03d" % i, [rand(rng, rng.randrange(200, 3000))]) for i in range(120)]
    docs.append((b"long", [rand(rng, 70000)]))
    img = cb.build_compact(docs, cb.IndexParams(block_size=50), device=gpu)
    view = cb.open_image(img, gpu)
    pats = [docs[rng.randrange(len(docs))][1][0][:rng.randrange(20, 900)] for _ in range(60)]
    pats.insert(17, docs[-1][1][0][:66000])  # l > 65535: 32-bit scores for every query
    pats.insert(3, b"ACG")                    # DataError row
    one = cb.query_batch(view, pats, 0.3, 5, scores=True)
    os.environ["COBS_QUERY_BUDGET"] = "300000"
    try:
        split = cb.query_batch(view, pats, 0.3, 5, scores=True)
    finally:
        os.environ.pop("COBS_QUERY_BUDGET")
    assert split.launches > one.launches  # really ran as several sub-batches
    assert one.dense.dtype == split.dense.dtype == np.uint32
    assert np.array_equal(one.dense, split.dense)
    for f in ("ell", "skipped", "status", "hit_n"):
        assert np.array_equal(getattr(one, f), getattr(split, f)), f
    assert one.messages == split.messages
    for i in range(len(pats)):
        a, b = one.hits(i), split.hits(i)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    view.close()


def test_row_bytes_equal_reference_bytes_read(gpu, tmp_path):
    """The roofline's algorithmic bytes are the reference's own traffic
    accounting: the batch's row_bytes (k * sum(l) * sum_b row_bytes_b) equals
    the bytes the reference's random-access reader fetches for the same
    queries (bytes_read, storage.cpp:325-336; test_storage.cpp:157-190)."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    rng = random.Random(66)
    docs = [(b"b%03d" % i, [rand(rng, rng.randrange(100, 4000))]) for i in range(150)]
    path = str(tmp_path / "ra.cobs")
    for k, kind in ((1, cb.KIND_COMPACT), (3, cb.KIND_COMPACT), (2, cb.KIND_CLASSIC)):
        params = cb.IndexParams(k=k, block_size=40)
        cb.build_image(docs, params, kind, path=path, device=gpu)
        view = cb.open_resident(path, gpu)
        pats = [docs[rng.randrange(150)][1][0][:rng.randrange(31, 600)] for _ in range(25)] + [b"ACG"]
        ra = O.RefIndex.open(path, random_access=True)
        for p in pats:
            try:
                ra.query(p, 0.5)
            except O.OracleError:
                pass
        got = cb.query_batch(view, pats, 0.5)
        assert got.row_bytes == ra.bytes_read(), (k, kind)
        view.close()


def test_synth_c5_block_shards(gpu):
    """bench.py --shard blocks: block shards of the procedural config-5 index
    (synth_c5_blocks) hold exactly the full index's blocks, and their merged
    hit lists equal the unsharded index's (small instance)."""
    from paper_1905_09624_b200 import dist as D
    from workloads import synth
    cfg = synth.replace(synth.CONFIGS["c5"], n_docs=3000, block_size=256, c5_median=2e4, n_queries=64)
    args = (cfg.seed,)
    kw = dict(n_docs=cfg.n_docs, block_size=cfg.block_size, median=cfg.c5_median, sigma=cfg.c5_sigma, p=cfg.p)
    full = cb.synth_c5(cfg.seed, cfg.n_docs, cfg.block_size, cfg.c5_median, cfg.c5_sigma, cfg.p, device=gpu)
    nb = full.block_count()
    cuts = [0, 3, 7, nb]
    shards = [cb.synth_c5_blocks(*args, a, b, device=gpu, **kw) for a, b in zip(cuts, cuts[1:])]
    assert [s.column_offset() for s in shards] == [c * cfg.block_size for c in cuts[:-1]]
    for s, a in zip(shards, cuts):
        for b in range(s.block_count()):
            assert s.width(b) == full.width(a + b)
            for r in (0, s.width(b) // 2, s.width(b) - 1):
                assert s.row_data(b, r) == full.row_data(a + b, r)
    qb, qo = synth.queries(cfg)
    # random queries score only false positives (density ~0.3 per row), so
    # K around 0.3 gives a mix of hits and misses
    for K, top_t in ((0.3, 0), (0.32, 5), (1e-12, 3)):
        want = cb.query_batch_raw(full, qb, qo, K, top_t)
        parts = [cb.query_batch_raw(s, qb, qo, K, top_t) for s in shards]
        flat = [D.flat_hits(r) for r in parts]
        hn, cols, sc = D.merge_hits([(h, c + s.column_offset(), x) for (h, c, x), s in zip(flat, shards)],
                                    D.name_ranks(full.doc_names()), top_t)
        w_hn, w_cols, w_sc = D.flat_hits(want)
        assert np.array_equal(hn, w_hn), (K, top_t)
        assert np.array_equal(cols, w_cols) and np.array_equal(sc, w_sc)
        assert int(want.hit_n.sum()) > 0
    for v in shards + [full]:
        v.close()
