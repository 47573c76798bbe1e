"""Edge cases on the GPU against the oracle: empty batches, zero-window and
all-skipped patterns mixed with good ones, q = 1 / q > 32 / k = 5 (runtime-k
path), raw non-ASCII bytes, exact-integer thresholds, top_t beyond the hits."""
import random

import numpy as np
import pytest

import paper_1905_09624_b200 as cb
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def rb(rng, n, alphabet):
    return bytes(rng.choice(alphabet) for _ in range(n))


def check(img, pats, Ks=(1e-12, 0.5, 1.0), tops=(0, 2, 10**9)):
    view = cb.open_image(img, 0)
    idx = O.OracleIndex.parse(img)
    for K in Ks:
        for top in tops:
            b = cb.query_batch(view, pats, K, top, scores=True)
            for i, p in enumerate(pats):
                try:
                    ell, sk, hits, dense = idx.query(p, K, top, scores=True)
                except O.OracleError as e:
                    assert (int(b.status[i]), b.messages[i]) == (e.code, e.msg)
                    continue
                assert (int(b.ell[i]), int(b.skipped[i])) == (ell, sk)
                d, s = b.hits(i)
                assert [(int(x), int(y)) for x, y in zip(d, s)] == hits
                assert np.array_equal(b.dense[i].astype(np.uint32), dense)
    view.close()


def test_empty_batch(gpu):
    img = O.build_image([(b"a", [b"ACGT" * 20])])
    view = cb.open_image(img, 0)
    b = cb.query_batch(view, [], 0.5)
    assert len(b.ell) == 0 and len(b.docs) == 0
    view.close()


def test_mixed_error_and_good_patterns(gpu):
    rng = random.Random(1)
    docs = [(b"d%02d" % i, [rb(rng, 400, b"ACGT")]) for i in range(20)]
    for canonical in (False, True):
        img = O.build_image(docs, canonical=canonical, k=2)
        pats = [b"", b"ACGT", docs[3][1][0][:80], b"N" * 31, b"N" * 100 + docs[4][1][0][:60],
                docs[5][1][0][10:41], b"acgt" * 20, docs[6][1][0]]
        check(img, pats)


@pytest.mark.parametrize("q,k,alphabet,canonical", [
    (1, 1, b"ACGT", False), (2, 3, b"ACGTN", True), (31, 5, b"ACGT", False),
    (32, 2, b"ACGT", True), (40, 1, b"ACGT", True), (64, 2, b"ACGTN", False),
    (7, 2, bytes(range(256)), False), (12, 1, b"\x00\xffAC", False)])
def test_parameter_corners(gpu, q, k, alphabet, canonical):
    rng = random.Random(q * 100 + k)
    docs = [(b"doc%03d" % i, [rb(rng, rng.randint(0, 700), alphabet)]) for i in range(30)]
    img = O.build_image(docs, q=q, k=k, canonical=canonical, block_size=7, kind=1)
    assert cb.build_image(docs, cb.IndexParams(q=q, k=k, canonical=canonical, block_size=7), 1,
                          device=0) == img
    pats = []
    for i in range(24):
        src = docs[i][1][0]
        if i % 3 == 0 or len(src) < q:
            pats.append(rb(rng, rng.randint(0, 300), alphabet))
        else:
            st = rng.randrange(len(src) - q + 1)
            pats.append(src[st:st + rng.randint(q, 300)])
    check(img, pats)


def test_exact_integer_thresholds(gpu):
    """K * l an exact integer: tau must not be pushed up (bloom.cpp:120-123,
    test_bloom.cpp:256-265)."""
    rng = random.Random(9)
    base = rb(rng, 2000, b"ACGT")
    docs = [(b"x%d" % i, [base[: 100 * (i + 1)]]) for i in range(20)]
    img = O.build_image(docs)
    # patterns with l = 10, 20, 30, 100, 1000 distinct 31-mers
    pats = [base[:31 + ell - 1] for ell in (10, 20, 30, 100, 1000)]
    check(img, pats, Ks=(0.9, 0.1, 0.3, 0.7, 1.0), tops=(0,))


def test_forced_tag_collisions_stay_exact(gpu):
    """With the dedup tags narrowed to 2 bits (COBS_DEBUG_TAG_BITS, read per
    call), distinct byte-path terms collide on the tag all the time and the
    exact byte comparison must keep l, term counts and scores right."""
    import os
    rng = random.Random(77)
    docs = [(b"p%03d" % i, [rb(rng, rng.randint(50, 900), b"ACDEFGHIKLMNPQRSTVWY")]) for i in range(25)]
    dna = [(b"q%03d" % i, [rb(rng, rng.randint(50, 900), b"ACGTN")]) for i in range(25)]
    os.environ["COBS_DEBUG_TAG_BITS"] = "2"
    try:
        for corpus, q, canonical in [(docs, 10, False), (dna, 40, True), (dna, 31, False)]:
            img = O.build_image(corpus, q=q, k=2, canonical=canonical, block_size=6, kind=1)
            assert cb.build_image(corpus, cb.IndexParams(q=q, k=2, canonical=canonical, block_size=6), 1,
                                  device=0) == img
            pats = [corpus[i][1][0][: 60 + 10 * i] for i in range(len(corpus))]
            check(img, pats, Ks=(1e-12, 0.5), tops=(0,))
    finally:
        del os.environ["COBS_DEBUG_TAG_BITS"]


def test_tie_order_with_non_ascii_names(gpu, tmp_path):
    """Hit order (score desc, name asc) compares names as unsigned bytes
    (std::string <, query.cpp:156-160): names with bytes >= 0x80, prefixes
    of one another, all scoring the same -- the device order equals the
    reference's query() on the same file, with and without top_t.  (Build
    entry points take NUL-terminated names.)"""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    seq = b"ACGT" * 40 + b"TTGACA" * 20
    names = [b"\xff", b"\x80a", b"a\x01b", b"a", b"ab", b"A", b"\x7f", b"z\xc3\xa9", b"zz"]
    docs = [(n, [seq]) for n in names]
    path = str(tmp_path / "names.cobs")
    cb.build_compact(docs, cb.IndexParams(block_size=3), path=path, device=gpu)
    view = cb.open_resident(path, gpu)
    ref = O.RefIndex.open(path)
    for top_t in (0, 4):
        got = cb.query(view, seq[:120], cb.QueryOptions(K=0.5, top_t=top_t))
        _, _, want = ref.query(seq[:120], 0.5, top_t)
        all_names = view.doc_names()
        assert [(h.doc_name, h.score) for h in got.hits] == [(all_names[d], s) for d, s in want]
        assert len({h.score for h in got.hits}) == 1  # a genuine tie
    view.close()


@pytest.mark.parametrize("partition", ["0", "1"])
def test_q32_raw_poly_t_and_high_codes(gpu, partition):
    """q = 32 without canonicalisation: the poly-T 32-mer's 2-bit code is
    2^64-1 and G/T-leading codes have bit 63 set, so code keys would wrap to
    the empty marker / share the byte-path key space.  The reference dedups
    with sort + unique over the term bytes (termizer.cpp:120-127), so T^32
    is one term however often it occurs.  l, dense scores, hits and the
    built file bytes must equal the oracle on both count paths
    (COBS_COUNT_PARTITION=0/1, read per call)."""
    import os
    rng = random.Random(3232)
    T32 = b"T" * 32
    special = [b"T" * 40, T32 + b"N" + T32, b"G" * 33 + b"T" * 33, T32 + b"A" + T32 + b"N" + b"T" * 35,
               b"N".join(rb(rng, 40, b"GT") for _ in range(6))]
    docs = [(b"s%02d" % i, [s]) for i, s in enumerate(special)]
    docs += [(b"r%02d" % i, [rb(rng, rng.randint(32, 400), b"ACGTN" if i % 2 else b"GT"),
                              T32 * (i % 3)]) for i in range(20)]
    pats = special + [T32, T32 + T32, b"T" * 31, T32 + b"N" + T32 + b"G" * 40,
                      docs[7][1][0] + T32, rb(rng, 200, b"GTN")]
    os.environ["COBS_COUNT_PARTITION"] = partition
    try:
        for kind, block in ((0, 1024), (1, 6)):
            img = O.build_image(docs, q=32, k=2, canonical=False, block_size=block, kind=kind)
            params = cb.IndexParams(q=32, k=2, canonical=False, block_size=block)
            assert cb.build_image(docs, params, kind, device=0) == img
            idx = O.OracleIndex.parse(img)
            assert idx.term_counts()[idx.names().index(b"s00")] == 1  # T^40: nine windows, one term
            check(img, pats, Ks=(1e-12, 0.5, 1.0), tops=(0, 3))
    finally:
        del os.environ["COBS_COUNT_PARTITION"]


def test_hit_overflow_splits_batch(gpu):
    """More hits than one ordering pass may hold (CUB's int item count, the
    hit buffers): the batch is re-run in halves with identical answers
    (COBS_HIT_LIMIT lowers the limit per call for the test); a single
    pattern over the limit, or a device-input batch, is a usage error."""
    import os
    rng = random.Random(12)
    docs = [(b"h%03d" % i, [rb(rng, 400, b"ACGT")]) for i in range(60)]
    img = O.build_image(docs, k=1, block_size=16, kind=1)
    pats = [docs[i][1][0][:200] for i in range(0, 60, 3)] + [rb(rng, 150, b"ACGT") for _ in range(7)]
    view = cb.open_image(img, 0)
    want = cb.query_batch(view, pats, 1e-12, 5)
    os.environ["COBS_HIT_LIMIT"] = "100"   # each pattern hits ~every document
    try:
        got = cb.query_batch(view, pats, 1e-12, 5)
        for i in range(len(pats)):
            a, b = want.hits(i), got.hits(i)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
            assert want.ell[i] == got.ell[i]
        os.environ["COBS_HIT_LIMIT"] = "10"
        with pytest.raises(ValueError, match="hits of one pattern exceed one ordering pass"):
            cb.query_batch(view, pats[:2], 1e-12)
    finally:
        del os.environ["COBS_HIT_LIMIT"]
    view.close()
