"""The C restatement (oracle/cobs_oracle.c) against the reference itself
(oracle/_ref: /root/reference/proj sources compiled unmodified).  Skipped
where oracle/_ref was not built (it needs /root/reference at build time)."""
import os
import random
import tempfile

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def rand_dna(rng, n, alphabet=b"ACGT"):
    return bytes(rng.choice(alphabet) for _ in range(n))


def test_xxh64_and_math_vs_ref():
    rng = random.Random(1)
    R = O.ref()
    for n in range(0, 70):
        data = bytes(rng.randrange(256) for _ in range(n))
        assert O.xxh64(data, n) == R.ref_xxh64(data, n, n)
    for _ in range(300):
        v, k, p = rng.randint(0, 10**7), rng.randint(1, 6), rng.uniform(0.001, 0.95)
        w = O._u64()
        assert R.ref_size_filter(v, p, k, O.C.byref(w)) == 0
        assert O.size_filter(v, p, k) == w.value
        ell, K = rng.randint(1, 100000), rng.choice([0.1, 0.3, 0.5, 0.7, 0.8, 0.9, 1.0, rng.random()])
        assert O.score_threshold(ell, K) == R.ref_score_threshold(ell, K)


def test_extract_terms_vs_ref():
    rng = random.Random(2)
    for trial in range(60):
        q = rng.choice([1, 2, 3, 5, 10, 31, 32, 33])
        canonical = trial % 2 == 1
        content = [rand_dna(rng, rng.randint(0, 200), b"ACGTN" if trial % 3 == 0 else b"ACGT")
                   for _ in range(rng.randint(1, 4))]
        assert O.extract_terms(content, q, canonical) == O.ref_extract_terms(content, q, canonical)


def corpus(rng, n, lo, hi, canonical_noise=False):
    docs = []
    for i in range(n):
        alphabet = b"ACGTN" if canonical_noise and i % 5 == 0 else b"ACGT"
        segs = [rand_dna(rng, rng.randint(lo, hi), alphabet) for _ in range(1 + (i % 3 == 0))]
        docs.append((b"doc%04d" % i, segs))
    return docs


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("k,canonical", [(1, False), (2, True), (3, False)])
def test_build_bytes_vs_ref(kind, k, canonical):
    rng = random.Random(10 * k + kind)
    docs = corpus(rng, 23, 40, 900, canonical_noise=canonical)
    img = O.build_image(docs, k=k, canonical=canonical, block_size=5, kind=kind)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "r.cobs")
        O.ref_build_write(docs, path, k=k, canonical=canonical, block_size=5, kind=kind)
        assert open(path, "rb").read() == img


def test_query_vs_ref():
    rng = random.Random(7)
    for trial, (kind, k, canonical) in enumerate([(0, 1, False), (1, 2, True), (1, 3, False),
                                                   (0, 2, True)]):
        docs = corpus(rng, 17, 60, 2500, canonical_noise=canonical)
        img = O.build_image(docs, k=k, canonical=canonical, block_size=4, kind=kind)
        idx = O.OracleIndex.parse(img)
        with tempfile.TemporaryDirectory() as d:
            path = os.path.join(d, "q.cobs")
            open(path, "wb").write(img)
            ref = O.RefIndex.open(path)
            for pat_i in range(12):
                if pat_i % 3 == 0:
                    pat = rand_dna(rng, 150)
                else:
                    src = docs[pat_i % len(docs)][1][0]
                    ln = min(len(src), 100 + pat_i * 40)
                    st = rng.randrange(len(src) - ln + 1)
                    pat = src[st:st + ln]
                if pat_i == 5:
                    pat = pat[:40] + b"N" + pat[41:]
                for K, top_t in [(1.0, 0), (0.5, 0), (1e-12, 0), (0.3, 3)]:
                    try:
                        want = ref.query(pat, K, top_t)
                    except O.OracleError as e:
                        with pytest.raises(O.OracleError) as e2:
                            idx.query(pat, K, top_t)
                        assert (e2.value.code, e2.value.msg) == (e.code, e.msg)
                        continue
                    ell, sk, hits, _ = idx.query(pat, K, top_t)
                    assert (ell, sk, hits) == want


def test_reader_rejection_vs_ref():
    rng = random.Random(3)
    docs = corpus(rng, 9, 40, 300)
    img = O.build_image(docs, k=2, block_size=3, kind=1)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "m.cobs")
        for trial in range(150):
            m = bytearray(img)
            if trial % 3 == 0:
                m = m[: rng.randrange(len(m))]
            else:
                pos = rng.randrange(min(len(m), 400))
                m[pos] = rng.randrange(256)
            open(path, "wb").write(bytes(m))
            try:
                O.RefIndex.open(path).close()
                ref_ok = True
            except O.OracleError as e:
                ref_ok, ref_msg = False, e.msg
            try:
                O.OracleIndex.parse(bytes(m), path)
                orc_ok = True
            except O.OracleError as e:
                orc_ok, orc_msg = False, e.msg
            assert ref_ok == orc_ok
            if not ref_ok:
                assert orc_msg == ref_msg


def test_c5_header_and_rows_vs_ref():
    # the config-5 procedural index: oracle header == reference writer's
    seed, n, B, med, sig, p = 99, 2500, 1024, 3000.0, 0.5, 0.3
    orc = O.OracleIndex.c5(seed, n, B, med, sig, p)
    ref = O.RefIndex.c5(seed, n, B, med, sig, p)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "c5.cobs")
        ref.write(path)
        data = open(path, "rb").read()
    head = orc.header()
    assert data[: len(head)] == head
    parsed = O.OracleIndex.parse(data)
    assert parsed.blocks() == orc.blocks()
    rng = random.Random(4)
    for _ in range(5):
        pat = rand_dna(rng, 300)
        a = orc.query(pat, 0.25, scores=True)
        b = parsed.query(pat, 0.25, scores=True)
        assert a[:3] == b[:3] and np.array_equal(a[3], b[3])


def test_q32_poly_t_vs_ref():
    """q = 32, raw bytes: T^32 repeated is one term (sort + unique over the
    term strings, termizer.cpp:120-127); the oracle's term counts and built
    file equal the reference's (the GPU edge test checks against these)."""
    T32 = b"T" * 32
    content = [b"T" * 40, T32 + b"N" + T32, b"G" * 33 + b"T" * 33]
    for c in content:
        assert O.extract_terms([c], 32, False) == O.ref_extract_terms([c], 32, False)
    assert len(O.extract_terms([b"T" * 40], 32, False)[0]) == 1
    docs = [(b"s%02d" % i, [c]) for i, c in enumerate(content)]
    img = O.build_image(docs, q=32, k=2, canonical=False, block_size=2, kind=1)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "q32.cobs")
        O.ref_build_write(docs, path, q=32, k=2, canonical=False, block_size=2, kind=1)
        assert open(path, "rb").read() == img
