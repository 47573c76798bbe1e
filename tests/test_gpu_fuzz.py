"""Seeded fuzzing of the whole path against the CPU oracle: random index
parameters (q 1-40, k 1-4, p, canonical, classic/compact, block size), random
alphabets (DNA with N and lowercase, protein, arbitrary bytes), random
document and pattern shapes.  Every iteration: the GPU-built file equals the
oracle's byte for byte (with the default count and with the partitioned
count under random knobs), and the batch's l, skipped, status, dense scores
and ordered, top_t-cut hit lists equal the oracle's."""
import os
import random

import numpy as np
import pytest

import paper_1905_09624_b200 as cb
from oracle import oracle as O

pytestmark = pytest.mark.gpu

ALPHABETS = [b"ACGT", b"ACGTN", b"ACGTacgtN", b"ACDEFGHIKLMNPQRSTVWY", bytes(range(1, 256)), b"AC"]
ITERS = int(os.environ.get("COBS_FUZZ_ITERS", "40"))


def rbytes(rng, n, alphabet):
    return bytes(rng.choice(alphabet) for _ in range(n))


@pytest.mark.parametrize("it", range(ITERS))
def test_fuzz_build_and_query(gpu, it):
    rng = random.Random(0xC0B5 + it)
    q = rng.choice([1, 2, 5, 10, 16, 20, 31, 31, 32, 33, 40])
    k = rng.randint(1, 4)
    p = rng.choice([0.05, 0.1, 0.3, 0.5])
    canonical = rng.random() < 0.4
    kind = rng.randint(0, 1)
    B = rng.randint(1, 12)
    alphabet = rng.choice(ALPHABETS)
    n_docs = rng.randint(1, 30)
    names = rng.sample(range(10000), n_docs)
    docs = []
    for i in range(n_docs):
        segs = [rbytes(rng, rng.choice([0, rng.randint(1, 40), rng.randint(40, 900)]), alphabet)
                for _ in range(rng.randint(1, 3))]
        docs.append((b"f%04d" % names[i], segs))
    params = cb.IndexParams(q=q, k=k, p=p, canonical=canonical, block_size=B)
    img = cb.build_image(docs, params, kind, device=gpu)
    assert img == O.build_image(docs, q=q, k=k, p=p, canonical=canonical, block_size=B, kind=kind), \
        (it, q, k, canonical, kind, B)
    # the partitioned count (2-bit / symbol codes, fingerprint dedup sets) on
    # the same corpus, with random bucket sizes, narrowed fingerprints and
    # small waves -- the corpora are below its size threshold, so forced
    knobs = {"COBS_COUNT_PARTITION": "1", "COBS_PC_TARGET": str(rng.choice([64, 300, 4096])),
             "COBS_PC_FP_MASK": rng.choice(["0xffffffff", "0x30000", "0x0"]),
             "COBS_PC_WAVE_KEYS": str(rng.choice([2000, 1 << 30])),
             # dedup: straight-line first probes or the per-key loop, keys from global memory or staged
             "COBS_PC_DD_FAST": rng.choice(["1", "1", "0"]), "COBS_PC_DD_STAGE": rng.choice(["0", "0", "1"])}
    saved = {v: os.environ.get(v) for v in knobs}
    os.environ.update(knobs)
    try:
        assert cb.build_image(docs, params, kind, device=gpu) == img, (it, knobs)
    finally:
        for v, old in saved.items():
            if old is None:
                os.environ.pop(v, None)
            else:
                os.environ[v] = old
    view = cb.open_image(img, gpu)
    idx = O.OracleIndex.parse(img)
    pats = []
    for _ in range(rng.randint(1, 12)):
        d = docs[rng.randrange(n_docs)][1]
        src = d[rng.randrange(len(d))]
        if src and rng.random() < 0.7:
            a = rng.randrange(len(src))
            pats.append(src[a:a + rng.randint(1, 500)])
        else:
            pats.append(rbytes(rng, rng.randint(0, 300), alphabet))
    K = rng.choice([1e-12, 0.1, 0.5, 0.8, 1.0])
    top_t = rng.choice([0, 0, 1, 3])
    b = cb.query_batch(view, pats, K, top_t, scores=True)
    for i, pat in enumerate(pats):
        try:
            e, s, h, dense = idx.query(pat, K, top_t, scores=True)
        except O.OracleError as err:
            assert b.status[i] == 2 and b.messages[i] == err.msg, (it, i)
            continue
        assert b.status[i] == 0 and int(b.ell[i]) == e and int(b.skipped[i]) == s, (it, i)
        assert np.array_equal(b.dense[i].astype(np.uint32), dense), (it, i)
        d, sc = b.hits(i)
        assert [(int(x), int(y)) for x, y in zip(d, sc)] == h, (it, i)
    view.close()
