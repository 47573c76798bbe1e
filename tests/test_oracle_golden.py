"""Pin the CPU oracle (oracle/cobs_oracle.c) against the reference's own golden
vectors and known-answer tests.  CPU only."""
import math
import random
import struct

import pytest

from oracle import oracle as O

# proj/tests/test_termizer.cpp:29-46 and proj/FORMAT.md:122-132
XXH_GOLDEN = [
    (b"", 0, 0xEF46DB3751D8E999),
    (b"abc", 0, 0x44BC2CF5AD770999),
    (b"1234", 0, 0xD8316E61D84F6BA4),
    (b"12345678", 7, 0xDE04D6794DDCD8A6),
    (b"A" * 31, 0, 0x04D4645EC33F5384),
    (b"A" * 31, 1, 0x04CAEAB334EEB221),
    (b"q" * 33, 0, 0x40149E1612102FB7),
    (b"Nobody inspects the spammish repetition", 0, 0xFBCEA83C8A378BF1),
    (b"ACGT" * 9, 0, 0xD0B5650968777664),
    (bytes(range(47)), 42, 0x5D21F13EBD0D4A6C),
]


@pytest.mark.parametrize("data,seed,want", XXH_GOLDEN)
def test_xxh64_golden(data, seed, want):
    assert O.xxh64(data, seed) == want


def test_xxh64_matches_python_xxhash():
    xxhash = pytest.importorskip("xxhash")
    rng = random.Random(5)
    for n in list(range(0, 80)) + [127, 128, 129, 1000]:
        data = bytes(rng.randrange(256) for _ in range(n))
        for seed in (0, 1, 2, 2**63 + 5):
            assert O.xxh64(data, seed) == xxhash.xxh64_intdigest(data, seed)


def test_hash_rows_golden():
    # test_termizer.cpp:149-152: XXH64("A"*31, 0) mod 2^61
    assert O.xxh64(b"A" * 31, 0) % (1 << 61) == 348013429379781508


def test_size_filter_pinned():
    # test_bloom.cpp:108-112
    assert O.size_filter(0, 0.3, 1) == 1
    assert O.size_filter(1, 0.3, 1) == 3
    assert O.size_filter(1000, 0.3, 1) == 2804


def test_size_filter_minimal():
    # test_bloom.cpp:114-130 (own random grid)
    rng = random.Random(11)
    for _ in range(200):
        v = rng.randint(1, 20000)
        k = rng.randint(1, 8)
        p = rng.uniform(0.001, 0.9)
        w = O.size_filter(v, p, k)
        assert O.fpr_approx(w, k, v) <= p
        if w > 1:
            assert O.fpr_approx(w - 1, k, v) > p


def test_size_filter_rejects():
    with pytest.raises(ValueError):
        O.size_filter(10, 0.0, 1)
    with pytest.raises(ValueError):
        O.size_filter(10, 1.0, 1)


def test_score_threshold():
    # test_bloom.cpp:254-265
    assert O.score_threshold(1, 1.0) == 1
    assert O.score_threshold(50, 1.0) == 50
    assert O.score_threshold(10, 0.9) == 9
    assert O.score_threshold(70, 0.5) == 35
    assert O.score_threshold(70, 0.51) == 36
    assert O.score_threshold(1, 0.3) == 1
    assert O.score_threshold(3, 0.01) == 1
    for ell in (10, 20, 30, 100, 1000):
        assert O.score_threshold(ell, 0.9) == ell * 9 // 10
    # the config thresholds quoted in SURVEY.md §8(a) a4
    assert O.score_threshold(970, 0.8) == 776
    assert O.score_threshold(91, 0.9) == 82


def test_extract_terms_cases():
    # test_termizer.cpp:63-106
    t, sk, occ = O.extract_terms([b"ABCDE"], 3, False)
    assert t == [b"ABC", b"BCD", b"CDE"] and occ == 3 and sk == 0
    assert O.extract_terms([b"TTT"], 3, True)[0] == [b"AAA"]
    assert O.extract_terms([b"ACGT"], 4, True)[0] == [b"ACGT"]
    t, sk, occ = O.extract_terms([b"ABCD", b"EFGH"], 3, False)
    assert t == [b"ABC", b"BCD", b"EFG", b"FGH"] and occ == 4
    t, sk, occ = O.extract_terms([b"AAAA"], 2, False)
    assert t == [b"AA"] and occ == 3
    t, sk, occ = O.extract_terms([b"ACGNACG"], 3, True)
    assert t == [b"ACG"] and sk == 3 and occ == 2
    t, sk, occ = O.extract_terms([b"ACGNACG"], 3, False)
    assert sk == 0 and occ == 5 and len(t) == 4
    t, sk, occ = O.extract_terms([b"AB", b"", b"ABCD"], 3, False)
    assert occ == 2 and t == [b"ABC", b"BCD"]
    # lowercase is not ACGT under canonicalisation (termizer.cpp:18-30)
    t, sk, occ = O.extract_terms([b"acgt"], 4, True)
    assert t == [] and sk == 1


def _revcomp(s: bytes) -> bytes:
    return s[::-1].translate(bytes.maketrans(b"ACGT", b"TGCA"))


def test_canonical_fixed_points():
    # test_termizer.cpp:131-141
    rng = random.Random(23)
    for _ in range(10):
        s = bytes(rng.choice(b"ACGT") for _ in range(500))
        terms, _, _ = O.extract_terms([s], 31, True)
        assert terms == sorted(set(terms))
        for t in terms:
            assert t == min(t, _revcomp(t))


def golden_90() -> bytes:
    """FORMAT.md:134-160 worked example, byte for byte."""
    return bytes.fromhex(
        "434f425349445831" "01000000" "1f000000" "01000000" "333333333333d33f"
        "0004000000000000" "0100000000000000" "0100000000000000" "0100000000000000"
        "0300000000000000" "0100" "64" "0100000000000000" "5700000000000000"
        "00" "01" "00")


def test_golden_90_byte_file():
    # test_storage.cpp:61-91 / FORMAT.md:134-160; the one-term document is
    # built from content "A"*31
    img = O.build_image([(b"d", [b"A" * 31])])
    assert len(img) == 90
    assert img == golden_90()
    assert struct.unpack_from("<d", img, 20)[0] == 0.3


def test_parse_golden_and_rejections():
    # test_storage.cpp:192-235
    img = golden_90()
    idx = O.OracleIndex.parse(img)
    assert idx.num_docs == 1 and idx.blocks() == [(1, 3, 0)]

    def reject(mut):
        with pytest.raises(O.OracleError) as e:
            O.OracleIndex.parse(mut)
        assert e.value.code == 2

    for off, val in [(0, ord("X")), (8, 2), (9, 7), (10, 1), (11, 2), (12, 0), (16, 0), (36, 2),
                     (44, 9), (60, 9), (79, 12)]:
        m = bytearray(img)
        m[off] = val
        reject(bytes(m))
    m = bytearray(img)
    m[20:28] = struct.pack("<d", 2.0)
    reject(bytes(m))
    for cut in (0, 7, 51, 70, 86, 89):
        reject(img[:cut])
    reject(img + b"Z")


def test_bit_matrix_lsb_first():
    # test_index.cpp:67-87 semantics through a built file: documents 0..12 in
    # one block; document 9's bits live in bit 1 of byte 1 of its rows
    docs = [(b"d%02d" % i, [b"A" * 31] if i == 9 else []) for i in range(13)]
    img = O.build_image(docs)
    idx = O.OracleIndex.parse(img)
    (dc, w, _), = idx.blocks()
    assert dc == 13
    row = O.xxh64(b"A" * 31, 0) % w
    payload = img[len(img) - w * 2:]
    for r in range(w):
        assert payload[2 * r] == 0
        assert payload[2 * r + 1] == (0x02 if r == row else 0)


def _make_doc(name: bytes, n_terms: int, q: int = 8):
    # n distinct q-grams, as test_index.cpp's make_doc does with synthetic terms
    rng = random.Random(hash(name) & 0xFFFF)
    terms = set()
    while len(terms) < n_terms:
        terms.add(bytes(rng.choice(b"ACGT") for _ in range(q)))
    return name, list(terms)


def test_compact_sort_and_staircase():
    # test_index.cpp:261-322
    docs = [_make_doc(b"zeta", 40), _make_doc(b"alpha", 40), _make_doc(b"mid", 7),
            _make_doc(b"tiny", 2), _make_doc(b"big", 900), _make_doc(b"beta", 40)]
    img = O.build_image(docs, q=8, block_size=4, kind=1)
    idx = O.OracleIndex.parse(img)
    assert list(zip(idx.term_counts(), idx.names())) == [
        (2, b"tiny"), (7, b"mid"), (40, b"alpha"), (40, b"beta"), (40, b"zeta"), (900, b"big")]
    docs = [_make_doc(b"d%03d" % i, i) for i in range(1, 101)]
    random.Random(31).shuffle(docs)
    img = O.build_image(docs, q=8, block_size=8, kind=1)
    idx = O.OracleIndex.parse(img)
    blocks = idx.blocks()
    assert len(blocks) == 13
    tcs = idx.term_counts()
    prev_w = 0
    for b, (dc, w, base) in enumerate(blocks):
        assert dc == (8 if b < 12 else 4)
        mx = max(tcs[base:base + dc])
        assert w == O.size_filter(mx, 0.3, 1) and w >= prev_w
        prev_w = w


def test_compact_single_block_equals_sorted_classic():
    # test_index.cpp:324-342
    rng = random.Random(37)
    docs = []
    for i in range(21):
        n = rng.randint(100, 120)
        docs.append((b"doc%04d" % i, [bytes(rng.choice(b"ACGT") for _ in range(n))]))
    comp = O.build_image(docs, block_size=64, kind=1)
    srt = sorted(docs, key=lambda d: (len(O.extract_terms(d[1], 31, False)[0]), d[0]))
    clas = O.build_image(srt, block_size=64, kind=0)
    # identical except the kind byte and block_size field stay as given
    assert comp[9] == 1 and clas[9] == 0
    c2 = bytearray(comp)
    c2[9] = 0
    assert bytes(c2) == clas


def test_query_ties_and_top_t():
    # test_query.cpp:90-115
    rng = random.Random(11)
    dna = bytes(rng.choice(b"ACGT") for _ in range(400))
    docs = [(n, [dna]) for n in (b"zebra", b"apple", b"mango")]
    docs.append((b"other", [bytes(rng.choice(b"ACGT") for _ in range(400))]))
    idx = O.OracleIndex.parse(O.build_image(docs))
    names = idx.names()
    ell, sk, hits, _ = idx.query(dna[:200], 1.0)
    assert [names[d] for d, _ in hits[:3]] == [b"apple", b"mango", b"zebra"]
    assert all(s == ell for _, s in hits[:3])
    ell2, _, capped, _ = idx.query(dna[:200], 1.0, top_t=2)
    assert capped == hits[:2]


def test_query_errors():
    # test_query.cpp:117-148, query.cpp:125-138
    rng = random.Random(13)
    docs = [(b"doc%04d" % i, [bytes(rng.choice(b"ACGT") for _ in range(150))]) for i in range(4)]
    idx = O.OracleIndex.parse(O.build_image(docs))
    with pytest.raises(O.OracleError) as e:
        idx.query(b"ACGT", 0.5)
    assert e.value.code == 2 and e.value.msg == "query: pattern shorter than q = 31"
    with pytest.raises(O.OracleError) as e:
        idx.query(b"A" * 40, 0.0)
    assert e.value.code == 1
    cidx = O.OracleIndex.parse(O.build_image(docs, canonical=True))
    with pytest.raises(O.OracleError) as e:
        cidx.query(b"N" * 40, 0.5)
    assert e.value.msg == "query: all 10 pattern grams were skipped by canonicalization"
    base = docs[0][1][0]
    pat = base[:60] + b"N" + base[60:120]
    ell, sk, _, _ = cidx.query(pat, 1.0)
    assert sk == 31


def test_fixture_files_match_oracle():
    """tests/golden/*.cobs were written by the reference (make_golden.py); the
    oracle rebuilds them byte for byte and reproduces the reference's query
    results recorded in golden.json."""
    import json
    import os
    gdir = os.path.join(os.path.dirname(__file__), "golden")
    g = json.load(open(os.path.join(gdir, "golden.json")))
    assert open(os.path.join(gdir, "tiny.cobs"), "rb").read() == golden_90()
    for name, spec in g["files"].items():
        docs = [(d[0].encode(), [s.encode() for s in d[1]]) for d in spec["docs"]]
        img = open(os.path.join(gdir, name + ".cobs"), "rb").read()
        assert O.build_image(docs, **spec["params"]) == img, name
        idx = O.OracleIndex.parse(img)
        for r in g["results"][name]:
            pat = r["pat"].encode()
            if "error" in r:
                with pytest.raises(O.OracleError) as e:
                    idx.query(pat, r["K"], r["top_t"])
                assert (e.value.code, e.value.msg) == (r["error"], r["msg"])
            else:
                ell, sk, hits, _ = idx.query(pat, r["K"], r["top_t"])
                assert (ell, sk) == (r["ell"], r["skipped"])
                assert [list(h) for h in hits] == r["hits"]
