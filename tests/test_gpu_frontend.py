"""File front ends on the GPU vs the reference: the FASTA batch query's TSV
(cli.cpp:192-223) and document ingestion for builds (cli.cpp:112-166)."""
import os
import random

import pytest

import paper_1905_09624_b200 as cb
from oracle import oracle as O

GDIR = os.path.join(os.path.dirname(__file__), "golden")


def rand(rng, n, a=b"ACGT"):
    return bytes(rng.choice(a) for _ in range(n))


def write_tricky_fasta(path, docs_seqs, rng):
    s1 = docs_seqs[0][:120]
    s2 = docs_seqs[1][40:300]
    lines = [
        rand(rng, 50),                               # headerless leading sequence -> query_0
        b">first record with spaces",
        s1[:60].lower(), s1[60:],                    # lowercase is uppercased by the reader
        b"",                                         # empty line skipped
        b">\ttab-led",                               # name = "" -> query_2
        s2[:100] + b"\r", s2[100:] + b"\r",          # CRLF
        b">short",
        b"ACGT",                                     # shorter than q -> ERR line
        b">withN",
        s2[:50] + b"NNN" + s2[50:120],
        b">alien",
        rand(rng, 200),
        b">last_no_newline",
        s1[:90],
    ]
    with open(path, "wb") as f:
        f.write(b"\n".join(lines))


def write_cr_edge_fasta(path, docs_seqs, rng):
    """Line-ending corners of the reader (termizer.cpp:48-88): a '\r' inside
    a line stays, one before '\n' goes, a final line without '\n' keeps its
    '\r'; a line "\r>..." is sequence, not a header; "\r\n" alone is an empty
    line; bytes >= 0x80 are not uppercased; chunk-crossing long lines."""
    s1 = docs_seqs[0][:200]
    body = (b"\r\n" + s1[:70] + b"\r\n" + b">h1\rmid  tail\r\n" + s1[10:110].lower() + b"\r" + s1[110:150]
            + b"\n\r>" + s1[:80] + b"\n>h\xe9\xff x\n" + b"acgt\xe9" * 30 + b"\n>long\n"
            + (s1 * 6000) + b"\n>" + b"\n" + rand(rng, 90) + b"\n>endcr\n" + s1[:64] + b"\r")
    with open(path, "wb") as f:
        f.write(body)


@pytest.mark.gpu
def test_query_fasta_line_ending_corners(gpu, tmp_path):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    import json
    g = json.load(open(os.path.join(GDIR, "golden.json")))
    rng = random.Random(9)
    for name in ("compact_canon", "classic_k2"):
        path = os.path.join(GDIR, name + ".cobs")
        seqs = [s.encode() for d in g["files"][name]["docs"] for s in d[1]]
        fa = str(tmp_path / (name + "_cr.fa"))
        write_cr_edge_fasta(fa, seqs, rng)
        view = cb.open_resident(path, gpu)
        ref = O.RefIndex.open(path)
        for K, top_t in [(0.5, 0), (1e-12, 2)]:
            assert cb.query_fasta(view, fa, K, top_t) == ref.query_fasta_tsv(fa, K, top_t), (name, K, top_t)
        view.close()


@pytest.mark.gpu
def test_query_fasta_tsv_matches_reference(gpu, tmp_path):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    import json
    g = json.load(open(os.path.join(GDIR, "golden.json")))
    rng = random.Random(8)
    for name in ("compact_canon", "classic_k2"):
        path = os.path.join(GDIR, name + ".cobs")
        seqs = [s.encode() for d in g["files"][name]["docs"] for s in d[1]]
        fa = str(tmp_path / (name + ".fa"))
        write_tricky_fasta(fa, seqs, rng)
        view = cb.open_resident(path, gpu)
        ref = O.RefIndex.open(path)
        for K, top_t in [(0.5, 0), (1e-12, 3), (1.0, 0)]:
            got = cb.query_fasta(view, fa, K, top_t)
            want = ref.query_fasta_tsv(fa, K, top_t)
            assert got == want, (name, K, top_t)
        assert b"*query_0\t" in got and b"*short\tERR\tquery: pattern shorter than q = 31\n" in got
        with pytest.raises(ValueError, match=r"^K must be in \(0,1\]$"):
            cb.query_fasta(view, fa, 1.5)
        with pytest.raises(cb.DataError, match="cannot open input file"):
            cb.query_fasta(view, str(tmp_path / "missing.fa"), 0.5)
        view.close()


def make_corpus_dir(root, rng):
    os.makedirs(os.path.join(root, "b", "nested"))
    os.makedirs(os.path.join(root, "a"))
    files = {
        "a/s1.fa": b">r1 desc\n" + rand(rng, 300) + b"\n>r2\n" + rand(rng, 200).lower() + b"\n",
        "a/s2.FASTA": rand(rng, 400) + b"\n",                   # headerless record
        "b/s3.fna": b">x\r\n" + rand(rng, 150) + b"\r\n" + rand(rng, 150) + b"\r\n",
        "b/nested/s4.txt": rand(rng, 500),                       # text: the whole file
        "b/nested/s5.txt": rand(rng, 100) + b"\n" + rand(rng, 100),
        "c_short.fa": b">tiny\nACGTACGT\n",                     # zero terms
        "b/s6.fa": b"\r\n" + rand(rng, 40) + b"\r" + rand(rng, 60).lower() + b"\n\r>" + rand(rng, 70)
                   + b"\n>y\n" + rand(rng, 80) + b"\r",                # line-ending corners
        "b/s7.fa": b"",                                          # no records: a document with no strings
    }
    for rel, data in files.items():
        with open(os.path.join(root, rel), "wb") as f:
            f.write(data)
    return [os.path.join(root, "a"), os.path.join(root, "b"), os.path.join(root, "c_short.fa")]


@pytest.mark.gpu
@pytest.mark.parametrize("kind,fmt,canonical", [(1, 0, True), (0, 0, False), (1, 2, False),
                                                (0, 1, True)])
def test_build_files_matches_reference(gpu, tmp_path, kind, fmt, canonical):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    rng = random.Random(kind * 10 + fmt)
    inputs = make_corpus_dir(str(tmp_path / "corpus"), rng)
    params = cb.IndexParams(canonical=canonical, block_size=2)
    img = cb.build_files(inputs, params, kind=kind, format=fmt, device=gpu)
    out = str(tmp_path / "ref.cobs")
    O.ref_build_files(inputs, out, canonical=canonical, block_size=2, kind=kind, format=fmt)
    assert img == open(out, "rb").read()


def test_build_files_input_errors(tmp_path):
    """expand_inputs' errors (cli.cpp:60-82) are raised before any device use."""
    with pytest.raises(cb.DataError, match="input not found: " + str(tmp_path / "nope")):
        cb.build_files([str(tmp_path / "nope")])
    (tmp_path / "empty").mkdir()
    with pytest.raises(cb.DataError, match="^no input files$"):
        cb.build_files([str(tmp_path / "empty")])
    with pytest.raises(ValueError, match="params: q must be >= 1"):
        cb.build_files([str(tmp_path)], cb.IndexParams(q=0))
