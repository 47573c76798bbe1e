"""The C-ABI library loads and exports every symbol include/cobs_gpu.h
declares; host-side logic reachable without a GPU (parse/reject before any
device call).  CPU only."""
import ctypes as C
import os
import re
import struct

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "cobs_gpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cobs_gpu_\w+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = C.CDLL(os.path.join(ROOT, "paper_1905_09624_b200", "_lib", "libcobs_gpu.so"))
    syms = header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), s


def test_binding_covers_header():
    from paper_1905_09624_b200 import _native as N
    assert sorted(N.SIGNATURES) == header_symbols()


def test_version():
    from paper_1905_09624_b200 import _native as N
    assert b"sm_100a" in N.lib.cobs_gpu_version()


def golden_90():
    from tests.test_oracle_golden import golden_90 as g
    return g()


def test_reader_rejects_before_device(tmp_path):
    """The host parser rejects exactly what parse_index rejects
    (test_storage.cpp:192-235); no device is touched for a rejected file."""
    import paper_1905_09624_b200 as cb
    img = golden_90()
    cases = [(0, ord("X"), "bad magic"), (8, 2, "unsupported format version 2"),
             (9, 7, "unknown index kind 7"), (10, 1, "unknown hash scheme 1"),
             (11, 2, "bad canonical flag"), (12, 0, "bad q/k parameters"),
             (16, 0, "bad q/k parameters"),
             (36, 2, "classic index must have exactly one block"),
             (44, 9, "document count mismatch"), (60, 9, "payload exceeds file size"),
             (79, 12, "payload offsets not contiguous")]
    path = str(tmp_path / "m.cobs")
    for off, val, msg in cases:
        m = bytearray(img)
        m[off] = val
        open(path, "wb").write(bytes(m))
        with pytest.raises(cb.DataError) as e:
            cb.open_resident(path)
        assert str(e.value) == f"index file {path}: {msg}"
    m = bytearray(img)
    m[20:28] = struct.pack("<d", 2.0)
    open(path, "wb").write(bytes(m))
    with pytest.raises(cb.DataError, match="target FPR out of range"):
        cb.open_resident(path)
    for cut in (0, 7, 51, 70, 86, 89):
        open(path, "wb").write(img[:cut])
        with pytest.raises(cb.DataError):
            cb.open_resident(path)
    open(path, "wb").write(img + b"Z")
    with pytest.raises(cb.DataError, match="trailing bytes after payload"):
        cb.open_resident(path)
    with pytest.raises(cb.DataError, match="cannot open index file"):
        cb.open_resident(str(tmp_path / "nonexistent.cobs"))


def test_reader_matches_oracle_on_random_corruptions(tmp_path):
    """Same accept/reject decision and message as the oracle (and hence the
    reference, tests/test_oracle_vs_ref.py) on random mutations."""
    import random
    import paper_1905_09624_b200 as cb
    from oracle import oracle as O
    rng = random.Random(3)
    docs = [(b"doc%04d" % i, [bytes(rng.choice(b"ACGT") for _ in range(rng.randint(40, 300)))])
            for i in range(9)]
    img = O.build_image(docs, k=2, block_size=3, kind=1)
    path = str(tmp_path / "m.cobs")
    for trial in range(150):
        m = bytearray(img)
        if trial % 3 == 0:
            m = m[: rng.randrange(len(m))]
        else:
            pos = rng.randrange(min(len(m), 400))
            m[pos] = rng.randrange(256)
        open(path, "wb").write(bytes(m))
        try:
            O.OracleIndex.parse(bytes(m), path)
            continue  # accepted files need a device to finish opening
        except O.OracleError as e:
            want = e.msg
        with pytest.raises(cb.DataError) as got:
            cb.open_resident(path)
        assert str(got.value) == want


def test_build_usage_errors_without_device():
    import paper_1905_09624_b200 as cb
    with pytest.raises(cb.DataError, match="build: no documents"):
        cb.build_classic([])
    with pytest.raises(ValueError, match="params: k must be >= 1"):
        cb.build_classic([(b"a", [b"ACGT" * 10])], cb.IndexParams(k=0))
    with pytest.raises(cb.DataError, match="duplicate document name: x"):
        cb.build_compact([(b"x", [b"ACGT" * 10]), (b"x", [b"ACGT" * 10])])


def test_build_segment_ptrs_rejects_device_input():
    """COBS_B_SEGMENT_PTRS (host pointer per string) with COBS_B_DEVICE_INPUT
    is a usage error, reported before any device call; the Python packer
    hands the library one pointer per string (no packed copy)."""
    import paper_1905_09624_b200 as cb
    from paper_1905_09624_b200 import _native as N
    names, ptrs, seg_off, doc_segs = cb._pack_docs([(b"a", [b"ACGT" * 10, b"GG"]), ("b", ["TTTT" * 9])])
    assert [C.string_at(ptrs[i], int(seg_off[i + 1] - seg_off[i])) for i in range(3)] == \
        [b"ACGT" * 10, b"GG", b"TTTT" * 9]
    assert list(doc_segs) == [0, 2, 3] and names == [b"a", b"b"]
    nm = (C.c_char_p * 2)(*names)
    err = C.create_string_buffer(512)
    cp = cb.IndexParams()._c()
    rc = N.lib.cobs_gpu_build_ex(C.cast(ptrs, C.c_void_p), seg_off.ctypes.data, 3, doc_segs.ctypes.data, nm, 2,
                                 C.byref(cp), cb.KIND_CLASSIC, 0, 0, N.B_SEGMENT_PTRS | N.B_DEVICE_INPUT, None,
                                 None, None, None, err, len(err))
    assert rc == 1 and b"COBS_B_SEGMENT_PTRS" in err.value
