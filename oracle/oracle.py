"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes wrappers over
  * oracle/_build/libcobs_oracle.so : our plain-C restatement of the
    reference path (cobs_oracle.c, every function citing reference file:line)
  * oracle/_ref/libcobs_ref.so      : the UNMODIFIED reference sources
    (/root/reference/proj/src) compiled here by oracle/Makefile.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or
the reference CPU baseline -- never as the thing measured or shipped.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import List, Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libcobs_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcobs_ref.so")


def ensure_built() -> None:
    """Build the C restatement if missing (gcc is on the GPU box too)."""
    if not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-C", HERE, "oracle"], check=True, capture_output=True)


class OrcParams(C.Structure):
    _fields_ = [("q", C.c_uint32), ("k", C.c_uint32), ("p", C.c_double), ("canonical", C.c_int),
                ("block_size", C.c_uint64), ("hash_scheme", C.c_uint8)]


class OrcBlock(C.Structure):
    _fields_ = [("doc_count", C.c_uint64), ("w", C.c_uint64), ("row_bytes", C.c_uint64),
                ("offset", C.c_uint64), ("doc_base", C.c_uint64)]


class OrcIndex(C.Structure):
    _fields_ = [("params", OrcParams), ("kind", C.c_uint8), ("num_blocks", C.c_uint64),
                ("num_docs", C.c_uint64), ("blocks", C.POINTER(OrcBlock)),
                ("names", C.POINTER(C.c_void_p)), ("name_len", C.POINTER(C.c_uint16)),
                ("term_count", C.POINTER(C.c_uint64)), ("payload", C.c_void_p),
                ("payload_start", C.c_uint64), ("file_size", C.c_uint64),
                ("name_pool", C.c_void_p), ("c5_seed", C.c_uint64),
                ("c5_thr16", C.POINTER(C.c_uint32))]


class OrcStreamSpec(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("alpha", C.c_int), ("n_docs", C.c_uint64), ("doc_len", C.c_void_p),
                ("params", OrcParams), ("kind", C.c_int)]


class OrcStreamReport(C.Structure):
    _fields_ = [("header_equal", C.c_int), ("header_len", C.c_uint64), ("image_len_expected", C.c_uint64),
                ("term_count_mismatch", C.c_uint64), ("payload_bad_bytes", C.c_uint64),
                ("bad_block", C.c_uint64), ("bad_row", C.c_uint64), ("bad_byte", C.c_uint64),
                ("windows", C.c_uint64)]


class OrcHit(C.Structure):
    _fields_ = [("doc", C.c_uint64), ("score", C.c_uint64)]


_vp = C.c_void_p
_u64 = C.c_uint64


def _take(ptr, n: int) -> bytes:
    # ctypes.string_at truncates its size to a C int; copy through numpy
    if n == 0:
        return b""
    return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint8)), shape=(n,)).tobytes()


def _load_oracle():
    ensure_built()
    L = C.CDLL(ORACLE_SO)
    L.orc_xxh64.restype = _u64
    L.orc_xxh64.argtypes = [C.c_char_p, C.c_size_t, _u64]
    L.orc_fpr_approx.restype = C.c_double
    L.orc_fpr_approx.argtypes = [_u64, C.c_uint32, _u64]
    L.orc_size_filter.argtypes = [_u64, C.c_double, C.c_uint32, C.POINTER(_u64)]
    L.orc_score_threshold.restype = _u64
    L.orc_score_threshold.argtypes = [_u64, C.c_double]
    L.orc_extract_terms.argtypes = [_vp, _vp, C.c_size_t, C.c_uint32, C.c_int, C.POINTER(_vp),
                                    C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64)]
    L.orc_parse.argtypes = [_vp, _u64, C.c_char_p, C.POINTER(OrcIndex), C.c_char_p, C.c_size_t]
    L.orc_index_free.argtypes = [C.POINTER(OrcIndex)]
    L.orc_query.argtypes = [C.POINTER(OrcIndex), _vp, _u64, C.c_double, _u64, _vp, C.POINTER(_u64),
                            C.POINTER(_u64), C.POINTER(C.POINTER(OrcHit)), C.POINTER(_u64),
                            C.c_char_p, C.c_size_t]
    L.orc_query_batch.argtypes = [C.POINTER(OrcIndex), _vp, _vp, C.c_size_t, C.c_double, _vp, _vp,
                                  _vp, _vp, _vp, C.c_int]
    L.orc_build_image.argtypes = [_vp, _vp, _vp, _vp, C.c_size_t, C.POINTER(OrcParams), C.c_int,
                                  _u64, C.POINTER(_vp), C.POINTER(_u64), C.c_char_p, C.c_size_t]
    L.orc_c5_make.argtypes = [_u64, _u64, _u64, C.c_double, C.c_double, C.c_double,
                              C.POINTER(OrcIndex)]
    L.orc_header_image.argtypes = [C.POINTER(OrcIndex), C.POINTER(_vp), C.POINTER(_u64)]
    L.orc_stream_check.argtypes = [C.POINTER(OrcStreamSpec), _vp, _u64, C.c_int, C.POINTER(OrcStreamReport),
                                   _vp, C.c_char_p, C.c_size_t]
    L.orc_free.argtypes = [_vp]
    return L


_orc = None


def orc():
    global _orc
    if _orc is None:
        _orc = _load_oracle()
    return _orc


def xxh64(data: bytes, seed: int = 0) -> int:
    return orc().orc_xxh64(data, len(data), seed)


def size_filter(v: int, p: float, k: int) -> int:
    w = _u64()
    if orc().orc_size_filter(v, p, k, C.byref(w)):
        raise ValueError("size_filter: invalid argument")
    return w.value


def fpr_approx(w: int, k: int, v: int) -> float:
    return orc().orc_fpr_approx(w, k, v)


def score_threshold(ell: int, K: float) -> int:
    return orc().orc_score_threshold(ell, K)


def _segs(content: Sequence[bytes]):
    keep = [np.frombuffer(c, dtype=np.uint8) if len(c) else np.zeros(1, np.uint8) for c in content]
    ptrs = (C.c_void_p * max(len(keep), 1))(*[k.ctypes.data for k in keep])
    lens = (C.c_uint64 * max(len(keep), 1))(*[len(c) for c in content])
    return keep, ptrs, lens


def extract_terms(content: Sequence[bytes], q: int, canonical: bool) -> Tuple[List[bytes], int, int]:
    """(sorted distinct terms, skipped, occurrences) — termizer.cpp:103-129."""
    keep, ptrs, lens = _segs(content)
    terms = C.c_void_p()
    ell, sk, occ = _u64(), _u64(), _u64()
    orc().orc_extract_terms(ptrs, lens, len(content), q, 1 if canonical else 0, C.byref(terms),
                            C.byref(ell), C.byref(sk), C.byref(occ))
    raw = _take(terms, ell.value * q)
    orc().orc_free(terms)
    return [raw[i * q:(i + 1) * q] for i in range(ell.value)], sk.value, occ.value


class OracleIndex:
    """A parsed index image (or the config-5 procedural index)."""

    def __init__(self):
        self.x = OrcIndex()
        self._img = None

    @classmethod
    def parse(cls, image: bytes, path: str = "<memory>") -> "OracleIndex":
        o = cls()
        o._img = np.frombuffer(image, dtype=np.uint8).copy()
        err = C.create_string_buffer(1024)
        rc = orc().orc_parse(o._img.ctypes.data, len(image), path.encode(), C.byref(o.x), err, 1024)
        if rc:
            o.x = OrcIndex()
            raise OracleError(rc, err.value.decode())
        return o

    @classmethod
    def parse_array(cls, image: np.ndarray, path: str = "<memory>") -> "OracleIndex":
        """parse() over a uint8 array without copying it (full-size images)."""
        o = cls()
        o._img = np.ascontiguousarray(image, dtype=np.uint8)
        err = C.create_string_buffer(1024)
        rc = orc().orc_parse(o._img.ctypes.data, len(o._img), path.encode(), C.byref(o.x), err, 1024)
        if rc:
            o.x = OrcIndex()
            raise OracleError(rc, err.value.decode())
        return o

    @classmethod
    def c5(cls, seed: int, n_docs: int, block_size: int, median: float, sigma: float,
           p: float) -> "OracleIndex":
        o = cls()
        orc().orc_c5_make(seed, n_docs, block_size, median, sigma, p, C.byref(o.x))
        return o

    def __del__(self):
        try:
            orc().orc_index_free(C.byref(self.x))
        except Exception:
            pass

    @property
    def num_docs(self) -> int:
        return self.x.num_docs

    def blocks(self) -> List[Tuple[int, int, int]]:
        return [(self.x.blocks[b].doc_count, self.x.blocks[b].w, self.x.blocks[b].doc_base)
                for b in range(self.x.num_blocks)]

    def names(self) -> List[bytes]:
        return [C.string_at(self.x.names[i], self.x.name_len[i]) for i in range(self.x.num_docs)]

    def term_counts(self) -> List[int]:
        return [self.x.term_count[i] for i in range(self.x.num_docs)]

    def header(self) -> bytes:
        p = C.c_void_p()
        n = _u64()
        orc().orc_header_image(C.byref(self.x), C.byref(p), C.byref(n))
        out = _take(p, n.value)
        orc().orc_free(p)
        return out

    def query(self, pattern: bytes, K: float, top_t: int = 0, scores: bool = False):
        """-> (ell, skipped, hits[(doc, score)], dense scores or None); raises
        OracleError(1|2) like query.cpp:125-138."""
        buf = np.frombuffer(pattern, dtype=np.uint8) if pattern else np.zeros(1, np.uint8)
        dense = np.zeros(self.x.num_docs, dtype=np.uint32) if scores else None
        ell, sk, nh = _u64(), _u64(), _u64()
        hits = C.POINTER(OrcHit)()
        err = C.create_string_buffer(512)
        rc = orc().orc_query(C.byref(self.x), buf.ctypes.data, len(pattern), K, top_t,
                             dense.ctypes.data if scores else None, C.byref(ell), C.byref(sk),
                             C.byref(hits), C.byref(nh), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode(), ell=ell.value, skipped=sk.value)
        out = [(hits[i].doc, hits[i].score) for i in range(nh.value)]
        orc().orc_free(C.cast(hits, C.c_void_p))
        return ell.value, sk.value, out, dense

    def query_batch(self, buf: np.ndarray, off: np.ndarray, K: float, scores: bool = False,
                    threads: int = 0):
        """Batch on `threads` host threads -> (ell, skipped, status, n_hits, dense)."""
        n = len(off) - 1
        ell = np.zeros(n, np.uint64)
        sk = np.zeros(n, np.uint64)
        st = np.zeros(n, np.int32)
        nh = np.zeros(n, np.uint64)
        dense = np.zeros((n, self.x.num_docs), np.uint32) if scores else None
        buf = np.ascontiguousarray(buf, np.uint8)
        off = np.ascontiguousarray(off, np.uint64)
        orc().orc_query_batch(C.byref(self.x), buf.ctypes.data, off.ctypes.data, n, K,
                              dense.ctypes.data if scores else None, ell.ctypes.data,
                              sk.ctypes.data, st.ctypes.data, nh.ctypes.data,
                              threads or (os.cpu_count() or 1))
        return ell, sk, st, nh, dense


class OracleError(Exception):
    def __init__(self, code: int, msg: str, **kw):
        super().__init__(msg)
        self.code = code
        self.msg = msg
        self.__dict__.update(kw)


def build_image(docs: Sequence[Tuple[bytes, Sequence[bytes]]], q=31, k=1, p=0.3, canonical=False,
                block_size=1024, kind=0, forced_w=0) -> bytes:
    """orc_build_image: classic_index.cpp + compact_index.cpp + storage.cpp."""
    segs, doc_seg, names = [], [0], []
    for name, content in docs:
        names.append(name)
        segs.extend(content)
        doc_seg.append(len(segs))
    keep, ptrs, lens = _segs(segs)
    ds = (C.c_uint64 * len(doc_seg))(*doc_seg)
    nm = (C.c_char_p * max(len(names), 1))(*names)
    prm = OrcParams(q, k, p, 1 if canonical else 0, block_size, 0)
    img = C.c_void_p()
    n = _u64()
    err = C.create_string_buffer(512)
    rc = orc().orc_build_image(ptrs, lens, ds, nm, len(names), C.byref(prm), kind, forced_w,
                               C.byref(img), C.byref(n), err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    out = _take(img, n.value)
    orc().orc_free(img)
    return out


def stream_check(seed: int, alpha: int, doc_len: np.ndarray, image, q=31, k=1, p=0.3, canonical=False,
                 block_size=1024, kind=0, threads: int = 0) -> dict:
    """orc_stream_check (oracle/cobs_stream.c): the index image (bytes or a
    uint8 array) of the seeded synthetic corpus against the build the
    reference would make of it, every payload byte and the whole header,
    streamed one 64-document column group at a time.  Returns the report
    plus the oracle's term counts by draw index."""
    arr = np.frombuffer(image, np.uint8) if isinstance(image, (bytes, bytearray)) else image
    arr = np.ascontiguousarray(arr, dtype=np.uint8)
    lens = np.ascontiguousarray(doc_len, dtype=np.uint64)
    spec = OrcStreamSpec(seed, alpha, len(lens), lens.ctypes.data,
                         OrcParams(q, k, p, 1 if canonical else 0, block_size, 0), kind)
    rep = OrcStreamReport()
    tc = np.zeros(len(lens), np.uint64)
    err = C.create_string_buffer(512)
    rc = orc().orc_stream_check(C.byref(spec), arr.ctypes.data, len(arr), threads or (os.cpu_count() or 1),
                                C.byref(rep), tc.ctypes.data, err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    out = {f: getattr(rep, f) for f, _ in OrcStreamReport._fields_}
    out["header_equal"] = bool(out["header_equal"])
    out["term_counts"] = tc
    return out


# ---- the reference itself (oracle/_ref) ----------------------------------

def ref_available() -> bool:
    return os.path.exists(REF_SO)


_ref = None


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise FileNotFoundError(REF_SO)
        L = C.CDLL(REF_SO)
        L.ref_xxh64.restype = _u64
        L.ref_xxh64.argtypes = [C.c_char_p, C.c_size_t, _u64]
        L.ref_size_filter.argtypes = [_u64, C.c_double, C.c_uint32, C.POINTER(_u64)]
        L.ref_fpr_approx.restype = C.c_double
        L.ref_fpr_approx.argtypes = [_u64, C.c_uint32, _u64]
        L.ref_score_threshold.restype = _u64
        L.ref_score_threshold.argtypes = [_u64, C.c_double]
        L.ref_extract_terms.argtypes = [_vp, _vp, C.c_size_t, C.c_uint32, C.c_int, C.POINTER(_vp),
                                        C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64)]
        L.ref_free.argtypes = [_vp]
        L.ref_build_write.argtypes = [_vp, _vp, _vp, _vp, C.c_size_t, C.c_uint32, C.c_uint32,
                                      C.c_double, C.c_int, _u64, C.c_int, _u64, C.c_uint32,
                                      C.c_char_p, C.c_char_p, C.c_size_t]
        L.ref_build_terms_write.argtypes = L.ref_build_write.argtypes
        L.ref_open_random_access.argtypes = [C.c_char_p, C.POINTER(_vp), C.c_char_p, C.c_size_t]
        L.ref_bytes_read.argtypes = [_vp]
        L.ref_bytes_read.restype = _u64
        L.ref_open.argtypes = [C.c_char_p, C.POINTER(_vp), C.c_char_p, C.c_size_t]
        L.ref_query_fasta_tsv.argtypes = [_vp, C.c_char_p, C.c_double, _u64, C.POINTER(_vp),
                                          C.c_char_p, C.c_size_t]
        L.ref_build_files.argtypes = [C.POINTER(C.c_char_p), C.c_size_t, C.c_uint32, C.c_uint32,
                                      C.c_double, C.c_int, _u64, C.c_int, C.c_int, C.c_char_p,
                                      C.c_char_p, C.c_size_t]
        L.ref_merge_write.argtypes = [_vp, _vp, _vp, _vp, C.c_size_t, C.c_size_t, C.c_uint32,
                                      C.c_uint32, C.c_double, C.c_int, _u64, C.c_char_p, C.c_char_p,
                                      C.c_size_t]
        L.ref_c5_open.argtypes = [_u64, _u64, _u64, C.c_double, C.c_double, C.c_double, C.c_int,
                                  C.c_int, C.POINTER(_vp), C.c_char_p, C.c_size_t]
        L.ref_close.argtypes = [_vp]
        L.ref_total_docs.restype = _u64
        L.ref_total_docs.argtypes = [_vp]
        L.ref_write.argtypes = [_vp, C.c_char_p, C.c_char_p, C.c_size_t]
        L.ref_query.argtypes = [_vp, _vp, _u64, C.c_double, _u64, C.c_uint32, C.POINTER(_u64),
                                C.POINTER(_u64), C.POINTER(C.POINTER(_u64)),
                                C.POINTER(C.POINTER(_u64)), C.POINTER(_u64), C.c_char_p, C.c_size_t]
        L.ref_query_batch.argtypes = [_vp, _vp, _vp, C.c_size_t, C.c_double, C.c_int, _vp, _vp, _vp,
                                      _vp, _vp]
        _ref = L
    return _ref


class RefIndex:
    """A view opened through the reference's own API (open_resident or the
    config-5 IndexView)."""

    def __init__(self, h):
        self.h = h

    @classmethod
    def open(cls, path: str, random_access: bool = False) -> "RefIndex":
        """open_resident, or open_random_access (rows pread on demand,
        counted by bytes_read())."""
        h = C.c_void_p()
        err = C.create_string_buffer(1024)
        fn = ref().ref_open_random_access if random_access else ref().ref_open
        rc = fn(path.encode(), C.byref(h), err, 1024)
        if rc:
            raise OracleError(rc, err.value.decode())
        return cls(h)

    def bytes_read(self) -> int:
        """IndexView::bytes_read (index_view.hpp:44-46, storage.cpp:325-336)."""
        return int(ref().ref_bytes_read(self.h))

    @classmethod
    def c5(cls, seed, n_docs, block_size, median, sigma, p, materialise=False, threads=0):
        h = C.c_void_p()
        err = C.create_string_buffer(1024)
        rc = ref().ref_c5_open(seed, n_docs, block_size, median, sigma, p, 1 if materialise else 0,
                               threads or (os.cpu_count() or 1), C.byref(h), err, 1024)
        if rc:
            raise OracleError(rc, err.value.decode())
        return cls(h)

    def query_fasta_tsv(self, path: str, K: float, top_t: int = 0) -> bytes:
        out = C.c_void_p()
        err = C.create_string_buffer(1024)
        rc = ref().ref_query_fasta_tsv(self.h, path.encode(), K, top_t, C.byref(out), err, 1024)
        if rc:
            raise OracleError(rc, err.value.decode())
        try:
            return C.string_at(out)
        finally:
            ref().ref_free(out)

    def close(self):
        if self.h:
            ref().ref_close(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def total_docs(self) -> int:
        return ref().ref_total_docs(self.h)

    def write(self, path: str):
        err = C.create_string_buffer(1024)
        rc = ref().ref_write(self.h, path.encode(), err, 1024)
        if rc:
            raise OracleError(rc, err.value.decode())

    def query(self, pattern: bytes, K: float, top_t: int = 0, workers: int = 1):
        buf = np.frombuffer(pattern, dtype=np.uint8) if pattern else np.zeros(1, np.uint8)
        ell, sk, nh = _u64(), _u64(), _u64()
        docs = C.POINTER(_u64)()
        scores = C.POINTER(_u64)()
        err = C.create_string_buffer(1024)
        rc = ref().ref_query(self.h, buf.ctypes.data, len(pattern), K, top_t, workers, C.byref(ell),
                             C.byref(sk), C.byref(docs), C.byref(scores), C.byref(nh), err, 1024)
        if rc:
            raise OracleError(rc, err.value.decode())
        out = [(docs[i], scores[i]) for i in range(nh.value)]
        ref().ref_free(C.cast(docs, C.c_void_p))
        ref().ref_free(C.cast(scores, C.c_void_p))
        return ell.value, sk.value, out

    def query_batch(self, buf, off, K: float, scores: bool = False, threads: int = 0):
        n = len(off) - 1
        ell = np.zeros(n, np.uint64)
        sk = np.zeros(n, np.uint64)
        st = np.zeros(n, np.int32)
        nh = np.zeros(n, np.uint64)
        dense = np.zeros((n, self.total_docs()), np.uint32) if scores else None
        buf = np.ascontiguousarray(buf, np.uint8)
        off = np.ascontiguousarray(off, np.uint64)
        ref().ref_query_batch(self.h, buf.ctypes.data, off.ctypes.data, n, K,
                              threads or (os.cpu_count() or 1), ell.ctypes.data, sk.ctypes.data,
                              st.ctypes.data, nh.ctypes.data,
                              dense.ctypes.data if scores else None)
        return ell, sk, st, nh, dense


def ref_build_write(docs, path: str, q=31, k=1, p=0.3, canonical=False, block_size=1024, kind=0,
                    forced_w=0, workers=0):
    segs, doc_seg, names = [], [0], []
    for name, content in docs:
        names.append(name)
        segs.extend(content)
        doc_seg.append(len(segs))
    keep, ptrs, lens = _segs(segs)
    ds = (C.c_uint64 * len(doc_seg))(*doc_seg)
    nm = (C.c_char_p * max(len(names), 1))(*names)
    err = C.create_string_buffer(1024)
    rc = ref().ref_build_write(ptrs, lens, ds, nm, len(names), q, k, p, 1 if canonical else 0,
                               block_size, kind, forced_w, workers or (os.cpu_count() or 1),
                               path.encode(), err, 1024)
    if rc:
        raise OracleError(rc, err.value.decode())


def ref_build_terms_write(termsets, path: str, q=31, k=1, p=0.3, canonical=False, block_size=1024,
                          kind=0, forced_w=0, workers=1):
    """The reference's build_classic / build_compact over TermSets given as
    (name, [term, ...]) (terms kept as given) + write_index."""
    segs, doc_seg, names = [], [0], []
    for name, terms in termsets:
        names.append(name)
        segs.extend(terms)
        doc_seg.append(len(segs))
    keep, ptrs, lens = _segs(segs)
    ds = (C.c_uint64 * len(doc_seg))(*doc_seg)
    nm = (C.c_char_p * max(len(names), 1))(*names)
    err = C.create_string_buffer(1024)
    rc = ref().ref_build_terms_write(ptrs, lens, ds, nm, len(names), q, k, p, 1 if canonical else 0,
                                     block_size, kind, forced_w, workers, path.encode(), err, len(err))
    if rc:
        raise OracleError(rc, err.value.decode())


def ref_extract_terms(content: Sequence[bytes], q: int, canonical: bool):
    keep, ptrs, lens = _segs(content)
    terms = C.c_void_p()
    ell, sk, occ = _u64(), _u64(), _u64()
    rc = ref().ref_extract_terms(ptrs, lens, len(content), q, 1 if canonical else 0,
                                 C.byref(terms), C.byref(ell), C.byref(sk), C.byref(occ))
    if rc:
        raise OracleError(rc, "extract_terms")
    raw = _take(terms, ell.value * q)
    ref().ref_free(terms)
    return [raw[i * q:(i + 1) * q] for i in range(ell.value)], sk.value, occ.value


def ref_merge_write(docs, split: int, path: str, forced_w: int, q=31, k=1, p=0.3, canonical=False):
    """The reference's merge_classic of docs[:split] and docs[split:] built at
    a common forced width, written by its write_index."""
    segs, doc_seg, names = [], [0], []
    for name, content in docs:
        names.append(name)
        segs.extend(content)
        doc_seg.append(len(segs))
    keep, ptrs, lens = _segs(segs)
    ds = (C.c_uint64 * len(doc_seg))(*doc_seg)
    nm = (C.c_char_p * max(len(names), 1))(*names)
    err = C.create_string_buffer(1024)
    rc = ref().ref_merge_write(ptrs, lens, ds, nm, len(names), split, q, k, p, 1 if canonical else 0,
                               forced_w, path.encode(), err, 1024)
    if rc:
        raise OracleError(rc, err.value.decode())


def ref_build_files(inputs, out_path: str, q=31, k=1, p=0.3, canonical=False, block_size=1024,
                    kind=1, format=0):
    arr = (C.c_char_p * max(len(inputs), 1))(*[str(i).encode() for i in inputs])
    err = C.create_string_buffer(1024)
    rc = ref().ref_build_files(arr, len(inputs), q, k, p, 1 if canonical else 0, block_size, kind,
                               format, out_path.encode(), err, 1024)
    if rc:
        raise OracleError(rc, err.value.decode())
