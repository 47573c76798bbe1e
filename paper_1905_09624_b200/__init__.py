"""cobs-b200: B200-native COBS (Compact Bit-sliced Signature index) query
path and index construction.

Python host mirror of the reference's C++ interface for this path
(/root/reference/proj/include/cobs): ``open_resident`` / ``query`` /
``build_classic`` / ``build_compact`` / ``write_index`` with the same argument
meaning and error behaviour -- ``DataError`` where the reference throws
``cobs::DataError`` and ``ValueError`` where it throws
``std::invalid_argument``.  All compute goes through the C-ABI of
``include/cobs_gpu.h`` into hand-written sm_100a kernels; there is no CPU
fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Iterable, List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N

__all__ = [
    "DataError", "IndexParams", "QueryOptions", "ScoredHit", "QueryResult", "BatchResult",
    "DeviceIndexView", "open_resident", "open_image", "synth_c5", "query", "query_batch",
    "build_classic", "build_compact", "build_image", "write_index", "KIND_CLASSIC",
    "KIND_COMPACT",
]

KIND_CLASSIC = 0  # proj/include/cobs/index_view.hpp:13
KIND_COMPACT = 1  # proj/include/cobs/index_view.hpp:14


class DataError(RuntimeError):
    """cobs::DataError (proj/include/cobs/error.hpp:12-14)."""


class CudaError(RuntimeError):
    """Device failure (no reference equivalent)."""


def _raise(code: int, err: C.Array) -> None:
    msg = err.value.decode(errors="replace")
    if code == N.EDATA:
        raise DataError(msg)
    if code == N.EUSAGE:
        raise ValueError(msg)
    raise CudaError(msg)


def _errbuf() -> C.Array:
    return C.create_string_buffer(1024)


def _take_bytes(ptr: C.c_void_p, n: int) -> bytes:
    """Copy n bytes from a library buffer (ctypes.string_at truncates sizes
    to a C int, so go through a numpy view)."""
    if n == 0:
        return b""
    return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint8)), shape=(n,)).tobytes()


@dataclass
class IndexParams:
    """proj/include/cobs/params.hpp:17-38."""
    q: int = 31
    k: int = 1
    p: float = 0.3
    canonical: bool = False
    block_size: int = 1024
    hash_scheme: int = 0

    def _c(self) -> N.IndexParamsC:
        c = N.IndexParamsC()
        c.q, c.k, c.p = self.q, self.k, self.p
        c.block_size = self.block_size
        c.canonical = 1 if self.canonical else 0
        c.hash_scheme = self.hash_scheme
        return c


@dataclass
class QueryOptions:
    """proj/include/cobs/query.hpp:22-29 (``workers`` has no GPU meaning)."""
    K: float = 0.9
    top_t: int = 0
    workers: int = 1


@dataclass
class ScoredHit:
    """proj/include/cobs/query.hpp:15-20."""
    doc_name: bytes
    score: int


@dataclass
class QueryResult:
    """proj/include/cobs/query.hpp:31-39."""
    ell: int = 0
    skipped: int = 0
    hits: List[ScoredHit] = field(default_factory=list)


@dataclass
class BatchResult:
    """One batched call: per-query arrays plus hit lists (global columns)."""
    ell: np.ndarray
    skipped: np.ndarray
    status: np.ndarray
    messages: List[str]
    hit_off: np.ndarray
    hit_n: np.ndarray
    docs: np.ndarray
    scores: np.ndarray
    dense: Optional[np.ndarray]  # n x total_docs, uint16/uint32, or None
    ms_termize: float
    ms_gather: float
    ms_order: float
    ms_total: float
    launches: int
    row_bytes: int
    h2d_index_bytes: int = 0
    gather_path: int = 0  # rows read from: 0 HBM, 1 host memory over PCIe (zero-copy), 2 streamed via HBM

    def hits(self, i: int) -> Tuple[np.ndarray, np.ndarray]:
        o, n = int(self.hit_off[i]), int(self.hit_n[i])
        return self.docs[o:o + n], self.scores[o:o + n]


class DeviceIndexView:
    """An index resident in HBM; the IndexView accessors of
    proj/include/cobs/index_view.hpp:18-47."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        self._names: Optional[List[bytes]] = None

    def close(self) -> None:
        if self._h:
            N.lib.cobs_gpu_index_close(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def column_offset(self) -> int:
        """File column of this index's first document (non-zero for a block
        shard opened with open_blocks)."""
        return int(N.lib.cobs_gpu_index_column_offset(self._h))

    def set_stream(self, stream_ptr: int) -> None:
        """Run this index's batches on a caller-owned cudaStream_t."""
        N.lib.cobs_gpu_index_set_stream(self._h, C.c_void_p(stream_ptr or None))

    # IndexView accessors
    def params(self) -> IndexParams:
        c = N.IndexParamsC()
        N.lib.cobs_gpu_index_params(self._h, C.byref(c))
        return IndexParams(c.q, c.k, c.p, bool(c.canonical), c.block_size, c.hash_scheme)

    def kind(self) -> int:
        return int(N.lib.cobs_gpu_index_kind(self._h))

    def block_count(self) -> int:
        return int(N.lib.cobs_gpu_index_block_count(self._h))

    def doc_count(self, b: int) -> int:
        return int(N.lib.cobs_gpu_index_doc_count(self._h, b))

    def width(self, b: int) -> int:
        return int(N.lib.cobs_gpu_index_width(self._h, b))

    def row_bytes(self, b: int) -> int:
        return int(N.lib.cobs_gpu_index_row_bytes(self._h, b))

    def total_docs(self) -> int:
        return int(N.lib.cobs_gpu_index_total_docs(self._h))

    def streaming(self) -> bool:
        return bool(N.lib.cobs_gpu_index_streaming(self._h))

    def device_bytes(self) -> int:
        return int(N.lib.cobs_gpu_index_device_bytes(self._h))

    def doc(self, b: int, i: int) -> Tuple[bytes, int]:
        name = C.c_char_p()
        ln = C.c_uint64()
        tc = C.c_uint64()
        rc = N.lib.cobs_gpu_index_doc(self._h, b, i, C.byref(name), C.byref(ln), C.byref(tc))
        if rc:
            raise IndexError((b, i))
        return C.string_at(name, ln.value), int(tc.value)

    def doc_names(self) -> List[bytes]:
        """Names of all documents in file column order."""
        if self._names is None:
            self._names = [self.doc(b, i)[0] for b in range(self.block_count())
                           for i in range(self.doc_count(b))]
        return self._names

    def row_data(self, b: int, r: int, byte_lo: int = 0, byte_hi: Optional[int] = None) -> bytes:
        hi = self.row_bytes(b) if byte_hi is None else byte_hi
        buf = (C.c_uint8 * max(hi - byte_lo, 1))()
        rc = N.lib.cobs_gpu_index_row(self._h, b, r, byte_lo, hi, buf)
        if rc:
            raise IndexError((b, r, byte_lo, hi))
        return bytes(buf)[: hi - byte_lo]


def open_resident(path: str, device: int = 0) -> DeviceIndexView:
    """cobs::open_resident (storage.hpp:19): parse, validate, upload to HBM."""
    h = C.c_void_p()
    err = _errbuf()
    rc = N.lib.cobs_gpu_index_open(str(path).encode(), device, C.byref(h), err, len(err))
    if rc:
        _raise(rc, err)
    return DeviceIndexView(h.value)


def open_random_access(path: str, hbm_budget: int, device: int = 0,
                       from_file: bool = False) -> DeviceIndexView:
    """Streaming mode when the pitched payload exceeds hbm_budget (the
    counterpart of cobs::open_random_access, storage.hpp:23): the payload in
    pinned host memory, or with from_file=True read from the file every
    batch (no host copy)."""
    h = C.c_void_p()
    err = _errbuf()
    fn = N.lib.cobs_gpu_index_open_file if from_file else N.lib.cobs_gpu_index_open_ex
    rc = fn(str(path).encode(), device, hbm_budget, C.byref(h), err, len(err))
    if rc:
        _raise(rc, err)
    return DeviceIndexView(h.value)


def open_blocks(path: str, block_lo: int, block_hi: int, device: int = 0) -> DeviceIndexView:
    """Blocks [block_lo, block_hi) of a compact index file as a standalone
    compact index in HBM -- one shard of a block-sharded index (SURVEY.md
    §8e).  Its hit columns are local; column_offset() maps them to file
    columns.  Merge shard results with dist.merge_block_shards."""
    h = C.c_void_p()
    err = _errbuf()
    rc = N.lib.cobs_gpu_index_open_blocks(str(path).encode(), device, block_lo, block_hi, C.byref(h),
                                          err, len(err))
    if rc:
        _raise(rc, err)
    return DeviceIndexView(h.value)


def open_image(image: bytes, device: int = 0, path: str = "<memory>",
               hbm_budget: int = 0) -> DeviceIndexView:
    """open_resident over an in-memory file image (streaming mode when the
    pitched payload exceeds a non-zero hbm_budget)."""
    h = C.c_void_p()
    err = _errbuf()
    buf = np.frombuffer(image, dtype=np.uint8)
    rc = N.lib.cobs_gpu_index_open_image_ex(buf.ctypes.data, len(image), path.encode(), device,
                                            hbm_budget, C.byref(h), err, len(err))
    if rc:
        _raise(rc, err)
    return DeviceIndexView(h.value)


def synth_c5(seed: int, n_docs: int = 100_000, block_size: int = 1024, median: float = 2.4e6,
             sigma: float = 0.5, p: float = 0.3, device: int = 0) -> DeviceIndexView:
    """The config-5 procedural compact index, generated directly in HBM."""
    h = C.c_void_p()
    err = _errbuf()
    rc = N.lib.cobs_gpu_index_synth_c5(seed, n_docs, block_size, median, sigma, p, device,
                                       C.byref(h), err, len(err))
    if rc:
        _raise(rc, err)
    return DeviceIndexView(h.value)


def synth_c5_blocks(seed: int, block_lo: int, block_hi: int, n_docs: int = 100_000,
                    block_size: int = 1024, median: float = 2.4e6, sigma: float = 0.5, p: float = 0.3,
                    device: int = 0) -> DeviceIndexView:
    """Blocks [block_lo, block_hi) of the config-5 index as a block shard
    (like open_blocks: hit columns are local, column_offset() maps them)."""
    h = C.c_void_p()
    err = _errbuf()
    rc = N.lib.cobs_gpu_index_synth_c5_blocks(seed, n_docs, block_size, median, sigma, p, block_lo,
                                              block_hi, device, C.byref(h), err, len(err))
    if rc:
        _raise(rc, err)
    return DeviceIndexView(h.value)


def write_index(view: DeviceIndexView, path: str) -> None:
    """cobs::write_index(const IndexView&, path) (storage.hpp:14)."""
    err = _errbuf()
    rc = N.lib.cobs_gpu_index_write(view._h, str(path).encode(), err, len(err))
    if rc:
        _raise(rc, err)


def index_image(view: DeviceIndexView) -> bytes:
    """The file image of a device-resident index (write_index into memory)."""
    img = C.c_void_p()
    ln = C.c_uint64()
    err = _errbuf()
    rc = N.lib.cobs_gpu_index_image(view._h, C.byref(img), C.byref(ln), err, len(err))
    if rc:
        _raise(rc, err)
    try:
        return _take_bytes(img, ln.value)
    finally:
        N.lib.cobs_gpu_free(img)


def index_image_array(view: DeviceIndexView) -> np.ndarray:
    """index_image into one uint8 array (no intermediate copies: images of
    tens of GB)."""
    ln = C.c_uint64()
    err = _errbuf()
    N.lib.cobs_gpu_index_image_into(view._h, None, 0, C.byref(ln), err, len(err))
    out = np.empty(ln.value, dtype=np.uint8)
    rc = N.lib.cobs_gpu_index_image_into(view._h, out.ctypes.data, ln.value, None, err, len(err))
    if rc:
        _raise(rc, err)
    return out


def pack_patterns(patterns: Sequence[bytes]) -> Tuple[np.ndarray, np.ndarray]:
    """Concatenate patterns into (bytes, offsets[n+1])."""
    lens = np.fromiter((len(p) for p in patterns), dtype=np.uint64, count=len(patterns))
    off = np.zeros(len(patterns) + 1, dtype=np.uint64)
    np.cumsum(lens, out=off[1:])
    buf = np.frombuffer(b"".join(patterns), dtype=np.uint8) if patterns else np.zeros(0, np.uint8)
    return buf, off


def query_batch_raw(view: DeviceIndexView, buf, offsets, K: float = 0.9, top_t: int = 0,
                    scores: bool = False, hits: bool = True, device_input: bool = False,
                    keep_device: bool = False, prune: bool = False) -> BatchResult:
    """Batched cobs::query over packed patterns.  ``buf``/``offsets`` are
    numpy arrays (host) or integer device addresses with device_input."""
    n = (len(offsets) - 1) if not device_input else int(offsets[1])
    if device_input:
        pbuf, poff = buf, offsets[0]
    else:
        buf = np.ascontiguousarray(buf, dtype=np.uint8)
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        pbuf, poff = buf.ctypes.data, offsets.ctypes.data
    flags = (N.Q_HITS if hits else 0) | (N.Q_SCORES if scores else 0)
    if device_input:
        flags |= N.Q_DEVICE_INPUT
    if keep_device:
        flags |= N.Q_KEEP_DEVICE
    if prune:
        flags |= N.Q_PRUNE
    r = C.c_void_p()
    err = _errbuf()
    rc = N.lib.cobs_gpu_query_batch(view._h, pbuf, poff, n, K, top_t, flags, C.byref(r), err,
                                    len(err))
    if rc:
        _raise(rc, err)
    owner = _Results(r)
    ell, sk, st, ho, hn, dd, ss = (N.u32p(), N.u64p(), C.POINTER(C.c_int)(), N.u64p(),
                                   N.u64p(), N.u32p(), N.u32p())
    total = C.c_uint64()
    N.lib.cobs_gpu_results_arrays(r, C.byref(ell), C.byref(sk), C.byref(st), C.byref(ho),
                                  C.byref(hn), C.byref(dd), C.byref(ss), C.byref(total))

    def arr(ptr, count, dtype):
        if count == 0 or not ptr:
            return np.zeros(0, dtype=dtype)
        return np.ctypeslib.as_array(ptr, shape=(count,)).astype(dtype, copy=True)

    def wrap(ptr, count, ctype):
        """The library's result array itself (no copy): the numpy array
        keeps the results alive, which are freed with the last such array."""
        if count == 0 or not ptr:
            return np.zeros(0, dtype=np.uint16 if ctype is C.c_uint16 else np.uint32)
        buf = (ctype * count).from_address(C.cast(ptr, C.c_void_p).value)
        buf._owner = owner
        return np.ctypeslib.as_array(buf)

    res_ell = arr(ell, n, np.uint32)
    res_sk = arr(sk, n, np.uint64)
    res_st = arr(st, n, np.int32)
    messages = [""] * n
    for i in np.nonzero(res_st)[0].tolist():  # only the failed queries carry text
        msg = C.c_char_p()
        N.lib.cobs_gpu_results_query(r, i, None, None, None, C.byref(msg), None)
        messages[i] = msg.value.decode()
    dense = None
    if scores and not keep_device:
        sb = C.c_uint32()
        p = N.lib.cobs_gpu_results_scores(r, C.byref(sb))
        D = view.total_docs()
        dt = np.uint16 if sb.value == 2 else np.uint32
        if p and n * D:
            dense = wrap(p, n * D, C.c_uint16 if sb.value == 2 else C.c_uint32).reshape(n, D)
        else:
            dense = np.zeros((n, D), dtype=dt)
    t = [C.c_double(), C.c_double(), C.c_double(), C.c_double()]
    N.lib.cobs_gpu_results_timing(r, *(C.byref(x) for x in t))
    return BatchResult(
        ell=res_ell, skipped=res_sk, status=res_st, messages=messages,
        hit_off=arr(ho, n, np.uint64), hit_n=arr(hn, n, np.uint64),
        docs=wrap(dd, total.value, C.c_uint32), scores=wrap(ss, total.value, C.c_uint32),
        dense=dense, ms_termize=t[0].value, ms_gather=t[1].value, ms_order=t[2].value,
        ms_total=t[3].value, launches=int(N.lib.cobs_gpu_results_launches(r)),
        row_bytes=int(N.lib.cobs_gpu_results_row_bytes(r)),
        h2d_index_bytes=int(N.lib.cobs_gpu_results_h2d_index_bytes(r)),
        gather_path=int(N.lib.cobs_gpu_results_gather_path(r)))


class _Results:
    """Owns a cobs_gpu_results handle; freed when the last array viewing
    its hit / score buffers is gone."""
    def __init__(self, handle: C.c_void_p):
        self._h = handle

    def __del__(self):
        if self._h:
            N.lib.cobs_gpu_results_free(self._h)
            self._h = None


def query_batch(view: DeviceIndexView, patterns: Sequence[bytes], K: float = 0.9,
                top_t: int = 0, scores: bool = False) -> BatchResult:
    buf, off = pack_patterns(patterns)
    return query_batch_raw(view, buf, off, K, top_t, scores=scores)


def query(view: DeviceIndexView, pattern: bytes, opts: QueryOptions = QueryOptions()) -> QueryResult:
    """cobs::query (query.hpp:46-47): raises ValueError for K outside (0,1],
    DataError when the pattern yields no terms (query.cpp:125-138)."""
    if isinstance(pattern, str):
        pattern = pattern.encode()
    b = query_batch(view, [pattern], opts.K, opts.top_t)
    if b.status[0]:
        raise DataError(b.messages[0])
    names = view.doc_names()
    d, s = b.hits(0)
    return QueryResult(int(b.ell[0]), int(b.skipped[0]),
                       [ScoredHit(names[int(x)], int(y)) for x, y in zip(d, s)])


Document = Tuple[bytes, Sequence[bytes]]  # (name, content strings)


def _pack_docs(docs: Sequence[Document]):
    """Names, one host pointer per content string (COBS_B_SEGMENT_PTRS: the
    library gathers the strings into HBM itself, no packed copy here), the
    strings' packed offsets and each document's string range."""
    names, segs, doc_segs = [], [], [0]
    for name, content in docs:
        names.append(name if isinstance(name, bytes) else name.encode())
        for c in content:
            segs.append(bytes(c) if not isinstance(c, (bytes, str)) else c if isinstance(c, bytes) else c.encode())
        doc_segs.append(len(segs))
    lens = np.fromiter((len(s) for s in segs), dtype=np.uint64, count=len(segs))
    seg_off = np.zeros(len(segs) + 1, dtype=np.uint64)
    np.cumsum(lens, out=seg_off[1:])
    ptrs = (C.c_char_p * max(len(segs), 1))(*segs)  # (keeps the strings alive)
    return names, ptrs, seg_off, np.asarray(doc_segs, dtype=np.uint64)


def build_image(docs: Sequence[Document], params: IndexParams, kind: int, forced_w: int = 0,
                path: Optional[str] = None, device: int = 0) -> bytes:
    """extract_terms + build_{classic,compact} + write_index on the device;
    returns the file image (byte-identical to the reference writer's)."""
    names, buf, seg_off, doc_segs = _pack_docs(docs)
    name_arr = (C.c_char_p * max(len(names), 1))(*names)
    img = C.c_void_p()
    ln = C.c_uint64()
    err = _errbuf()
    cp = params._c()
    rc = N.lib.cobs_gpu_build_ex(C.cast(buf, C.c_void_p), seg_off.ctypes.data, len(seg_off) - 1,
                                 doc_segs.ctypes.data, name_arr, len(names), C.byref(cp), kind,
                                 forced_w, device, N.B_SEGMENT_PTRS, str(path).encode() if path else None,
                                 C.byref(img), C.byref(ln), None, err, len(err))
    if rc:
        _raise(rc, err)
    try:
        return _take_bytes(img, ln.value)
    finally:
        N.lib.cobs_gpu_free(img)


def build_classic(docs: Sequence[Document], params: IndexParams = IndexParams(),
                  forced_w: int = 0, path: Optional[str] = None, device: int = 0) -> bytes:
    """build_classic (classic_index.hpp:37-39) + write_index."""
    return build_image(docs, params, KIND_CLASSIC, forced_w, path, device)


def build_compact(docs: Sequence[Document], params: IndexParams = IndexParams(),
                  path: Optional[str] = None, device: int = 0) -> bytes:
    """build_compact (compact_index.hpp:26-27) + write_index."""
    return build_image(docs, params, KIND_COMPACT, 0, path, device)


def build_device(seqs, seg_off: np.ndarray, doc_segs: np.ndarray, names: Sequence[bytes],
                 params: IndexParams, kind: int, forced_w: int = 0, device: int = 0,
                 seqs_on_device: bool = False, want_image: bool = False,
                 path: Optional[str] = None) -> Tuple[DeviceIndexView, Optional[bytes]]:
    """Build and keep the index resident in HBM (ready to query).  ``seqs`` is
    a host numpy uint8 array or, with seqs_on_device, a device address."""
    seg_off = np.ascontiguousarray(seg_off, np.uint64)
    doc_segs = np.ascontiguousarray(doc_segs, np.uint64)
    nm = (C.c_char_p * max(len(names), 1))(*[n if isinstance(n, bytes) else n.encode() for n in names])
    h = C.c_void_p()
    img = C.c_void_p()
    ln = C.c_uint64()
    err = _errbuf()
    cp = params._c()
    sp = seqs if seqs_on_device else np.ascontiguousarray(seqs, np.uint8).ctypes.data
    rc = N.lib.cobs_gpu_build_ex(sp, seg_off.ctypes.data, len(seg_off) - 1, doc_segs.ctypes.data,
                                 nm, len(names), C.byref(cp), kind, forced_w, device,
                                 N.B_DEVICE_INPUT if seqs_on_device else 0,
                                 str(path).encode() if path else None,
                                 C.byref(img) if want_image else None,
                                 C.byref(ln) if want_image else None, C.byref(h), err, len(err))
    if rc:
        _raise(rc, err)
    image = None
    if want_image:
        try:
            image = _take_bytes(img, ln.value)
        finally:
            N.lib.cobs_gpu_free(img)
    return DeviceIndexView(h.value), image


def build_from_terms(termsets: Sequence[Tuple[bytes, Sequence[bytes]]], params: IndexParams,
                     kind: int, forced_w: int = 0, path: Optional[str] = None,
                     device: int = 0) -> bytes:
    """build_classic / build_compact over pre-extracted TermSets
    (classic_index.hpp:37-44, compact_index.hpp:26-27): each (name, terms)
    pair is a TermSet; terms are hashed as given and term_count = len(terms).
    A term whose length is not q raises ValueError with the reference's
    message (classic_index.cpp:49-56).  Returns the file image."""
    names, buf, seg_off, doc_segs = _pack_docs(termsets)
    nm = (C.c_char_p * max(len(names), 1))(*names)
    img = C.c_void_p()
    ln = C.c_uint64()
    err = _errbuf()
    cp = params._c()
    rc = N.lib.cobs_gpu_build_ex(C.cast(buf, C.c_void_p), seg_off.ctypes.data, len(seg_off) - 1,
                                 doc_segs.ctypes.data, nm, len(names), C.byref(cp), kind, forced_w,
                                 device, N.B_TERMS | N.B_SEGMENT_PTRS, str(path).encode() if path else None,
                                 C.byref(img), C.byref(ln), None, err, len(err))
    if rc:
        _raise(rc, err)
    try:
        return _take_bytes(img, ln.value)
    finally:
        N.lib.cobs_gpu_free(img)


def calibrate(device: int = 0, nbytes: int = 16 << 30) -> Tuple[float, float]:
    """(streaming read GB/s, random 128-byte line GB/s) on this GPU: the
    same-box ceiling the gather kernel is compared against in bench.py."""
    a, b = C.c_double(), C.c_double()
    rc = N.lib.cobs_gpu_calibrate(device, nbytes, C.byref(a), C.byref(b))
    if rc:
        raise CudaError("calibration failed")
    return a.value, b.value


def synth_docs_device(seed: int, alpha: int, lengths: np.ndarray, dev_ptr: int, device: int = 0,
                      lo: int = 0, hi: Optional[int] = None) -> None:
    """Generate seeded documents [lo, hi) straight into device memory."""
    lengths = np.ascontiguousarray(lengths, np.uint64)
    hi = len(lengths) if hi is None else hi
    rc = N.lib.cobs_gpu_synth_docs(seed, alpha, lengths.ctypes.data, lo, hi, dev_ptr, device)
    if rc:
        raise CudaError("synth_docs failed")


def merge_classic(a: DeviceIndexView, b: DeviceIndexView, device: int = 0) -> DeviceIndexView:
    """merge_classic (classic_index.hpp:46-49) on the device."""
    h = C.c_void_p()
    err = _errbuf()
    rc = N.lib.cobs_gpu_merge_classic(a._h, b._h, device, C.byref(h), err, len(err))
    if rc:
        _raise(rc, err)
    return DeviceIndexView(h.value)


FORMAT_AUTO, FORMAT_FASTA, FORMAT_TEXT = 0, 1, 2


def query_fasta(view: DeviceIndexView, fasta_path: str, K: float = 0.9, top_t: int = 0) -> bytes:
    """`cobs query index -F queries.fa`: the CLI's batch TSV, byte for byte."""
    out = C.c_void_p()
    ln = C.c_uint64()
    err = _errbuf()
    rc = N.lib.cobs_gpu_query_fasta(view._h, str(fasta_path).encode(), K, top_t, C.byref(out),
                                    C.byref(ln), err, len(err))
    if rc:
        _raise(rc, err)
    try:
        return _take_bytes(out, ln.value)
    finally:
        N.lib.cobs_gpu_free(out)


def build_files(inputs: Sequence[str], params: IndexParams = IndexParams(), kind: int = KIND_COMPACT,
                format: int = FORMAT_AUTO, path: Optional[str] = None, device: int = 0) -> bytes:
    """`cobs build inputs... --mode classic|compact`: returns the file image."""
    arr = (C.c_char_p * max(len(inputs), 1))(*[str(i).encode() for i in inputs])
    img = C.c_void_p()
    ln = C.c_uint64()
    err = _errbuf()
    cp = params._c()
    rc = N.lib.cobs_gpu_build_files(arr, len(inputs), C.byref(cp), kind, format, device,
                                    str(path).encode() if path else None, C.byref(img),
                                    C.byref(ln), err, len(err))
    if rc:
        _raise(rc, err)
    try:
        return _take_bytes(img, ln.value)
    finally:
        N.lib.cobs_gpu_free(img)


def last_build_timing() -> Tuple[float, float, float]:
    a, b, c = C.c_double(), C.c_double(), C.c_double()
    N.lib.cobs_gpu_build_timing(C.byref(a), C.byref(b), C.byref(c))
    return a.value, b.value, c.value


def trim() -> int:
    """Release the device memory kept between calls (the build's count
    workspace); returns the bytes released."""
    return int(N.lib.cobs_gpu_trim())


def last_build_timing_ex() -> dict:
    """ms of the last build's legs: h2d, count, fill, d2h, total."""
    v = [C.c_double() for _ in range(5)]
    N.lib.cobs_gpu_build_timing_ex(*(C.byref(x) for x in v))
    t = dict(zip(("ms_h2d", "ms_count", "ms_fill", "ms_d2h", "ms_total"), (x.value for x in v)))
    w = [C.c_double() for _ in range(3)]  # the count leg: kernels alone, workspace cudaMalloc / cudaFree
    N.lib.cobs_gpu_build_timing_count(*(C.byref(x) for x in w))
    t.update(zip(("ms_count_kernels", "ms_count_alloc", "ms_count_free"), (x.value for x in w)))
    return t
