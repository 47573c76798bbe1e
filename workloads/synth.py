"""Seeded synthetic workloads for the five BASELINE.json configs.

Input generation only (paper_1905_09624_b200/csrc/synth.h through
workloads/_lib/libcobs_synth.so); the same header drives the device
generators, so host and device see identical bytes.
No public dataset is used: the paper's 100k-sample McCortex corpus and its
query sets are absent, and these seeded inputs take their shapes instead
(DESIGN.md §7).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, replace
from typing import Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_lib", "libcobs_synth.so")


class _Lib:
    """The generator's C ABI (workloads/synth_host.c over csrc/synth.h),
    bound on first use.  `bind(path)` selects another build of the same
    functions: bench.py's reference arm binds the oracle library's copy so
    that process loads nothing outside oracle/ (no product code)."""
    def __init__(self):
        self.h = None

    def bind(self, path: str) -> None:
        h = C.CDLL(path)
        _declare(h)
        self.h = h

    def __getattr__(self, name):
        if self.h is None:
            if not os.path.exists(_SO):
                raise ImportError(f"{_SO} missing: run `make lib`")
            self.bind(_SO)
        return getattr(self.h, name)


_lib = _Lib()


def bind(path: str) -> None:
    _lib.bind(path)

DNA, AA = 0, 1
Q_RANDOM, Q_SUBST, Q_INDEL = 0, 1, 2
LEN_FIXED, LEN_LOGUNIFORM, LEN_LOGNORMAL = 0, 1, 2


class QuerySpecC(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("alpha", C.c_int), ("n_queries", C.c_uint64),
                ("qlen", C.c_uint64), ("kind", C.c_int), ("edit_per_65536", C.c_uint32),
                ("mixed", C.c_int)]


def _declare(h) -> None:
    h.syn_c_doc_lengths.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_double, C.c_double,
                                    C.c_uint64, C.c_void_p]
    h.syn_c_c5_term_counts.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_double, C.c_void_p]
    h.syn_c_c5_thr16.argtypes = [C.c_uint64, C.c_uint64]
    h.syn_c_c5_thr16.restype = C.c_uint32
    h.syn_c_c5_row.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32,
                               C.c_uint64, C.c_void_p]
    h.syn_c_docs.argtypes = [C.c_uint64, C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p,
                             C.c_int]
    h.syn_c_queries.argtypes = [C.POINTER(QuerySpecC), C.c_void_p, C.c_uint64, C.c_void_p,
                                C.c_uint64, C.c_void_p, C.c_int]


@dataclass(frozen=True)
class Config:
    name: str
    kind: int                 # 0 classic, 1 compact
    n_docs: int
    alpha: int
    len_dist: int
    len_a: float
    len_b: float
    q: int
    k: int
    p: float
    canonical: bool
    block_size: int
    n_queries: int
    qlen: int
    qkind: int
    edit: float
    K: float
    seed: int = 1905_09624
    # config 5 only (procedural index): log-normal term counts
    c5_median: float = 0.0
    c5_sigma: float = 0.0


# The five BASELINE.json configs.  C5 holds the "~100 GB resident" total and
# the log-normal shape with median 2.4M distinct 31-mers (sigma 0.5): the
# stated 4.5M median would need >= 158 GB even with zero spread.
CONFIGS = {
    "c1": Config("c1", 0, 1000, DNA, LEN_FIXED, 100_000, 0, 31, 1, 0.3, False, 1024,
                 1000, 1000, Q_SUBST, 0.01, 0.8),
    "c2": Config("c2", 0, 10_000, DNA, LEN_LOGUNIFORM, 5e4, 5e6, 31, 3, 0.3, False, 1024,
                 10_000, 200, Q_SUBST, 0.02, 0.7),
    "c3": Config("c3", 1, 20_000, DNA, LEN_LOGNORMAL, 3e6, 0.6, 31, 1, 0.3, True, 1024,
                 5000, 10_000, Q_INDEL, 0.08, 0.5),
    "c4": Config("c4", 0, 50_000, AA, LEN_FIXED, 300_000, 0, 10, 2, 0.1, False, 1024,
                 50_000, 100, Q_SUBST, 0.05, 0.9),
    "c5": Config("c5", 1, 100_000, DNA, LEN_FIXED, 0, 0, 31, 1, 0.3, False, 1024,
                 100_000, 1000, Q_RANDOM, 0.0, 0.8, c5_median=2.4e6, c5_sigma=0.5),
}


def scaled(cfg: Config, n_docs: int, len_scale: float = 1.0, n_queries: Optional[int] = None,
           **kw) -> Config:
    """A smaller instance of a config with the same shape (for parity tests)."""
    c = replace(cfg, n_docs=n_docs,
                n_queries=n_queries if n_queries is not None else cfg.n_queries, **kw)
    if cfg.len_dist == LEN_FIXED:
        c = replace(c, len_a=max(cfg.q, int(cfg.len_a * len_scale)))
    elif cfg.len_dist == LEN_LOGUNIFORM:
        c = replace(c, len_a=cfg.len_a * len_scale, len_b=cfg.len_b * len_scale)
    else:
        c = replace(c, len_a=cfg.len_a * len_scale)
    return c


def doc_lengths(cfg: Config) -> np.ndarray:
    out = np.zeros(cfg.n_docs, dtype=np.uint64)
    _lib.syn_c_doc_lengths(cfg.seed, cfg.n_docs, cfg.len_dist, float(cfg.len_a),
                           float(cfg.len_b), cfg.q, out.ctypes.data)
    return out


def doc_names(cfg: Config, ids: Optional[Sequence[int]] = None) -> list:
    width = max(4, len(str(cfg.n_docs - 1)))
    ids = range(cfg.n_docs) if ids is None else ids
    return [b"doc" + str(i).zfill(width).encode() for i in ids]


def docs(cfg: Config, ids: Optional[Sequence[int]] = None, lengths: Optional[np.ndarray] = None,
         threads: int = 0) -> Tuple[np.ndarray, np.ndarray]:
    """Bytes of documents `ids` concatenated, and offsets[n+1]."""
    lengths = doc_lengths(cfg) if lengths is None else lengths
    ids = np.arange(cfg.n_docs, dtype=np.uint64) if ids is None else np.asarray(ids, np.uint64)
    off = np.zeros(len(ids) + 1, dtype=np.uint64)
    np.cumsum(lengths[ids.astype(np.int64)], out=off[1:])
    buf = np.empty(int(off[-1]), dtype=np.uint8)
    _lib.syn_c_docs(cfg.seed, cfg.alpha, ids.ctypes.data, off.ctypes.data, len(ids),
                    buf.ctypes.data, threads or (os.cpu_count() or 1))
    return buf, off


def queries(cfg: Config, ids: Optional[Sequence[int]] = None, lengths: Optional[np.ndarray] = None,
            threads: int = 0) -> Tuple[np.ndarray, np.ndarray]:
    """Query batch (or the subset `ids`): packed bytes and offsets[n+1].
    C5's query-only documents have no sequences: all its queries are random."""
    ids = np.arange(cfg.n_queries, dtype=np.uint64) if ids is None else np.asarray(ids, np.uint64)
    if lengths is None:
        lengths = doc_lengths(cfg) if cfg.qkind != Q_RANDOM else np.ones(1, np.uint64)
    spec = QuerySpecC(cfg.seed, cfg.alpha, cfg.n_queries, cfg.qlen,
                      cfg.qkind if cfg.qkind != Q_RANDOM else Q_SUBST,
                      int(round(cfg.edit * 65536)), 1 if cfg.qkind != Q_RANDOM else 0)
    buf = np.empty(len(ids) * cfg.qlen, dtype=np.uint8)
    _lib.syn_c_queries(C.byref(spec), lengths.ctypes.data, len(lengths), ids.ctypes.data,
                       len(ids), buf.ctypes.data, threads or (os.cpu_count() or 1))
    off = np.arange(len(ids) + 1, dtype=np.uint64) * np.uint64(cfg.qlen)
    return buf, off


def c5_term_counts(cfg: Config) -> np.ndarray:
    out = np.zeros(cfg.n_docs, dtype=np.uint64)
    _lib.syn_c_c5_term_counts(cfg.seed, cfg.n_docs, cfg.c5_median, cfg.c5_sigma, out.ctypes.data)
    return out


def c5_row(seed: int, block: int, row: int, rb: int, thr16: int, dc: int) -> bytes:
    out = (C.c_uint8 * rb)()
    _lib.syn_c_c5_row(seed, block, row, rb, thr16, dc, out)
    return bytes(out)


def c5_thr16(w: int, n: int) -> int:
    return int(_lib.syn_c_c5_thr16(w, n))
