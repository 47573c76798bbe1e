"""ctypes binding of the C-ABI in include/cobs_gpu.h.

The product path has no fallback: if ``_lib/libcobs_gpu.so`` is missing the
import fails loudly (build it with ``python -c "import __graft_entry__ as g;
g.build()"`` or ``make lib``).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("COBS_GPU_LIB") or os.path.join(_HERE, "_lib", "libcobs_gpu.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"cobs-b200 native library not built: {LIB_PATH} is missing "
        "(run `make lib` or __graft_entry__.build()); there is no CPU fallback")

lib = C.CDLL(LIB_PATH)

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
vp = C.c_void_p


class IndexParamsC(C.Structure):
    _fields_ = [("q", C.c_uint32), ("k", C.c_uint32), ("p", C.c_double),
                ("block_size", C.c_uint64), ("canonical", C.c_uint8),
                ("hash_scheme", C.c_uint8), ("reserved", C.c_uint8 * 6)]


def _sig(name, res, args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = args
    return f


# Every symbol declared in include/cobs_gpu.h (tests/test_capi_symbols.py checks
# this list against the header).
SIGNATURES = {
    "cobs_gpu_version": (C.c_char_p, []),
    "cobs_gpu_index_open": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(vp), C.c_char_p, C.c_size_t]),
    "cobs_gpu_index_open_image": (C.c_int, [vp, C.c_uint64, C.c_char_p, C.c_int, C.POINTER(vp),
                                            C.c_char_p, C.c_size_t]),
    "cobs_gpu_index_open_ex": (C.c_int, [C.c_char_p, C.c_int, C.c_uint64, C.POINTER(vp), C.c_char_p,
                                         C.c_size_t]),
    "cobs_gpu_index_open_image_ex": (C.c_int, [vp, C.c_uint64, C.c_char_p, C.c_int, C.c_uint64,
                                               C.POINTER(vp), C.c_char_p, C.c_size_t]),
    "cobs_gpu_index_streaming": (C.c_int, [vp]),
    "cobs_gpu_index_close": (None, [vp]),
    "cobs_gpu_index_set_stream": (C.c_int, [vp, vp]),
    "cobs_gpu_index_params": (C.c_int, [vp, C.POINTER(IndexParamsC)]),
    "cobs_gpu_index_kind": (C.c_uint8, [vp]),
    "cobs_gpu_index_block_count": (C.c_uint64, [vp]),
    "cobs_gpu_index_doc_count": (C.c_uint64, [vp, C.c_uint64]),
    "cobs_gpu_index_width": (C.c_uint64, [vp, C.c_uint64]),
    "cobs_gpu_index_row_bytes": (C.c_uint64, [vp, C.c_uint64]),
    "cobs_gpu_index_total_docs": (C.c_uint64, [vp]),
    "cobs_gpu_index_doc": (C.c_int, [vp, C.c_uint64, C.c_uint64, C.POINTER(C.c_char_p),
                                     C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "cobs_gpu_index_doc_global": (C.c_uint64, [vp, C.c_uint64, C.c_uint64]),
    "cobs_gpu_index_device_bytes": (C.c_uint64, [vp]),
    "cobs_gpu_index_row": (C.c_int, [vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, vp]),
    "cobs_gpu_index_write": (C.c_int, [vp, C.c_char_p, C.c_char_p, C.c_size_t]),
    "cobs_gpu_index_image_into": (C.c_int, [vp, vp, C.c_uint64, C.POINTER(C.c_uint64), C.c_char_p,
                                            C.c_size_t]),
    "cobs_gpu_index_image": (C.c_int, [vp, C.POINTER(vp), C.POINTER(C.c_uint64), C.c_char_p,
                                       C.c_size_t]),
    "cobs_gpu_query_batch": (C.c_int, [vp, vp, vp, C.c_uint64, C.c_double, C.c_uint64, C.c_uint32,
                                       C.POINTER(vp), C.c_char_p, C.c_size_t]),
    "cobs_gpu_results_count": (C.c_uint64, [vp]),
    "cobs_gpu_results_query": (C.c_int, [vp, C.c_uint64, C.POINTER(C.c_uint64),
                                         C.POINTER(C.c_uint64), C.POINTER(C.c_int),
                                         C.POINTER(C.c_char_p), C.POINTER(C.c_uint64)]),
    "cobs_gpu_results_hits": (C.c_int, [vp, C.c_uint64, C.POINTER(u32p), C.POINTER(u32p)]),
    "cobs_gpu_results_arrays": (C.c_int, [vp, C.POINTER(u32p), C.POINTER(u64p),
                                          C.POINTER(C.POINTER(C.c_int)), C.POINTER(u64p),
                                          C.POINTER(u64p), C.POINTER(u32p), C.POINTER(u32p),
                                          C.POINTER(C.c_uint64)]),
    "cobs_gpu_results_scores": (vp, [vp, C.POINTER(C.c_uint32)]),
    "cobs_gpu_results_timing": (C.c_int, [vp, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                          C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "cobs_gpu_results_launches": (C.c_uint32, [vp]),
    "cobs_gpu_results_row_bytes": (C.c_uint64, [vp]),
    "cobs_gpu_results_gather_path": (C.c_uint32, [vp]),
    "cobs_gpu_results_h2d_index_bytes": (C.c_uint64, [vp]),
    "cobs_gpu_results_free": (None, [vp]),
    "cobs_gpu_build": (C.c_int, [vp, vp, C.c_uint64, vp, C.POINTER(C.c_char_p), C.c_uint64,
                                 C.POINTER(IndexParamsC), C.c_int, C.c_uint64, C.c_int, C.c_char_p,
                                 C.POINTER(vp), C.POINTER(C.c_uint64), C.c_char_p, C.c_size_t]),
    "cobs_gpu_build_ex": (C.c_int, [vp, vp, C.c_uint64, vp, C.POINTER(C.c_char_p), C.c_uint64,
                                    C.POINTER(IndexParamsC), C.c_int, C.c_uint64, C.c_int,
                                    C.c_uint32, C.c_char_p, C.POINTER(vp), C.POINTER(C.c_uint64),
                                    C.POINTER(vp), C.c_char_p, C.c_size_t]),
    "cobs_gpu_merge_classic": (C.c_int, [vp, vp, C.c_int, C.POINTER(vp), C.c_char_p, C.c_size_t]),
    "cobs_gpu_query_fasta": (C.c_int, [vp, C.c_char_p, C.c_double, C.c_uint64, C.POINTER(vp),
                                       C.POINTER(C.c_uint64), C.c_char_p, C.c_size_t]),
    "cobs_gpu_build_files": (C.c_int, [C.POINTER(C.c_char_p), C.c_uint64, C.POINTER(IndexParamsC),
                                       C.c_int, C.c_int, C.c_int, C.c_char_p, C.POINTER(vp),
                                       C.POINTER(C.c_uint64), C.c_char_p, C.c_size_t]),
    "cobs_gpu_build_timing": (C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_double),
                                        C.POINTER(C.c_double)]),
    "cobs_gpu_build_timing_ex": (C.c_int, [C.POINTER(C.c_double)] * 5),
    "cobs_gpu_build_timing_count": (C.c_int, [C.POINTER(C.c_double)] * 3),
    "cobs_gpu_trim": (C.c_uint64, []),
    "cobs_gpu_free": (None, [vp]),
    "cobs_gpu_index_synth_c5": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_double,
                                          C.c_double, C.c_double, C.c_int, C.POINTER(vp),
                                          C.c_char_p, C.c_size_t]),
    "cobs_gpu_index_synth_c5_blocks": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_double,
                                                 C.c_double, C.c_double, C.c_uint64, C.c_uint64,
                                                 C.c_int, C.POINTER(vp), C.c_char_p, C.c_size_t]),
    "cobs_gpu_index_open_file": (C.c_int, [C.c_char_p, C.c_int, C.c_uint64, C.POINTER(vp), C.c_char_p,
                                           C.c_size_t]),
    "cobs_gpu_index_open_blocks": (C.c_int, [C.c_char_p, C.c_int, C.c_uint64, C.c_uint64, C.POINTER(vp),
                                             C.c_char_p, C.c_size_t]),
    "cobs_gpu_index_column_offset": (C.c_uint64, [vp]),
    "cobs_gpu_calibrate": (C.c_int, [C.c_int, C.c_uint64, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "cobs_gpu_synth_docs": (C.c_int, [C.c_uint64, C.c_int, vp, C.c_uint64, C.c_uint64, vp,
                                      C.c_int]),
}

for _name, (_res, _args) in SIGNATURES.items():
    _sig(_name, _res, _args)

OK, EUSAGE, EDATA, ECUDA = 0, 1, 2, 4
Q_HITS, Q_SCORES, Q_DEVICE_INPUT, Q_KEEP_DEVICE, Q_PRUNE = 1, 2, 4, 8, 16
B_DEVICE_INPUT, B_TERMS, B_SEGMENT_PTRS = 1, 2, 4
