"""ctypes bindings for the two native libraries of the package.

* ``lib/libtrigpu.so``  -- the sm_100a engine behind ``include/trigpu.h``.
* ``lib/libtrihost.so`` -- host input prep: the reference's orderings and cost
  report (compiled unchanged) plus the synthetic generators
  (``csrc/host/trihost.h``).

Both are built in-tree by ``make`` (``__graft_entry__.build()``). There is no
fallback: a missing library raises ``NativeLibraryMissing``.
"""
from __future__ import annotations

import ctypes as C
import os
from functools import lru_cache

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_HERE, "lib")
# TRIGPU_LIB_SUFFIX selects an experimental build (e.g. "_win") for A/B timing
TRIGPU_PATH = os.path.join(LIB_DIR, "libtrigpu%s.so" % os.environ.get("TRIGPU_LIB_SUFFIX", ""))
TRIHOST_PATH = os.path.join(LIB_DIR, "libtrihost.so")

# include/trigpu.h
TL_OK = 0
TL_ERR_INVALID_ARGUMENT = 1
TL_ERR_CUDA = 2
TL_ERR_OUT_OF_MEMORY = 3
TL_ERR_STATE = 4
TL_ERR_CAPACITY = 5
TL_ALGO_APP = 0
TL_ALGO_APM = 1
TL_ORDER_DEGREE = 0
TL_ORDER_SPLIT = 1
TL_ORDER_CORE = 2
TL_OUT_COUNT = 0
TL_OUT_CHECKSUM = 1
TL_OUT_VERTEX_COUNTS = 2
TL_OUT_LIST = 4
TL_DEBUG_BM_SHRINK = 1
TL_DEBUG_VARIANT = 2
TL_DEBUG_CLASS_WORK = 3
TL_DEBUG_H_WIDE_MIN_N = 4
TL_DEBUG_H_SPLIT = 5

# every exported symbol of include/trigpu.h (tests check the .so exports all)
TRIGPU_SYMBOLS = (
    "tl_version", "tl_create", "tl_destroy", "tl_last_error", "tl_orient",
    "tl_orient_device", "tl_check_sizes", "tl_list", "tl_fetch_triangles",
    "tl_fetch_vertex_counts", "tl_fetch_oriented", "tl_cost_report",
    "tl_host_register", "tl_host_unregister", "tl_phase_times", "tl_phase_name",
    "tl_timer_start", "tl_timer_stop", "tl_order", "tl_order_device", "tl_orient_ordered",
    "tl_fetch_ranks", "tl_normalize", "tl_fetch_graph", "tl_orient_normalized",
    "tl_fetch_triangles_range", "tl_fetch_triangle_labels", "tl_debug_set", "tl_list_range",
    "tl_core_decompose", "tl_core_decompose_device",
)


class NativeLibraryMissing(RuntimeError):
    pass


class TlStats(C.Structure):
    _fields_ = [
        ("triangle_count", C.c_uint64),
        ("inner_ops", C.c_uint64),
        ("mark_ops", C.c_uint64),
        ("checksum", C.c_uint64),
        ("c_pp", C.c_uint64),
        ("c_pm", C.c_uint64),
        ("c_mm", C.c_uint64),
        ("sum_deg_sq", C.c_uint64),
        ("orient_ms", C.c_double),
        ("list_ms", C.c_double),
        ("h2d_ms", C.c_double),
        ("kernel_launches", C.c_uint64),
    ]


class ThCsr(C.Structure):
    _fields_ = [
        ("n", C.c_uint32),
        ("m", C.c_uint64),
        ("offsets", C.POINTER(C.c_uint64)),
        ("adj", C.POINTER(C.c_uint32)),
    ]


_vp = C.c_void_p
_u32 = C.c_uint32
_u64 = C.c_uint64


def use_library_variant(suffix: str) -> None:
    """Switch later trigpu() calls to lib/libtrigpu<suffix>.so (A/B timing of
    tuning builds, tools/ab.py); contexts created before keep their library."""
    global TRIGPU_PATH
    TRIGPU_PATH = os.path.join(LIB_DIR, "libtrigpu%s.so" % suffix)
    trigpu.cache_clear()


@lru_cache(maxsize=None)
def trigpu() -> C.CDLL:
    if not os.path.exists(TRIGPU_PATH):
        raise NativeLibraryMissing(
            f"{TRIGPU_PATH} is missing: run `make gpu` (or __graft_entry__.build()); "
            "there is no CPU fallback for the listing engine")
    lib = C.CDLL(TRIGPU_PATH)
    lib.tl_version.restype = C.c_int
    lib.tl_create.argtypes = [C.POINTER(_vp), C.c_int]
    lib.tl_create.restype = C.c_int
    lib.tl_destroy.argtypes = [_vp]
    lib.tl_destroy.restype = None
    lib.tl_last_error.argtypes = [_vp]
    lib.tl_last_error.restype = C.c_char_p
    lib.tl_orient.argtypes = [_vp, _u32, _u64, _vp, _vp, _vp]
    lib.tl_orient.restype = C.c_int
    lib.tl_orient_device.argtypes = [_vp, _u32, _u64, _vp, _vp, _vp]
    lib.tl_orient_device.restype = C.c_int
    lib.tl_check_sizes.argtypes = [_u32, _u32]
    lib.tl_check_sizes.restype = C.c_int
    lib.tl_list.argtypes = [_vp, C.c_int, C.c_uint, C.POINTER(TlStats)]
    lib.tl_list.restype = C.c_int
    lib.tl_list_range.argtypes = [_vp, C.c_int, C.c_uint, C.c_uint32, C.c_uint32, C.POINTER(TlStats)]
    lib.tl_list_range.restype = C.c_int
    lib.tl_fetch_triangles.argtypes = [_vp, _vp, _u64, C.POINTER(_u64)]
    lib.tl_fetch_triangles.restype = C.c_int
    lib.tl_fetch_vertex_counts.argtypes = [_vp, _vp]
    lib.tl_fetch_vertex_counts.restype = C.c_int
    lib.tl_fetch_oriented.argtypes = [_vp, _vp, _vp, _vp, _vp]
    lib.tl_fetch_oriented.restype = C.c_int
    lib.tl_cost_report.argtypes = [_vp, _vp]
    lib.tl_cost_report.restype = C.c_int
    lib.tl_host_register.argtypes = [_vp, _vp, C.c_size_t]
    lib.tl_host_register.restype = C.c_int
    lib.tl_host_unregister.argtypes = [_vp, _vp]
    lib.tl_host_unregister.restype = C.c_int
    lib.tl_timer_start.argtypes = [_vp]
    lib.tl_timer_start.restype = C.c_int
    lib.tl_timer_stop.argtypes = [_vp, C.POINTER(C.c_double)]
    lib.tl_timer_stop.restype = C.c_int
    lib.tl_phase_times.argtypes = [_vp, C.POINTER(C.c_double), C.c_int]
    lib.tl_phase_times.restype = C.c_int
    lib.tl_order.argtypes = [_vp, _u32, _vp, C.c_int, _vp]
    lib.tl_order.restype = C.c_int
    lib.tl_order_device.argtypes = [_vp, _u32, _vp, C.c_int, _vp]
    lib.tl_order_device.restype = C.c_int
    lib.tl_orient_ordered.argtypes = [_vp, _u32, _u64, _vp, _vp, C.c_int]
    lib.tl_orient_ordered.restype = C.c_int
    lib.tl_core_decompose.argtypes = [_vp, _u32, _u64, _vp, _vp, _vp, _vp, C.POINTER(_u32)]
    lib.tl_core_decompose.restype = C.c_int
    lib.tl_core_decompose_device.argtypes = [_vp, _u32, _u64, _vp, _vp, _vp, _vp, C.POINTER(_u32)]
    lib.tl_core_decompose_device.restype = C.c_int
    lib.tl_fetch_ranks.argtypes = [_vp, _vp]
    lib.tl_fetch_ranks.restype = C.c_int
    lib.tl_normalize.argtypes = [_vp, _u64, _vp, C.POINTER(_u32), C.POINTER(_u64), C.POINTER(_u64),
                                 C.POINTER(_u64)]
    lib.tl_normalize.restype = C.c_int
    lib.tl_fetch_graph.argtypes = [_vp, _vp, _vp, _vp]
    lib.tl_fetch_graph.restype = C.c_int
    lib.tl_fetch_triangles_range.argtypes = [_vp, _u64, _u64, _vp, C.POINTER(_u64)]
    lib.tl_fetch_triangles_range.restype = C.c_int
    lib.tl_fetch_triangle_labels.argtypes = [_vp, _u64, _u64, _vp, _vp, C.POINTER(_u64)]
    lib.tl_fetch_triangle_labels.restype = C.c_int
    lib.tl_orient_normalized.argtypes = [_vp, C.c_int]
    lib.tl_orient_normalized.restype = C.c_int
    lib.tl_phase_name.argtypes = [C.c_int]
    lib.tl_phase_name.restype = C.c_char_p
    lib.tl_debug_set.argtypes = [_vp, C.c_int, C.c_int]
    lib.tl_debug_set.restype = C.c_int
    return lib


@lru_cache(maxsize=None)
def trihost() -> C.CDLL:
    if not os.path.exists(TRIHOST_PATH):
        raise NativeLibraryMissing(
            f"{TRIHOST_PATH} is missing: run `make host` (needs the reference sources)")
    lib = C.CDLL(TRIHOST_PATH)
    lib.th_last_error.restype = C.c_char_p
    lib.th_threads.restype = C.c_int
    P = C.POINTER(ThCsr)
    lib.th_gen_gnm.argtypes = [_u32, _u64, _u64, P]
    lib.th_gen_rmat.argtypes = [_u32, _u32, _u64, P]
    lib.th_gen_rmat_raw.argtypes = [_u32, _u32, _u64, _vp]
    lib.th_gen_rmat_raw.restype = C.c_int
    lib.th_gen_chung_lu.argtypes = [_u32, _u64, C.c_double, C.c_double, C.c_double, _u64, P]
    lib.th_gen_ws.argtypes = [_u32, _u32, C.c_double, _u64, P]
    lib.th_csr_from_pairs.argtypes = [_u32, _u64, _vp, P]
    for f in (lib.th_gen_gnm, lib.th_gen_rmat, lib.th_gen_chung_lu, lib.th_gen_ws,
              lib.th_csr_from_pairs):
        f.restype = C.c_int
    lib.th_csr_free.argtypes = [P]
    lib.th_csr_free.restype = None
    lib.th_csr_check.argtypes = [P]
    lib.th_csr_check.restype = C.c_int
    lib.th_graph_new.argtypes = [P]
    lib.th_graph_new.restype = _vp
    lib.th_graph_free.argtypes = [_vp]
    lib.th_graph_free.restype = None
    lib.th_graph_load.argtypes = [C.c_char_p, C.POINTER(_u64), C.POINTER(_u64)]
    lib.th_graph_load.restype = _vp
    lib.th_graph_to_csr.argtypes = [_vp, P]
    lib.th_graph_to_csr.restype = C.c_int
    lib.th_graph_labels.argtypes = [_vp, _vp]
    lib.th_graph_labels.restype = None
    lib.th_parse_edgelist.argtypes = [C.c_char_p, C.POINTER(C.POINTER(C.c_int64)), C.POINTER(_u64)]
    lib.th_parse_edgelist.restype = C.c_int
    lib.th_free.argtypes = [_vp]
    lib.th_free.restype = None
    lib.th_order.argtypes = [_vp, C.c_char_p, _u64, _vp, C.POINTER(C.c_double)]
    lib.th_order.restype = C.c_int
    lib.th_cost.argtypes = [_vp, _vp, _vp]
    lib.th_cost.restype = C.c_int
    lib.th_bench_csv.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_uint,
                                 _u64, _u64, _u64, _u64, _u64, _u64, C.c_double, C.c_double,
                                 C.c_double, C.c_char_p, _u64]
    lib.th_bench_csv.restype = C.c_int
    lib.th_bench_csv_header.restype = C.c_char_p
    return lib
