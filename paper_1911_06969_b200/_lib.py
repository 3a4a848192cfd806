"""ctypes binding of libgpm.so (the C ABI in include/gpm.h).

The product path has no fallback: if the CUDA library is not built, importing
the package raises.  Build with ``python -c "import __graft_entry__ as g; g.build()"``
or ``make -C paper_1911_06969_b200/csrc``.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, os.environ.get("GPM_LIB_VARIANT", "libgpm.so"))  # variant: A/B builds in-tree

GPM_OK, GPM_EINVAL, GPM_EPARSE, GPM_ENOMEM, GPM_ECUDA, GPM_ENCCL, GPM_ECONFIG = range(7)
APP_TC, APP_CF, APP_MC, APP_FSM = range(4)

EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_int, C.c_void_p)

EXPORTS = [
    "gpm_config_default", "gpm_graph_create_csr", "gpm_graph_create_dag_csr", "gpm_graph_orient_dag", "gpm_graph_info", "gpm_graph_download",
    "gpm_graph_is_connected", "gpm_level1", "gpm_graph_free", "gpm_mine", "gpm_result_total",
    "gpm_result_num_patterns", "gpm_result_pattern", "gpm_result_stats", "gpm_result_free",
    "gpm_load_edge_list", "gpm_load_labeled_graph", "gpm_csr_from_edges", "gpm_generate_rmat", "gpm_csr_free",
    "gpm_last_error", "gpm_version", "gpm_steal_create", "gpm_steal_open", "gpm_steal_reset", "gpm_steal_release",
    "gpm_release_cached", "gpm_csr_save", "gpm_csr_load", "gpm_load_cached",
    "gpm_canonicalize_batch", "gpm_nccl_unique_id", "gpm_exchange_nccl_create", "gpm_exchange_nccl_wrap",
    "gpm_exchange_nccl_fn", "gpm_exchange_nccl_destroy", "gpm_probe_read_bandwidth",
]


# gpm_list_fn(ctx, const uint32_t* verts, uint64_t n, int k) -> int
LIST_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint32), C.c_uint64, C.c_int)


class Config(C.Structure):
    _fields_ = [("app", C.c_int), ("k", C.c_int), ("min_support", C.c_uint64), ("mem_budget", C.c_uint64),
                ("no_orient", C.c_int), ("rank", C.c_int), ("world", C.c_int), ("root_lo", C.c_uint64),
                ("root_hi", C.c_uint64), ("stream", C.c_void_p), ("exchange", EXCHANGE_FN),
                ("exchange_ctx", C.c_void_p), ("steal_ctrs", C.c_void_p), ("steal_chunk", C.c_uint64),
                ("list_fn", LIST_FN), ("list_ctx", C.c_void_p), ("mni_mode", C.c_int)]


# gpm_stats.paths bits (include/gpm.h)
PATH_GENERIC, PATH_CF_EDGE_CHUNK, PATH_CF_SIBLINGS, PATH_MC3_WARP, PATH_MC3_BLOCK, PATH_MC3_MULTITILE, \
    PATH_MC4_STAGED, PATH_MC4_HBM_SETS, PATH_PLANNER_CHUNKS, PATH_FSM_ROUNDS, PATH_FSM_FUSED_LAST, \
    PATH_FSM_GROUPED, PATH_FSM_FAN, PATH_FSM_SPARSE, PATH_CF_LOCAL, PATH_CF_LOCAL_BIG = (1 << i for i in range(16))


class Stats(C.Structure):
    _fields_ = [("n_levels", C.c_int), ("level_sizes", C.c_uint64 * 16), ("candidates", C.c_uint64 * 16),
                ("survivors", C.c_uint64 * 16), ("n_explored", C.c_uint64), ("b_alg", C.c_double),
                ("ms_total", C.c_double), ("ms_extend", C.c_double), ("ms_dominant", C.c_double),
                ("b_dominant", C.c_double), ("launches", C.c_uint64), ("chunks", C.c_uint64),
                ("dominant", C.c_char * 64), ("b_moved_dominant", C.c_double), ("n_counted", C.c_uint64),
                ("paths", C.c_uint32)]


class CsrStruct(C.Structure):
    _fields_ = [("n", C.c_uint32), ("m", C.c_uint64), ("row_offsets", C.c_void_p), ("col", C.c_void_p),
                ("labels", C.c_void_p), ("original_ids", C.c_void_p)]


class GpmError(RuntimeError):
    """Raised for any non-zero gpm_status (mirrors gpmine::error, error.hpp:10-13)."""

    def __init__(self, code: int, msg: str, line: int = 0):
        super().__init__(msg)
        self.code = code
        self.line = line


class ParseError(GpmError):
    """gpmine::parse_error (error.hpp:16-25): carries the 1-based line number."""


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    vp, u64, u32, i32 = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int
    sig = {
        "gpm_config_default": (None, [C.POINTER(Config)]),
        "gpm_graph_create_csr": (i32, [vp, vp, vp, u32, u64, i32, i32, C.POINTER(vp)]),
        "gpm_graph_create_dag_csr": (i32, [vp, vp, vp, u32, u64, i32, C.POINTER(vp)]),
        "gpm_graph_orient_dag": (i32, [vp, C.POINTER(vp)]),
        "gpm_graph_info": (i32, [vp, C.POINTER(u32), C.POINTER(u64), C.POINTER(i32), C.POINTER(i32)]),
        "gpm_graph_download": (i32, [vp, vp, vp]),
        "gpm_graph_is_connected": (i32, [vp, vp, vp, u64, vp]),
        "gpm_level1": (i32, [vp, vp, vp, u64, C.POINTER(u64)]),
        "gpm_graph_free": (None, [vp]),
        "gpm_mine": (i32, [vp, C.POINTER(Config), C.POINTER(vp)]),
        "gpm_result_total": (i32, [vp, C.POINTER(u64)]),
        "gpm_result_num_patterns": (i32, [vp, C.POINTER(u64)]),
        "gpm_result_pattern": (i32, [vp, u64, C.c_char_p, C.c_size_t, C.POINTER(u64), C.POINTER(i32)]),
        "gpm_result_stats": (i32, [vp, C.POINTER(Stats)]),
        "gpm_result_free": (None, [vp]),
        "gpm_load_edge_list": (i32, [C.c_char_p, C.POINTER(CsrStruct), C.POINTER(u64)]),
        "gpm_load_labeled_graph": (i32, [C.c_char_p, C.POINTER(CsrStruct), C.POINTER(u64)]),
        "gpm_csr_from_edges": (i32, [vp, vp, u64, C.POINTER(CsrStruct)]),
        "gpm_generate_rmat": (i32, [i32, C.c_double, C.c_double, C.c_double, C.c_double, u64, u32, u64,
                                    C.POINTER(CsrStruct)]),
        "gpm_csr_free": (None, [C.POINTER(CsrStruct)]),
        "gpm_nccl_unique_id": (i32, [vp]),
        "gpm_exchange_nccl_create": (i32, [vp, i32, i32, i32, C.POINTER(vp)]),
        "gpm_exchange_nccl_wrap": (i32, [vp, C.POINTER(vp)]),
        "gpm_exchange_nccl_fn": (EXCHANGE_FN, []),
        "gpm_exchange_nccl_destroy": (i32, [vp]),
        "gpm_canonicalize_batch": (i32, [i32, i32, u64, vp, vp, vp, vp, vp]),
        "gpm_csr_save": (i32, [C.c_char_p, C.POINTER(CsrStruct), C.c_char_p]),
        "gpm_csr_load": (i32, [C.c_char_p, C.POINTER(CsrStruct)]),
        "gpm_load_cached": (i32, [C.c_char_p, i32, C.c_char_p, C.POINTER(CsrStruct), C.POINTER(u64),
                                  C.POINTER(i32)]),
        "gpm_last_error": (C.c_char_p, []),
        "gpm_steal_create": (i32, [i32, i32, C.POINTER(vp), vp]),
        "gpm_steal_open": (i32, [i32, vp, C.POINTER(vp)]),
        "gpm_steal_reset": (i32, [vp, i32, vp]),
        "gpm_steal_release": (i32, [vp, i32]),
        "gpm_release_cached": (i32, [i32]),
        "gpm_probe_read_bandwidth": (i32, [i32, u64, i32, C.POINTER(C.c_double)]),
        "gpm_version": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(rc: int, line: int = 0):
    if rc != GPM_OK:
        msg = lib().gpm_last_error().decode()
        if rc == GPM_EPARSE:
            raise ParseError(rc, msg, line)
        raise GpmError(rc, msg, line)
