"""ctypes declarations for libhm.so (include/hm.h).  Marshalling only.

The library is the product path; if it is missing this module raises -- there
is no fallback implementation anywhere in the package.
"""
import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhm.so")

HM_OK, HM_EINVAL, HM_ERANGE, HM_ENOMEM, HM_ECUDA, HM_ESTATE = 0, -1, -2, -3, -4, -5
HM_NAIVE, HM_CC1, HM_CC2, HM_CC2_AVG, HM_CC1_RARY = 0, 1, 2, 3, 4
STATUS_NAMES = {0: "HM_OK", -1: "HM_EINVAL", -2: "HM_ERANGE", -3: "HM_ENOMEM", -4: "HM_ECUDA",
                -5: "HM_ESTATE"}

c_i32p = ctypes.POINTER(ctypes.c_int32)
c_i64p = ctypes.POINTER(ctypes.c_int64)
vp = ctypes.c_void_p


class HmStats(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_int64), ("bfs_launches", ctypes.c_int64), ("bfs_ms", ctypes.c_double),
                ("bfs_levels", ctypes.c_int64), ("bfs_batches", ctypes.c_int64),
                ("bfs_model_bytes", ctypes.c_double), ("bfs_row_commits", ctypes.c_int64),
                ("bfs_csr_bytes", ctypes.c_double), ("bfs_td_levels", ctypes.c_int64),
                ("bfs_state_bytes", ctypes.c_double), ("host_syncs", ctypes.c_int64),
                ("phase_ms", ctypes.c_double * 10), ("bfs_gathers", ctypes.c_int64),
                ("bfs_own_reads", ctypes.c_int64)]


# name -> (restype, argtypes); must match include/hm.h (tests/test_abi.py checks the names)
SIGNATURES = {
    "hm_create": (ctypes.c_int32, [ctypes.POINTER(vp), ctypes.c_int, vp]),
    "hm_destroy": (None, [vp]),
    "hm_last_error": (ctypes.c_char_p, [vp]),
    "hm_set_param": (ctypes.c_int32, [vp, ctypes.c_char_p, ctypes.c_int64]),
    "hm_load_layers": (ctypes.c_int32, [vp, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(vp), c_i64p, c_i64p]),
    "hm_graph_info": (ctypes.c_int32, [vp, ctypes.c_int32, c_i32p, c_i64p, ctypes.POINTER(vp), ctypes.POINTER(vp)]),
    "hm_graph_csr": (ctypes.c_int32, [vp, ctypes.c_int32, vp, vp]),
    "hm_and_aggregate": (ctypes.c_int32, [vp, c_i32p, ctypes.c_int32, c_i32p]),
    "hm_or_aggregate": (ctypes.c_int32, [vp, c_i32p, ctypes.c_int32, c_i32p]),
    "hm_free_graph": (ctypes.c_int32, [vp, ctypes.c_int32]),
    "hm_closeness": (ctypes.c_int32, [vp, ctypes.c_int32, vp, vp, vp, vp]),
    "hm_closeness_multi": (ctypes.c_int32, [vp, c_i32p, ctypes.c_int32]),
    "hm_closeness_results": (ctypes.c_int32, [vp, ctypes.c_int32, vp, vp, vp, vp]),
    "hm_closeness_partial": (ctypes.c_int32, [vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, vp]),
    "hm_closeness_combine": (ctypes.c_int32, [vp, ctypes.c_int32, vp]),
    "hm_cc_nodes": (ctypes.c_int32, [vp, ctypes.c_int32, vp, c_i32p, ctypes.POINTER(ctypes.c_double)]),
    "hm_degrees": (ctypes.c_int32, [vp, ctypes.c_int32, vp]),
    "hm_topk_closeness": (ctypes.c_int32, [vp, ctypes.c_int32, ctypes.c_int32, vp]),
    "hm_compose": (ctypes.c_int32, [vp, ctypes.c_int32, c_i32p, ctypes.c_int32, ctypes.c_int32, vp, c_i32p]),
    "hm_set_metrics": (ctypes.c_int32, [vp, ctypes.c_int32, vp, ctypes.c_int64, vp, ctypes.c_int64,
                                        ctypes.POINTER(ctypes.c_double)]),
    "hm_exact_mean": (ctypes.c_int32, [vp, vp, ctypes.c_int64, vp, ctypes.POINTER(ctypes.c_double), c_i32p]),
    "hm_sync": (ctypes.c_int32, [vp]),
    "hm_debug_counts": (ctypes.c_int32, [vp, vp, ctypes.c_int32]),
    "hm_get_stats": (ctypes.c_int32, [vp, ctypes.POINTER(HmStats), ctypes.c_int]),
}

_lib = None


def load(path=LIB_PATH):
    """Load libhm.so and declare every entry point.  Raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"libhm.so not found at {path}: build it with `python -m paper_2207_11662_b200.build` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L
