"""ctypes binding of libcpg.so (include/cpg.h).  Fails loudly when the library is missing.

There is no CPU fallback anywhere in this package: every query runs the sm_100a
kernels inside libcpg.so.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_uint32, c_uint64, c_void_p

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CPG_LIB_PATH") or os.path.join(PKG, "libcpg.so")  # override: A/B builds

CPG_OK, CPG_EINVAL, CPG_ECUDA, CPG_ENCCL, CPG_ENOMEM, CPG_ESTRUCT, CPG_EPARSE, CPG_EIO = 0, 1, 2, 3, 4, 5, 6, 7


class cpg_stats(ctypes.Structure):
    _fields_ = [("iterations", c_uint32), ("push_work", c_uint64), ("wall_seconds", c_double),
                ("device_ms", c_double), ("mass_err_max", c_double), ("bytes_model", c_double),
                ("launches", c_uint32), ("step_ms", c_double), ("step_launches", c_uint32)]


class cpg_plan(ctypes.Structure):
    _fields_ = [("cheby_steps", c_uint64), ("taylor_steps", c_uint64), ("epsilon", c_double),
                ("tail_bound", c_double)]


class cpg_graph_info(ctypes.Structure):
    _fields_ = [("n", c_uint32), ("nnz", c_uint64), ("n_local", c_uint32), ("nnz_local", c_uint64),
                ("row_begin", c_uint32), ("n_padded", c_uint32), ("n_hubs", c_uint32),
                ("n_items", c_uint32), ("max_degree", c_uint32), ("rank", c_int), ("nranks", c_int),
                ("device", c_int), ("structure_hash", c_uint64), ("chunks", c_int), ("fused_allgather", c_int)]


class cpg_error_report(ctypes.Structure):  # ErrorReport, eval.hpp:15-20
    _fields_ = [("l1", c_double), ("l2", c_double), ("deg_norm_inf", c_double), ("argmax_node", c_uint32)]


_u64p = POINTER(c_uint64)
_u32p = POINTER(c_uint32)
_f64p = POINTER(c_double)
_G = c_void_p

# name -> (restype, argtypes); the full export list of include/cpg.h.
SIGNATURES = {
    "cpg_last_error": (c_char_p, []),
    "cpg_version": (c_char_p, []),
    "cpg_set_profiling": (None, [c_int]),
    "cpg_ppr_cheby_coeffs": (c_int, [c_double, c_uint64, _f64p]),
    "cpg_hkpr_cheby_coeffs": (c_int, [c_double, c_uint64, _f64p]),
    "cpg_cheby_coeffs": (c_int, [c_int, c_double, c_uint64, _f64p]),
    "cpg_plan_truncation": (c_int, [c_int, c_double, c_double, POINTER(cpg_plan)]),
    "cpg_parse_kernel_spec": (c_int, [c_char_p, POINTER(c_int), POINTER(c_double)]),
    "cpg_taylor_coeffs": (c_int, [c_int, c_double, c_uint64, _f64p]),
    "cpg_ground_truth_steps": (c_uint64, [c_int, c_double]),
    "cpg_power_method": (c_int, [_G, _f64p, c_uint32, _u32p, c_uint32, c_void_p, POINTER(cpg_stats)]),
    "cpg_validate_csr": (c_int, [_u64p, _u32p, c_uint64, c_uint64, _u64p]),
    "cpg_graph_create": (c_int, [_u64p, _u32p, c_uint32, c_uint64, c_int, c_int, POINTER(_G)]),
    "cpg_graph_create_device": (c_int, [c_void_p, c_void_p, c_uint32, c_uint64, c_int, POINTER(_G)]),
    "cpg_nccl_unique_id": (c_int, [c_void_p]),
    "cpg_graph_create_sharded": (c_int, [c_void_p, c_void_p, c_uint32, c_uint64, c_int, c_int, c_int,
                                         c_int, c_void_p, POINTER(_G)]),
    "cpg_loopback_group_create": (c_int, [c_int, POINTER(c_void_p)]),
    "cpg_graph_create_multi": (c_int, [_u64p, _u32p, c_uint32, c_uint64, POINTER(c_int), c_int, POINTER(_G)]),
    "cpg_graph_create_multi_loopback": (c_int, [_u64p, _u32p, c_uint32, c_uint64, c_int, c_int, POINTER(_G)]),
    "cpg_loopback_group_destroy": (c_int, [c_void_p]),
    "cpg_graph_create_loopback": (c_int, [c_void_p, c_void_p, c_uint32, c_uint64, c_int, c_int, c_int, c_void_p,
                                          POINTER(_G)]),
    "cpg_shard_plan": (c_int, [_u64p, c_uint32, c_int, c_int, _u32p, _u32p]),
    "cpg_graph_info_get": (c_int, [_G, POINTER(cpg_graph_info)]),
    "cpg_graph_destroy": (c_int, [_G]),
    "cpg_chebypower": (c_int, [_G, _f64p, c_uint32, _u32p, c_uint32, c_void_p, POINTER(cpg_stats)]),
    "cpg_chebypower_device": (c_int, [_G, _f64p, c_uint32, _u32p, c_uint32, c_void_p, c_void_p,
                                      POINTER(cpg_stats)]),
    "cpg_chebypower_vec": (c_int, [_G, _f64p, c_uint32, _f64p, c_uint32, c_void_p, POINTER(cpg_stats)]),
    "cpg_chebypower_batched": (c_int, [_G, _f64p, c_uint32, _u32p, c_uint32, c_uint32, c_void_p,
                                       POINTER(cpg_stats)]),
    "cpg_chebypower_batched_device": (c_int, [_G, _f64p, c_uint32, _u32p, c_uint32, c_uint32, c_void_p,
                                              c_void_p, POINTER(cpg_stats)]),
    "cpg_chebypower_batched_async": (c_int, [_G, _f64p, c_uint32, _u32p, c_uint32, c_uint32, c_void_p,
                                             POINTER(cpg_stats)]),
    "cpg_graph_sync": (c_int, [_G]),
    "cpg_chebypower_trace": (c_int, [_G, _f64p, c_uint32, c_uint32, c_void_p, c_void_p, c_void_p]),
    "cpg_chebypower_vec_trace": (c_int, [_G, _f64p, c_uint32, _f64p, c_void_p, c_void_p, c_void_p]),
    "cpg_apply_walk": (c_int, [_G, _f64p, _f64p]),
    "cpg_chebypower_topk": (c_int, [_G, _f64p, c_uint32, _u32p, c_uint32, c_uint32, _u32p, _f64p,
                                    POINTER(cpg_stats)]),
    "cpg_general_gp": (c_int, [_G, _f64p, c_uint32, c_double, _f64p, c_uint32, c_uint32, c_void_p,
                               POINTER(cpg_stats)]),
    "cpg_bytes_per_step": (c_double, [_G, c_uint32]),
    "cpg_sparse_early_steps": (c_uint32, [_G, c_uint32, c_uint32]),
    "cpg_last_split_profile": (c_int, [_G, POINTER(c_double), POINTER(c_double), POINTER(c_uint32)]),
    "cpg_gen_rmat": (c_int, [c_uint32, c_uint64, c_double, c_double, c_double, c_uint64, c_int,
                             POINTER(c_void_p), POINTER(c_void_p), _u32p, _u64p]),
    "cpg_gen_chunglu": (c_int, [c_uint32, c_uint64, c_double, c_double, c_uint32, c_uint64, c_int,
                                POINTER(c_void_p), POINTER(c_void_p), _u32p, _u64p]),
    "cpg_free_csr": (c_int, [c_void_p, c_void_p, c_int]),
    "cpg_ingest_edges": (c_int, [POINTER(ctypes.c_int64), c_uint64, c_int, POINTER(c_void_p), POINTER(c_void_p),
                                 _u32p, _u64p, POINTER(ctypes.c_int64), c_uint64]),
    "cpg_csr_to_host": (c_int, [c_void_p, c_void_p, c_uint32, c_uint64, c_int, _u64p, _u32p]),
    "cpg_measure": (c_int, [_G, c_void_p, c_void_p, c_uint32, c_int, POINTER(cpg_error_report)]),
    "cpg_chebypower_measure": (c_int, [_G, _f64p, c_uint32, _u32p, c_uint32, c_void_p, c_int,
                                       POINTER(cpg_error_report), POINTER(cpg_stats)]),
    "cpg_parse_edge_text": (c_int, [c_void_p, c_uint64, ctypes.c_char, c_void_p, c_uint64, _u64p, c_int]),
    "cpg_csr_cache_write": (c_int, [c_char_p, _u64p, _u32p, c_uint64, c_uint64]),
    "cpg_csr_cache_info": (c_int, [c_char_p, _u64p, _u64p]),
    "cpg_csr_cache_read": (c_int, [c_char_p, _u64p, _u32p, c_uint64, c_uint64]),
    "cpg_truth_cache_write": (c_int, [c_char_p, c_char_p, c_uint64, _f64p, c_uint64]),
    "cpg_truth_cache_info": (c_int, [c_char_p, c_char_p, c_uint64, _u64p, _u64p]),
    "cpg_truth_cache_read": (c_int, [c_char_p, _f64p, c_uint64]),
    "cpg_truth_cache_filename": (c_int, [c_uint64, c_char_p, c_uint64, c_char_p, c_uint64]),
}

_lib = None


def lib():
    """Load libcpg.so (built by ``python -m paper_2412_10789_b200._build``)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build the CUDA library first "
                "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            if os.environ.get("CPG_LIB_PATH") and not hasattr(L, name):
                continue  # A/B against an older build: its missing entries stay unbound
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return lib().cpg_last_error().decode(errors="replace")
