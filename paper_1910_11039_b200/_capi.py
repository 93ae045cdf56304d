"""ctypes declarations for include/ebc_b200.h (the C ABI of libebc_b200.so).

The library is loaded from this package directory.  There is no pure-Python or
CPU fallback: if the shared library is missing and cannot be built, importing
anything that needs it raises.
"""
from __future__ import annotations

import ctypes as C
import os

from . import build as _build

u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)
f64p = C.POINTER(C.c_double)

EBC_OK, EBC_ERR_CONFIG, EBC_ERR_PARSE, EBC_ERR_BACKEND, EBC_ERR_CUDA = 0, 2, 3, 4, 5

ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p)


class RunConfig(C.Structure):
    _fields_ = [
        ("eps", C.c_double), ("delta", C.c_double), ("seed", C.c_uint64),
        ("bound", C.c_int), ("allocator", C.c_int),
        ("omega_override", C.c_uint64), ("calib_samples", C.c_uint64),
        ("diameter_sweeps", C.c_int), ("vertex_diameter_override", C.c_uint64),
        ("epoch_samples", C.c_uint64), ("max_epochs", C.c_uint64),
        ("device", C.c_int), ("rank", C.c_int), ("world_size", C.c_int),
        ("allreduce", ALLREDUCE_FN), ("allreduce_user", C.c_void_p),
        ("block_threads", C.c_uint32), ("slots", C.c_uint32), ("slot_capacity", C.c_uint64),
        ("overlap", C.c_int), ("items_per_thread", C.c_uint32), ("materialize_final_level", C.c_int), ("renumber", C.c_int), ("reserved_sms", C.c_int), ("work_counters", C.c_int),
    ]


class RunStats(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in ("epochs", "samples", "tau", "omega", "calibration_samples",
                                          "discarded_samples", "n0", "n", "m", "diameter_upper_bound",
                                          "vertex_diameter_bound")] + \
               [(k, C.c_double) for k in ("adaptive_s", "diameter_s", "calibration_s", "reduce_s",
                                          "check_s", "upload_s", "wall_s")] + \
               [("overflow_samples", C.c_uint64), ("work", C.c_uint64 * 12)]


class SampleRecord(C.Structure):
    _fields_ = [("s", C.c_uint32), ("t", C.c_uint32), ("dist", C.c_uint32), ("meet", C.c_uint32),
                ("meet_count", C.c_uint32), ("draws", C.c_uint32), ("path_len", C.c_uint32),
                ("flags", C.c_uint32), ("weight_lo", C.c_uint64), ("weight_hi", C.c_uint64)]


class CompareReport(C.Structure):
    _fields_ = [("max_abs_error", C.c_double), ("vertices_above_eps", C.c_uint64), ("top10_overlap", C.c_double),
                ("top100_overlap", C.c_double), ("vertices", C.c_uint64)]


# name -> (restype, argtypes); every symbol include/ebc_b200.h declares.
SIGNATURES = {
    "ebc_last_error": (C.c_char_p, []),
    "ebc_version": (C.c_char_p, []),
    "ebc_graph_from_csr": (C.c_int, [C.c_uint64, u64p, u32p, u64p, C.c_int, C.POINTER(C.c_void_p)]),
    "ebc_graph_from_edges": (C.c_int, [C.c_uint64, u64p, u64p, C.c_uint64, C.POINTER(C.c_void_p)]),
    "ebc_graph_load": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]),
    "ebc_graph_save": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int]),
    "ebc_graph_lcc": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "ebc_graph_lcc_device": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]),
    "ebc_graph_from_edges_device": (C.c_int, [C.c_uint64, u64p, u64p, C.c_uint64, C.c_int, C.c_int,
                                              C.POINTER(C.c_void_p)]),
    "ebc_gen_rmat_device": (C.c_int, [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                                      C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "ebc_graph_num_vertices": (C.c_uint64, [C.c_void_p]),
    "ebc_graph_num_edges": (C.c_uint64, [C.c_void_p]),
    "ebc_graph_offsets": (u64p, [C.c_void_p]),
    "ebc_graph_targets": (u32p, [C.c_void_p]),
    "ebc_graph_original_ids": (u64p, [C.c_void_p]),
    "ebc_graph_free": (None, [C.c_void_p]),
    "ebc_gen_erdos_renyi": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(C.c_void_p)]),
    "ebc_gen_rmat": (C.c_int, [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                               C.c_uint64, C.POINTER(C.c_void_p)]),
    "ebc_gen_grid": (C.c_int, [C.c_uint64, C.c_uint64, C.c_double, C.c_double, C.c_uint64,
                               C.POINTER(C.c_void_p)]),
    "ebc_compute_omega": (C.c_int, [C.c_uint64, C.c_double, C.c_double, u64p]),
    "ebc_epoch_length": (C.c_int, [C.c_int, C.c_int, C.c_double, C.c_double, u64p]),
    "ebc_calibrate": (C.c_int, [u64p, C.c_uint64, C.c_double, C.c_int, f64p, f64p]),
    "ebc_diameter_upper_bound": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64, u64p]),
    "ebc_shard_range": (None, [C.c_uint64, C.c_uint64, C.c_int, C.c_int, u64p, u64p]),
    "ebc_run_config_default": (None, [C.POINTER(RunConfig)]),
    "ebc_run": (C.c_int, [C.c_void_p, C.POINTER(RunConfig), C.POINTER(C.c_void_p)]),
    "ebc_result_scores": (C.c_int, [C.c_void_p, C.POINTER(f64p), u64p]),
    "ebc_result_counts": (C.c_int, [C.c_void_p, C.POINTER(u64p), u64p]),
    "ebc_result_tau": (C.c_uint64, [C.c_void_p]),
    "ebc_result_original_ids": (C.c_int, [C.c_void_p, C.POINTER(u64p), u64p]),
    "ebc_result_stats": (C.c_int, [C.c_void_p, C.POINTER(RunStats)]),
    "ebc_result_free": (None, [C.c_void_p]),
    "ebc_sampler_create": (C.c_int, [C.c_void_p, C.POINTER(RunConfig), C.POINTER(C.c_void_p)]),
    "ebc_sampler_free": (None, [C.c_void_p]),
    "ebc_sampler_sample": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_int]),
    "ebc_sampler_sample_debug": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64,
                                           u32p, C.c_int, C.POINTER(SampleRecord), u32p, C.c_uint64]),
    "ebc_sampler_last_state": (C.c_int, [C.c_void_p, C.c_int, u32p, u64p]),
    "ebc_sampler_set_stopping": (C.c_int, [C.c_void_p, C.c_double, C.c_uint64, f64p, f64p, C.c_int]),
    "ebc_sampler_fold_and_check": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int)]),
    "ebc_sampler_read_frame": (C.c_int, [C.c_void_p, C.c_int, u64p]),
    "ebc_sampler_write_state": (C.c_int, [C.c_void_p, u64p]),
    "ebc_sampler_clear": (C.c_int, [C.c_void_p]),
    "ebc_sampler_work": (C.c_int, [C.c_void_p, u64p, C.c_int]),
    "ebc_sampler_mark": (C.c_int, [C.c_void_p, C.c_int]),
    "ebc_sampler_elapsed_ms": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_float)]),
    "ebc_sampler_sync": (C.c_int, [C.c_void_p]),
    "ebc_sampler_info": (C.c_int, [C.c_void_p, u64p]),
    "ebc_sampler_stream": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "ebc_sampler_frame_ptr": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_void_p), u64p]),
    "ebc_sampler_bfs": (C.c_int, [C.c_void_p, C.c_uint32, u32p, u64p]),
    "ebc_sampler_flush_l2": (C.c_int, [C.c_void_p]),
    "ebc_release_device_cache": (None, []),
    "ebc_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "ebc_nccl_comm_create": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "ebc_nccl_allreduce": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]),
    "ebc_nccl_comm_free": (None, [C.c_void_p]),
    "ebc_scores_write": (C.c_int, [C.c_char_p, u64p, f64p, C.c_uint64, C.POINTER(C.c_char_p), C.POINTER(C.c_char_p),
                                   C.c_uint64]),
    "ebc_result_write_scores": (C.c_int, [C.c_void_p, C.POINTER(RunConfig), C.c_char_p]),
    "ebc_scores_read": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "ebc_scores_data": (C.c_int, [C.c_void_p, C.POINTER(u64p), C.POINTER(f64p), u64p]),
    "ebc_scores_meta": (C.c_char_p, [C.c_void_p, C.c_char_p]),
    "ebc_scores_free": (None, [C.c_void_p]),
    "ebc_scores_compare": (C.c_int, [C.c_void_p, C.c_void_p, C.c_double, C.POINTER(CompareReport)]),
    "ebc_result_stats_json": (C.c_int, [C.c_void_p, C.POINTER(RunConfig), C.c_char_p, C.c_uint64, u64p]),
}

_lib = None


def lib_path() -> str:
    return _build.LIB


def load():
    """Loads (building first if the sources are newer) libebc_b200.so.  Raises if unavailable."""
    global _lib
    if _lib is None:
        path = os.environ.get("EBC_LIB")  # experiment hook: an alternative build of the same library (A/B runs)
        if not path:
            if not os.path.exists(_build.LIB) or (_build.is_stale() and _have_nvcc()):
                _build.build()
            path = _build.LIB
        L = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)  # AttributeError if a declared symbol is not exported
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _have_nvcc() -> bool:
    try:
        _build.nvcc_path()
        return True
    except RuntimeError:
        return False
