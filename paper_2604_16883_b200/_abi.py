"""ctypes binding of include/sinkr_cuda.h (the C-ABI of libsinkr_cuda.so).

The library is the product: there is no Python or CPU fallback.  If the
shared object is missing, importing the package still works (so the CPU test
suite can inspect the host logic), but every call that needs the engine
raises loudly.
"""
from __future__ import annotations

import ctypes as C
import os

from .build import LIB

c_size_t = C.c_size_t


class CacheConfigC(C.Structure):
    _fields_ = [("num_layers", c_size_t), ("num_q_heads", c_size_t),
                ("num_kv_heads", c_size_t), ("head_dim", c_size_t),
                ("capacity", c_size_t), ("num_seqs", c_size_t)]


class ThresholdProfileC(C.Structure):
    _fields_ = [("coeffs", C.c_double * 4), ("length_normalizer", C.c_double),
                ("clamp_lo", C.c_double), ("clamp_hi", C.c_double)]


class RoutingConfigC(C.Structure):
    _fields_ = [("gamma", C.c_double), ("profile", ThresholdProfileC),
                ("excluded_layers", C.POINTER(c_size_t)), ("num_excluded_layers", c_size_t),
                ("sink_on_tie", C.c_int)]


class EngineOptionsC(C.Structure):
    _fields_ = [("num_splits", c_size_t), ("block_size", c_size_t),
                ("observe_only", C.c_int), ("global_context_len", c_size_t)]


class LoadCountersC(C.Structure):
    _fields_ = [("kv_floats_loaded", C.c_uint64), ("anchor_floats_loaded", C.c_uint64),
                ("groups_active", C.c_uint64), ("groups_skipped", C.c_uint64),
                ("routing_seconds", C.c_double), ("attention_seconds", C.c_double),
                ("merge_seconds", C.c_double)]


class GroupInfoC(C.Structure):
    _fields_ = [("layer", c_size_t), ("kv_head", c_size_t), ("group_score", C.c_double),
                ("threshold", C.c_double), ("sink", C.c_int32), ("degenerate", C.c_int32),
                ("kv_floats_loaded", C.c_uint64), ("tokens_loaded", C.c_uint64)]


class CalibrationPointC(C.Structure):
    _fields_ = [("length", c_size_t), ("tau", C.c_double), ("skip", C.c_double)]


MAX_EXCLUDED_LAYERS = 32
MAX_CALIBRATION_POINTS = 64


class ProfileC(C.Structure):
    _fields_ = [("threshold", ThresholdProfileC), ("target_skip", C.c_double),
                ("gamma", C.c_double), ("excluded_layers", c_size_t * MAX_EXCLUDED_LAYERS),
                ("num_excluded_layers", c_size_t),
                ("points", CalibrationPointC * MAX_CALIBRATION_POINTS),
                ("num_points", c_size_t)]


# sinkr_status -> the Python analogue of the reference's exception classes
SINKR_OK = 0
_EXC = {
    1: ValueError,        # std::invalid_argument
    2: IndexError,        # std::out_of_range
    3: RuntimeError,      # std::runtime_error
    4: AssertionError,    # std::logic_error (ragged cache)
}


class SinkrCudaError(RuntimeError):
    """CUDA failure (status 5) or no sm_100 device (status 6)."""


class LogicError(AssertionError):
    """std::logic_error (status 4)."""


_EXC[4] = LogicError
_EXC[5] = SinkrCudaError
_EXC[6] = SinkrCudaError

# Every symbol include/sinkr_cuda.h declares (checked by the CPU test suite).
EXPORTS = (
    "sinkr_last_error", "sinkr_version", "sinkr_engine_create", "sinkr_engine_destroy",
    "sinkr_engine_stream", "sinkr_kv_append", "sinkr_kv_append_device_bf16",
    "sinkr_kv_append_synthetic", "sinkr_kv_length", "sinkr_kv_token_count", "sinkr_kv_anchor",
    "sinkr_kv_set_anchor", "sinkr_kv_read", "sinkr_threshold_for_length", "sinkr_route",
    "sinkr_auto_num_splits", "sinkr_split_ranges", "sinkr_routed_decode_step",
    "sinkr_routed_decode_batch", "sinkr_routed_decode_async", "sinkr_fetch_step_info",
    "sinkr_rank_partial_floats", "sinkr_decode_rank_partial_async",
    "sinkr_merge_rank_partials_async", "sinkr_last_step_stats", "sinkr_set_timing",
    "sinkr_decode_grid", "sinkr_step_io_bytes", "sinkr_step_io_buffers", "sinkr_engine_config",
    # calibration (f1)
    "sinkr_profile_default", "sinkr_profile_constant", "sinkr_sweep", "sinkr_skip_ratio_at",
    "sinkr_solve_threshold", "sinkr_fit_cubic", "sinkr_calibrate", "sinkr_save_profile",
    "sinkr_load_profile", "sinkr_collect_scores", "sinkr_collect_scores_batch",
    # snapshots / device prefill (f2)
    "sinkr_write_tensor", "sinkr_read_tensor", "sinkr_snkt_file_size", "sinkr_save_snapshot",
    "sinkr_load_snapshot", "sinkr_load_snapshot_into", "sinkr_kv_append_device_f32",
    # analysis (f4)
    "sinkr_attention_bos_mass", "sinkr_attention_weights", "sinkr_attention_last_kernel_seconds",
    "sinkr_group_attention", "sinkr_routed_decode_peer", "sinkr_oracle_labels",
    "sinkr_pr_curve",
    # fused sequence-sharded peer merge
    "sinkr_peer_setup", "sinkr_peer_ipc_handle", "sinkr_peer_open", "sinkr_peer_set_blocks",
    "sinkr_peer_block", "sinkr_routed_decode_peer_async",
    # span-level attention operators (attention.hpp:14-85)
    "sinkr_attend_chunk", "sinkr_attend_chunk_cached", "sinkr_merge_partials",
    "sinkr_merge_partials_async", "sinkr_splitk_attention", "sinkr_online_attention",
    "sinkr_dense_attention",
    # per-token append (the decode loop's KvCache::append)
    "sinkr_kv_append_token_async", "sinkr_decode_append_step",
)

_lib = None


def lib():
    """Load libsinkr_cuda.so; raise (never fall back) if it is not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError(
                f"{LIB} is not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the engine has no CPU fallback)")
        L = C.CDLL(LIB)
        L.sinkr_last_error.restype = C.c_char_p
        L.sinkr_version.restype = C.c_char_p
        L.sinkr_engine_stream.restype = C.c_void_p
        L.sinkr_engine_stream.argtypes = [C.c_void_p]
        L.sinkr_auto_num_splits.restype = c_size_t
        L.sinkr_auto_num_splits.argtypes = [c_size_t]
        L.sinkr_rank_partial_floats.restype = c_size_t
        L.sinkr_rank_partial_floats.argtypes = [C.c_void_p]
        L.sinkr_decode_grid.restype = C.c_int
        L.sinkr_decode_grid.argtypes = [C.c_void_p]
        L.sinkr_engine_destroy.argtypes = [C.c_void_p]
        L.sinkr_peer_block.restype = C.c_void_p
        L.sinkr_peer_block.argtypes = [C.c_void_p]
        L.sinkr_snkt_file_size.restype = C.c_uint64
        L.sinkr_snkt_file_size.argtypes = [C.c_void_p, c_size_t]
        L.sinkr_profile_default.restype = None
        L.sinkr_profile_constant.restype = None
        L.sinkr_profile_constant.argtypes = [C.c_double, C.c_void_p]
        for name in ("sinkr_skip_ratio_at", "sinkr_solve_threshold"):
            getattr(L, name).argtypes = [C.c_void_p, c_size_t, C.c_double, C.c_void_p]
        L.sinkr_calibrate.argtypes = [C.c_void_p, c_size_t, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_double, C.c_double, C.c_void_p, c_size_t, C.c_void_p]
        L.sinkr_oracle_labels.argtypes = [C.c_void_p, c_size_t, c_size_t, C.c_double, C.c_int,
                                          C.c_void_p, C.c_void_p]
        vp, sz = C.c_void_p, c_size_t
        for name, at in {
            "sinkr_sweep": [vp, sz, vp, sz, vp],
            "sinkr_fit_cubic": [vp, vp, sz, vp, vp],
            "sinkr_save_profile": [C.c_char_p, vp],
            "sinkr_load_profile": [C.c_char_p, vp],
            "sinkr_profile_default": [vp],
            "sinkr_collect_scores": [vp, vp, sz, vp, vp, vp, vp],
            "sinkr_collect_scores_batch": [vp, vp, sz, sz, vp, vp, vp, vp],
            "sinkr_write_tensor": [C.c_char_p, vp, sz, vp],
            "sinkr_read_tensor": [C.c_char_p, vp, vp, vp, sz],
            "sinkr_save_snapshot": [vp, sz, C.c_char_p],
            "sinkr_load_snapshot": [C.c_char_p, C.c_int, vp],
            "sinkr_load_snapshot_into": [vp, sz, C.c_char_p],
            "sinkr_kv_append_device_f32": [vp, sz, sz, sz, vp, vp, sz],
            "sinkr_engine_config": [vp, vp],
            "sinkr_step_io_buffers": [vp, vp, vp],
            "sinkr_attention_bos_mass": [vp, vp, sz, vp],
            "sinkr_attention_weights": [vp, vp, sz, sz, sz, vp],
            "sinkr_attention_last_kernel_seconds": [vp, vp],
            "sinkr_group_attention": [vp, vp, sz, sz, sz, sz, vp, vp],
            "sinkr_routed_decode_peer": [vp, vp, sz, vp, vp, vp, vp, vp, vp],
            "sinkr_pr_curve": [vp, vp, sz, vp, vp, vp],
            "sinkr_peer_setup": [vp, C.c_uint32, C.c_uint32, vp],
            "sinkr_peer_ipc_handle": [vp, vp],
            "sinkr_peer_open": [vp, vp],
            "sinkr_peer_set_blocks": [vp, vp],
            "sinkr_routed_decode_peer_async": [vp, vp, sz, vp, vp, vp],
            "sinkr_attend_chunk": [vp, sz, sz, vp, vp, sz, sz, vp, vp, vp, vp],
            "sinkr_attend_chunk_cached": [vp, vp, sz, sz, sz, sz, sz, sz, vp, vp, vp, vp],
            "sinkr_merge_partials": [sz, vp, vp, vp, vp, sz, sz, vp],
            "sinkr_merge_partials_async": [sz, vp, vp, vp, vp, sz, sz, vp, vp],
            "sinkr_splitk_attention": [vp, sz, sz, vp, vp, sz, sz, sz, vp, vp],
            "sinkr_online_attention": [vp, sz, sz, vp, vp, sz, sz, vp],
            "sinkr_dense_attention": [vp, sz, sz, vp, vp, sz, vp],
            "sinkr_kv_append_token_async": [vp, sz, vp, vp],
            "sinkr_decode_append_step": [vp, vp, vp, vp, sz, vp, vp, vp, vp, vp, vp],
        }.items():
            getattr(L, name).argtypes = at
            getattr(L, name).restype = C.c_int if name != "sinkr_profile_default" else None
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != SINKR_OK:
        msg = lib().sinkr_last_error().decode(errors="replace")
        raise _EXC.get(rc, SinkrCudaError)(msg)
