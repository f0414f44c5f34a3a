"""Host-side mirror of the reference's operator API (router.hpp, kv_cache.hpp,
calibration.hpp's ThresholdProfile, counters.hpp), backed by the sm_100a engine
through the C-ABI in include/sinkr_cuda.h.

Names, argument meaning and error behaviour follow the reference:

=============================  ===============================================
reference                      here
=============================  ===============================================
CacheConfig (kv_cache.hpp:13)  CacheConfig (+ num_seqs for batched caches)
KvCache (kv_cache.hpp:42-80)   KvCache — bf16 K/V resident in HBM
ThresholdProfile (calib.:21)   ThresholdProfile, ThresholdProfile.constant
RoutingConfig (router.hpp:16)  RoutingConfig, RoutingConfig.from_profile
EngineOptions (router.hpp:69)  EngineOptions (+ global_context_len)
threshold_for_length / route   threshold_for_length / route (host scalar logic)
auto_num_splits / split_ranges auto_num_splits / split_ranges
routed_decode_step (:84-86)    routed_decode_step  -> LayerStepResult
=============================  ===============================================

Exceptions: std::invalid_argument -> ValueError, std::out_of_range ->
IndexError, std::runtime_error -> RuntimeError, std::logic_error ->
LogicError (an AssertionError subclass).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _abi
from ._abi import check, lib

kDefaultBlockSize = 128  # attention.hpp:35


# ----------------------------------------------------------------------------
# configuration types
@dataclass
class CacheConfig:
    num_layers: int = 0
    num_q_heads: int = 0
    num_kv_heads: int = 0
    head_dim: int = 0
    capacity: int = 0
    num_seqs: int = 1

    def group_width(self) -> int:
        return self.num_q_heads // self.num_kv_heads


@dataclass
class ThresholdProfile:
    coeffs: Sequence[float] = (0.0, 0.0, 0.0, 0.0)
    length_normalizer: float = 1.0
    clamp_lo: float = 0.0
    clamp_hi: float = 1.0
    target_skip: float = 0.60
    gamma: float = 0.65
    excluded_layers: Sequence[int] = (0, 1)
    points: list = field(default_factory=list)

    @staticmethod
    def constant(tau: float) -> "ThresholdProfile":
        """calibration.cpp:29-35 — clamp widened so tau outside [0,1] holds."""
        return ThresholdProfile(coeffs=(0.0, 0.0, 0.0, float(tau)),
                                clamp_lo=min(tau, 0.0), clamp_hi=max(tau, 1.0))

    def _c(self) -> _abi.ThresholdProfileC:
        p = _abi.ThresholdProfileC()
        for i in range(4):
            p.coeffs[i] = float(self.coeffs[i])
        p.length_normalizer = float(self.length_normalizer)
        p.clamp_lo = float(self.clamp_lo)
        p.clamp_hi = float(self.clamp_hi)
        return p


@dataclass
class RoutingConfig:
    gamma: float = 0.65
    profile: ThresholdProfile = field(default_factory=ThresholdProfile)
    excluded_layers: Sequence[int] = (0, 1)
    sink_on_tie: bool = False

    @staticmethod
    def from_profile(profile: ThresholdProfile) -> "RoutingConfig":
        """router.cpp:23-29."""
        return RoutingConfig(gamma=profile.gamma, profile=profile,
                             excluded_layers=tuple(profile.excluded_layers))

    def layer_excluded(self, layer: int) -> bool:
        return layer in tuple(self.excluded_layers)

    def _c(self):
        arr = (C.c_size_t * max(1, len(self.excluded_layers)))(*self.excluded_layers)
        c = _abi.RoutingConfigC()
        c.gamma = float(self.gamma)
        c.profile = self.profile._c()
        c.excluded_layers = C.cast(arr, C.POINTER(C.c_size_t))
        c.num_excluded_layers = len(self.excluded_layers)
        c.sink_on_tie = int(bool(self.sink_on_tie))
        return c, arr  # keep `arr` alive for the duration of the call


@dataclass
class EngineOptions:
    num_splits: int = 0
    block_size: int = kDefaultBlockSize
    observe_only: bool = False
    global_context_len: int = 0

    def _c(self) -> _abi.EngineOptionsC:
        o = _abi.EngineOptionsC()
        o.num_splits = int(self.num_splits)
        o.block_size = int(self.block_size)
        o.observe_only = int(bool(self.observe_only))
        o.global_context_len = int(self.global_context_len)
        return o


# ----------------------------------------------------------------------------
# result types (router.hpp:28-39,56-67; counters.hpp:9-28)
@dataclass
class LoadCounters:
    kv_floats_loaded: int = 0
    anchor_floats_loaded: int = 0
    groups_active: int = 0
    groups_skipped: int = 0
    routing_seconds: float = 0.0
    attention_seconds: float = 0.0
    merge_seconds: float = 0.0


@dataclass
class RouteDecision:
    group_score: float = 0.0
    threshold: float = 0.0
    sink: bool = False
    degenerate: bool = False
    head_scores: List[float] = field(default_factory=list)


@dataclass
class GroupStepInfo:
    layer: int = 0
    kv_head: int = 0
    decision: RouteDecision = field(default_factory=RouteDecision)
    kv_floats_loaded: int = 0
    tokens_loaded: int = 0
    seq: int = 0


@dataclass
class LayerStepResult:
    outputs: np.ndarray  # [H_q, D] (or [B, H_q, D] for batched caches)
    groups: List[GroupStepInfo]
    counters: LoadCounters

    @property
    def route_bitmap(self) -> np.ndarray:
        """Sink bit per group (the routing decision the probe kernel emits)."""
        return np.array([g.decision.sink for g in self.groups], dtype=bool)


# ----------------------------------------------------------------------------
# host scalar helpers (router.hpp:47-54,78; attention.hpp:82-85)
def threshold_for_length(context_len: int, profile: ThresholdProfile) -> float:
    out = C.c_double()
    p = profile._c()
    check(lib().sinkr_threshold_for_length(C.c_size_t(context_len), C.byref(p), C.byref(out)))
    return out.value


def route(layer: int, score: float, context_len: int, config: RoutingConfig) -> RouteDecision:
    c, keep = config._c()
    sink, tau = C.c_int(), C.c_double()
    check(lib().sinkr_route(C.c_size_t(layer), C.c_double(score), C.c_size_t(context_len),
                            C.byref(c), C.byref(sink), C.byref(tau)))
    del keep
    return RouteDecision(group_score=score, threshold=tau.value, sink=bool(sink.value))


def auto_num_splits(context_len: int) -> int:
    return int(lib().sinkr_auto_num_splits(C.c_size_t(context_len)))


def split_ranges(length: int, num_splits: int):
    buf = (C.c_size_t * (2 * max(1, num_splits)))()
    check(lib().sinkr_split_ranges(C.c_size_t(length), C.c_size_t(num_splits), buf))
    return [(buf[2 * i], buf[2 * i + 1]) for i in range(num_splits)]


# ----------------------------------------------------------------------------
class KvCache:
    """kv_cache.hpp:42-80 on the GPU: bf16 K/V [layer][seq][kv_head][cap][D] in
    HBM, f32 anchors captured at first append (kv_cache.cpp:71-77)."""

    def __init__(self, config: CacheConfig, device: int = 0):
        self._h = None
        self._config = config
        cc = _abi.CacheConfigC(config.num_layers, config.num_q_heads, config.num_kv_heads,
                               config.head_dim, config.capacity, config.num_seqs or 1)
        h = C.c_void_p()
        check(lib().sinkr_engine_create(C.byref(cc), C.c_int(device), C.byref(h)))
        self._h = h
        self.device = device
        self.B = config.num_seqs or 1
        self._keep = []

    # -- lifetime
    def close(self):
        if self._h:
            lib().sinkr_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self):
        return self._h

    def config(self) -> CacheConfig:
        return self._config

    @property
    def stream(self) -> int:
        return int(lib().sinkr_engine_stream(self._h) or 0)

    def decode_grid(self) -> int:
        return int(lib().sinkr_decode_grid(self._h))

    # -- KvCache API
    def append(self, layer: int, kv_head: int, k, v, seq: int = 0) -> None:
        """Append one row (D,) or rows (n, D) of f32 keys/values."""
        d = self._config.head_dim
        k = np.ascontiguousarray(k, dtype=np.float32).reshape(-1)
        v = np.ascontiguousarray(v, dtype=np.float32).reshape(-1)
        if k.size != v.size or k.size % d != 0 or k.size == 0:
            raise ValueError("k/v row size does not match head_dim")
        check(lib().sinkr_kv_append(self._h, C.c_size_t(seq), C.c_size_t(layer),
                                    C.c_size_t(kv_head), k.ctypes.data_as(C.c_void_p),
                                    v.ctypes.data_as(C.c_void_p), C.c_size_t(k.size // d)))

    def append_device_bf16(self, layer: int, kv_head: int, k_ptr: int, v_ptr: int, rows: int,
                           seq: int = 0) -> None:
        check(lib().sinkr_kv_append_device_bf16(self._h, C.c_size_t(seq), C.c_size_t(layer),
                                                C.c_size_t(kv_head), C.c_void_p(k_ptr),
                                                C.c_void_p(v_ptr), C.c_size_t(rows)))

    def append_synthetic(self, layer: int, kv_head: int, key_k: int, key_v: int, rows: int,
                         k_scale: float = 1.0, v_scale: float = 1.0, seq: int = 0,
                         global_row0: int = None) -> None:
        """Append `rows` device-generated rows; their values are those of global
        rows global_row0.. (default: the slot's current length)."""
        if global_row0 is None:
            global_row0 = self.length(layer, kv_head, seq)
        check(lib().sinkr_kv_append_synthetic(
            self._h, C.c_size_t(seq), C.c_size_t(layer), C.c_size_t(kv_head),
            C.c_uint64(key_k), C.c_uint64(key_v), C.c_float(k_scale), C.c_float(v_scale),
            C.c_size_t(global_row0), C.c_size_t(rows)))

    def append_token_async(self, layer: int, d_k_new: int, d_v_new: int) -> None:
        """The decode loop's append: one new row to every (seq, kv_head) slot of
        `layer` from device f32 [B][H_kv][D] buffers, enqueued on the engine
        stream (no host sync after the first row)."""
        check(lib().sinkr_kv_append_token_async(self.handle, layer, C.c_void_p(d_k_new),
                                                C.c_void_p(d_v_new)))

    def step_io_bytes(self):
        h2d, d2h = C.c_size_t(), C.c_size_t()
        check(lib().sinkr_step_io_bytes(self._h, C.byref(h2d), C.byref(d2h)))
        return h2d.value, d2h.value

    def length(self, layer: int, kv_head: int, seq: int = 0) -> int:
        out = C.c_size_t()
        check(lib().sinkr_kv_length(self._h, C.c_size_t(seq), C.c_size_t(layer),
                                    C.c_size_t(kv_head), C.byref(out)))
        return out.value

    def token_count(self, seq: int = 0) -> int:
        out = C.c_size_t()
        check(lib().sinkr_kv_token_count(self._h, C.c_size_t(seq), C.byref(out)))
        return out.value

    def anchor(self, layer: int, kv_head: int, seq: int = 0):
        k0 = np.zeros(self._config.head_dim, dtype=np.float32)
        n = C.c_float()
        check(lib().sinkr_kv_anchor(self._h, C.c_size_t(seq), C.c_size_t(layer),
                                    C.c_size_t(kv_head), k0.ctypes.data_as(C.c_void_p),
                                    C.byref(n)))
        return k0, n.value

    def set_anchor(self, layer: int, kv_head: int, k0, k0_norm: float, seq: int = 0) -> None:
        k0 = np.ascontiguousarray(k0, dtype=np.float32)
        check(lib().sinkr_kv_set_anchor(self._h, C.c_size_t(seq), C.c_size_t(layer),
                                        C.c_size_t(kv_head), k0.ctypes.data_as(C.c_void_p),
                                        C.c_float(k0_norm)))

    def append_device_f32(self, layer: int, kv_head: int, k_ptr: int, v_ptr: int, rows: int,
                          seq: int = 0) -> None:
        """Device prefill: f32 rows already in device memory, converted to bf16
        on the device (16-byte aligned pointers)."""
        check(lib().sinkr_kv_append_device_f32(self._h, C.c_size_t(seq), C.c_size_t(layer),
                                               C.c_size_t(kv_head), C.c_void_p(k_ptr),
                                               C.c_void_p(v_ptr), C.c_size_t(rows)))

    # -- snapshots (kv_cache.hpp:72-80; SNKT files + manifest.json)
    def save_snapshot(self, directory, seq: int = 0) -> None:
        """KvCache::save_snapshot for sequence `seq` (kv_cache.cpp:123-153)."""
        check(lib().sinkr_save_snapshot(self._h, C.c_size_t(seq), str(directory).encode()))

    def load_snapshot_into(self, directory, seq: int = 0) -> None:
        """Replays a snapshot into sequence `seq` of this (empty) cache."""
        check(lib().sinkr_load_snapshot_into(self._h, C.c_size_t(seq), str(directory).encode()))

    @staticmethod
    def load_snapshot(directory, device: int = 0) -> "KvCache":
        """KvCache::load_snapshot (kv_cache.cpp:155-191): a single-sequence
        cache sized by the manifest, rows replayed on the device."""
        h = C.c_void_p()
        check(lib().sinkr_load_snapshot(str(directory).encode(), C.c_int(device), C.byref(h)))
        cc = _abi.CacheConfigC()
        check(lib().sinkr_engine_config(h, C.byref(cc)))
        self = KvCache.__new__(KvCache)
        self._h = h
        self._config = CacheConfig(cc.num_layers, cc.num_q_heads, cc.num_kv_heads, cc.head_dim,
                                   cc.capacity, cc.num_seqs)
        self.device = device
        self.B = cc.num_seqs
        self._keep = []
        return self

    def historical(self, layer: int, kv_head: int, frm: int, to: int, seq: int = 0):
        """Rows [frm, to) of K and V as f32 (exact upcast of the stored bf16)."""
        d = self._config.head_dim
        k = np.zeros((to - frm, d), dtype=np.float32)
        v = np.zeros((to - frm, d), dtype=np.float32)
        check(lib().sinkr_kv_read(self._h, C.c_size_t(seq), C.c_size_t(layer),
                                  C.c_size_t(kv_head), C.c_size_t(frm), C.c_size_t(to),
                                  k.ctypes.data_as(C.c_void_p), v.ctypes.data_as(C.c_void_p)))
        return k, v


# ----------------------------------------------------------------------------
def _step_buffers(cache: KvCache):
    cc = cache.config()
    B = cache.B
    out = np.zeros((B, cc.num_q_heads, cc.head_dim), dtype=np.float32)
    groups = (_abi.GroupInfoC * (B * cc.num_kv_heads))()
    hs = np.zeros(B * cc.num_q_heads, dtype=np.float64)
    ctr = _abi.LoadCountersC()
    return out, groups, hs, ctr


def _to_result(cache: KvCache, out, groups, hs, ctr, batched: bool) -> LayerStepResult:
    cc = cache.config()
    r = cc.group_width()
    infos = []
    for u in range(cache.B * cc.num_kv_heads):
        g = groups[u]
        seq = u // cc.num_kv_heads
        h0 = seq * cc.num_q_heads + g.kv_head * r
        dec = RouteDecision(group_score=g.group_score, threshold=g.threshold, sink=bool(g.sink),
                            degenerate=bool(g.degenerate), head_scores=list(hs[h0:h0 + r]))
        infos.append(GroupStepInfo(layer=g.layer, kv_head=g.kv_head, decision=dec,
                                   kv_floats_loaded=int(g.kv_floats_loaded),
                                   tokens_loaded=int(g.tokens_loaded), seq=seq))
    counters = LoadCounters(int(ctr.kv_floats_loaded), int(ctr.anchor_floats_loaded),
                            int(ctr.groups_active), int(ctr.groups_skipped),
                            ctr.routing_seconds, ctr.attention_seconds, ctr.merge_seconds)
    return LayerStepResult(outputs=out if batched else out[0], groups=infos, counters=counters)


def routed_decode_step(queries, layer: int, cache: KvCache, config: RoutingConfig,
                       options: Optional[EngineOptions] = None) -> LayerStepResult:
    """router.hpp:84-86 — one decode step for one layer (all B sequences).

    queries: f32 [H_q, D] (or [B, H_q, D] for a batched cache), host memory.
    """
    cc = cache.config()
    q = np.ascontiguousarray(queries, dtype=np.float32)
    if q.size != cache.B * cc.num_q_heads * cc.head_dim:
        raise ValueError("queries span must be H_q x D for one layer")
    out, groups, hs, ctr = _step_buffers(cache)
    c, keep = config._c()
    o = (options or EngineOptions())._c()
    check(lib().sinkr_routed_decode_batch(cache.handle, q.ctypes.data_as(C.c_void_p),
                                          C.c_size_t(layer), C.byref(c), C.byref(o),
                                          out.ctypes.data_as(C.c_void_p), groups,
                                          hs.ctypes.data_as(C.c_void_p), C.byref(ctr)))
    del keep
    return _to_result(cache, out, groups, hs, ctr, batched=cache.B > 1 or q.ndim == 3)


@dataclass
class SplitkResult:
    """SplitkResult (attention.hpp:71-74)."""
    out: np.ndarray            # [r, D] f32
    counters: LoadCounters


def splitk_attention(cache, group_queries, layer=None, kv_head=None,
                     num_splits=1, seq=0, **kw) -> SplitkResult:
    """splitk_attention (attention.cpp:204-235) of one cached group on the GPU:
    the group's r query heads over all of its cached rows.  num_splits is
    validated like split_ranges; the kernel picks its own split.  Replaces the
    engine's last routing record.

    Called with a QueryGroup (or a [heads, dim] array) and host K/V spans
    instead of a KvCache, this is the reference's span overload
    (attention.hpp:76-85): see attention.splitk_attention."""
    if not isinstance(cache, KvCache):
        from . import attention as _A

        # (qg, keys, values, len, num_splits, pool, block_size)
        return _A.splitk_attention(cache, group_queries, layer, kv_head, num_splits, seq, **kw)
    if layer is None or kv_head is None:
        raise TypeError("splitk_attention(cache, group_queries, layer, kv_head, num_splits, ...)")
    cc = cache.config()
    r = cc.num_q_heads // cc.num_kv_heads
    q = np.ascontiguousarray(group_queries, dtype=np.float32)
    if q.size != r * cc.head_dim:
        raise ValueError("query span size does not match heads x dim")
    out = np.zeros((r, cc.head_dim), dtype=np.float32)
    ctr = _abi.LoadCountersC()
    check(lib().sinkr_group_attention(cache.handle, q.ctypes.data_as(C.c_void_p), C.c_size_t(seq),
                                      C.c_size_t(layer), C.c_size_t(kv_head),
                                      C.c_size_t(num_splits), out.ctypes.data_as(C.c_void_p),
                                      C.byref(ctr)))
    return SplitkResult(out=out, counters=LoadCounters(int(ctr.kv_floats_loaded)))


def dense_attention(cache, group_queries, layer=None, kv_head=None,
                    seq: int = 0) -> np.ndarray:
    """dense_attention (attention.cpp:42-73) of one cached group: [r, D] f32
    (the GPU group attention; exact softmax to fp32 accumulation).  With a
    QueryGroup / array and host spans (qg, keys, values[, len]): the span
    overload (attention.dense_attention)."""
    if not isinstance(cache, KvCache):
        from . import attention as _A

        return _A.dense_attention(cache, group_queries, layer, kv_head)
    if layer is None or kv_head is None:
        raise TypeError("dense_attention(cache, group_queries, layer, kv_head, ...)")
    return splitk_attention(cache, group_queries, layer, kv_head, 1, seq).out


def online_attention(cache, group_queries, layer=None, kv_head=None,
                     block_size: int = kDefaultBlockSize, seq: int = 0) -> np.ndarray:
    """online_attention (attention.cpp:144-157) of one cached group: [r, D] f32.
    block_size is validated like attend_chunk (attention.cpp:107); the GPU
    streams in its own 64-token stages.  With a QueryGroup / array and host
    spans (qg, keys, values[, len[, block_size]]): the span overload
    (attention.online_attention)."""
    if not isinstance(cache, KvCache):
        from . import attention as _A

        return _A.online_attention(cache, group_queries, layer, kv_head, block_size)
    if layer is None or kv_head is None:
        raise TypeError("online_attention(cache, group_queries, layer, kv_head, ...)")
    if block_size == 0:
        raise ValueError("block_size must be positive")
    return splitk_attention(cache, group_queries, layer, kv_head, 1, seq).out


def routed_decode_async(d_queries: int, layer: int, cache: KvCache, config: RoutingConfig,
                        options: Optional[EngineOptions] = None, d_outputs: int = 0) -> None:
    """Device-resident step: enqueue on the engine stream, no host sync."""
    c, keep = config._c()
    o = (options or EngineOptions())._c()
    check(lib().sinkr_routed_decode_async(cache.handle, C.c_void_p(d_queries),
                                          C.c_size_t(layer), C.byref(c), C.byref(o),
                                          C.c_void_p(d_outputs)))
    del keep


def fetch_step_info(cache: KvCache) -> LayerStepResult:
    out, groups, hs, ctr = _step_buffers(cache)
    check(lib().sinkr_fetch_step_info(cache.handle, groups, hs.ctypes.data_as(C.c_void_p),
                                      C.byref(ctr)))
    return _to_result(cache, None, groups, hs, ctr, batched=True)


def last_step_stats(cache: KvCache):
    n = C.c_uint32()
    dms, sms = C.c_float(), C.c_float()
    check(lib().sinkr_last_step_stats(cache.handle, C.byref(n), C.byref(dms), C.byref(sms)))
    return int(n.value), float(dms.value), float(sms.value)


def set_timing(cache: KvCache, enabled: bool) -> None:
    check(lib().sinkr_set_timing(cache.handle, C.c_int(int(enabled))))


# ----------------------------------------------------------------------------
# sequence-sharded multi-GPU split (sharding.py)
def rank_partial_floats(cache: KvCache) -> int:
    return int(lib().sinkr_rank_partial_floats(cache.handle))


def decode_rank_partial_async(d_queries: int, layer: int, cache: KvCache, config: RoutingConfig,
                              options: Optional[EngineOptions], d_partial: int) -> None:
    c, keep = config._c()
    o = (options or EngineOptions())._c()
    check(lib().sinkr_decode_rank_partial_async(cache.handle, C.c_void_p(d_queries),
                                                C.c_size_t(layer), C.byref(c), C.byref(o),
                                                C.c_void_p(d_partial)))
    del keep


def merge_rank_partials_async(cache: KvCache, d_gathered: int, num_ranks: int,
                              d_outputs: int) -> None:
    check(lib().sinkr_merge_rank_partials_async(cache.handle, C.c_void_p(d_gathered),
                                                C.c_size_t(num_ranks), C.c_void_p(d_outputs)))


def routed_decode_peer_async(d_queries: int, layer: int, cache: KvCache, config: RoutingConfig,
                             options: Optional[EngineOptions], d_outputs: int) -> None:
    """Sequence-sharded step with the merge fused into the kernel (peer memory);
    needs sharding.PeerMerge set up on every rank."""
    c, keep = config._c()
    o = (options or EngineOptions())._c()
    check(lib().sinkr_routed_decode_peer_async(cache.handle, C.c_void_p(d_queries),
                                               C.c_size_t(layer), C.byref(c), C.byref(o),
                                               C.c_void_p(d_outputs)))
    del keep


KvCache.rank_partial_floats = rank_partial_floats


class StepRunner:
    """Lean repeated-call form of routed_decode_step for serving loops: all
    host buffers and C structs are allocated once, each call is one C-ABI call
    (sinkr_routed_decode_batch: H2D queries -> graph -> D2H results, blocking).
    Returns the reused output buffer; `result()` builds the full
    LayerStepResult of the last call on demand."""

    def __init__(self, cache: KvCache, config: RoutingConfig, options: Optional[EngineOptions] = None,
                 layer: int = 0, pinned_io: bool = False):
        self.cache = cache
        self.layer = layer
        self.out, self.groups, self.hs, self.ctr = _step_buffers(cache)
        self.queries = None
        if pinned_io:
            # the engine's own pinned buffers (sinkr_step_io_buffers): fill
            # `self.queries`, call with no argument, read the returned outputs;
            # no host copy on either side
            qp, op = C.c_void_p(), C.c_void_p()
            check(lib().sinkr_step_io_buffers(cache.handle, C.byref(qp), C.byref(op)))
            shape, n = self.out.shape, self.out.size
            self.queries = np.ctypeslib.as_array((C.c_float * n).from_address(qp.value)).reshape(shape)
            self.out = np.ctypeslib.as_array((C.c_float * n).from_address(op.value)).reshape(shape)
        self._cfg, self._keep = config._c()
        self._opt = (options or EngineOptions())._c()
        L = lib()
        self._fn = L.sinkr_routed_decode_batch
        self._fn.restype = C.c_int
        self._fn.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p,
                             C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        self._args = (cache.handle, None, layer, C.addressof(self._cfg), C.addressof(self._opt),
                      self.out.ctypes.data, C.addressof(self.groups), self.hs.ctypes.data,
                      C.addressof(self.ctr))
        self._qsize = self.out.size

    def __call__(self, queries: Optional[np.ndarray] = None) -> np.ndarray:
        if queries is None:
            if self.queries is None:
                raise ValueError("no queries: pass them, or build the runner with pinned_io=True")
            queries = self.queries
        if queries.dtype != np.float32 or not queries.flags.c_contiguous or \
                queries.size != self._qsize:
            queries = np.ascontiguousarray(queries, dtype=np.float32)
            if queries.size != self._qsize:
                raise ValueError("queries span must be H_q x D for one layer")
        h, _, layer, cfg, opt, out, groups, hs, ctr = self._args
        rc = self._fn(h, queries.ctypes.data, layer, cfg, opt, out, groups, hs, ctr)
        if rc:
            check(rc)
        return self.out

    def result(self) -> LayerStepResult:
        return _to_result(self.cache, self.out.copy(), self.groups, self.hs, self.ctr,
                          batched=self.cache.B > 1)


class AppendStepRunner(StepRunner):
    """StepRunner whose calls first append the new token's K/V rows (host f32
    [B][H_kv][D]) to every slot of the layer, then step over the grown cache:
    sinkr_decode_append_step, one graph per call."""

    def __init__(self, cache: KvCache, config: RoutingConfig, options: Optional[EngineOptions] = None,
                 layer: int = 0, pinned_io: bool = False):
        super().__init__(cache, config, options, layer, pinned_io)
        self._fa = lib().sinkr_decode_append_step
        cc = cache.config()
        self._kvsize = cache.B * cc.num_kv_heads * cc.head_dim

    def __call__(self, k_new, v_new, queries: Optional[np.ndarray] = None) -> np.ndarray:
        if queries is None:
            if self.queries is None:
                raise ValueError("no queries: pass them, or build the runner with pinned_io=True")
            queries = self.queries
        queries = np.ascontiguousarray(queries, dtype=np.float32)
        k = np.ascontiguousarray(k_new, dtype=np.float32)
        v = np.ascontiguousarray(v_new, dtype=np.float32)
        if queries.size != self._qsize:
            raise ValueError("queries span must be H_q x D for one layer")
        if k.size != self._kvsize or v.size != self._kvsize:
            raise ValueError("k/v row size does not match head_dim")
        h, _, layer, cfg, opt, out, groups, hs, ctr = self._args
        rc = self._fa(h, queries.ctypes.data, k.ctypes.data, v.ctypes.data, layer, cfg, opt, out,
                      groups, hs, ctr)
        if rc:
            check(rc)
        return self.out
