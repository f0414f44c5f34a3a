"""The reference's span-level attention API (attention.hpp:14-85) on the GPU.

=====================================  ========================================
reference (attention.hpp)              here
=====================================  ========================================
QueryGroup::over (:14-21)              QueryGroup.over
SplitPartial (:26-33)                  SplitPartial (fp64 m, l, acc; tokens)
attend_chunk (:55-60)                  attend_chunk(qg, keys, values, len, block)
merge_partials (:62-64)                merge_partials(parts, heads, dim)
splitk_attention (:76-85)              splitk_attention(qg, keys, values, ...)
dense_attention (:38-42)               dense_attention(qg, keys, values, len)
online_attention (:48-53)              online_attention(qg, keys, values, ...)
=====================================  ========================================

Spans are host arrays (uploaded per call).  `attend_chunk_cached` runs
attend_chunk over a cached range of an engine (KvCache::historical +
attend_chunk, router.cpp:149-160) without a copy.  The cached-group forms of
splitk/dense/online_attention live in router.py and dispatch here when given
a QueryGroup / array instead of a KvCache.

Errors follow check_shapes (attention.cpp:13-23): ValueError for empty query
groups, len 0, mismatched span sizes, block_size 0, num_splits outside
[1, len], and an all-empty merge.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from ._abi import check, lib

kDefaultBlockSize = 128  # attention.hpp:35


@dataclass
class QueryGroup:
    """QueryGroup (attention.hpp:14-21): r query rows sharing a KV head."""
    q: np.ndarray          # [heads, dim] f32
    heads: int
    dim: int
    scale: float

    @staticmethod
    def over(q, heads: int, dim: int) -> "QueryGroup":
        """attention.cpp:33-40: scale = 1.0f / sqrt((float)dim)."""
        if dim == 0:
            raise ValueError("head_dim must be positive")
        a = np.ascontiguousarray(q, dtype=np.float32).reshape(-1)
        scale = float(np.float32(1.0) / np.float32(math.sqrt(np.float32(dim))))
        if a.size != heads * dim:
            raise ValueError("query span size does not match heads x dim")
        return QueryGroup(a.reshape(heads, dim) if heads else a, heads, dim, scale)


@dataclass
class SplitPartial:
    """SplitPartial (attention.hpp:26-33): fp64 online-softmax state."""
    m: np.ndarray = field(default_factory=lambda: np.zeros(0))    # [heads]
    l: np.ndarray = field(default_factory=lambda: np.zeros(0))    # [heads]
    acc: np.ndarray = field(default_factory=lambda: np.zeros(0))  # [heads, dim]
    tokens: int = 0

    def empty(self) -> bool:
        return self.tokens == 0


def _group(qg) -> QueryGroup:
    if isinstance(qg, QueryGroup):
        return qg
    a = np.asarray(qg, dtype=np.float32)
    if a.ndim != 2:
        raise ValueError("query group must be [heads, dim]")
    return QueryGroup.over(a, a.shape[0], a.shape[1])


def _span(x, length: Optional[int], dim: int, what: str):
    a = np.ascontiguousarray(x, dtype=np.float32).reshape(-1)
    n = a.size // dim if dim else 0
    if length is None:
        length = n
    if a.size != length * dim:
        raise ValueError(f"{what} span size does not match len x dim")
    return a, length


def _p(a) -> C.c_void_p:
    return a.ctypes.data_as(C.c_void_p)


def attend_chunk(qg, keys, values, length: Optional[int] = None,
                 block_size: int = kDefaultBlockSize) -> SplitPartial:
    """attend_chunk (attention.cpp:101-142) on the GPU."""
    g = _group(qg)
    k, length = _span(keys, length, g.dim, "key")
    v, _ = _span(values, length, g.dim, "value")
    m = np.zeros(g.heads)
    lsum = np.zeros(g.heads)
    acc = np.zeros((g.heads, g.dim))
    tok = C.c_uint64()
    check(lib().sinkr_attend_chunk(_p(np.ascontiguousarray(g.q, dtype=np.float32)), g.heads, g.dim,
                                   _p(k), _p(v), length, block_size, _p(m), _p(lsum), _p(acc),
                                   C.byref(tok)))
    return SplitPartial(m, lsum, acc, int(tok.value))


def attend_chunk_cached(cache, group_queries, layer: int, kv_head: int, frm: int, to: int,
                        seq: int = 0, block_size: int = kDefaultBlockSize) -> SplitPartial:
    """attend_chunk over the cached rows [frm, to) of (seq, layer, kv_head)."""
    cc = cache.config()
    r, d = cc.num_q_heads // cc.num_kv_heads, cc.head_dim
    q = np.ascontiguousarray(group_queries, dtype=np.float32)
    if q.size != r * d:
        raise ValueError("query span size does not match heads x dim")
    m = np.zeros(r)
    lsum = np.zeros(r)
    acc = np.zeros((r, d))
    tok = C.c_uint64()
    check(lib().sinkr_attend_chunk_cached(cache.handle, _p(q), seq, layer, kv_head, frm, to,
                                          block_size, _p(m), _p(lsum), _p(acc), C.byref(tok)))
    return SplitPartial(m, lsum, acc, int(tok.value))


def merge_partials(parts: Sequence[SplitPartial], heads: int, dim: int) -> np.ndarray:
    """merge_partials (attention.cpp:159-183): LSE combine on the GPU; empty
    partials are skipped, all-empty raises ValueError."""
    live = [p for p in parts if not p.empty()]
    for p in live:
        if (np.asarray(p.m).size != heads or np.asarray(p.l).size != heads
                or np.asarray(p.acc).size != heads * dim):
            raise ValueError("partial shape does not match heads x dim")
    n = len(parts)
    m = np.zeros((max(n, 1), heads))
    lsum = np.zeros((max(n, 1), heads))
    acc = np.zeros((max(n, 1), heads, dim))
    tok = np.zeros(max(n, 1), dtype=np.uint64)
    for i, p in enumerate(parts):
        tok[i] = p.tokens
        if not p.empty():
            m[i] = p.m
            lsum[i] = p.l
            acc[i] = np.asarray(p.acc).reshape(heads, dim)
    out = np.zeros((heads, dim), dtype=np.float32)
    check(lib().sinkr_merge_partials(n, _p(m), _p(lsum), _p(acc), _p(tok), heads, dim, _p(out)))
    return out


def splitk_attention(qg, keys, values, length: Optional[int] = None, num_splits: int = 1,
                     pool=None, block_size: int = kDefaultBlockSize):
    """splitk_attention (attention.cpp:204-235) over host spans -> SplitkResult.
    `pool` (a ThreadPool in the reference) is accepted and ignored: the split
    runs on the GPU."""
    from .router import LoadCounters, SplitkResult

    g = _group(qg)
    k, length = _span(keys, length, g.dim, "key")
    v, _ = _span(values, length, g.dim, "value")
    out = np.zeros((g.heads, g.dim), dtype=np.float32)
    from ._abi import LoadCountersC

    ctr = LoadCountersC()
    check(lib().sinkr_splitk_attention(_p(np.ascontiguousarray(g.q, dtype=np.float32)), g.heads,
                                       g.dim, _p(k), _p(v), length, num_splits, block_size,
                                       _p(out), C.byref(ctr)))
    return SplitkResult(out=out, counters=LoadCounters(int(ctr.kv_floats_loaded)))


def online_attention(qg, keys, values, length: Optional[int] = None,
                     block_size: int = kDefaultBlockSize) -> np.ndarray:
    """online_attention (attention.cpp:144-157) over host spans."""
    g = _group(qg)
    k, length = _span(keys, length, g.dim, "key")
    v, _ = _span(values, length, g.dim, "value")
    out = np.zeros((g.heads, g.dim), dtype=np.float32)
    check(lib().sinkr_online_attention(_p(np.ascontiguousarray(g.q, dtype=np.float32)), g.heads,
                                       g.dim, _p(k), _p(v), length, block_size, _p(out)))
    return out


def dense_attention(qg, keys, values, length: Optional[int] = None) -> np.ndarray:
    """dense_attention (attention.cpp:42-73) over host spans."""
    g = _group(qg)
    k, length = _span(keys, length, g.dim, "key")
    v, _ = _span(values, length, g.dim, "value")
    out = np.zeros((g.heads, g.dim), dtype=np.float32)
    check(lib().sinkr_dense_attention(_p(np.ascontiguousarray(g.q, dtype=np.float32)), g.heads,
                                      g.dim, _p(k), _p(v), length, _p(out)))
    return out
