"""Proxy-reliability analysis: full-attention BOS mass on
the GPU and the oracle-label / precision-recall machinery of analysis.hpp.

=============================================  ====================================
reference                                      here
=============================================  ====================================
attention_weights (attention.cpp:75-99)        attention_weights(cache, q, ...) [GPU]
  (its token-0 column, for every head)         attention_bos_mass(cache, q, layer) [GPU]
OracleMode / OracleLabel / oracle_labels       OracleMode / OracleLabel / oracle_labels
  (analysis.hpp:10-22)                         oracle_labels_from_alpha0
PrPoint / PrCurve / pr_curve (:24-39)          PrPoint / PrCurve / pr_curve
=============================================  ====================================

The reference declares oracle_labels / pr_curve without an implementation;
the semantics follow SPEC.md's analysis-oracle module (strict alpha0 > gamma,
group label from the mean alpha0, operating points at every distinct score,
AUPRC as average precision).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List

import numpy as np

from ._abi import check, lib
from .router import KvCache


class OracleMode(enum.IntEnum):
    Head = 0
    GroupMean = 1


@dataclass
class OracleLabel:
    alpha0: float = 0.0
    is_sink: bool = False


@dataclass
class PrPoint:
    threshold: float = 0.0
    precision: float = 0.0
    recall: float = 0.0
    f1: float = 0.0


@dataclass
class PrCurve:
    points: List[PrPoint] = field(default_factory=list)
    auprc: float = 0.0


def attention_bos_mass(cache: KvCache, queries, layer: int) -> np.ndarray:
    """alpha0 = softmax(scale q.K^T)[0] over the whole context of `layer` for
    every query head of every sequence: one K-only streaming pass on the GPU.
    Returns [B, H_q] float64."""
    cc = cache.config()
    q = np.ascontiguousarray(queries, dtype=np.float32)
    if q.size != cache.B * cc.num_q_heads * cc.head_dim:
        raise ValueError("queries span must be B x H_q x D for one layer")
    out = np.zeros((cache.B, cc.num_q_heads), dtype=np.float64)
    check(lib().sinkr_attention_bos_mass(cache.handle, q.ctypes.data, C.c_size_t(layer),
                                         out.ctypes.data))
    return out


def last_kernel_seconds(cache: KvCache) -> float:
    """Device time of the last attention_bos_mass / attention_weights call's
    kernels (CUDA events on the engine stream; host staging excluded)."""
    out = C.c_double()
    check(lib().sinkr_attention_last_kernel_seconds(cache.handle, C.byref(out)))
    return out.value


def attention_weights(cache: KvCache, group_queries, layer: int, kv_head: int,
                      seq: int = 0) -> np.ndarray:
    """attention_weights (attention.cpp:75-99) for one GQA group over the
    slot's cached rows, on the GPU: [r, L] float32."""
    cc = cache.config()
    r = cc.num_q_heads // cc.num_kv_heads
    q = np.ascontiguousarray(group_queries, dtype=np.float32)
    if q.size != r * cc.head_dim:
        raise ValueError("group queries must be r x D")
    L = cache.length(layer, kv_head, seq)
    out = np.zeros((r, L), dtype=np.float32)
    check(lib().sinkr_attention_weights(cache.handle, q.ctypes.data, C.c_size_t(seq),
                                        C.c_size_t(layer), C.c_size_t(kv_head), out.ctypes.data))
    return out


def oracle_labels_from_alpha0(alpha0, gamma: float, mode: OracleMode = OracleMode.Head,
                              group: int = 1) -> List[OracleLabel]:
    a = np.ascontiguousarray(alpha0, dtype=np.float64).ravel()
    n_out = a.size if mode == OracleMode.Head else (a.size // max(group, 1))
    la = np.zeros(max(n_out, 1), dtype=np.float64)
    sk = np.zeros(max(n_out, 1), dtype=np.uint8)
    check(lib().sinkr_oracle_labels(a.ctypes.data, C.c_size_t(a.size), C.c_size_t(group),
                                    C.c_double(gamma), C.c_int(int(mode)), la.ctypes.data,
                                    sk.ctypes.data))
    return [OracleLabel(float(la[i]), bool(sk[i])) for i in range(n_out)]


def oracle_labels(weights, heads: int, length: int, gamma: float,
                  mode: OracleMode) -> List[OracleLabel]:
    """analysis.hpp:17-19: one label per weight row (Head) or one for the
    group from the mean alpha0 over its rows (GroupMean); rows must sum to 1
    within 1e-4."""
    w = np.asarray(weights, dtype=np.float64).reshape(heads, length)
    sums = w.sum(axis=1)
    if np.any(np.abs(sums - 1.0) > 1e-4):
        raise ValueError("attention weight rows must sum to 1 within 1e-4")
    return oracle_labels_from_alpha0(w[:, 0], gamma, mode, heads)


def pr_curve(scores, labels) -> PrCurve:
    s = np.ascontiguousarray(scores, dtype=np.float64).ravel()
    l = np.ascontiguousarray(np.asarray(labels).astype(bool), dtype=np.uint8).ravel()
    if s.size != l.size:
        raise ValueError("scores and labels must have equal length")
    pts = np.zeros((max(s.size, 1), 4), dtype=np.float64)
    n = C.c_size_t()
    ap = C.c_double()
    check(lib().sinkr_pr_curve(s.ctypes.data, l.ctypes.data, C.c_size_t(s.size), pts.ctypes.data,
                               C.byref(n), C.byref(ap)))
    return PrCurve([PrPoint(*pts[i]) for i in range(n.value)], ap.value)
