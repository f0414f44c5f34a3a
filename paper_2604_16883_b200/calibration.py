"""Threshold calibration: the reference's calibration.hpp
API over the C-ABI, with score collection on the GPU.

=============================================  ====================================
reference (calibration.hpp)                    here
=============================================  ====================================
CalibrationPoint (:14-18)                      CalibrationPoint
ScoreSample / ScorePopulation (:36-50)         ScoreSample / ScorePopulation
sweep / skip_ratio_at / solve_threshold        sweep / skip_ratio_at / solve_threshold
CubicFit / fit_cubic (:63-70)                  CubicFit / fit_cubic
ScoreCollector / calibrate (:72-83)            calibrate(collect, lengths, ...)
save_profile / load_profile (:85-86)           save_profile / load_profile
router score-collection mode     collect_scores(cache, queries, layer)
=============================================  ====================================

The statistics and the fit run in the library's host C++ (bit-identical to
the reference: same expression order, no FMA contraction); ``collect_scores``
runs the routing phase alone on the GPU — no K/V streaming — so a calibration
sample costs one probe launch.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import _abi
from ._abi import check, lib
from .router import KvCache, RoutingConfig, ThresholdProfile


@dataclass
class CalibrationPoint:
    length: int = 0
    tau: float = 0.0
    skip: float = 0.0


@dataclass
class ScoreSample:
    score: float = 0.0
    layer: int = 0
    length: int = 0


@dataclass
class ScorePopulation:
    samples: List[ScoreSample] = field(default_factory=list)

    def add(self, score: float, layer: int, length: int) -> None:
        self.samples.append(ScoreSample(float(score), int(layer), int(length)))

    def extend(self, scores, layer: int, length: int) -> None:
        for s in np.asarray(scores, dtype=np.float64).ravel():
            self.add(s, layer, length)

    def size(self) -> int:
        return len(self.samples)

    def empty(self) -> bool:
        return not self.samples

    def scores(self) -> np.ndarray:
        return np.array([s.score for s in self.samples], dtype=np.float64)

    def layers(self) -> np.ndarray:
        return np.array([s.layer for s in self.samples], dtype=np.uint64)


@dataclass
class CubicFit:
    coeffs: Tuple[float, float, float, float] = (0.0, 0.0, 0.0, 0.0)
    residual: float = 0.0


def _scores(pop) -> np.ndarray:
    a = pop.scores() if isinstance(pop, ScorePopulation) else np.asarray(pop, dtype=np.float64)
    return np.ascontiguousarray(a, dtype=np.float64)


def sweep(pop, thresholds: Sequence[float]):
    """Fraction of scores strictly greater than each threshold (calibration.cpp:37-47)."""
    s = _scores(pop)
    t = np.ascontiguousarray(thresholds, dtype=np.float64)
    out = np.zeros(len(t))
    check(lib().sinkr_sweep(s.ctypes.data, C.c_size_t(s.size), t.ctypes.data, C.c_size_t(t.size),
                            out.ctypes.data))
    return list(zip(t.tolist(), out.tolist()))


def skip_ratio_at(pop, threshold: float) -> float:
    s = _scores(pop)
    out = C.c_double()
    check(lib().sinkr_skip_ratio_at(s.ctypes.data, s.size, float(threshold), C.byref(out)))
    return out.value


def solve_threshold(pop, target_skip: float) -> float:
    """Lower (1 - target) empirical quantile (calibration.cpp:58-71)."""
    s = _scores(pop)
    out = C.c_double()
    check(lib().sinkr_solve_threshold(s.ctypes.data, s.size, float(target_skip), C.byref(out)))
    return out.value


def fit_cubic(points: Sequence[Tuple[float, float]]) -> CubicFit:
    pts = list(points)
    x = np.ascontiguousarray([p[0] for p in pts], dtype=np.float64)
    y = np.ascontiguousarray([p[1] for p in pts], dtype=np.float64)
    co = (C.c_double * 4)()
    res = C.c_double()
    check(lib().sinkr_fit_cubic(x.ctypes.data, y.ctypes.data, C.c_size_t(len(pts)), co, C.byref(res)))
    return CubicFit(tuple(co), res.value)


def _profile_from_c(p: _abi.ProfileC) -> ThresholdProfile:
    t = p.threshold
    return ThresholdProfile(
        coeffs=tuple(t.coeffs), length_normalizer=t.length_normalizer, clamp_lo=t.clamp_lo,
        clamp_hi=t.clamp_hi, target_skip=p.target_skip, gamma=p.gamma,
        excluded_layers=tuple(int(p.excluded_layers[i]) for i in range(p.num_excluded_layers)),
        points=[CalibrationPoint(int(p.points[i].length), p.points[i].tau, p.points[i].skip)
                for i in range(p.num_points)])


def _profile_to_c(prof: ThresholdProfile) -> _abi.ProfileC:
    p = _abi.ProfileC()
    p.threshold = prof._c()
    p.target_skip = float(prof.target_skip)
    p.gamma = float(prof.gamma)
    ex = list(prof.excluded_layers)
    if len(ex) > _abi.MAX_EXCLUDED_LAYERS:
        raise ValueError("too many excluded layers")
    for i, l in enumerate(ex):
        p.excluded_layers[i] = int(l)
    p.num_excluded_layers = len(ex)
    pts = list(prof.points)
    if len(pts) > _abi.MAX_CALIBRATION_POINTS:
        raise ValueError("too many calibration points")
    for i, q in enumerate(pts):
        p.points[i].length = int(q.length)
        p.points[i].tau = float(q.tau)
        p.points[i].skip = float(q.skip)
    p.num_points = len(pts)
    return p


ScoreCollector = Callable[[int], ScorePopulation]


def calibrate(collect: ScoreCollector, lengths: Sequence[int], target_skip: float,
              gamma: float, excluded_layers: Sequence[int] = (0, 1)) -> ThresholdProfile:
    """calibrate (calibration.cpp:119-172): per distinct length (ascending) the
    collector's population is filtered to routable layers, the threshold that
    realises `target_skip` is solved, and tau is fitted as a cubic in
    x = L / max(lengths).  The collector is called once per distinct length."""
    lengths = [int(x) for x in lengths]
    if len(set(lengths)) < 4:
        raise ValueError("calibration needs at least 4 distinct lengths")
    pops = {}
    for L in sorted(set(lengths)):
        pops[L] = collect(L)
    uniq = sorted(pops)
    scores, layers, offsets = [], [], [0]
    for L in uniq:
        p = pops[L]
        scores.append(p.scores())
        layers.append(p.layers())
        offsets.append(offsets[-1] + p.size())
    s = np.ascontiguousarray(np.concatenate(scores) if scores else np.zeros(0), dtype=np.float64)
    ly = np.ascontiguousarray(np.concatenate(layers) if layers else np.zeros(0), dtype=np.uint64)
    off = np.ascontiguousarray(offsets, dtype=np.uint64)
    ln = np.ascontiguousarray(uniq, dtype=np.uint64)
    ex = np.ascontiguousarray(list(excluded_layers) or [0], dtype=np.uint64)
    out = _abi.ProfileC()
    check(lib().sinkr_calibrate(ln.ctypes.data, C.c_size_t(ln.size), s.ctypes.data, ly.ctypes.data,
                                off.ctypes.data, float(target_skip), float(gamma), ex.ctypes.data,
                                C.c_size_t(len(excluded_layers)), C.byref(out)))
    return _profile_from_c(out)


def save_profile(path: str, profile: ThresholdProfile) -> None:
    p = _profile_to_c(profile)
    check(lib().sinkr_save_profile(str(path).encode(), C.byref(p)))


def load_profile(path: str) -> ThresholdProfile:
    p = _abi.ProfileC()
    check(lib().sinkr_load_profile(str(path).encode(), C.byref(p)))
    return _profile_from_c(p)


def collect_scores(cache: KvCache, queries, layer: int, config: Optional[RoutingConfig] = None):
    """Score-collection mode on the GPU: the routing phase alone.  Returns
    (head_scores [B*H_q], group_scores [B*H_kv], sink [B*H_kv] bool)."""
    cfg = cache.config()
    B = cfg.num_seqs
    q = np.ascontiguousarray(queries, dtype=np.float32)
    if q.size != B * cfg.num_q_heads * cfg.head_dim:
        raise ValueError("queries span must be B x H_q x D for one layer")
    hs = np.zeros(B * cfg.num_q_heads, dtype=np.float64)
    gs = np.zeros(B * cfg.num_kv_heads, dtype=np.float64)
    sk = np.zeros(B * cfg.num_kv_heads, dtype=np.int32)
    keep = None
    cptr = None
    if config is not None:
        c, keep = config._c()
        cptr = C.byref(c)
    check(lib().sinkr_collect_scores(cache.handle, q.ctypes.data, C.c_size_t(layer), cptr,
                                     hs.ctypes.data, gs.ctypes.data, sk.ctypes.data))
    del keep
    return hs, gs, sk.astype(bool)


def collect_scores_batch(cache: KvCache, queries, layer: int, config: Optional[RoutingConfig] = None):
    """collect_scores for n query samples over the same cache layer in ONE
    launch (sinkr_collect_scores_batch): queries [n][B][H_q][D] ->
    (head_scores [n][B*H_q], group_scores [n][B*H_kv], sink [n][B*H_kv] bool),
    bit-identical to n collect_scores calls."""
    cfg = cache.config()
    B = cfg.num_seqs
    per = B * cfg.num_q_heads * cfg.head_dim
    q = np.ascontiguousarray(queries, dtype=np.float32)
    if q.size == 0 or q.size % per:
        raise ValueError("queries must be n x B x H_q x D for one layer")
    n = q.size // per
    hs = np.zeros((n, B * cfg.num_q_heads), dtype=np.float64)
    gs = np.zeros((n, B * cfg.num_kv_heads), dtype=np.float64)
    sk = np.zeros((n, B * cfg.num_kv_heads), dtype=np.int32)
    keep = None
    cptr = None
    if config is not None:
        c, keep = config._c()
        cptr = C.byref(c)
    check(lib().sinkr_collect_scores_batch(cache.handle, q.ctypes.data, C.c_size_t(n),
                                           C.c_size_t(layer), cptr, hs.ctypes.data,
                                           gs.ctypes.data, sk.ctypes.data))
    del keep
    return hs, gs, sk.astype(bool)


def gpu_score_collector(cache: KvCache, query_source: Callable[[int, int], np.ndarray],
                        layers: Sequence[int], samples: int) -> ScoreCollector:
    """A ScoreCollector over an engine whose cache is (re)filled per length by
    `query_source(length, sample)` -> queries [B][H_q][D]; every group score of
    every sample and layer joins the population (skipping disabled)."""
    def collect(length: int) -> ScorePopulation:
        # all samples of a length in one launch per layer; the population
        # keeps the reference's order (sample-major, then layer)
        pop = ScorePopulation()
        qs = np.stack([np.asarray(query_source(length, s), dtype=np.float32) for s in range(samples)])
        per_layer = [collect_scores_batch(cache, qs, layer)[1] for layer in layers]
        for s in range(samples):
            for li, layer in enumerate(layers):
                pop.extend(per_layer[li][s], layer, length)
        return pop
    return collect
