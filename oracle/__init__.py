"""TEST INFRASTRUCTURE ONLY — the checker, never the product.

ctypes bindings for
  * ``oracle/_ref/libsinkr_ref.so`` — the UNMODIFIED reference library compiled
    from ``/root/reference/proj/src`` (recipe: ``oracle/Makefile``), reached
    through ``oracle/ref_shim.cpp``;
  * ``oracle/_build/libsinkr_oracle.so`` — the plain-C restatement
    (``oracle/sinkr_oracle.c``), pinned bit-exactly against the former.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s reference /
cpu_baseline legs import this package.  The product package
(``paper_2604_16883_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libsinkr_ref.so")
ORC_SO = os.path.join(HERE, "_build", "libsinkr_oracle.so")

_ERR = {1: ValueError, 2: IndexError, 3: RuntimeError, 4: AssertionError}


def build(ref: bool = True) -> None:
    """Compile the restatement (and the reference when its sources exist)."""
    targets = ["oracle"]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


# ----------------------------------------------------------------------------
# Profiles (calibration.hpp:21-34)
@dataclass
class Profile:
    coeffs: tuple = (0.0, 0.0, 0.0, 0.0)
    normalizer: float = 1.0
    lo: float = 0.0
    hi: float = 1.0

    @staticmethod
    def constant(tau: float) -> "Profile":
        # calibration.cpp:29-35
        return Profile((0.0, 0.0, 0.0, float(tau)), 1.0, min(tau, 0.0), max(tau, 1.0))


@dataclass
class StepResult:
    outputs: np.ndarray
    group_scores: np.ndarray
    thresholds: np.ndarray
    sink: np.ndarray
    degenerate: np.ndarray
    group_kv_floats: np.ndarray
    head_scores: np.ndarray
    counters: dict = field(default_factory=dict)


class _Lib:
    prefix = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            build(ref=self.prefix == "ref_")
        self.lib = C.CDLL(path)
        self.path = path

    def _fn(self, name, restype=C.c_int):
        f = getattr(self.lib, self.prefix + name)
        f.restype = restype
        return f

    def _check(self, rc):
        if rc:
            msg = ""
            if self.prefix == "ref_":
                self.lib.ref_last_error.restype = C.c_char_p
                msg = self.lib.ref_last_error().decode()
            raise _ERR.get(rc, RuntimeError)(msg or f"oracle error {rc}")

    # -- scalar helpers --------------------------------------------------------
    def proxy_score(self, q, k0, k0_norm):
        q, k0 = _f32(q), _f32(k0)
        s, dg = C.c_double(), C.c_int()
        self._check(self._fn("proxy_score")(_p(q), _p(k0), C.c_float(k0_norm),
                                            C.c_size_t(q.size), C.byref(s), C.byref(dg)))
        return s.value, bool(dg.value)

    def group_score(self, scores, width):
        s = _f64(scores)
        out = C.c_double()
        self._check(self._fn("group_score")(_p(s), C.c_size_t(s.size), C.c_size_t(width),
                                            C.byref(out)))
        return out.value

    def threshold_for_length(self, length, prof: Profile):
        c = _f64(prof.coeffs)
        out = C.c_double()
        self._check(self._fn("threshold_for_length")(
            C.c_size_t(length), _p(c), C.c_double(prof.normalizer), C.c_double(prof.lo),
            C.c_double(prof.hi), C.byref(out)))
        return out.value

    def route(self, layer, score, length, prof: Profile, excluded=(0, 1), sink_on_tie=False):
        c = _f64(prof.coeffs)
        ex = np.ascontiguousarray(excluded, dtype=np.uint64)
        sink, tau = C.c_int(), C.c_double()
        self._check(self._fn("route")(
            C.c_size_t(layer), C.c_double(score), C.c_size_t(length), _p(c),
            C.c_double(prof.normalizer), C.c_double(prof.lo), C.c_double(prof.hi), _p(ex),
            C.c_size_t(ex.size), C.c_int(int(sink_on_tie)), C.byref(sink), C.byref(tau)))
        return bool(sink.value), tau.value

    def auto_num_splits(self, length):
        return int(self._fn("auto_num_splits", C.c_size_t)(C.c_size_t(length)))

    def split_ranges(self, length, n):
        out = np.zeros(2 * max(n, 1), dtype=np.uint64)
        self._check(self._fn("split_ranges")(C.c_size_t(length), C.c_size_t(n), _p(out)))
        return [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(n)]

    # -- attention -------------------------------------------------------------
    def attend_chunk(self, q, k, v, block=128):
        q, k, v = _f32(q), _f32(k), _f32(v)
        heads, dim = q.shape
        length = k.shape[0]
        m = np.zeros(heads)
        lsum = np.zeros(heads)
        acc = np.zeros((heads, dim))
        if self.prefix == "ref_":
            tok = C.c_size_t()
            rc = self._fn("attend_chunk")(_p(q), C.c_size_t(heads), C.c_size_t(dim), _p(k),
                                          _p(v), C.c_size_t(length), C.c_size_t(block),
                                          _p(m), _p(lsum), _p(acc), C.byref(tok))
        else:
            rc = self._fn("attend_chunk")(_p(q), C.c_size_t(heads), C.c_size_t(dim), _p(k),
                                          _p(v), C.c_size_t(length), C.c_size_t(block),
                                          _p(m), _p(lsum), _p(acc))
        self._check(rc)
        return m, lsum, acc

    def merge_partials(self, parts, heads, dim):
        """parts: list of (m[heads], l[heads], acc[heads,dim], tokens)."""
        n = len(parts)
        m = _f64([p[0] for p in parts]) if n else np.zeros(0)
        lsum = _f64([p[1] for p in parts]) if n else np.zeros(0)
        acc = _f64([p[2] for p in parts]) if n else np.zeros(0)
        tok = np.ascontiguousarray([p[3] for p in parts], dtype=np.uint64)
        out = np.zeros((heads, dim), dtype=np.float32)
        self._check(self._fn("merge_partials")(C.c_size_t(n), _p(m), _p(lsum), _p(acc), _p(tok),
                                               C.c_size_t(heads), C.c_size_t(dim), _p(out)))
        return out

    def dense_attention(self, q, k, v):
        q, k, v = _f32(q), _f32(k), _f32(v)
        heads, dim = q.shape
        out = np.zeros((heads, dim), dtype=np.float32)
        self._check(self._fn("dense_attention")(_p(q), C.c_size_t(heads), C.c_size_t(dim),
                                                _p(k), _p(v), C.c_size_t(k.shape[0]), _p(out)))
        return out


class RefLib(_Lib):
    """The compiled reference (oracle/_ref)."""

    prefix = "ref_"

    def __init__(self):
        super().__init__(REF_SO)
        self.lib.ref_pool_create.restype = C.c_void_p
        self.lib.ref_pool_destroy.argtypes = [C.c_void_p]
        self.lib.ref_cache_destroy.argtypes = [C.c_void_p]

    def online_attention(self, q, k, v, block=128):
        q, k, v = _f32(q), _f32(k), _f32(v)
        heads, dim = q.shape
        out = np.zeros((heads, dim), dtype=np.float32)
        self._check(self.lib.ref_online_attention(_p(q), C.c_size_t(heads), C.c_size_t(dim),
                                                  _p(k), _p(v), C.c_size_t(k.shape[0]),
                                                  C.c_size_t(block), _p(out)))
        return out

    def splitk_attention(self, q, k, v, splits, workers=1, block=128):
        q, k, v = _f32(q), _f32(k), _f32(v)
        heads, dim = q.shape
        out = np.zeros((heads, dim), dtype=np.float32)
        kvf = C.c_uint64()
        pool = self.lib.ref_pool_create(C.c_uint(workers)) if workers > 1 else None
        try:
            self._check(self.lib.ref_splitk_attention(
                _p(q), C.c_size_t(heads), C.c_size_t(dim), _p(k), _p(v),
                C.c_size_t(k.shape[0]), C.c_size_t(splits), C.c_void_p(pool),
                C.c_size_t(block), _p(out), C.byref(kvf)))
        finally:
            if pool:
                self.lib.ref_pool_destroy(C.c_void_p(pool))
        return out, int(kvf.value)

    def attention_weights(self, q, k):
        q, k = _f32(q), _f32(k)
        heads, dim = q.shape
        out = np.zeros((heads, k.shape[0]), dtype=np.float32)
        self._check(self.lib.ref_attention_weights(_p(q), C.c_size_t(heads), C.c_size_t(dim),
                                                   _p(k), C.c_size_t(k.shape[0]), _p(out)))
        return out

    # -- calibration (calibration.hpp:36-90) -----------------------------------
    def sweep(self, scores, thresholds):
        s, t = _f64(scores), _f64(thresholds)
        out = np.zeros(t.size)
        self._check(self.lib.ref_sweep(_p(s), C.c_size_t(s.size), _p(t), C.c_size_t(t.size), _p(out)))
        return out

    def skip_ratio_at(self, scores, thr):
        s = _f64(scores)
        out = C.c_double()
        self._check(self.lib.ref_skip_ratio_at(_p(s), C.c_size_t(s.size), C.c_double(thr), C.byref(out)))
        return out.value

    def solve_threshold(self, scores, target):
        s = _f64(scores)
        out = C.c_double()
        self._check(self.lib.ref_solve_threshold(_p(s), C.c_size_t(s.size), C.c_double(target),
                                                 C.byref(out)))
        return out.value

    def fit_cubic(self, x, y):
        x, y = _f64(x), _f64(y)
        co = np.zeros(4)
        res = C.c_double()
        self._check(self.lib.ref_fit_cubic(_p(x), _p(y), C.c_size_t(x.size), _p(co), C.byref(res)))
        return co, res.value

    @staticmethod
    def _profile_dict(f8, ex, nex, pts, npts):
        return {"coeffs": f8[:4].copy(), "normalizer": f8[4], "lo": f8[5], "hi": f8[6],
                "target_skip": f8[7], "gamma": f8[8], "excluded": [int(x) for x in ex[:nex]],
                "points": [(int(pts[3 * i]), pts[3 * i + 1], pts[3 * i + 2]) for i in range(npts)]}

    def calibrate(self, lengths, populations, target, gamma, excluded=(0, 1)):
        """populations[i] = (scores, layers) for lengths[i]."""
        ln = np.ascontiguousarray(lengths, dtype=np.uint64)
        sc = _f64(np.concatenate([np.asarray(p[0], dtype=np.float64) for p in populations]))
        ly = np.ascontiguousarray(np.concatenate([np.asarray(p[1]) for p in populations]),
                                  dtype=np.uint64)
        off = np.ascontiguousarray(np.cumsum([0] + [len(p[0]) for p in populations]), dtype=np.uint64)
        ex = np.ascontiguousarray(list(excluded) or [0], dtype=np.uint64)
        f8 = np.zeros(9)
        exo = np.zeros(64, dtype=np.uint64)
        pts = np.zeros(3 * 256)
        nex, npts, calls = C.c_size_t(), C.c_size_t(), C.c_size_t()
        self._check(self.lib.ref_calibrate(_p(ln), C.c_size_t(ln.size), _p(sc), _p(ly), _p(off),
                                           C.c_double(target), C.c_double(gamma), _p(ex),
                                           C.c_size_t(len(excluded)), _p(f8), _p(exo), C.byref(nex),
                                           _p(pts), C.byref(npts), C.byref(calls)))
        d = self._profile_dict(f8, exo, nex.value, pts, npts.value)
        d["collector_calls"] = calls.value
        return d

    def save_profile(self, path, d):
        f8 = np.array(list(d["coeffs"]) + [d["normalizer"], d["lo"], d["hi"], d["target_skip"],
                                           d["gamma"]], dtype=np.float64)
        ex = np.ascontiguousarray(d["excluded"] or [0], dtype=np.uint64)
        pts = _f64([x for p in d["points"] for x in p] or [0.0])
        self._check(self.lib.ref_save_profile(str(path).encode(), _p(f8), _p(ex),
                                              C.c_size_t(len(d["excluded"])), _p(pts),
                                              C.c_size_t(len(d["points"]))))

    def load_profile(self, path):
        f8 = np.zeros(9)
        exo = np.zeros(64, dtype=np.uint64)
        pts = np.zeros(3 * 256)
        nex, npts = C.c_size_t(), C.c_size_t()
        self._check(self.lib.ref_load_profile(str(path).encode(), _p(f8), _p(exo), C.byref(nex),
                                              _p(pts), C.byref(npts)))
        return self._profile_dict(f8, exo, nex.value, pts, npts.value)

    # -- SNKT (tensor.hpp:86-96) ----------------------------------------------------
    def write_tensor(self, path, arr):
        a = _f32(arr)
        dims = np.ascontiguousarray(a.shape, dtype=np.uint64)
        self._check(self.lib.ref_write_tensor(str(path).encode(), _p(dims), C.c_size_t(dims.size),
                                              _p(a)))

    def read_tensor(self, path):
        dims = np.zeros(64, dtype=np.uint64)
        nd = C.c_size_t()
        self._check(self.lib.ref_read_tensor(str(path).encode(), _p(dims), C.byref(nd), None,
                                             C.c_size_t(0)))
        shape = tuple(int(x) for x in dims[:nd.value])
        out = np.zeros(shape, dtype=np.float32)
        self._check(self.lib.ref_read_tensor(str(path).encode(), _p(dims), C.byref(nd), _p(out),
                                             C.c_size_t(out.size)))
        return out

    def snkt_file_size(self, dims):
        d = np.ascontiguousarray(dims, dtype=np.uint64)
        self.lib.ref_snkt_file_size.restype = C.c_uint64
        return int(self.lib.ref_snkt_file_size(_p(d), C.c_size_t(d.size)))

    def load_snapshot(self, path, layers, hq, hkv, dim):
        h = C.c_void_p()
        self._check(self.lib.ref_cache_load_snapshot(str(path).encode(), C.byref(h)))
        c = RefCache.__new__(RefCache)
        c.ref, c.hq, c.hkv, c.dim, c.h = self, hq, hkv, dim, h
        return c


class RefCache:
    """sinkr::KvCache (kv_cache.hpp:42-80) owned by the compiled reference."""

    def __init__(self, ref: RefLib, layers, hq, hkv, dim, capacity):
        self.ref, self.hq, self.hkv, self.dim = ref, hq, hkv, dim
        h = C.c_void_p()
        ref._check(ref.lib.ref_cache_create(C.c_size_t(layers), C.c_size_t(hq),
                                            C.c_size_t(hkv), C.c_size_t(dim),
                                            C.c_size_t(capacity), C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            self.ref.lib.ref_cache_destroy(self.h)
            self.h = None

    __del__ = close

    def append_rows(self, layer, head, k, v):
        k, v = _f32(k), _f32(v)
        self.ref._check(self.ref.lib.ref_cache_append_rows(
            self.h, C.c_size_t(layer), C.c_size_t(head), _p(k), _p(v),
            C.c_size_t(k.shape[0])))

    def save_snapshot(self, path):
        self.ref._check(self.ref.lib.ref_cache_save_snapshot(self.h, str(path).encode()))

    def token_count(self):
        n = C.c_size_t()
        self.ref._check(self.ref.lib.ref_cache_token_count(self.h, C.byref(n)))
        return n.value

    def historical(self, layer, head, frm, to):
        k = np.zeros((to - frm, self.dim), dtype=np.float32)
        v = np.zeros((to - frm, self.dim), dtype=np.float32)
        self.ref._check(self.ref.lib.ref_cache_historical(self.h, C.c_size_t(layer), C.c_size_t(head),
                                                          C.c_size_t(frm), C.c_size_t(to), _p(k), _p(v)))
        return k, v

    def anchor(self, layer, head):
        k0 = np.zeros(self.dim, dtype=np.float32)
        n = C.c_float()
        self.ref._check(self.ref.lib.ref_cache_anchor(self.h, C.c_size_t(layer),
                                                      C.c_size_t(head), _p(k0), C.byref(n)))
        return k0, n.value

    def routed_decode_step(self, queries, layer, prof: Profile, excluded=(0, 1),
                           sink_on_tie=False, num_splits=0, block=128, workers=1,
                           observe_only=False) -> StepResult:
        q = _f32(queries).reshape(-1)
        hkv, r, d = self.hkv, self.hq // self.hkv, self.dim
        res = _alloc_result(self.hq, hkv, d)
        c = _f64(prof.coeffs)
        ex = np.ascontiguousarray(excluded, dtype=np.uint64)
        cnt = np.zeros(4, dtype=np.uint64)
        secs = np.zeros(3)
        pool = self.ref.lib.ref_pool_create(C.c_uint(workers)) if workers > 1 else None
        try:
            self.ref._check(self.ref.lib.ref_routed_decode_step(
                self.h, _p(q), C.c_size_t(layer), _p(c), C.c_double(prof.normalizer),
                C.c_double(prof.lo), C.c_double(prof.hi), _p(ex), C.c_size_t(ex.size),
                C.c_int(int(sink_on_tie)), C.c_size_t(num_splits), C.c_size_t(block),
                C.c_void_p(pool), C.c_int(int(observe_only)), _p(res.outputs),
                _p(res.group_scores), _p(res.thresholds), _p(res.sink), _p(res.degenerate),
                _p(res.group_kv_floats), _p(res.head_scores), _p(cnt), _p(secs)))
        finally:
            if pool:
                self.ref.lib.ref_pool_destroy(C.c_void_p(pool))
        res.counters = _counters(cnt, secs)
        res.outputs = res.outputs.reshape(self.hq, d)
        return res


def _alloc_result(hq, hkv, d):
    return StepResult(
        outputs=np.zeros(hq * d, dtype=np.float32),
        group_scores=np.zeros(hkv),
        thresholds=np.zeros(hkv),
        sink=np.zeros(hkv, dtype=np.int32),
        degenerate=np.zeros(hkv, dtype=np.int32),
        group_kv_floats=np.zeros(hkv, dtype=np.uint64),
        head_scores=np.zeros(hq),
    )


def _counters(cnt, secs=None):
    out = dict(kv_floats_loaded=int(cnt[0]), anchor_floats_loaded=int(cnt[1]),
               groups_active=int(cnt[2]), groups_skipped=int(cnt[3]))
    if secs is not None:
        out.update(routing_seconds=float(secs[0]), attention_seconds=float(secs[1]),
                   merge_seconds=float(secs[2]))
    return out


class OracleLib(_Lib):
    """The plain-C restatement (oracle/_build)."""

    prefix = "orc_"

    def __init__(self):
        super().__init__(ORC_SO)
        self.lib.orc_mix_seed.restype = C.c_uint64
        self.lib.orc_gauss12.restype = C.c_float
        self.lib.orc_round_bf16.restype = C.c_float
        self.lib.orc_round_bf16.argtypes = [C.c_float]

    def anchor_norm(self, k):
        k = _f32(k)
        n = C.c_float()
        self._check(self.lib.orc_anchor_norm(_p(k), C.c_size_t(k.size), C.byref(n)))
        return n.value

    def routed_decode_step(self, k, v, k0, k0_norm, queries, layer, prof: Profile,
                           excluded=(0, 1), sink_on_tie=False, num_splits=0, block=128,
                           observe_only=False, threads=1) -> StepResult:
        """k, v: [H_kv, L, D] f32; k0: [H_kv, D]; k0_norm: [H_kv]; queries [H_q, D]."""
        k, v, k0 = _f32(k), _f32(v), _f32(k0)
        kn = _f32(k0_norm)
        q = _f32(queries)
        hkv, length, d = k.shape
        hq = q.shape[0]
        res = _alloc_result(hq, hkv, d)
        c = _f64(prof.coeffs)
        ex = np.ascontiguousarray(excluded, dtype=np.uint64)
        cnt = np.zeros(4, dtype=np.uint64)
        self._check(self.lib.orc_routed_decode_step(
            _p(k), _p(v), _p(k0), _p(kn), C.c_size_t(hq), C.c_size_t(hkv), C.c_size_t(d),
            C.c_size_t(length), C.c_size_t(layer), _p(q), _p(c), C.c_double(prof.normalizer),
            C.c_double(prof.lo), C.c_double(prof.hi), _p(ex), C.c_size_t(ex.size),
            C.c_int(int(sink_on_tie)), C.c_size_t(num_splits), C.c_size_t(block),
            C.c_int(int(observe_only)), C.c_int(threads), _p(res.outputs),
            _p(res.group_scores), _p(res.thresholds), _p(res.sink), _p(res.degenerate),
            _p(res.group_kv_floats), _p(res.head_scores), _p(cnt)))
        res.counters = _counters(cnt)
        res.outputs = res.outputs.reshape(hq, d)
        return res

    def mix_seed(self, seed, tags):
        t = np.ascontiguousarray(tags, dtype=np.uint64)
        return int(self.lib.orc_mix_seed(C.c_uint64(seed), _p(t), C.c_size_t(t.size)))

    def fill_rows(self, key, row0, rows, d, scale=1.0):
        out = np.zeros((rows, d), dtype=np.float32)
        self.lib.orc_fill_rows(C.c_uint64(key), C.c_size_t(row0), C.c_size_t(rows),
                               C.c_size_t(d), C.c_float(scale), _p(out))
        return out

    def round_bf16(self, x):
        return float(self.lib.orc_round_bf16(C.c_float(x)))


_REF = None
_ORC = None


def ref() -> RefLib:
    global _REF
    if _REF is None:
        _REF = RefLib()
    return _REF


def orc() -> OracleLib:
    global _ORC
    if _ORC is None:
        _ORC = OracleLib()
    return _ORC
