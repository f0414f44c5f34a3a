"""Synthetic planted-sink decode workload.

Every (seq, kv_head) slot gets a planted BOS sink: token 0's key has a large
norm (k0_scale) and its value is near zero (v0_scale).  A fraction p of the
groups of each sequence -- floor(p * H_kv), chosen by a seeded permutation --
get queries aligned with their anchor (cosine rho_sink), so they route Sink
under tau = 0.5; the other groups get queries orthogonal to the anchor
(cosine ~ 0) and route Active.

Rows 1.. of K and V are N(0,1)-like values from the counter-based generator
restated in oracle/sinkr_oracle.c:orc_fill_rows: the device generator
(`KvCache.append_synthetic`) and `host_rows` below produce bit-identical
bf16 values, so the CPU checker can see exactly the cache the GPU reads.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)
TAG_K, TAG_V, TAG_Q, TAG_ANCHOR, TAG_IMG_K, TAG_IMG_V = 1, 2, 3, 4, 5, 6


def _sm64_final(z):
    z = (z ^ (z >> np.uint64(30))) * M1
    z = (z ^ (z >> np.uint64(27))) * M2
    return z ^ (z >> np.uint64(31))


def sm64_draw(key, n):
    """n-th output of the reference SplitMix64 seeded with key (tensor.hpp:15-25)."""
    with np.errstate(over="ignore"):
        return _sm64_final(np.uint64(key) + (np.asarray(n, dtype=np.uint64) + np.uint64(1)) * GOLDEN)


def mix_seed(seed: int, tags) -> int:
    """tensor.cpp:53-61."""
    with np.errstate(over="ignore"):
        h = sm64_draw(np.uint64(seed), 0)
        for t in tags:
            h = sm64_draw(h ^ (np.uint64(t) + GOLDEN), 0)
    return int(h)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """f32 -> bf16 (RNE) -> f32, finite inputs."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    with np.errstate(over="ignore"):
        r = (b + np.uint32(0x7FFF) + ((b >> np.uint32(16)) & np.uint32(1))) & np.uint32(0xFFFF0000)
    return r.view(np.float32)


def gauss12(key: int, e: np.ndarray) -> np.ndarray:
    """Irwin-Hall(12) - 6 from 24-bit uniforms, exact integer arithmetic."""
    e = np.asarray(e, dtype=np.uint64)
    s = np.zeros(e.shape, dtype=np.uint64)
    with np.errstate(over="ignore"):
        for j in range(6):
            h = sm64_draw(key, e * np.uint64(6) + np.uint64(j))
            s += (h >> np.uint64(40)) + ((h >> np.uint64(16)) & np.uint64(0xFFFFFF))
    return (s.astype(np.float64) * 2.0 ** -24 - 6.0).astype(np.float32)


def host_rows(key: int, row0: int, rows: int, d: int, scale: float = 1.0) -> np.ndarray:
    e = (np.arange(row0, row0 + rows, dtype=np.uint64)[:, None] * np.uint64(d)
         + np.arange(d, dtype=np.uint64)[None, :])
    return round_bf16(np.float32(scale) * gauss12(key, e))


@dataclass
class WorkloadSpec:
    num_q_heads: int = 32
    num_kv_heads: int = 8
    head_dim: int = 128
    length: int = 32768
    num_seqs: int = 1
    sink_fraction: float = 0.0     # p: floor(p * H_kv) groups per sequence route Sink
    seed: int = 42
    layer: int = 0
    num_layers: int = 1
    k0_scale: float = 24.0
    v0_scale: float = 1e-3
    rho_sink: float = 0.8
    capacity: int = 0              # 0 -> length
    image_tokens: int = 0          # LLaVA-style image block: rows 1..image_tokens
    image_scale: float = 1.5       # ... drawn from a separate, wider stream

    @property
    def r(self) -> int:
        return self.num_q_heads // self.num_kv_heads

    def n_sink(self) -> int:
        return int(np.floor(self.sink_fraction * self.num_kv_heads + 1e-9))

    def slot_keys(self, seq: int, head: int, layer: int = None):
        layer = self.layer if layer is None else layer
        return (mix_seed(self.seed, (layer, seq, head, TAG_K)),
                mix_seed(self.seed, (layer, seq, head, TAG_V)))

    def sink_groups(self, seq: int) -> np.ndarray:
        rng = np.random.default_rng(mix_seed(self.seed, (self.layer, seq, 0, TAG_Q)) >> 1)
        perm = rng.permutation(self.num_kv_heads)
        mask = np.zeros(self.num_kv_heads, dtype=bool)
        mask[perm[: self.n_sink()]] = True
        return mask

    def first_rows(self, seq: int, head: int, layer: int = None):
        """Planted BOS row: (k0, v0) as f32 (bf16-representable) rows."""
        layer = self.layer if layer is None else layer
        rng = np.random.default_rng(mix_seed(self.seed, (layer, seq, head, TAG_ANCHOR)) >> 1)
        z = rng.standard_normal(self.head_dim)
        k0 = round_bf16((z / np.linalg.norm(z) * self.k0_scale).astype(np.float32))
        v0 = round_bf16((self.v0_scale * rng.standard_normal(self.head_dim)).astype(np.float32))
        return k0, v0

    def queries(self) -> np.ndarray:
        """f32 [B, H_q, D]."""
        D, r = self.head_dim, self.r
        out = np.zeros((self.num_seqs, self.num_q_heads, D), dtype=np.float32)
        for s in range(self.num_seqs):
            sinks = self.sink_groups(s)
            rng = np.random.default_rng(mix_seed(self.seed, (self.layer, s, 1, TAG_Q)) >> 1)
            for g in range(self.num_kv_heads):
                k0, _ = self.first_rows(s, g)
                kh = k0.astype(np.float64) / np.linalg.norm(k0.astype(np.float64))
                for i in range(r):
                    n = rng.standard_normal(D)
                    n -= (n @ kh) * kh
                    n /= np.linalg.norm(n)
                    rho = self.rho_sink if sinks[g] else 0.0
                    q = np.sqrt(D) * (rho * kh + np.sqrt(1.0 - rho * rho) * n)
                    out[s, g * r + i] = q.astype(np.float32)
        return out

    # -- materialisation --------------------------------------------------------
    def segments(self, seq: int, head: int):
        """Row segments after the planted row 0: (row0, rows, key_k, key_v, scale)."""
        kk, kv = self.slot_keys(seq, head)
        n_img = max(0, min(self.image_tokens, self.length - 1))
        out = []
        if n_img:
            out.append((1, n_img, mix_seed(self.seed, (self.layer, seq, head, TAG_IMG_K)),
                        mix_seed(self.seed, (self.layer, seq, head, TAG_IMG_V)),
                        self.image_scale))
        if self.length > 1 + n_img:
            out.append((1 + n_img, self.length - 1 - n_img, kk, kv, 1.0))
        return out

    def host_slot(self, seq: int, head: int):
        """f32 K, V [L, D] exactly as stored by the device cache."""
        k0, v0 = self.first_rows(seq, head)
        k = np.empty((self.length, self.head_dim), dtype=np.float32)
        v = np.empty_like(k)
        k[0], v[0] = k0, v0
        for row0, rows, key_k, key_v, scale in self.segments(seq, head):
            k[row0:row0 + rows] = host_rows(key_k, row0, rows, self.head_dim, scale)
            v[row0:row0 + rows] = host_rows(key_v, row0, rows, self.head_dim, scale)
        return k, v

    def host_cache(self, seq: int = 0):
        """(K [H_kv, L, D], V [H_kv, L, D]) for one sequence."""
        ks, vs = zip(*(self.host_slot(seq, g) for g in range(self.num_kv_heads)))
        return np.stack(ks), np.stack(vs)

    def fill(self, cache) -> None:
        """Fill an engine KvCache: planted row 0 from the host, rows 1.. on device."""
        for s in range(self.num_seqs):
            for g in range(self.num_kv_heads):
                k0, v0 = self.first_rows(s, g)
                cache.append(self.layer, g, k0, v0, seq=s)
                for row0, rows, key_k, key_v, scale in self.segments(s, g):
                    cache.append_synthetic(self.layer, g, key_k, key_v, rows, k_scale=scale,
                                           v_scale=scale, seq=s, global_row0=row0)
