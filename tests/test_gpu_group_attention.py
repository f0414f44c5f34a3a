"""splitk_attention of one cached group on the GPU (sinkr_group_attention)
against the compiled reference's splitk_attention (attention.cpp:204-235):
outputs within the hot path's tolerance, the reference's kv-float count, its
argument errors, and a routed step after it routing as before (the forced
route must not leak into the next step's parameters)."""
import os

import numpy as np
import pytest

import oracle
import paper_2604_16883_b200 as P
from paper_2604_16883_b200.workload import WorkloadSpec, round_bf16

pytestmark = pytest.mark.gpu

MAX_ABS, REL_L2 = 2e-3, 1e-3  # SURVEY.md §8c output tolerance


@pytest.fixture(scope="module")
def ref():
    if not os.path.exists(oracle.REF_SO):
        pytest.skip("oracle/_ref not built")
    return oracle.ref()


def _close(a, b):
    err = np.abs(a - b).max()
    rel = np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)
    return err <= MAX_ABS and rel <= REL_L2, (err, rel)


@pytest.mark.parametrize("B,hq,hkv,D", [(1, 32, 8, 128), (2, 32, 4, 128), (3, 8, 8, 64), (1, 16, 4, 32)])
def test_group_attention_vs_reference(ref, B, hq, hkv, D):
    rng = np.random.default_rng(hq * 10 + B + D)
    r, cap = hq // hkv, 6000
    lens = rng.integers(1, cap, size=B)  # one length per sequence (the reference's cache is not ragged)
    lens[0] = 1
    kv = {}
    with P.KvCache(P.CacheConfig(2, hq, hkv, D, cap, B)) as cache:
        for s in range(B):
            for g in range(hkv):
                k = round_bf16(rng.standard_normal((lens[s], D)).astype(np.float32) * 2.0)
                v = round_bf16(rng.standard_normal((lens[s], D)).astype(np.float32))
                cache.append(1, g, k, v, seq=s)
                kv[s, g] = (k, v)
        for s in range(B):
            for g in sorted({0, hkv - 1, hkv // 2}):
                q = (rng.standard_normal((r, D)) * 1.5).astype(np.float32)
                k, v = kv[s, g]
                splits = int(rng.integers(1, min(16, lens[s]) + 1))
                res = P.splitk_attention(cache, q, 1, g, splits, seq=s)
                want, kvf = ref.splitk_attention(q, k, v, splits)
                ok, err = _close(res.out, want)
                assert ok, (s, g, err)
                assert res.counters.kv_floats_loaded == kvf == 2 * lens[s] * D


def test_group_attention_errors_and_next_step(ref):
    spec = WorkloadSpec(length=3000, sink_fraction=0.5, seed=7)
    q = spec.queries()[0]
    r = spec.r
    with P.KvCache(P.CacheConfig(1, 32, 8, 128, 4000)) as cache:
        spec.fill(cache)
        cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
        before = P.routed_decode_step(q, 0, cache, cfg)
        k, v = spec.host_cache(0)
        res = P.splitk_attention(cache, q[2 * r:3 * r], 0, 2, 4)
        want, _ = ref.splitk_attention(q[2 * r:3 * r], k[2], v[2], 4)
        assert _close(res.out, want)[0]
        # the reference's split_ranges message (attention.cpp:187-190)
        for bad in (0, 3001):
            with pytest.raises(ValueError, match=r"num_splits must be in \[1, len\], got %d for len 3000" % bad):
                P.splitk_attention(cache, q[:r], 0, 0, bad)
        with pytest.raises(IndexError):
            P.splitk_attention(cache, q[:r], 0, 8, 1)
        with pytest.raises(ValueError):
            P.splitk_attention(cache, q[:r + 1], 0, 0, 1)
        # a routed step afterwards routes again (same result as before; the
        # Split-K merge order may differ, so the outputs agree to rounding)
        after = P.routed_decode_step(q, 0, cache, cfg)
        assert np.abs(after.outputs - before.outputs).max() <= 1e-6
        assert [g.decision.sink for g in after.groups] == [g.decision.sink for g in before.groups]
        assert after.counters.kv_floats_loaded == before.counters.kv_floats_loaded


@pytest.mark.parametrize("B", [2, 8])  # 16 units (lean routing) / 64 units (distributed)
def test_group_attention_other_slots_empty(ref, B):
    """Only (seq 1, layer 0, head 3) holds rows: the rest of the cache is empty."""
    rng = np.random.default_rng(5)
    with P.KvCache(P.CacheConfig(1, 32, 8, 128, 2048, B)) as cache:
        k = round_bf16(rng.standard_normal((777, 128)).astype(np.float32))
        v = round_bf16(rng.standard_normal((777, 128)).astype(np.float32))
        cache.append(0, 3, k, v, seq=1)
        q = rng.standard_normal((4, 128)).astype(np.float32)
        res = P.splitk_attention(cache, q, 0, 3, 2, seq=1)
        want, _ = ref.splitk_attention(q, k, v, 2)
        assert _close(res.out, want)[0]
        with pytest.raises(ValueError, match="at least one token"):
            P.splitk_attention(cache, q, 0, 2, 1, seq=1)


def test_dense_and_online_attention_vs_reference(ref):
    rng = np.random.default_rng(11)
    with P.KvCache(P.CacheConfig(1, 32, 8, 128, 5000)) as cache:
        ks = {}
        for g in range(8):
            k = round_bf16(rng.standard_normal((4321, 128)).astype(np.float32) * 2.0)
            v = round_bf16(rng.standard_normal((4321, 128)).astype(np.float32))
            cache.append(0, g, k, v)
            ks[g] = (k, v)
        q = (rng.standard_normal((4, 128)) * 1.5).astype(np.float32)
        k, v = ks[5]
        assert _close(P.dense_attention(cache, q, 0, 5), ref.dense_attention(q, k, v))[0]
        assert _close(P.online_attention(cache, q, 0, 5, 96), ref.online_attention(q, k, v, 96))[0]
        with pytest.raises(ValueError, match="block_size must be positive"):
            P.online_attention(cache, q, 0, 5, 0)
