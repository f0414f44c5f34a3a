"""GPU: the §8 "next" rows on the B200 engine, each against the compiled
reference.
  f1  score collection (routing phase alone) bit-exact with the reference's
      routed_decode_step scores; the calibration closed loop of SPEC.md
      acceptance 4 driven by GPU-collected populations.
  f2  snapshots: reference-written snapshots replay into the engine (rows,
      anchors and a routed step identical to the reference's on the same
      snapshot), engine-written snapshots load in the reference; device f32
      prefill equals host append.
  f4  full-attention BOS mass and attention_weights on the GPU vs the
      reference's attention_weights; the planted workload's proxy separates
      the oracle labels perfectly (AUPRC 1.0)."""
import numpy as np
import pytest

import oracle
import paper_2604_16883_b200 as P
from paper_2604_16883_b200 import analysis as A
from paper_2604_16883_b200 import calibration as cal
from paper_2604_16883_b200.workload import WorkloadSpec, round_bf16

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    if not __import__("os").path.exists(oracle.REF_SO):
        pytest.skip("reference library not built")
    return oracle.ref()


def _ref_cache_from(spec, k, v):
    rc = oracle.RefCache(oracle.ref(), 1, spec.num_q_heads, spec.num_kv_heads, spec.head_dim,
                         spec.length)
    for g in range(spec.num_kv_heads):
        rc.append_rows(0, g, k[g], v[g])
    return rc


# ---------------------------------------------------------------- f1
def test_collect_scores_bit_exact(ref):
    spec = WorkloadSpec(length=3000, sink_fraction=0.5, seed=5)
    q = spec.queries()[0]
    k, v = spec.host_cache(0)
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
    with P.KvCache(P.CacheConfig(1, 32, 8, 128, spec.length)) as cache:
        spec.fill(cache)
        hs, gs, sink = cal.collect_scores(cache, q, 0, cfg)
        _, gs0, sink0 = cal.collect_scores(cache, q, 0, None)
    rc = _ref_cache_from(spec, k, v)
    r = rc.routed_decode_step(q, 0, oracle.Profile.constant(0.5), excluded=())
    assert hs.tobytes() == r.head_scores.tobytes()
    assert gs.tobytes() == r.group_scores.tobytes() == gs0.tobytes()
    assert np.array_equal(sink, r.sink.astype(bool)) and sink.sum() == 4
    assert not sink0.any()


@pytest.mark.parametrize("hq,hkv", [(32, 8), (128, 8)])
def test_collect_scores_batch_vs_reference(ref, hq, hkv):
    """Batched score collection against the compiled reference's
    routed_decode_step scores directly, per sample (r = 4 and the WIDE r = 16)."""
    spec = WorkloadSpec(num_q_heads=hq, num_kv_heads=hkv, length=2000, sink_fraction=0.5, seed=15)
    k, v = spec.host_cache(0)
    rng = np.random.default_rng(hq)
    qs = np.stack([spec.queries()[0]] + [rng.standard_normal((hq, 128)).astype(np.float32) * 3
                                          for _ in range(4)])
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
    with P.KvCache(P.CacheConfig(1, hq, hkv, 128, spec.length)) as cache:
        spec.fill(cache)
        hb, gb, sb = cal.collect_scores_batch(cache, qs, 0, cfg)
    rc = oracle.RefCache(oracle.ref(), 1, hq, hkv, 128, spec.length)
    for g in range(hkv):
        rc.append_rows(0, g, k[g], v[g])
    for i, q in enumerate(qs):
        r = rc.routed_decode_step(q, 0, oracle.Profile.constant(0.5), excluded=())
        assert hb[i].tobytes() == r.head_scores.tobytes()
        assert gb[i].tobytes() == r.group_scores.tobytes()
        assert np.array_equal(sb[i], r.sink.astype(bool))
    rc.close()


@pytest.mark.parametrize("hq,hkv,D,B", [(32, 8, 128, 1), (40, 8, 64, 2), (8, 8, 32, 3), (64, 8, 128, 1),
                                         (35, 7, 128, 1), (128, 8, 128, 1), (24, 2, 64, 2)])
def test_collect_scores_batch_matches_single(hq, hkv, D, B):
    """sinkr_collect_scores_batch over n samples == n sinkr_collect_scores
    calls, byte for byte (head/group scores, sink flags), including a
    degenerate (zero) query head, sink_on_tie and an excluded layer; B = 1-3,
    r = 1, 4, 5, 8, 12, 16 and D = 32 / 64 / 128 (the single call is pinned to the
    reference by test_collect_scores_bit_exact)."""
    rng = np.random.default_rng(hq * 131 + D)
    L = 700
    n = 37
    with P.KvCache(P.CacheConfig(2, hq, hkv, D, L, B)) as cache:
        for layer in range(2):
            for s in range(B):
                for g in range(hkv):
                    k = rng.standard_normal((L, D)).astype(np.float32)
                    cache.append(layer, g, k, k * 0.5, seq=s)
        qs = rng.standard_normal((n, B, hq, D)).astype(np.float32)
        qs[3, 0, 1] = 0.0  # degenerate head: never sinks
        cfgs = [None,
                P.RoutingConfig(profile=P.ThresholdProfile.constant(0.02), excluded_layers=()),
                P.RoutingConfig(profile=P.ThresholdProfile.constant(0.0), excluded_layers=(),
                                sink_on_tie=True),
                P.RoutingConfig(profile=P.ThresholdProfile.constant(-0.5), excluded_layers=(1,))]
        for layer in range(2):
            for cfg in cfgs:
                hb, gb, sb = cal.collect_scores_batch(cache, qs, layer, cfg)
                for i in range(n):
                    h1, g1, s1 = cal.collect_scores(cache, qs[i], layer, cfg)
                    assert hb[i].tobytes() == h1.tobytes()
                    assert gb[i].tobytes() == g1.tobytes()
                    assert np.array_equal(sb[i], s1)


def _aligned_queries(rng, k0s, r, cosines, D):
    """queries whose cosine with their group's anchor is exactly `cosines`."""
    out = np.zeros((len(k0s) * r, D), dtype=np.float32)
    for g, k0 in enumerate(k0s):
        kh = k0.astype(np.float64) / np.linalg.norm(k0.astype(np.float64))
        for i in range(r):
            n = rng.standard_normal(D)
            n -= (n @ kh) * kh
            n /= np.linalg.norm(n)
            c = cosines[g * r + i]
            out[g * r + i] = (np.sqrt(D) * (c * kh + np.sqrt(1 - c * c) * n)).astype(np.float32)
    return out


def test_calibration_closed_loop():
    """SPEC.md acceptance 4: a length-dependent planted score shift; the
    fitted cubic profile realises 60 % +- 3 pp skip at every calibration length
    when the GPU routes with it."""
    lengths = [4096, 8192, 16384, 32768, 65536]
    D, Hq, Hkv = 128, 32, 8
    r = Hq // Hkv
    spec = WorkloadSpec(length=max(lengths), sink_fraction=0.0, seed=11)
    k0s = [spec.first_rows(0, g)[0] for g in range(Hkv)]
    rng = np.random.default_rng(0)
    samples = 100
    qs = {}
    for L in lengths:
        mu = 0.15 + 0.35 * L / lengths[-1]
        qs[L] = [_aligned_queries(rng, k0s, r, np.clip(rng.normal(mu, 0.15, Hq), -0.95, 0.95), D)
                 for _ in range(samples)]
    caches = {}
    for L in lengths:  # one engine per length: tau(L) reads token_count()
        c = P.KvCache(P.CacheConfig(1, Hq, Hkv, D, L))
        for g in range(Hkv):
            k0, v0 = spec.first_rows(0, g)
            c.append(0, g, k0, v0)
            kk, kv = spec.slot_keys(0, g)
            c.append_synthetic(0, g, kk, kv, L - 1, global_row0=1)
        caches[L] = c
    calls = []

    def collect(L):
        calls.append(L)
        pop = cal.ScorePopulation()
        _, gss, _ = cal.collect_scores_batch(caches[L], np.stack(qs[L]), 0)
        for gs in gss:
            pop.extend(gs, 0, L)
        return pop

    prof = cal.calibrate(collect, lengths, 0.6, 0.65, excluded_layers=())
    assert calls == lengths
    taus = [p.tau for p in prof.points]
    assert taus == sorted(taus)  # the planted shift moves the threshold up with L
    cfg = P.RoutingConfig.from_profile(prof)
    for L in lengths:
        sinks = [cal.collect_scores(caches[L], q, 0, cfg)[2] for q in qs[L]]
        realised = float(np.mean(sinks))
        assert abs(realised - 0.6) <= 0.03, (L, realised)
    for c in caches.values():
        c.close()


# ---------------------------------------------------------------- f2
def test_snapshot_interop(ref, tmp_path):
    spec = WorkloadSpec(length=1500, sink_fraction=0.375, seed=9)
    k, v = spec.host_cache(0)
    q = spec.queries()[0]
    rc = _ref_cache_from(spec, k, v)
    rdir = tmp_path / "ref_snap"
    rc.save_snapshot(rdir)
    cache = P.KvCache.load_snapshot(rdir)
    assert cache.config().capacity == spec.length and cache.token_count() == spec.length
    for g in range(spec.num_kv_heads):
        kk, vv = cache.historical(0, g, 0, spec.length)
        assert np.array_equal(kk, k[g]) and np.array_equal(vv, v[g])
        a, n = cache.anchor(0, g)
        ra, rn = rc.anchor(0, g)
        assert np.array_equal(a, ra) and n == rn
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
    res = P.routed_decode_step(q, 0, cache, cfg)
    rr = rc.routed_decode_step(q, 0, oracle.Profile.constant(0.5), excluded=())
    assert np.array_equal(res.route_bitmap, rr.sink.astype(bool))
    assert np.abs(res.outputs - rr.outputs).max() <= 2e-3
    # engine -> reference
    odir = tmp_path / "our_snap"
    cache.save_snapshot(odir)
    back = ref.load_snapshot(odir, 1, spec.num_q_heads, spec.num_kv_heads, spec.head_dim)
    assert back.token_count() == spec.length
    for g in range(spec.num_kv_heads):
        kk, vv = back.historical(0, g, 0, spec.length)
        assert np.array_equal(kk, k[g]) and np.array_equal(vv, v[g])
    for f in sorted(p.name for p in rdir.iterdir() if p.suffix == ".snkt"):
        assert (rdir / f).read_bytes() == (odir / f).read_bytes()
    # replay into sequence 1 of a batched engine
    with P.KvCache(P.CacheConfig(1, 32, 8, 128, spec.length, num_seqs=2)) as b2:
        b2.load_snapshot_into(odir, seq=1)
        assert b2.length(0, 3, seq=1) == spec.length and b2.length(0, 3, seq=0) == 0
        kk, _ = b2.historical(0, 3, 0, spec.length, seq=1)
        assert np.array_equal(kk, k[3])
    cache.close()


def test_snapshot_errors(tmp_path):
    with pytest.raises(RuntimeError, match="manifest"):
        P.KvCache.load_snapshot(tmp_path / "nowhere")
    spec = WorkloadSpec(length=64, seed=1)
    with P.KvCache(P.CacheConfig(1, 32, 8, 128, 64)) as c:
        spec.fill(c)
        c.save_snapshot(tmp_path / "s")
    (tmp_path / "s" / "v_l0_h2.snkt").write_bytes(b"SNKX")
    with pytest.raises(RuntimeError, match="bad magic"):
        P.KvCache.load_snapshot(tmp_path / "s")


def test_device_f32_prefill_matches_host_append():
    import torch

    rng = np.random.default_rng(4)
    L, D = 777, 128
    k = (rng.standard_normal((L, D)) * 2).astype(np.float32)
    v = rng.standard_normal((L, D)).astype(np.float32)
    with P.KvCache(P.CacheConfig(1, 4, 1, D, 1024)) as a, P.KvCache(P.CacheConfig(1, 4, 1, D, 1024)) as b:
        a.append(0, 0, k, v)
        dk, dv = torch.from_numpy(k).cuda(), torch.from_numpy(v).cuda()
        b.append_device_f32(0, 0, dk.data_ptr(), dv.data_ptr(), 500)
        b.append_device_f32(0, 0, dk[500:].data_ptr(), dv[500:].data_ptr(), L - 500)
        ka, va = a.historical(0, 0, 0, L)
        kb, vb = b.historical(0, 0, 0, L)
        assert np.array_equal(ka, kb) and np.array_equal(va, vb)
        assert np.array_equal(kb, round_bf16(k))
        assert a.anchor(0, 0)[1] == b.anchor(0, 0)[1]
        assert np.array_equal(a.anchor(0, 0)[0], b.anchor(0, 0)[0])


# ---------------------------------------------------------------- f4
@pytest.mark.parametrize("L,p,seed", [(1, 0.5, 1), (300, 0.5, 2), (5000, 0.25, 3), (40000, 0.625, 4)])
def test_bos_mass_and_weights_vs_reference(ref, L, p, seed):
    spec = WorkloadSpec(length=L, sink_fraction=p, seed=seed)
    q = spec.queries()[0]
    k, v = spec.host_cache(0)
    r = spec.r
    with P.KvCache(P.CacheConfig(1, 32, 8, 128, L)) as cache:
        spec.fill(cache)
        a0 = A.attention_bos_mass(cache, q, 0)[0]
        for g in (0, 5):
            w = A.attention_weights(cache, q[g * r:(g + 1) * r], 0, g)
            rw = ref.attention_weights(q[g * r:(g + 1) * r], k[g])
            assert w.shape == rw.shape
            assert np.abs(w - rw).max() <= 1e-6, np.abs(w - rw).max()
            assert np.abs(a0[g * r:(g + 1) * r] - rw[:, 0]).max() <= 1e-6
    for g in range(8):
        rw = ref.attention_weights(q[g * r:(g + 1) * r], k[g])
        assert np.abs(a0[g * r:(g + 1) * r] - rw[:, 0]).max() <= 1e-6


@pytest.mark.parametrize("B,hq,hkv,D", [(2, 32, 4, 128), (3, 8, 8, 64), (1, 16, 4, 32), (2, 64, 8, 128),
                                         (1, 128, 8, 128), (2, 24, 2, 64)])
def test_bos_mass_ragged_shapes(ref, B, hq, hkv, D):
    """BOS pass over ragged slots (units of different lengths share the flat
    token space and CTA ranges straddle units), r = 8, r = 1, the two-tile
    widths r = 16 / 12 and D = 64/32; alpha0 and weights against
    attention_weights (attention.cpp:75-99) per group, layer 1 of 2."""
    rng = np.random.default_rng(B * 1000 + hq + D)
    r = hq // hkv
    cap = 9000
    lens = rng.integers(1, cap, size=(B, hkv))
    lens[0, 0] = 1
    lens[-1, -1] = cap
    ks = {}
    with P.KvCache(P.CacheConfig(2, hq, hkv, D, cap, B)) as cache:
        for s in range(B):
            for g in range(hkv):
                k = (rng.standard_normal((lens[s, g], D)) * 1.5).astype(np.float32)
                k[0] *= 6.0
                k = round_bf16(k)  # the cache stores bf16: compare on representable rows
                v = round_bf16(rng.standard_normal((lens[s, g], D)).astype(np.float32))
                cache.append(1, g, k, v, seq=s)
                ks[s, g] = k
        q = (rng.standard_normal((B, hq, D)) * np.sqrt(D) * 0.3).astype(np.float32)
        a0 = A.attention_bos_mass(cache, q, 1)
        for s in range(B):
            for g in range(hkv):
                rw = ref.attention_weights(q[s, g * r:(g + 1) * r], ks[s, g])
                assert np.abs(a0[s, g * r:(g + 1) * r] - rw[:, 0]).max() <= 1e-6, (s, g)
        for s, g in [(0, 0), (B - 1, hkv - 1), (B // 2, hkv // 2)]:
            w = A.attention_weights(cache, q[s, g * r:(g + 1) * r], 1, g, seq=s)
            rw = ref.attention_weights(q[s, g * r:(g + 1) * r], ks[s, g])
            assert np.abs(w - rw).max() <= 1e-6, (s, g, np.abs(w - rw).max())


def test_attention_weights_after_length_change(ref):
    """attention_weights twice on one unit whose length changed in between,
    after a longer unit sized the scratch (no reallocation): the captured
    graph must follow the new token count (its weights offset moves with T)."""
    rng = np.random.default_rng(77)
    D, cap = 128, 12000
    with P.KvCache(P.CacheConfig(1, 32, 8, D, cap)) as cache:
        ks = {}
        for g, n in ((1, 11000), (0, 2000)):
            k = round_bf16((rng.standard_normal((n, D)) * 1.5).astype(np.float32))
            k[0] *= 6.0
            v = round_bf16(rng.standard_normal((n, D)).astype(np.float32))
            cache.append(0, g, k, v)
            ks[g] = k
        q = (rng.standard_normal((4, D)) * 3.0).astype(np.float32)
        A.attention_weights(cache, q, 0, 1)  # the scratch covers 11,000 tokens
        for extra in (0, 37, 1500, 16):
            if extra:
                k = round_bf16((rng.standard_normal((extra, D)) * 1.5).astype(np.float32))
                v = round_bf16(rng.standard_normal((extra, D)).astype(np.float32))
                cache.append(0, 0, k, v)
                ks[0] = np.concatenate([ks[0], k])
            w = A.attention_weights(cache, q, 0, 0)
            rw = ref.attention_weights(q, ks[0])
            assert w.shape == rw.shape
            assert np.abs(w - rw).max() <= 1e-6, (extra, np.abs(w - rw).max())


def test_route_eval_planted_workload():
    """SPEC.md analysis invariant: on the planted workload the proxy at tau 0.5
    gives precision = recall = 1 against oracle labels with gamma 0.65, and the
    group-score PR curve has AUPRC 1.0."""
    scores, labels = [], []
    for seed in range(4):
        spec = WorkloadSpec(length=20000, sink_fraction=[0.25, 0.5, 0.625, 0.875][seed], seed=seed)
        q = spec.queries()[0]
        with P.KvCache(P.CacheConfig(1, 32, 8, 128, spec.length)) as cache:
            spec.fill(cache)
            _, gs, _ = cal.collect_scores(cache, q, 0)
            a0 = A.attention_bos_mass(cache, q, 0)[0]
        labs = A.oracle_labels_from_alpha0(a0, 0.65, A.OracleMode.GroupMean, spec.r)
        assert [l.is_sink for l in labs] == spec.sink_groups(0).tolist()
        assert all(l.alpha0 > 0.99 for l in labs if l.is_sink)
        scores += gs.tolist()
        labels += [l.is_sink for l in labs]
    curve = A.pr_curve(scores, labels)
    assert curve.auprc == 1.0
    pred = np.array(scores) > 0.5
    lab = np.array(labels)
    assert (pred == lab).all()
