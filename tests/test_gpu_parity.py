"""Parity of the sm_100a engine (through the C-ABI) with the CPU oracle.

Bar (north star): route bitmaps, group/head scores and per-group loaded-token
counts bit-exact; outputs within max-abs 2e-3 and rel-L2 1e-3 of the
reference; Sink rows bitwise zero.  The oracle is the C restatement, itself
pinned bit-exactly to the compiled reference in tests/test_oracle.py; a few
cases also run the compiled reference (oracle/_ref) directly.
"""
import os

import numpy as np
import pytest

import paper_2604_16883_b200 as P
from paper_2604_16883_b200.workload import WorkloadSpec

pytestmark = pytest.mark.gpu

MAX_ABS = 2e-3
REL_L2 = 1e-3


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / den if den > 0 else np.linalg.norm(a - b)


def oracle_profile(prof):
    import oracle

    return oracle.Profile(tuple(prof.coeffs), prof.length_normalizer, prof.clamp_lo,
                          prof.clamp_hi)


def make_cache(spec: WorkloadSpec):
    cc = P.CacheConfig(spec.num_layers, spec.num_q_heads, spec.num_kv_heads, spec.head_dim,
                       spec.capacity or spec.length, spec.num_seqs)
    cache = P.KvCache(cc)
    spec.fill(cache)
    return cache


def oracle_step(orc, spec, seq, q, cfg: P.RoutingConfig, opts: P.EngineOptions, kv=None,
                length=None):
    k, v = kv if kv is not None else spec.host_cache(seq)
    k0 = k[:, 0, :].copy()
    k0n = np.array([orc.anchor_norm(k0[g]) for g in range(k.shape[0])], dtype=np.float32)
    return orc.routed_decode_step(
        k, v, k0, k0n, q, spec.layer, oracle_profile(cfg.profile),
        excluded=tuple(cfg.excluded_layers), sink_on_tie=cfg.sink_on_tie,
        num_splits=opts.num_splits, block=opts.block_size, observe_only=opts.observe_only,
        threads=8)


def assert_parity(res, ref, r, D, seq_groups):
    # routing: bit-exact
    sink = np.array([g.decision.sink for g in seq_groups], dtype=np.int32)
    np.testing.assert_array_equal(sink, ref.sink)
    np.testing.assert_array_equal([g.decision.degenerate for g in seq_groups], ref.degenerate)
    gs = np.array([g.decision.group_score for g in seq_groups])
    assert gs.tobytes() == ref.group_scores.tobytes(), (gs, ref.group_scores)
    th = np.array([g.decision.threshold for g in seq_groups])
    assert th.tobytes() == ref.thresholds.tobytes()
    hs = np.concatenate([g.decision.head_scores for g in seq_groups])
    assert hs.tobytes() == ref.head_scores.tobytes()
    # skipped-block record: per-group loaded floats exact
    np.testing.assert_array_equal([g.kv_floats_loaded for g in seq_groups], ref.group_kv_floats)
    # outputs
    out = np.asarray(res, np.float32)
    for gi, g in enumerate(seq_groups):
        rows = slice(gi * r, (gi + 1) * r)
        if ref.sink[gi] and not ref.group_kv_floats[gi]:
            assert not np.any(out[rows].view(np.uint32)), "Sink rows must be bitwise +0"
    err = np.abs(out - ref.outputs).max()
    assert err <= MAX_ABS, err
    assert rel_l2(out, ref.outputs) <= REL_L2


CASES = [
    # (hq, hkv, D, L, p)
    (32, 8, 128, 1, 0.0),
    (32, 8, 128, 7, 0.0),
    (32, 8, 128, 64, 0.5),
    (32, 8, 128, 1000, 0.5),
    (32, 8, 128, 4096, 0.625),
    (32, 4, 128, 3000, 0.5),     # r = 8 (Yi / 70B width)
    (40, 40, 128, 2048, 0.5),    # r = 1 (MHA, LLaVA)
    (8, 8, 64, 1500, 0.25),      # D = 64
    (16, 4, 32, 777, 0.5),       # D = 32
    (12, 4, 128, 333, 0.5),      # r = 3 (padded MMA rows)
    # wide GQA (the step kernel's WIDE form: two 8-head tiles per group)
    (128, 8, 128, 4096, 0.625),  # r = 16 (Llama-3.1-405B attention shape)
    (16, 1, 64, 3000, 0.0),      # r = 16, one KV head, D = 64
    (96, 8, 128, 2000, 0.5),     # r = 12 (second tile half full)
    (20, 2, 32, 500, 0.5),       # r = 10, D = 32
]


@pytest.mark.parametrize("hq,hkv,D,L,p", CASES)
def test_planted_parity(oracle_libs, hq, hkv, D, L, p):
    _, orc = oracle_libs
    spec = WorkloadSpec(num_q_heads=hq, num_kv_heads=hkv, head_dim=D, length=L, sink_fraction=p,
                        seed=L + hq)
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
    opts = P.EngineOptions()
    q = spec.queries()[0]
    with make_cache(spec) as cache:
        res = P.routed_decode_step(q, spec.layer, cache, cfg, opts)
        ref = oracle_step(orc, spec, 0, q, cfg, opts)
        assert_parity(res.outputs, ref, spec.r, D, res.groups)
        assert res.counters.kv_floats_loaded == ref.counters["kv_floats_loaded"]
        assert res.counters.groups_active == ref.counters["groups_active"]
        assert res.counters.groups_skipped == ref.counters["groups_skipped"]
        assert res.counters.anchor_floats_loaded == ref.counters["anchor_floats_loaded"]


def test_device_generator_matches_host(oracle_libs):
    spec = WorkloadSpec(num_q_heads=8, num_kv_heads=2, head_dim=128, length=300, seed=7)
    with make_cache(spec) as cache:
        for g in range(2):
            k, v = cache.historical(spec.layer, g, 0, spec.length)
            hk, hv = spec.host_slot(0, g)
            assert k.tobytes() == hk.tobytes() and v.tobytes() == hv.tobytes()
            k0, n = cache.anchor(spec.layer, g)
            assert k0.tobytes() == hk[0].tobytes()
            assert n == np.float32(oracle_libs[1].anchor_norm(hk[0]))


def test_random_dense_vs_reference(oracle_libs):
    """Diffuse random caches (no planted sink), tau > 1: compare with the
    compiled reference's routed_decode_step directly."""
    import oracle

    ref_lib, _ = oracle_libs
    if ref_lib is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(3)
    hq, hkv, D, L = 32, 8, 128, 2500
    k = rng.standard_normal((hkv, L, D)).astype(np.float32)
    v = rng.standard_normal((hkv, L, D)).astype(np.float32)
    from paper_2604_16883_b200.workload import round_bf16

    k, v = round_bf16(k).reshape(k.shape), round_bf16(v).reshape(v.shape)
    q = rng.standard_normal((hq, D)).astype(np.float32) * 3
    rc = oracle.RefCache(ref_lib, 1, hq, hkv, D, L)
    with P.KvCache(P.CacheConfig(1, hq, hkv, D, L)) as cache:
        for g in range(hkv):
            cache.append(0, g, k[g], v[g])
            rc.append_rows(0, g, k[g], v[g])
        cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(2.0))
        res = P.routed_decode_step(q, 0, cache, cfg)
        ref = rc.routed_decode_step(q, 0, oracle.Profile.constant(2.0), workers=8)
        assert_parity(res.outputs, ref, hq // hkv, D, res.groups)


@pytest.mark.parametrize("tau,expect_all_sink", [(2.0, False), (-2.0, True)])
def test_routing_limits(oracle_libs, tau, expect_all_sink):
    """tau > 1 -> all Active; tau < -1 -> all Sink, zeros,
    kv_floats == 0."""
    spec = WorkloadSpec(num_q_heads=32, num_kv_heads=8, head_dim=128, length=513,
                        sink_fraction=0.5)
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(tau), excluded_layers=())
    with make_cache(spec) as cache:
        res = P.routed_decode_step(spec.queries()[0], 0, cache, cfg)
        sinks = res.route_bitmap
        assert sinks.all() == expect_all_sink and sinks.any() == expect_all_sink
        if expect_all_sink:
            assert not np.any(res.outputs.view(np.uint32))
            assert res.counters.kv_floats_loaded == 0
            assert res.counters.groups_skipped == 8
        else:
            assert res.counters.kv_floats_loaded == 8 * 2 * 513 * 128


def test_excluded_layers_and_observe_only(oracle_libs):
    _, orc = oracle_libs
    spec = WorkloadSpec(num_q_heads=32, num_kv_heads=8, head_dim=128, length=900,
                        sink_fraction=0.5)
    q = spec.queries()[0]
    with make_cache(spec) as cache:
        # default RoutingConfig excludes layers {0,1}: nothing skips on layer 0
        cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5))
        res = P.routed_decode_step(q, 0, cache, cfg)
        assert not res.route_bitmap.any()
        ref = oracle_step(orc, spec, 0, q, cfg, P.EngineOptions())
        assert_parity(res.outputs, ref, 4, 128, res.groups)
        # observe_only: decisions recorded, every group attends, none skipped
        cfg2 = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
        opts = P.EngineOptions(observe_only=True)
        res2 = P.routed_decode_step(q, 0, cache, cfg2, opts)
        ref2 = oracle_step(orc, spec, 0, q, cfg2, opts)
        assert res2.route_bitmap.sum() == 4
        assert res2.counters.groups_skipped == 0 and res2.counters.groups_active == 8
        assert_parity(res2.outputs, ref2, 4, 128, res2.groups)


def test_tie_and_sink_on_tie(oracle_libs):
    """q=[3,4,...], k0=[1,0,...] gives S == 0.6 exactly; tau = 0.6 ties."""
    _, orc = oracle_libs
    D, hq, hkv, L = 64, 4, 1, 80
    k0 = np.zeros(D, np.float32)
    k0[0] = 1.0
    rng = np.random.default_rng(5)
    k = np.vstack([k0, rng.standard_normal((L - 1, D)).astype(np.float32)])
    v = rng.standard_normal((L, D)).astype(np.float32)
    from paper_2604_16883_b200.workload import round_bf16

    k, v = round_bf16(k).reshape(L, D), round_bf16(v).reshape(L, D)
    q = np.zeros((hq, D), np.float32)
    q[:, 0], q[:, 1] = 3.0, 4.0
    with P.KvCache(P.CacheConfig(1, hq, hkv, D, L)) as cache:
        cache.append(0, 0, k, v)
        for tie in (False, True):
            cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.6), excluded_layers=(),
                                  sink_on_tie=tie)
            res = P.routed_decode_step(q, 0, cache, cfg)
            assert res.groups[0].decision.group_score == 0.6
            assert res.groups[0].decision.sink == tie
            ref = orc.routed_decode_step(k[None], v[None], k[None, 0], [orc.anchor_norm(k[0])], q,
                                         0, __import__("oracle").Profile.constant(0.6),
                                         excluded=(), sink_on_tie=tie)
            assert_parity(res.outputs, ref, hq, D, res.groups)


def test_degenerate_query_forces_active(oracle_libs):
    _, orc = oracle_libs
    spec = WorkloadSpec(num_q_heads=8, num_kv_heads=2, head_dim=128, length=200,
                        sink_fraction=1.0)
    q = spec.queries()[0]
    q[1] = 0.0  # head 1 of group 0 degenerate
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
    with make_cache(spec) as cache:
        res = P.routed_decode_step(q, 0, cache, cfg)
        assert res.groups[0].decision.degenerate and not res.groups[0].decision.sink
        assert res.groups[0].decision.head_scores[1] == 0.0
        assert res.groups[1].decision.sink
        ref = oracle_step(orc, spec, 0, q, cfg, P.EngineOptions())
        assert_parity(res.outputs, ref, 4, 128, res.groups)


def test_batched_sequences(oracle_libs):
    """B independent caches in one launch."""
    _, orc = oracle_libs
    spec = WorkloadSpec(num_q_heads=16, num_kv_heads=4, head_dim=128, length=640, num_seqs=3,
                        sink_fraction=0.5, seed=11)
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
    qs = spec.queries()
    with make_cache(spec) as cache:
        res = P.routed_decode_step(qs, 0, cache, cfg)
        assert res.outputs.shape == (3, 16, 128)
        for s in range(3):
            ref = oracle_step(orc, spec, s, qs[s], cfg, P.EngineOptions())
            assert_parity(res.outputs[s], ref, 4, 128, res.groups[s * 4:(s + 1) * 4])


def test_wide_gqa_envelope():
    """GQA width above 16 is rejected at creation (9-16 run on the WIDE step
    kernel and the two-tile analysis pass)."""
    with pytest.raises(ValueError, match="above 16"):
        P.KvCache(P.CacheConfig(1, 34, 2, 128, 16))


def test_errors_mirror_reference():
    spec = WorkloadSpec(num_q_heads=8, num_kv_heads=2, head_dim=64, length=10)
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5))
    with P.KvCache(P.CacheConfig(2, 8, 2, 64, 16)) as cache:
        q = spec.queries()[0]
        with pytest.raises(RuntimeError, match="empty cache"):
            P.routed_decode_step(q, 0, cache, cfg)
        with pytest.raises(IndexError):
            P.routed_decode_step(q, 5, cache, cfg)
        with pytest.raises(ValueError):
            P.routed_decode_step(q[:3], 0, cache, cfg)
        with pytest.raises(RuntimeError, match="degenerate anchor"):
            cache.append(0, 0, np.zeros(64), np.ones(64))
        cache.append(0, 0, np.ones((3, 64)), np.ones((3, 64)))
        from paper_2604_16883_b200._abi import LogicError

        with pytest.raises(LogicError):
            cache.token_count()
        with pytest.raises(RuntimeError, match="overflow"):
            cache.append(0, 0, np.ones((14, 64)), np.ones((14, 64)))


def test_timings_and_launch_count():
    spec = WorkloadSpec(num_q_heads=32, num_kv_heads=8, head_dim=128, length=4096,
                        sink_fraction=0.5)
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
    with make_cache(spec) as cache:
        res = P.routed_decode_step(spec.queries()[0], 0, cache, cfg)
        c = res.counters
        assert c.routing_seconds > 0 and c.attention_seconds > 0 and c.merge_seconds > 0
        n, dms, sms = P.last_step_stats(cache)
        assert n in (1, 3) and 0 < dms <= sms * 1.0001


# ---- golden fixtures from the compiled reference (tests/golden) ------------------
from golden_cases import case_ids, load_cases  # noqa: E402


@pytest.mark.parametrize("name", case_ids())
def test_golden_fixture_engine(name):
    meta, k, v, z = next(c for c in load_cases() if c[0]["name"] == name)
    hkv, L, D = k.shape
    hq = z["q"].shape[0]
    layers = max(2, meta["layer"] + 1)
    c, n, lo, hi = meta["prof"]
    prof = P.ThresholdProfile(coeffs=tuple(c), length_normalizer=n, clamp_lo=lo, clamp_hi=hi)
    cfg = P.RoutingConfig(profile=prof, excluded_layers=tuple(meta["excluded"]),
                          sink_on_tie=meta["sink_on_tie"])
    opts = P.EngineOptions(num_splits=meta["num_splits"], observe_only=meta["observe_only"])
    with P.KvCache(P.CacheConfig(layers, hq, hkv, D, L)) as cache:
        for layer in range(layers):
            for g in range(hkv):
                cache.append(layer, g, k[g], v[g])
        res = P.routed_decode_step(z["q"], meta["layer"], cache, cfg, opts)

    class Ref:
        pass

    ref = Ref()
    for f in ("outputs", "group_scores", "thresholds", "sink", "degenerate", "group_kv_floats",
              "head_scores"):
        setattr(ref, f, z[f])
    assert_parity(res.outputs, ref, hq // hkv, D, res.groups)
    cnt = z["counters"]
    assert res.counters.kv_floats_loaded == cnt[0]
    assert res.counters.anchor_floats_loaded == cnt[1]
    assert res.counters.groups_active == cnt[2] and res.counters.groups_skipped == cnt[3]


@pytest.mark.parametrize("slots", [2, 5])
def test_partial_spill_slot(oracle_libs, monkeypatch, slots):
    """Force a tiny partial-slot budget (SINKR_DEBUG_SLOTS) so most Split-K
    partials of a unit spill into the locked, LSE-combined last slot; the step
    must still match the oracle (routing bit-exact, outputs within tolerance)."""
    import oracle

    _, orc = oracle_libs
    monkeypatch.setenv("SINKR_DEBUG_SLOTS", str(slots))
    spec = WorkloadSpec(length=65536, sink_fraction=0.625, seed=slots)
    q = spec.queries()[0]
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
    with P.KvCache(P.CacheConfig(1, 32, 8, 128, spec.length)) as cache:
        spec.fill(cache)
        res = P.routed_decode_step(q, 0, cache, cfg)
        res2 = P.routed_decode_step(q, 0, cache, cfg)  # counters/locks reset between steps
    k, v = spec.host_cache(0)
    k0n = [orc.anchor_norm(k[g, 0]) for g in range(8)]
    ref = orc.routed_decode_step(k, v, k[:, 0].copy(), k0n, q, 0, oracle.Profile.constant(0.5),
                                 excluded=(), threads=8)
    for r_ in (res, res2):
        assert np.array_equal(r_.route_bitmap, ref.sink.astype(bool))
        assert [g.kv_floats_loaded for g in r_.groups] == list(ref.group_kv_floats)
        assert np.abs(r_.outputs - ref.outputs).max() <= 2e-3
        assert np.linalg.norm(r_.outputs - ref.outputs) <= 1e-3 * np.linalg.norm(ref.outputs)


@pytest.mark.parametrize("seed", range(int(os.environ.get("SINKR_PARITY_SEEDS", 100))))
def test_randomized_parity(oracle_libs, seed):
    """SPEC.md acceptance 1-2 style: random shapes (D 32/64/128, r 1-16, B 1-3,
    L 1-5000), random keys and queries at random cosines to the anchor (so
    groups land on both sides of tau and near it), random routing options
    (tau, sink_on_tie, observe_only, excluded layers) -- bit-exact routing,
    exact skipped-block record, outputs within tolerance of the oracle."""
    import oracle

    _, orc = oracle_libs
    rng = np.random.default_rng(1000 + seed)
    D = int(rng.choice([32, 64, 128]))
    r = int(rng.choice([1, 2, 3, 4, 8, 12, 16]))
    hkv = int(rng.choice([1, 2, 4, 8]))
    B = int(rng.choice([1, 1, 2, 3]))
    L = int(rng.choice([1, 2, 63, 64, 65, 777, 2048, 5000]))
    layers = 2
    layer = int(rng.integers(layers))
    hq = hkv * r
    cc = P.CacheConfig(layers, hq, hkv, D, L, B)
    k = rng.standard_normal((B, layers, hkv, L, D)).astype(np.float32) * np.float32(rng.uniform(0.5, 3))
    v = rng.standard_normal((B, layers, hkv, L, D)).astype(np.float32)
    q = np.zeros((B, hq, D), np.float32)
    for b in range(B):
        for g in range(hkv):
            kh = k[b, layer, g, 0].astype(np.float64)
            kh /= np.linalg.norm(kh)
            for i in range(r):
                n = rng.standard_normal(D)
                n -= (n @ kh) * kh
                n /= np.linalg.norm(n)
                c = rng.uniform(-0.5, 0.95)
                q[b, g * r + i] = (np.sqrt(D) * (c * kh + np.sqrt(1 - c * c) * n)).astype(np.float32)
    if seed % 7 == 3:
        q[0, 0] = 0.0  # degenerate query
    excl = [(), (0,), (1,), (0, 1)][int(rng.integers(4))] if seed % 3 else ()
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(float(rng.uniform(0.1, 0.6))),
                          excluded_layers=excl, sink_on_tie=bool(seed % 5 == 1))
    opts = P.EngineOptions(observe_only=bool(seed % 6 == 2))
    with P.KvCache(cc) as cache:
        for b in range(B):
            for l_ in range(layers):
                for g in range(hkv):
                    cache.append(l_, g, k[b, l_, g], v[b, l_, g], seq=b)
        res = P.routed_decode_step(q if B > 1 else q[0], layer, cache, cfg, opts)
        if seed % 4 == 0:  # a tie: tau equal to a group score (exact-first routing)
            tie = res.groups[0].decision.group_score
            cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(tie), excluded_layers=excl,
                                  sink_on_tie=cfg.sink_on_tie)
            res = P.routed_decode_step(q if B > 1 else q[0], layer, cache, cfg, opts)
        outs = res.outputs if B > 1 else res.outputs[None]
        for b in range(B):
            kb = np.stack([cache.historical(layer, g, 0, L, seq=b)[0] for g in range(hkv)])
            vb = np.stack([cache.historical(layer, g, 0, L, seq=b)[1] for g in range(hkv)])
            k0 = kb[:, 0, :].copy()
            k0n = np.array([orc.anchor_norm(k0[g]) for g in range(hkv)], dtype=np.float32)
            ref = orc.routed_decode_step(kb, vb, k0, k0n, q[b], layer, oracle_profile(cfg.profile),
                                         excluded=excl, sink_on_tie=cfg.sink_on_tie,
                                         observe_only=opts.observe_only, threads=8)
            assert_parity(outs[b], ref, r, D, res.groups[b * hkv:(b + 1) * hkv])


@pytest.mark.parametrize("hq,hkv,D,L,p", CASES[3:7])
def test_three_kernel_pipeline_parity(oracle_libs, monkeypatch, hq, hkv, D, L, p):
    """The A/B three-kernel form (probe -> decode -> combine, SINKR_FUSED=0)
    meets the same bar as the fused step kernel."""
    monkeypatch.setenv("SINKR_FUSED", "0")
    test_planted_parity(oracle_libs, hq, hkv, D, L, p)


@pytest.mark.parametrize("seed", range(int(os.environ.get("SINKR_BATCHED_SEEDS", 16))))
def test_randomized_batched_parity(oracle_libs, seed):
    """Batched steps across the kernel's batched regimes -- distributed routing
    (U > 32), unit-affine and flat global-token scheduling (Active units above
    the SM count), queue-mode and last-flusher merges -- with a different
    length per sequence and a length-dependent cubic tau(L): bit-exact routing
    and skipped-block record per sequence, outputs within tolerance."""
    _, orc = oracle_libs
    rng = np.random.default_rng(5000 + seed)
    D = int(rng.choice([64, 128]))
    r = int(rng.choice([1, 2, 4, 8, 16]))
    hkv = int(rng.choice([4, 8]))
    B = int(rng.choice([5, 12, 24, 40]))
    B = min(B, 4096 // (hkv * r))  # B * H_q <= 4096 per engine
    hq = hkv * r
    cap = 2600
    lens = rng.integers(1, cap + 1, size=B)
    cc = P.CacheConfig(1, hq, hkv, D, cap, B)
    # tau rises with L over the sampled range, so sequences route differently
    prof = P.ThresholdProfile(coeffs=(0.0, 0.0, 0.3, 0.2), length_normalizer=float(cap),
                              clamp_lo=0.0, clamp_hi=1.0)
    cfg = P.RoutingConfig(profile=prof, excluded_layers=(), sink_on_tie=bool(seed % 2))
    q = np.zeros((B, hq, D), np.float32)
    kv = []
    with P.KvCache(cc) as cache:
        for b in range(B):
            k = (rng.standard_normal((hkv, lens[b], D)) * rng.uniform(0.5, 2.0)).astype(np.float32)
            v = rng.standard_normal((hkv, lens[b], D)).astype(np.float32)
            for g in range(hkv):
                cache.append(0, g, k[g], v[g], seq=b)
                kh = k[g, 0].astype(np.float64) / np.linalg.norm(k[g, 0])
                for i in range(r):
                    n = rng.standard_normal(D)
                    n -= (n @ kh) * kh
                    n /= np.linalg.norm(n)
                    c = rng.uniform(-0.3, 0.95)
                    q[b, g * r + i] = (np.sqrt(D) * (c * kh + np.sqrt(1 - c * c) * n)).astype(np.float32)
            kv.append((k, v))
        res = P.routed_decode_step(q, 0, cache, cfg)
        for b in range(B):
            kb = np.stack([cache.historical(0, g, 0, int(lens[b]), seq=b)[0] for g in range(hkv)])
            vb = np.stack([cache.historical(0, g, 0, int(lens[b]), seq=b)[1] for g in range(hkv)])
            k0 = kb[:, 0, :].copy()
            k0n = np.array([orc.anchor_norm(k0[g]) for g in range(hkv)], dtype=np.float32)
            ref = orc.routed_decode_step(kb, vb, k0, k0n, q[b], 0, oracle_profile(prof), excluded=(),
                                         sink_on_tie=cfg.sink_on_tie, observe_only=False, threads=8)
            assert_parity(res.outputs[b], ref, r, D, res.groups[b * hkv:(b + 1) * hkv])


def test_step_runner_pinned_io_matches(oracle_libs):
    """StepRunner over the engine's pinned step buffers (sinkr_step_io_buffers,
    no host copies) returns what the copying form returns."""
    spec = WorkloadSpec(length=9000, sink_fraction=0.5, seed=21)
    q = spec.queries()[0]
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
    with make_cache(spec) as cache:
        plain = P.StepRunner(cache, cfg)
        want = plain(q).copy()
        info = plain.result()
        pin = P.StepRunner(cache, cfg, pinned_io=True)
        pin.queries[...] = q.reshape(pin.queries.shape)
        for _ in range(3):
            got = pin()
            assert np.abs(got - want).max() <= 1e-6
        res = pin.result()
        assert [g.decision.sink for g in res.groups] == [g.decision.sink for g in info.groups]
        assert res.counters.kv_floats_loaded == info.counters.kv_floats_loaded


def test_speculative_prefetch_changing_routes(oracle_libs):
    """The speculative L2 prefetch guesses each layer's Active set from its
    previous step: steps that alternate between routes (a hit, a miss, a
    different layer, the dense route) stay bit-exact in routing and within
    tolerance, on a cache long enough for the prefetch to run (>= 1,024 Active
    rows per CTA)."""
    _, orc = oracle_libs
    specs = [WorkloadSpec(num_layers=2, layer=l, length=80000, sink_fraction=0.5, seed=17)
             for l in (0, 1)]
    opts = P.EngineOptions()
    cfgs = {"routed": P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=()),
            "dense": P.RoutingConfig(profile=P.ThresholdProfile.constant(2.0), excluded_layers=()),
            "few": P.RoutingConfig(profile=P.ThresholdProfile.constant(-0.5), excluded_layers=(1,))}
    q = specs[0].queries()[0]
    refs = {}
    with make_cache(specs[0]) as cache:
        specs[1].fill(cache)
        for layer, name in [(0, "routed"), (0, "routed"), (0, "dense"), (0, "routed"), (1, "few"),
                            (0, "few"), (1, "routed"), (0, "routed")]:
            res = P.routed_decode_step(q, layer, cache, cfgs[name], opts)
            if (layer, name) not in refs:
                refs[layer, name] = oracle_step(orc, specs[layer], 0, q, cfgs[name], opts)
            assert_parity(res.outputs, refs[layer, name], specs[0].r, specs[0].head_dim, res.groups)
