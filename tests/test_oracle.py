"""CPU: pin the oracle.

1. SPEC.md known-answer examples on the compiled reference AND the C
   restatement.
2. The restatement is bit-identical to the compiled reference on randomized
   attend_chunk / merge / dense / routed_decode_step instances.
3. The restatement reproduces the committed golden fixtures (generated from
   the reference by tests/golden/make_golden.py) bit-exactly.
4. SPEC.md acceptance 1 (kernel equivalence, 1e-5) holds for the reference.
"""
import math

import numpy as np
import pytest

import oracle
from golden_cases import case_ids, load_cases
from paper_2604_16883_b200.workload import WorkloadSpec, round_bf16


@pytest.fixture(scope="module")
def libs(oracle_libs):
    ref, orc = oracle_libs
    if ref is None:
        pytest.skip("reference not built (oracle/_ref)")
    return ref, orc


def both(libs):
    return [("ref", libs[0]), ("orc", libs[1])]


# ---- 1. SPEC known answers ---------------------------------------------------
def test_proxy_score_kats(libs):
    for _, L in both(libs):
        s, dg = L.proxy_score([1, 1], [1, 0], 1.0)
        assert s == 0.70710678118654746 and not dg
        assert L.proxy_score([1, 0], [0, 1], 1.0) == (0.0, False)
        assert L.proxy_score([3, 4], [3, 4], 5.0) == (1.0, False)
        assert L.proxy_score([0, 0], [3, 4], 5.0) == (0.0, True)  # degenerate query
        # scale invariance: exact for power-of-two scales
        q = np.array([0.3, -1.2, 2.0], np.float32)
        a = L.proxy_score(q, [1.0, 2.0, -0.5], math.sqrt(5.25))[0]
        assert L.proxy_score(q * 4, [1.0, 2.0, -0.5], math.sqrt(5.25))[0] == a
        assert abs(L.proxy_score(q * 3.7, [1.0, 2.0, -0.5], math.sqrt(5.25))[0] - a) < 1e-6


def test_group_score_and_threshold_kats(libs):
    for _, L in both(libs):
        assert L.group_score([0.6, 0.5, 0.7, 0.4], 4) == 0.55
        assert L.group_score([0.3], 1) == 0.3
        with pytest.raises(ValueError):
            L.group_score([0.1, 0.2], 3)
        assert L.threshold_for_length(12345, oracle.Profile.constant(0.55)) == 0.55
        assert L.threshold_for_length(5, oracle.Profile((1, 0, 0, 0), 10, 0, 1)) == 0.125
        with pytest.raises(ValueError):
            L.threshold_for_length(0, oracle.Profile.constant(0.5))


def test_route_kats(libs):
    p = oracle.Profile.constant(0.55)
    for _, L in both(libs):
        assert L.route(5, 0.56, 100, p) == (True, 0.55)
        assert L.route(5, 0.55, 100, p) == (False, 0.55)       # tie -> Active
        assert L.route(5, 0.55, 100, p, sink_on_tie=True)[0]   # fault hook flips it
        assert not L.route(0, 0.99, 100, p)[0]                  # excluded layer 0
        assert not L.route(1, 0.99, 100, p)[0]
        assert L.route(0, 0.99, 100, p, excluded=())[0]
        # default RoutingConfig{} is tau = 0 (SURVEY gotcha 1)
        assert L.route(5, 0.01, 100, oracle.Profile())[0]


def test_split_kats(libs):
    for _, L in both(libs):
        assert L.split_ranges(10, 3) == [(0, 4), (4, 7), (7, 10)]
        assert [L.auto_num_splits(n) for n in (8192, 32768, 65536, 131072, 204800, 524288)] \
            == [1, 4, 8, 16, 16, 16]
        assert L.auto_num_splits(1) == 1
        with pytest.raises(ValueError):
            L.split_ranges(3, 4)
        with pytest.raises(ValueError):
            L.split_ranges(3, 0)


def test_anchor_capture_kats(libs):
    ref, orc = libs
    assert orc.anchor_norm([3.0, 4.0]) == 5.0
    with pytest.raises(RuntimeError):
        orc.anchor_norm([0.0, 0.0])
    rc = oracle.RefCache(ref, 1, 2, 1, 2, 4)
    rc.append_rows(0, 0, [[3.0, 4.0]], [[1.0, 1.0]])
    k0, n = rc.anchor(0, 0)
    assert n == 5.0 and list(k0) == [3.0, 4.0]
    with pytest.raises(RuntimeError, match="degenerate anchor"):
        oracle.RefCache(ref, 1, 2, 1, 2, 4).append_rows(0, 0, [[0.0, 0.0]], [[1.0, 1.0]])
    with pytest.raises(RuntimeError, match="overflow"):
        rc.append_rows(0, 0, np.ones((4, 2)), np.ones((4, 2)))


def test_merge_kats(libs):
    rng = np.random.default_rng(0)
    for _, L in both(libs):
        m, l, acc = rng.standard_normal(2), rng.random(2) + 0.5, rng.standard_normal((2, 3))
        out = L.merge_partials([(m, l, acc, 5)], 2, 3)  # single partial -> acc / l
        np.testing.assert_array_equal(out, (acc / l[:, None]).astype(np.float32))
        with pytest.raises(ValueError):
            L.merge_partials([(m, l, acc, 0)], 2, 3)  # all empty


# ---- 2. restatement == reference, bit for bit ---------------------------------
@pytest.mark.parametrize("length,dim,heads,block", [(1, 32, 1, 128), (7, 64, 4, 3),
                                                    (300, 128, 8, 128), (1000, 64, 4, 1000),
                                                    (513, 128, 1, 1)])
def test_attend_chunk_bit_exact(libs, length, dim, heads, block):
    ref, orc = libs
    rng = np.random.default_rng(length + dim)
    q = rng.standard_normal((heads, dim)).astype(np.float32)
    k = rng.standard_normal((length, dim)).astype(np.float32)
    v = rng.standard_normal((length, dim)).astype(np.float32)
    for a, b in zip(ref.attend_chunk(q, k, v, block), orc.attend_chunk(q, k, v, block)):
        assert a.tobytes() == b.tobytes()
    assert ref.dense_attention(q, k, v).tobytes() == orc.dense_attention(q, k, v).tobytes()


def test_merge_bit_exact(libs):
    ref, orc = libs
    rng = np.random.default_rng(4)
    parts = [(rng.standard_normal(4) * 5, rng.random(4) + 0.1, rng.standard_normal((4, 16)),
              int(t)) for t in (3, 0, 9, 1)]
    assert ref.merge_partials(parts, 4, 16).tobytes() == orc.merge_partials(parts, 4, 16).tobytes()


ROUTED = [
    # hq, hkv, D, L, p, tau, splits, observe, tie, layer, excluded
    (32, 8, 128, 1, 0.5, 0.5, 0, False, False, 2, (0, 1)),
    (32, 8, 128, 7, 0.5, 0.5, 0, False, False, 2, (0, 1)),
    (16, 4, 64, 64, 0.5, 0.5, 2, False, False, 0, ()),
    (8, 8, 32, 1024, 0.25, 0.5, 8, True, False, 0, ()),
    (32, 4, 128, 1500, 0.5, 0.5, 4, False, True, 3, (0, 1)),
    (32, 8, 128, 2000, 0.625, 2.0, 0, False, False, 0, ()),
    (32, 8, 128, 2000, 0.625, -2.0, 0, False, False, 0, ()),
    (40, 40, 128, 500, 0.5, 0.5, 1, False, False, 0, (0, 1)),
]


@pytest.mark.parametrize("hq,hkv,D,L,p,tau,splits,observe,tie,layer,excluded", ROUTED)
def test_routed_decode_step_bit_exact(libs, hq, hkv, D, L, p, tau, splits, observe, tie, layer,
                                      excluded):
    ref, orc = libs
    spec = WorkloadSpec(num_q_heads=hq, num_kv_heads=hkv, head_dim=D, length=L, sink_fraction=p,
                        seed=L * 7 + hq)
    k, v = spec.host_cache(0)
    q = spec.queries()[0]
    prof = oracle.Profile.constant(tau)
    rc = oracle.RefCache(ref, layer + 1, hq, hkv, D, L)
    for lay in range(layer + 1):
        for g in range(hkv):
            rc.append_rows(lay, g, k[g], v[g])
    a = rc.routed_decode_step(q, layer, prof, excluded=excluded, sink_on_tie=tie,
                              num_splits=splits, observe_only=observe, workers=4)
    k0 = np.stack([rc.anchor(layer, g)[0] for g in range(hkv)])
    kn = [rc.anchor(layer, g)[1] for g in range(hkv)]
    assert kn == [orc.anchor_norm(k[g, 0]) for g in range(hkv)]
    b = orc.routed_decode_step(k, v, k0, kn, q, layer, prof, excluded=excluded, sink_on_tie=tie,
                               num_splits=splits, observe_only=observe, threads=4)
    for f in ("outputs", "group_scores", "thresholds", "sink", "degenerate", "group_kv_floats",
              "head_scores"):
        assert getattr(a, f).tobytes() == getattr(b, f).tobytes(), f
    for key in ("kv_floats_loaded", "anchor_floats_loaded", "groups_active", "groups_skipped"):
        assert a.counters[key] == b.counters[key]
    # SPEC.md:322-323 invariants on the reference itself
    r = hq // hkv
    for g in range(hkv):
        if a.sink[g] and not observe:
            assert not np.any(a.outputs[g * r:(g + 1) * r].view(np.uint32))
            assert a.group_kv_floats[g] == 0
        else:
            assert a.group_kv_floats[g] == 2 * L * D


# ---- 3. golden fixtures --------------------------------------------------------
@pytest.mark.parametrize("name", case_ids())
def test_golden_fixture(libs, name):
    _, orc = libs
    meta, k, v, z = next(c for c in load_cases() if c[0]["name"] == name)
    c, n, lo, hi = meta["prof"]
    kn = [orc.anchor_norm(k[g, 0]) for g in range(k.shape[0])]
    res = orc.routed_decode_step(k, v, k[:, 0].copy(), kn, z["q"], meta["layer"],
                                 oracle.Profile(tuple(c), n, lo, hi),
                                 excluded=tuple(meta["excluded"]),
                                 sink_on_tie=meta["sink_on_tie"], num_splits=meta["num_splits"],
                                 observe_only=meta["observe_only"], threads=2)
    for f in ("outputs", "group_scores", "thresholds", "sink", "degenerate", "group_kv_floats",
              "head_scores"):
        assert getattr(res, f).reshape(-1).tobytes() == z[f].reshape(-1).tobytes(), f


# ---- 4. SPEC acceptance 1 on the reference -----------------------------------------
@pytest.mark.parametrize("L", [1, 7, 64, 1024])
@pytest.mark.parametrize("D,G", [(32, 1), (64, 4), (128, 8)])
def test_reference_kernel_equivalence(libs, L, D, G):
    ref, _ = libs
    rng = np.random.default_rng(L * D + G)
    q = rng.standard_normal((G, D)).astype(np.float32)
    k = rng.standard_normal((L, D)).astype(np.float32)
    v = rng.standard_normal((L, D)).astype(np.float32)
    dense = ref.dense_attention(q, k, v)
    assert np.abs(ref.online_attention(q, k, v) - dense).max() <= 1e-5
    for s in (1, 2, 4, 8):
        if s <= L:
            out, kvf = ref.splitk_attention(q, k, v, s)
            assert np.abs(out - dense).max() <= 1e-5
            assert kvf == 2 * L * D


def test_bf16_rounding_matches_c(libs):
    _, orc = libs
    rng = np.random.default_rng(1)
    x = (rng.standard_normal(2000) * 10).astype(np.float32)
    ours = round_bf16(x)
    assert all(orc.round_bf16(float(a)) == b for a, b in zip(x[:200], ours[:200]))
