"""The reference's span-level attention API (attention.hpp:14-85) on the GPU,
against the COMPILED REFERENCE on identical f32 inputs (GPU).

Bar: attend_chunk's block maxima m are bit-identical (logits are the
reference's sequential fp64 dots of exact f32 products), l and acc within
1e-12 relative (fp64 state, different tiling of the rescales); merged /
normalised f32 outputs within 1e-6; every error case raises the reference's
exception class with its message."""
import numpy as np
import pytest

import paper_2604_16883_b200 as P
from paper_2604_16883_b200 import attention as A
from paper_2604_16883_b200.workload import WorkloadSpec

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref(oracle_libs):
    r, _ = oracle_libs
    if r is None:
        pytest.skip("compiled reference not available")
    return r


def _case(seed, heads, dim, n, qscale=2.0, sink=False):
    rng = np.random.default_rng(seed)
    q = (rng.standard_normal((heads, dim)) * qscale).astype(np.float32)
    k = rng.standard_normal((n, dim)).astype(np.float32)
    v = rng.standard_normal((n, dim)).astype(np.float32)
    if sink:  # a planted BOS sink: large-logit key, tiny value
        k[0] = q[0] / np.linalg.norm(q[0]) * 30.0
        v[0] *= 1e-3
    return q, k, v


@pytest.mark.parametrize("heads,dim,n,block", [
    (1, 32, 1, 128), (4, 128, 7, 128), (8, 128, 1000, 64), (3, 80, 4097, 128),
    (8, 64, 20000, 128), (2, 256, 3000, 7), (16, 128, 513, 128), (1, 1000, 300, 128),
])
def test_attend_chunk_vs_reference(ref, heads, dim, n, block):
    q, k, v = _case(heads * 1000 + n, heads, dim, n, sink=n > 100)
    p = A.attend_chunk(q, k, v, n, block)
    m, lsum, acc = ref.attend_chunk(q, k, v, block)
    assert p.tokens == n and not p.empty()
    assert p.m.tobytes() == m.tobytes()  # bit-identical maxima
    np.testing.assert_allclose(p.l, lsum, rtol=1e-12)
    np.testing.assert_allclose(p.acc, acc, rtol=1e-12, atol=1e-12 * np.abs(acc).max())


@pytest.mark.parametrize("heads,dim,n,splits", [
    (4, 128, 1, 1), (4, 128, 10, 3), (8, 128, 5000, 8), (1, 32, 999, 16), (6, 96, 3001, 5),
    (8, 128, 131072, 16),
])
def test_splitk_online_dense_vs_reference(ref, heads, dim, n, splits):
    q, k, v = _case(n + splits, heads, dim, n, sink=True)
    res = P.splitk_attention(A.QueryGroup.over(q, heads, dim), k, v, n, splits)
    out_r, kvf = ref.splitk_attention(q, k, v, splits, workers=4)
    assert res.counters.kv_floats_loaded == kvf == 2 * n * dim
    assert np.abs(res.out - out_r).max() <= 1e-6
    on = P.online_attention(q, k, v, n)
    assert np.abs(on - ref.online_attention(q, k, v)).max() <= 1e-6
    de = P.dense_attention(q, k, v, n)
    assert np.abs(de - ref.dense_attention(q, k, v)).max() <= 1e-6
    # online / splitk agree with dense within 1e-5
    assert np.abs(on - de).max() <= 1e-5 and np.abs(res.out - de).max() <= 1e-5


def test_merge_partials_vs_reference(ref):
    """merge_partials (attention.cpp:159-183) on partials of real chunks,
    with empty partials interleaved (skipped), in several orders
    (permutation-invariant within 1e-6)."""
    heads, dim, n = 4, 128, 6000
    q, k, v = _case(5, heads, dim, n, sink=True)
    parts = []
    for a, b in P.split_ranges(n, 7):
        parts.append(A.attend_chunk(q, k[a:b], v[a:b]))
    parts.insert(2, A.SplitPartial())
    parts.append(A.SplitPartial())
    out = A.merge_partials(parts, heads, dim)
    rp = [(p.m, p.l, p.acc, p.tokens) for p in parts if not p.empty()] + [
        (np.zeros(heads), np.zeros(heads), np.zeros((heads, dim)), 0)]
    out_r = ref.merge_partials(rp, heads, dim)
    assert np.abs(out - out_r).max() <= 1e-6
    assert np.abs(out - ref.dense_attention(q, k, v)).max() <= 1e-5
    rng = np.random.default_rng(0)
    for _ in range(3):
        perm = [parts[i] for i in rng.permutation(len(parts))]
        assert np.abs(A.merge_partials(perm, heads, dim) - out).max() <= 1e-6
    # a single partial merges to acc / l
    one = A.merge_partials([parts[0]], heads, dim)
    np.testing.assert_allclose(one, (parts[0].acc / parts[0].l[:, None]).astype(np.float32), rtol=1e-6)


def test_span_errors_match_reference(ref):
    q, k, v = _case(1, 4, 64, 10)
    with pytest.raises(ValueError, match="merge needs at least one non-empty partial"):
        A.merge_partials([A.SplitPartial(), A.SplitPartial()], 4, 64)
    with pytest.raises(ValueError, match="merge needs at least one non-empty partial"):
        A.merge_partials([], 4, 64)
    good = A.attend_chunk(q, k, v)
    with pytest.raises(ValueError, match="partial shape does not match heads x dim"):
        A.merge_partials([good], 4, 32)
    with pytest.raises(ValueError, match="block_size must be positive"):
        A.attend_chunk(q, k, v, 10, 0)
    with pytest.raises(ValueError, match="attention needs at least one token"):
        A.attend_chunk(q, k[:0], v[:0], 0)
    with pytest.raises(ValueError, match="num_splits must be in"):
        P.splitk_attention(q, k, v, 10, 0)
    with pytest.raises(ValueError, match="num_splits must be in"):
        P.splitk_attention(q, k, v, 10, 11)
    with pytest.raises(ValueError, match="key span size does not match len x dim"):
        P.dense_attention(q, k[:5], v, 10)
    with pytest.raises(ValueError, match="value span size does not match len x dim"):
        P.online_attention(q, k, v[:5], 10)
    with pytest.raises(ValueError, match="empty query group"):
        A.attend_chunk(np.zeros((0, 64), np.float32), k, v)


@pytest.mark.parametrize("frm,to", [(0, 1), (0, 5000), (1, 4096), (1234, 4321), (4999, 5000)])
def test_attend_chunk_cached_vs_reference(ref, frm, to):
    """attend_chunk over the cached bf16 rows [frm, to) of one group, read in
    place, against the reference's attend_chunk over those rows (exact f32
    upcast): KvCache::historical + attend_chunk, router.cpp:149-160."""
    spec = WorkloadSpec(length=5000, sink_fraction=0.5, seed=21)
    q = spec.queries()[0]
    with P.KvCache(P.CacheConfig(1, 32, 8, 128, spec.length)) as cache:
        spec.fill(cache)
        for g in (0, 5):
            gq = q[g * 4:(g + 1) * 4]
            p = A.attend_chunk_cached(cache, gq, 0, g, frm, to)
            k, v = cache.historical(0, g, frm, to)
            m, lsum, acc = ref.attend_chunk(gq, k, v)
            assert p.tokens == to - frm
            assert p.m.tobytes() == m.tobytes()
            np.testing.assert_allclose(p.l, lsum, rtol=1e-12)
            np.testing.assert_allclose(p.acc, acc, rtol=1e-12, atol=1e-12 * np.abs(acc).max())
        with pytest.raises(IndexError, match="exceeds length"):
            A.attend_chunk_cached(cache, q[:4], 0, 0, 10, 5001)
        with pytest.raises(ValueError, match="attention needs at least one token"):
            A.attend_chunk_cached(cache, q[:4], 0, 0, 10, 10)
        # the chunks of a split merge to the cached group's splitk_attention
        parts = [A.attend_chunk_cached(cache, q[:4], 0, 0, a, b) for a, b in P.split_ranges(5000, 5)]
        sk = P.splitk_attention(cache, q[:4], 0, 0, 5)
        assert np.abs(A.merge_partials(parts, 4, 128) - sk.out).max() <= 2e-6
