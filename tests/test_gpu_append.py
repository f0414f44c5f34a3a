"""The decode loop's per-token KV append (KvCache::append, kv_cache.cpp:61-84;
SPEC.md:331: the step attends over the just-appended token), stream-ordered
on the engine, against the COMPILED REFERENCE appending the same rows (GPU).

Bar per step: route bitmap and group-score bytes equal, per-group
kv_floats equal (the new row is counted for Active groups and skipped with
the rest of a Sink group), outputs within max-abs 2e-3 / rel-L2 1e-3, the
stored row equal to bf16(k_new)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2604_16883_b200 as P
from paper_2604_16883_b200.workload import WorkloadSpec, round_bf16

pytestmark = pytest.mark.gpu

CFG = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())


@pytest.fixture(scope="module")
def ref(oracle_libs):
    r, _ = oracle_libs
    if r is None:
        pytest.skip("compiled reference not available")
    return r


def _check(res, rr, r):
    sink = np.array([g.decision.sink for g in res.groups], dtype=np.int32)
    assert np.array_equal(sink, rr.sink)
    assert np.array([g.decision.group_score for g in res.groups]).tobytes() == rr.group_scores.tobytes()
    assert [g.kv_floats_loaded for g in res.groups] == [int(x) for x in rr.group_kv_floats]
    out = np.asarray(res.outputs).reshape(rr.outputs.shape)
    assert np.abs(out - rr.outputs).max() <= 2e-3
    assert np.linalg.norm(out - rr.outputs) <= 1e-3 * np.linalg.norm(rr.outputs)
    for gi in range(len(sink)):
        if sink[gi]:
            assert not np.any(out[gi * r:(gi + 1) * r].view(np.uint32))


@pytest.mark.parametrize("timing", [False, True])
def test_append_then_step_vs_reference(ref, timing):
    L0, steps = 3000, 9
    spec = WorkloadSpec(length=L0, sink_fraction=0.5, seed=31)
    q = spec.queries()[0]
    rng = np.random.default_rng(5)
    with P.KvCache(P.CacheConfig(1, 32, 8, 128, L0 + steps)) as cache:
        spec.fill(cache)
        P.set_timing(cache, timing)
        rc = oracle.RefCache(ref, 1, 32, 8, 128, L0 + steps)
        for g in range(8):
            k, v = cache.historical(0, g, 0, L0)
            rc.append_rows(0, g, k, v)
        runner = P.AppendStepRunner(cache, CFG)
        for step in range(steps):
            kn = round_bf16((rng.standard_normal((8, 128)) * 1.5).astype(np.float32))
            vn = round_bf16(rng.standard_normal((8, 128)).astype(np.float32))
            how = step % 3
            if how == 0:      # one graph: H2D + append kernel + step kernel
                runner(kn, vn, q)
                res = runner.result()
            elif how == 1:    # device rows, stream-ordered append, then a step
                dk = torch.from_numpy(kn).cuda()
                dv = torch.from_numpy(vn).cuda()
                torch.cuda.synchronize()
                cache.append_token_async(0, dk.data_ptr(), dv.data_ptr())
                res = P.routed_decode_step(q, 0, cache, CFG)
                del dk, dv
            else:             # the synchronous host append of every slot
                for g in range(8):
                    cache.append(0, g, kn[g:g + 1], vn[g:g + 1])
                res = P.routed_decode_step(q, 0, cache, CFG)
            for g in range(8):
                rc.append_rows(0, g, kn[g:g + 1], vn[g:g + 1])
            rr = rc.routed_decode_step(q, 0, oracle.Profile.constant(0.5), excluded=(), workers=8)
            L = L0 + step + 1
            assert cache.token_count() == L
            _check(res, rr, 4)
            for g in (0, 7):
                k, v = cache.historical(0, g, L - 1, L)
                assert np.array_equal(k[0], kn[g]) and np.array_equal(v[0], vn[g])
        rc.close()


def test_append_first_rows_and_errors():
    """First rows go through the host path (anchor capture from the stored
    row); overflow raises RuntimeError and a ragged multi-layer cache
    LogicError, both without appending anything."""
    rng = np.random.default_rng(9)
    with P.KvCache(P.CacheConfig(1, 8, 2, 64, 3)) as cache:
        runner = P.AppendStepRunner(cache, CFG)
        for n in range(3):
            kn = round_bf16((rng.standard_normal((2, 64)) + 2.0).astype(np.float32))
            vn = round_bf16(rng.standard_normal((2, 64)).astype(np.float32))
            runner(kn, vn, rng.standard_normal((8, 64)).astype(np.float32))
            assert cache.token_count() == n + 1
            if n == 0:
                k0, _ = cache.anchor(0, 1)
                assert np.array_equal(k0, kn[1])
        with pytest.raises(RuntimeError, match="kv cache overflow"):
            runner(kn, vn, rng.standard_normal((8, 64)).astype(np.float32))
        assert cache.token_count() == 3
    with P.KvCache(P.CacheConfig(2, 8, 2, 64, 10)) as cache:
        for layer in range(2):
            for g in range(2):
                cache.append(layer, g, rng.standard_normal((4, 64)).astype(np.float32) + 1.0,
                             rng.standard_normal((4, 64)).astype(np.float32))
        runner = P.AppendStepRunner(cache, CFG, layer=1)
        with pytest.raises(AssertionError, match="ragged"):
            runner(np.ones((2, 64), np.float32), np.ones((2, 64), np.float32),
                   np.ones((8, 64), np.float32))
        assert cache.length(1, 0) == 4 and cache.length(0, 0) == 4
        # the reference's order: append the token to every layer, then step
        dk = torch.ones((2, 64), device="cuda")
        for layer in range(2):
            cache.append_token_async(layer, dk.data_ptr(), dk.data_ptr())
        res = P.routed_decode_step(np.ones((8, 64), np.float32), 1, cache, CFG)
        assert cache.token_count() == 5 and np.isfinite(res.outputs).all()
