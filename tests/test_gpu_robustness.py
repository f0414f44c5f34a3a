"""GPU: a step's non-finite inputs stay in that step.

A NaN query head (or an inf K/V value) makes that step's outputs for the head
non-finite, as the reference's (router.cpp:82-188 attends whatever it is
given).  The Split-K partial slots of the engine are reused by later steps,
and a later step may produce fewer partials per unit than an earlier one: the
merge must not pick up an earlier step's stale slots, so the next clean step
of the same engine is exact again."""
import numpy as np
import pytest
import torch

import paper_2604_16883_b200 as P
from paper_2604_16883_b200.workload import WorkloadSpec

pytestmark = pytest.mark.gpu


def _cfg(tau):
    return P.RoutingConfig(profile=P.ThresholdProfile.constant(tau), excluded_layers=())


@pytest.mark.parametrize("hq", [32, 128])
def test_nan_query_does_not_poison_later_steps(hq):
    # routed first: 3 Active groups over the grid (~50 partials each); then
    # dense: 8 groups (~19 partials each), so slots 19..49 of a unit are the
    # routed step's
    spec = WorkloadSpec(num_q_heads=hq, num_kv_heads=8, length=65536, sink_fraction=0.625, seed=11)
    r = hq // 8
    with P.KvCache(P.CacheConfig(1, hq, 8, 128, spec.length)) as cache:
        spec.fill(cache)
        P.set_timing(cache, False)
        q = torch.from_numpy(spec.queries()[0]).cuda()
        out = torch.empty_like(q)

        def step(qq, tau):
            P.routed_decode_async(qq.data_ptr(), 0, cache, _cfg(tau), d_outputs=out.data_ptr())
            torch.cuda.synchronize()
            return out.clone(), P.fetch_step_info(cache)

        clean_dense, _ = step(q, 2.0)
        clean_routed, info = step(q, 0.5)
        assert torch.isfinite(clean_dense).all() and torch.isfinite(clean_routed).all()
        active = [u for u in range(8) if not info.groups[u].decision.sink]
        assert len(active) == 3
        # one head of every Active group NaN, one +inf
        bad = q.clone()
        for u in active:
            bad[u * r] = float("nan")
            bad[u * r + 1] = float("inf")
        nan_out, _ = step(bad, 0.5)
        assert not torch.isfinite(nan_out[active[0] * r]).any()
        for tau, ref in ((2.0, clean_dense), (0.5, clean_routed), (2.0, clean_dense)):
            got, _ = step(q, tau)
            assert torch.isfinite(got).all(), f"tau={tau}: non-finite outputs after a NaN step"
            assert torch.equal(got.isfinite(), ref.isfinite())
            err = float((got - ref).abs().max())
            assert err <= 1e-5, (tau, err)



def test_nan_query_does_not_poison_later_batched_steps():
    # batched (distributed routing, flat token-space schedule: more Active
    # groups than SMs, the last flusher merges): NaN heads in one step, then
    # clean steps with another routing
    spec = WorkloadSpec(num_q_heads=40, num_kv_heads=40, num_seqs=6, length=3000,
                        sink_fraction=0.5, seed=13)
    n = spec.num_seqs * spec.num_q_heads
    with P.KvCache(P.CacheConfig(1, 40, 40, 128, spec.length, spec.num_seqs)) as cache:
        spec.fill(cache)
        P.set_timing(cache, False)
        q = torch.from_numpy(spec.queries().reshape(n, 128)).cuda()
        out = torch.empty_like(q)

        def step(qq, tau):
            P.routed_decode_async(qq.data_ptr(), 0, cache, _cfg(tau), d_outputs=out.data_ptr())
            torch.cuda.synchronize()
            return out.clone()

        refs = {tau: step(q, tau) for tau in (2.0, 0.5)}
        assert all(torch.isfinite(x).all() for x in refs.values())
        bad = q.clone()
        bad[::7] = float("nan")
        step(bad, 2.0)
        for tau in (0.5, 2.0, 0.5):
            got = step(q, tau)
            assert torch.isfinite(got).all(), f"tau={tau}: non-finite outputs after a NaN step"
            assert float((got - refs[tau]).abs().max()) <= 1e-5
