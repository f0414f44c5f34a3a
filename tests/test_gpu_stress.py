"""GPU stress: many back-to-back steps across the kernel's code paths on one
engine set (lean / distributed routing, estimate-first / exact-first
decisions, unit-affine / global-token scheduling, queue / per-unit merge,
modes 0 / 1 / 3, the speculative prefetch hitting and missing, GQA width 16),
interleaved, each compared with a fresh single step and with
the previous replay of the same configuration.  Counters and locks must be
restored by every step; no step may report a kernel error."""
import os

import numpy as np
import pytest
import torch

import paper_2604_16883_b200 as P
from paper_2604_16883_b200 import sharding
from paper_2604_16883_b200.workload import WorkloadSpec

pytestmark = pytest.mark.gpu


def _cfg(tau, **kw):
    return P.RoutingConfig(profile=P.ThresholdProfile.constant(tau), excluded_layers=(), **kw)


def test_interleaved_paths_stay_consistent():
    rng = np.random.default_rng(0)
    specs = {
        "lean": WorkloadSpec(length=20000, sink_fraction=0.5, seed=1),
        "lean-r8": WorkloadSpec(num_q_heads=64, num_kv_heads=8, length=9000, sink_fraction=0.375, seed=2),
        "dist": WorkloadSpec(num_q_heads=32, num_kv_heads=4, num_seqs=6, length=7000, sink_fraction=0.5, seed=3),
        "flat": WorkloadSpec(num_q_heads=40, num_kv_heads=40, num_seqs=6, length=3000, sink_fraction=0.25, seed=4),
        # long enough for the speculative L2 prefetch (>= 1,024 Active rows per CTA)
        "long": WorkloadSpec(length=80000, sink_fraction=0.5, seed=5),
        # GQA width 16: the WIDE instantiation, single-sequence and distributed
        "wide": WorkloadSpec(num_q_heads=16, num_kv_heads=1, length=30000, sink_fraction=0.0, seed=6),
        "wide-dist": WorkloadSpec(num_q_heads=128, num_kv_heads=8, length=5000, sink_fraction=0.5, seed=7),
    }
    caches, qs, refs, outs = {}, {}, {}, {}
    cfgs = {"routed": _cfg(0.5), "dense": _cfg(2.0), "tie_exact": None}
    try:
        for name, spec in specs.items():
            c = P.KvCache(P.CacheConfig(1, spec.num_q_heads, spec.num_kv_heads, 128, spec.length,
                                        spec.num_seqs))
            spec.fill(c)
            P.set_timing(c, False)
            caches[name] = c
            q = spec.queries().reshape(spec.num_seqs * spec.num_q_heads, 128)
            qs[name] = torch.from_numpy(q).cuda()
            outs[name] = torch.empty_like(qs[name])
            # a tau equal to a group score forces the exact-first path
            g0 = P.routed_decode_step(q if spec.num_seqs > 1 else q, 0, c, cfgs["routed"]).groups[0]
            cfgs_local = dict(cfgs, tie_exact=_cfg(g0.decision.group_score))
            for k, cfg in cfgs_local.items():
                P.routed_decode_async(qs[name].data_ptr(), 0, c, cfg, d_outputs=outs[name].data_ptr())
                torch.cuda.synchronize()
                refs[(name, k)] = (outs[name].clone(), P.fetch_step_info(c))
            caches[name]._cfgs = cfgs_local
        (pm,) = sharding.peer_merge_in_process(P, [caches["lean"]])
        for it in range(int(os.environ.get("SINKR_STRESS_STEPS", 60))):
            name = list(specs)[rng.integers(len(specs))]
            c = caches[name]
            k = list(c._cfgs)[rng.integers(3)]
            out = outs[name]
            out.fill_(float("nan"))
            if name == "lean" and it % 5 == 0:
                pm.step(qs[name], out, c._cfgs[k], P.EngineOptions())
            else:
                P.routed_decode_async(qs[name].data_ptr(), 0, c, c._cfgs[k], d_outputs=out.data_ptr())
            torch.cuda.synchronize()
            ref, info0 = refs[(name, k)]
            assert torch.isfinite(out).all(), (it, name, k)
            assert (out - ref).abs().max().item() <= 1e-5, (it, name, k)
            info = P.fetch_step_info(c)  # raises on any step-kernel error
            assert [g.tokens_loaded for g in info.groups] == [g.tokens_loaded for g in info0.groups]
            assert [g.decision.sink for g in info.groups] == [g.decision.sink for g in info0.groups]
    finally:
        for c in caches.values():
            c.close()
