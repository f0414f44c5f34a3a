"""Dev tool: small routed steps (single-sequence with the code prewarm,
batched), score collection (single and batched), BOS mass, the span
operators, append+step and the fused peer merge, sized for compute-sanitizer
(memcheck / racecheck / synccheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2604_16883_b200 as P
from paper_2604_16883_b200 import analysis as A
from paper_2604_16883_b200.workload import WorkloadSpec

for B, L in ((1, 4096), (4, 3000), (40, 600)):
    spec = WorkloadSpec(length=L, num_seqs=B, sink_fraction=0.5, seed=3)
    with P.KvCache(P.CacheConfig(1, 32, 8, 128, L, B)) as cache:
        spec.fill(cache)
        q = spec.queries()
        cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
        for timing in (True, False):  # eager path, then the one-graph path (upload kernel + step)
            P.set_timing(cache, timing)
            for _ in range(3):  # both counter-set parities, twice
                res = P.routed_decode_step(q[0] if B == 1 else q, 0, cache, cfg)
            assert np.isfinite(res.outputs).all()
        g = P.splitk_attention(cache, q.reshape(B, 32, 128)[B - 1, 4:8], 0, 1, 1, seq=B - 1)
        assert np.isfinite(g.out).all()
        from paper_2604_16883_b200 import calibration as cal
        hs, gs, _ = cal.collect_scores(cache, q, 0)
        assert np.isfinite(hs).all() and np.isfinite(gs).all()
        hb, gb, _ = cal.collect_scores_batch(cache, np.stack([q, q * 0.5, -q]), 0)
        assert np.isfinite(hb).all() and np.isfinite(gb).all()
        a0 = A.attention_bos_mass(cache, q, 0)
        w = A.attention_weights(cache, q[0, :4], 0, 1)
        assert np.isfinite(a0).all() and np.isfinite(w).all()
# span operators (csrc/span.cu) on host spans
rng = np.random.default_rng(5)
kk = rng.standard_normal((700, 64)).astype(np.float32)
vv = rng.standard_normal((700, 64)).astype(np.float32)
qq = rng.standard_normal((3, 64)).astype(np.float32)
from paper_2604_16883_b200 import attention as SA
r1 = SA.splitk_attention(qq, kk, vv, num_splits=3)
parts = [SA.attend_chunk(qq, kk[a:b], vv[a:b]) for a, b in ((0, 300), (300, 700))]
mo = SA.merge_partials(parts + [SA.SplitPartial()], 3, 64)
assert np.isfinite(r1.out).all() and np.abs(mo - r1.out).max() < 1e-5
# per-token append + step (one graph) and the stream-ordered token append
spec = WorkloadSpec(length=1000, sink_fraction=0.5, seed=4)
with P.KvCache(P.CacheConfig(1, 32, 8, 128, 1003)) as cache:
    spec.fill(cache)
    P.set_timing(cache, False)
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
    run = P.AppendStepRunner(cache, cfg)
    for _ in range(3):
        o = run(rng.standard_normal((8, 128)).astype(np.float32),
                rng.standard_normal((8, 128)).astype(np.float32), spec.queries()[0])
        assert np.isfinite(o).all()
# the fused peer merge (mode 3, LL exchange) at world 1, several steps
import torch
from paper_2604_16883_b200 import sharding
spec = WorkloadSpec(length=5000, sink_fraction=0.5, seed=6)
with P.KvCache(P.CacheConfig(1, 32, 8, 128, spec.length)) as cache:
    spec.fill(cache)
    P.set_timing(cache, False)
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
    dq = torch.from_numpy(spec.queries()[0]).cuda()
    dout = torch.empty_like(dq)
    (pm,) = sharding.peer_merge_in_process(P, [cache])
    for _ in range(3):
        pm.step(dq, dout, cfg, P.EngineOptions())
    torch.cuda.synchronize()
    assert torch.isfinite(dout).all()
print("sanitize probe OK")
