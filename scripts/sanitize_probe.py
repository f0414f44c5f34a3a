"""Dev tool: one small routed step, one batched step and one BOS-mass pass,
sized for compute-sanitizer (memcheck / racecheck / synccheck)."""
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
        for _ in range(2):
            res = P.routed_decode_step(q[0] if B == 1 else q, 0, cache, cfg)
        assert np.isfinite(res.outputs).all()
        g = P.splitk_attention(cache, q.reshape(B, 32, 128)[B - 1, 4:8], 0, 1, 1, seq=B - 1)
        assert np.isfinite(g.out).all()
        from paper_2604_16883_b200 import calibration as cal
        hs, gs, _ = cal.collect_scores(cache, q, 0)
        assert np.isfinite(hs).all() and np.isfinite(gs).all()
        a0 = A.attention_bos_mass(cache, q, 0)
        w = A.attention_weights(cache, q[0, :4], 0, 1)
        assert np.isfinite(a0).all() and np.isfinite(w).all()
print("sanitize probe OK")
