"""Dev tool: one step-kernel case per process for ncu captures.

    python scripts/ncu_cases.py CASE        # CASE: routed512k dense512k peer64k c1routed c1dense
                                            #       c4routed (70B shape, 512K)
                                            #       c3routed / c5routed (batched: Yi-9B 200K B=16,
                                            #       LLaVA-13B 8K B=32), wide512krouted (r = 16)

Runs WARM (default 4) untimed steps, then 2 more; capture the last with
    ncu --set full --clock-control none --import-source on -k regex:step_kernel \
        -s $WARM -c 1 -o gpurun_out/<name> python scripts/ncu_cases.py CASE
ncu flushes the caches before every replay (--cache-control all), so every
capture is a cold-L2 step -- the realistic case between a model's GEMMs.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_16883_b200 as P
from paper_2604_16883_b200 import sharding
from paper_2604_16883_b200.workload import WorkloadSpec

CASES = {
    "routed512k": dict(length=524288, tau=0.5),
    "dense512k": dict(length=524288, tau=2.0),
    "peer64k": dict(length=65536, tau=0.5, peer=True),
    "c1routed": dict(length=32768, tau=0.5),
    "c1dense": dict(length=32768, tau=2.0),
    "c4routed": dict(length=524288, tau=0.5, hq=64),
    "wide512kdense": dict(length=524288, tau=2.0, hq=128),  # GQA width 16 (WIDE)
    "wide512krouted": dict(length=524288, tau=0.5, hq=128),
    # batched steps: distributed routing, flat / unit-affine schedules
    "c3routed": dict(length=204800, tau=0.5, hq=32, hkv=4, seqs=16),
    "c5routed": dict(length=8192, tau=0.5, hq=40, hkv=40, seqs=32, image=576),
}

case = CASES[sys.argv[1]]
warm = int(os.environ.get("WARM", 4))
hq, hkv, seqs = case.get("hq", 32), case.get("hkv", 8), case.get("seqs", 1)
spec = WorkloadSpec(num_q_heads=hq, num_kv_heads=hkv, head_dim=128, length=case["length"],
                    num_seqs=seqs, image_tokens=case.get("image", 0), sink_fraction=0.625)
cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(case["tau"]), excluded_layers=())
cache = P.KvCache(P.CacheConfig(1, hq, hkv, 128, case["length"], seqs))
spec.fill(cache)
P.set_timing(cache, False)
q = torch.from_numpy(spec.queries() if seqs > 1 else spec.queries()[0]).cuda()
out = torch.empty_like(q)
if case.get("peer"):
    (pm,) = sharding.peer_merge_in_process(P, [cache])
    opts = P.EngineOptions()

    def step():
        pm.step(q, out, cfg, opts)
else:
    def step():
        P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())

for _ in range(warm + 2):
    step()
torch.cuda.synchronize()
info = P.fetch_step_info(cache)
print(f"{sys.argv[1]}: groups_active={info.counters.groups_active} "
      f"kv_floats={info.counters.kv_floats_loaded}", flush=True)
cache.close()
