"""Dev tool: allsink step (no streaming) replayed as graphs, for ncu launch timing."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_16883_b200 as P
from paper_2604_16883_b200.workload import WorkloadSpec
L = 65536
spec = WorkloadSpec(length=L, sink_fraction=0.625)
cache = P.KvCache(P.CacheConfig(1, 32, 8, 128, L)); spec.fill(cache)
q = torch.from_numpy(spec.queries()[0]).cuda(); out = torch.zeros_like(q)
P.set_timing(cache, False)
cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(-2.0), excluded_layers=())
for _ in range(30): P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())
torch.cuda.synchronize()
st = torch.cuda.ExternalStream(cache.stream)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(100): P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())
e1.record(st); torch.cuda.synchronize()
print("allsink graph step us", e0.elapsed_time(e1) / 100 * 1e3)
