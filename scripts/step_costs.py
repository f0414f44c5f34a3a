"""Dev tool: graph-step time with kernels dropped (SINKR_DEBUG_KERNELS) to attribute fixed costs."""
import os, subprocess, sys
code = r'''
import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_2604_16883_b200 as P
from paper_2604_16883_b200.workload import WorkloadSpec
L = int(sys.argv[1]); spec = WorkloadSpec(length=L, sink_fraction=0.625)
cache = P.KvCache(P.CacheConfig(1, 32, 8, 128, L)); spec.fill(cache)
q = torch.from_numpy(spec.queries()[0]).cuda(); out = torch.zeros_like(q)
st = torch.cuda.ExternalStream(cache.stream); P.set_timing(cache, False)
res = []
for tau in (2.0, 0.5, -2.0):
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(tau), excluded_layers=())
    for _ in range(10): P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(50): P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())
    e1.record(st); torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1) / 50 * 1e3)
print(os.environ.get("SINKR_DEBUG_KERNELS", "7"), " ".join(f"{x:8.2f}" for x in res))
'''
L = sys.argv[1] if len(sys.argv) > 1 else "524288"
print("mask  dense(us) routed(us) allsink(us)")
for m in ("7", "1", "2", "4", "3", "6"):
    env = dict(os.environ, SINKR_DEBUG_KERNELS=m)
    r = subprocess.run([sys.executable, "-c", code, L], env=env, capture_output=True, text=True)
    print(r.stdout.strip() or r.stderr[-500:])
