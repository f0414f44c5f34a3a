"""Dev tool: what the fused peer merge (step mode 3) adds over a plain routed
step, at world 1 in one process: back-to-back step time and the per-CTA trace
(stream end, merge end).  LEN = tokens on this rank."""
import ctypes as C
import os
import sys

os.environ["SINKR_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2604_16883_b200 as P
from paper_2604_16883_b200 import _abi, sharding
from paper_2604_16883_b200.workload import WorkloadSpec

L = int(os.environ.get("LEN", 65536))
spec = WorkloadSpec(length=L, sink_fraction=0.625)
cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
cache = P.KvCache(P.CacheConfig(1, 32, 8, 128, L))
spec.fill(cache)
P.set_timing(cache, False)
q = torch.from_numpy(spec.queries()[0]).cuda()
out = torch.empty_like(q)
st = torch.cuda.ExternalStream(cache.stream)
G = cache.decode_grid()
(pm,) = sharding.peer_merge_in_process(P, [cache])
opts = P.EngineOptions()


def plain():
    P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())


def peer():
    pm.step(q, out, cfg, opts)


for name, fn in (("plain", plain), ("peer", peer)):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(50):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    b2b = e0.elapsed_time(e1) / 50 * 1e3
    buf = (C.c_ulonglong * (G * 8))()
    _abi.lib().sinkr_debug_trace(cache.handle, buf)
    fn()
    torch.cuda.synchronize()
    _abi.lib().sinkr_debug_trace(cache.handle, buf)
    stamps = (C.c_ulonglong * 24)()
    _abi.lib().sinkr_debug_stamps(cache.handle, stamps, 24)
    sv = np.array(stamps, dtype=np.int64)
    a = np.array(buf, dtype=np.float64).reshape(G, 8)
    t0 = a[:, 4].min()
    rel = lambda x: (x - t0) / 1e3
    print(f"{name:5s} L={L}: back-to-back {b2b:.2f} us; stream end max {rel(a[:, 1]).max():.2f}; "
          f"merge end max {rel(a[:, 2]).max():.2f} us")
