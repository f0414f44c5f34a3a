"""Dev tool: where the e2e (host buffers) step time goes, by variants of the
same step with parts of the host round trip removed."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2604_16883_b200 as P
from paper_2604_16883_b200.workload import WorkloadSpec

L = int(sys.argv[1]) if len(sys.argv) > 1 else 524288
spec = WorkloadSpec(length=L, sink_fraction=0.625)
cache = P.KvCache(P.CacheConfig(1, 32, 8, 128, L))
spec.fill(cache)
cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
P.set_timing(cache, False)
qh = spec.queries()[0]
q = torch.from_numpy(qh).cuda()
out = torch.zeros_like(q)
st = torch.cuda.ExternalStream(cache.stream)
qpin = torch.from_numpy(qh).pin_memory()
opin = torch.zeros_like(qpin).pin_memory()


def bench(name, fn, n=200):
    for _ in range(20):
        fn()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    us = (time.perf_counter() - t) / n * 1e6
    print(f"{name:48s} {us:8.2f} us")


def graph_only():
    P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())
    st.synchronize()


def h2d_graph():
    with torch.cuda.stream(st):
        q.copy_(qpin, non_blocking=True)
    P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())
    st.synchronize()


def h2d_graph_d2h():
    with torch.cuda.stream(st):
        q.copy_(qpin, non_blocking=True)
    P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())
    with torch.cuda.stream(st):
        opin.copy_(out, non_blocking=True)
    st.synchronize()


def launch_only():
    P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())


runner = P.StepRunner(cache, cfg)
bench("launch only (async, no sync; host rate)", launch_only)
st.synchronize()
bench("graph + stream sync", graph_only)
bench("H2D(q) + graph + sync", h2d_graph)
bench("H2D(q) + graph + D2H(out) + sync", h2d_graph_d2h)
bench("StepRunner (C-ABI blocking, full result)", lambda: runner(qh))
allsink = P.RoutingConfig(profile=P.ThresholdProfile.constant(-2.0), excluded_layers=())
r2 = P.StepRunner(cache, allsink)
bench("StepRunner all-sink (fixed cost only)", lambda: r2(qh))
bench("graph + sync all-sink", lambda: (P.routed_decode_async(q.data_ptr(), 0, cache, allsink, d_outputs=out.data_ptr()), st.synchronize()))
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(100):
    P.routed_decode_async(q.data_ptr(), 0, cache, allsink, d_outputs=out.data_ptr())
e1.record(st)
torch.cuda.synchronize()
print(f"{'device back-to-back all-sink':48s} {e0.elapsed_time(e1) / 100 * 1e3:8.2f} us")
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(100):
    P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())
e1.record(st)
torch.cuda.synchronize()
print(f"{'device back-to-back routed':48s} {e0.elapsed_time(e1) / 100 * 1e3:8.2f} us")
