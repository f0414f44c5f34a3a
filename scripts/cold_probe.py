"""Dev tool: what makes a cold step slow.  Per-step CUDA events around ONE
routed step, after different preludes (median of 15):

  warm        the previous op was the same step (KV, code, TLB warm)
  flush       256 MiB read-only L2 flush
  flush+sink  flush, then an all-sink step (warms code, descriptors, routing
              data; streams no KV)
  flush+tlbN  flush, then one 4-byte load every N bytes of the layer's K and V
              (warms address translation; leaves ~nothing in L2)
  flush+both  flush, all-sink step, touch every 64 KiB

    python scripts/cold_probe.py [L]
"""
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_16883_b200 as P
from paper_2604_16883_b200 import _abi
from paper_2604_16883_b200.workload import WorkloadSpec

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
spec = WorkloadSpec(length=L, sink_fraction=0.625)
cache = P.KvCache(P.CacheConfig(1, 32, 8, 128, L))
spec.fill(cache)
P.set_timing(cache, False)
q = torch.from_numpy(spec.queries()[0]).cuda()
out = torch.empty_like(q)
st = torch.cuda.ExternalStream(cache.stream)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
# a second cache of the same shape: a routed step over it runs the same code
# (warming instruction fetch paths in L2) without touching cache A's KV
cache_b = P.KvCache(P.CacheConfig(1, 32, 8, 128, L))
WorkloadSpec(length=L, sink_fraction=0.625, seed=7).fill(cache_b)
P.set_timing(cache_b, False)
out_b = torch.empty_like(q)
routed = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
allsink = P.RoutingConfig(profile=P.ThresholdProfile.constant(-2.0), excluded_layers=())
lib = _abi.lib()


def step(cfg):
    P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())


st_b = torch.cuda.ExternalStream(cache_b.stream)


def step_b(cfg):
    # ordered on A's stream: B's stream waits for what A enqueued, A waits for B
    ev = torch.cuda.Event()
    ev.record(st)
    st_b.wait_event(ev)
    P.routed_decode_async(q.data_ptr(), 0, cache_b, cfg, d_outputs=out_b.data_ptr())
    ev2 = torch.cuda.Event()
    ev2.record(st_b)
    st.wait_event(ev2)


def touch(stride):
    rc = lib.sinkr_debug_touch(cache.handle, C.c_size_t(0), C.c_size_t(stride))
    assert rc == 0


for cfg in (routed, allsink):
    for _ in range(5):
        step(cfg)
        step_b(cfg)
torch.cuda.synchronize()

preludes = {
    "warm": lambda: step(routed),
    "stepB": lambda: step_b(routed),
    "flush": lambda: flush.sum(),
    "flush+sink": lambda: (flush.sum(), step(allsink)),
    "flush+tlb2M": lambda: (flush.sum(), touch(2 << 20)),
    "flush+tlb64K": lambda: (flush.sum(), touch(64 << 10)),
    "flush+both": lambda: (flush.sum(), step(allsink), touch(64 << 10)),
    "flush+sink+tlb2M": lambda: (flush.sum(), step(allsink), touch(2 << 20)),
    "flush+stepB": lambda: (flush.sum(), step_b(routed)),
    "flush+stepB+tlb": lambda: (flush.sum(), step_b(routed), touch(64 << 10)),
}
print(f"L={L}: one routed step after each prelude (median of 15 per-step event pairs, us)")
for name, pre in preludes.items():
    evs = []
    with torch.cuda.stream(st):
        torch.cuda._sleep(4_000_000)
        for _ in range(15):
            pre()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(st)
            step(routed)
            b.record(st)
            evs.append((a, b))
    torch.cuda.synchronize()
    ts = sorted(x.elapsed_time(y) * 1e3 for x, y in evs)
    print(f"  {name:18s} median {statistics.median(ts):7.2f}  min {ts[0]:7.2f}  max {ts[-1]:7.2f}")
cache.close()
cache_b.close()
