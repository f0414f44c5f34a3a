"""Dev tool: where the cold step's time outside the kernel span goes.

For one routed step after (A) the bench's torch L2 flush, (B) the same flush
followed by a do-nothing 148-CTA kernel with the step kernel's shared-memory
size (SMs already configured for ~223 KB of smem), (C) the previous step
(back to back): event time, and from %globaltimer stamps the gap from the
preceding kernel's end to the first CTA start and the kernel span.

    python scripts/flush_kind_probe.py [L]
"""
import ctypes as C
import os
import sys

os.environ["SINKR_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_2604_16883_b200 as P
from paper_2604_16883_b200 import _abi
from paper_2604_16883_b200.workload import WorkloadSpec

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
fk = C.CDLL(os.path.join(ROOT, "scripts/micro/libflush_kind.so"))
spec = WorkloadSpec(length=L, sink_fraction=0.625)
cache = P.KvCache(P.CacheConfig(1, 32, 8, 128, L))
spec.fill(cache)
P.set_timing(cache, False)
q = torch.from_numpy(spec.queries()[0]).cuda()
out = torch.empty_like(q)
G = cache.decode_grid()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
st = torch.cuda.ExternalStream(cache.stream)
cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
stamp = torch.zeros(4, dtype=torch.int64, device="cuda")


def step():
    P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())


for kind in ("A torch flush", "B flush + big-smem kernel", "C back to back", "A torch flush", "B flush + big-smem kernel"):
    ev_us, gap, span, tail = [], [], [], []
    for _ in range(41):
        for _ in range(2):
            step()
        torch.cuda.synchronize()
        with torch.cuda.stream(st):
            torch.cuda._sleep(200000)
            if kind[0] in "AB":
                flush.sum()
            if kind[0] == "B":
                fk.touch_bigsmem(C.c_void_p(cache.stream), 223)
            if kind[0] == "C":
                step()
            fk.stamp(C.c_void_p(stamp.data_ptr()), C.c_void_p(cache.stream))
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            step()
            e1.record(st)
        torch.cuda.synchronize()
        buf = (C.c_ulonglong * (G * 8))()
        _abi.lib().sinkr_debug_trace(cache.handle, buf)
        a = np.array(buf, dtype=np.float64).reshape(G, 8)
        t_prev = float(stamp[0].item())
        ev_us.append(e0.elapsed_time(e1) * 1e3)
        gap.append((a[:, 4].min() - t_prev) / 1e3)
        span.append((a[:, 2].max() - a[:, 4].min()) / 1e3)
    print(f"L={L} {kind:28s} event {np.median(ev_us):6.2f} us | prev end -> first CTA start "
          f"{np.median(gap):5.2f} | CTA span {np.median(span):6.2f}", flush=True)
cache.close()
