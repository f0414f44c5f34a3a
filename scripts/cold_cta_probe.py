"""Dev tool: per-CTA phase stamps (%globaltimer, SINKR_TRACE) of ONE step,
back to back vs after a 256 MiB L2 flush: distribution (min / median / max
over the CTAs, us from the earliest CTA start) of routing end, producer done,
stream end, merge-wait done and exit.

    python scripts/cold_cta_probe.py [L] [tau]
"""
import ctypes as C
import os
import sys

os.environ["SINKR_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2604_16883_b200 as P
from paper_2604_16883_b200 import _abi
from paper_2604_16883_b200.workload import WorkloadSpec

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
tau = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
spec = WorkloadSpec(length=L, sink_fraction=0.625)
cache = P.KvCache(P.CacheConfig(1, 32, 8, 128, L))
spec.fill(cache)
P.set_timing(cache, False)
q = torch.from_numpy(spec.queries()[0]).cuda()
out = torch.empty_like(q)
G = cache.decode_grid()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
st = torch.cuda.ExternalStream(cache.stream)
cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(tau), excluded_layers=())
# a second cache of the same shape: a step over it runs the same code
# (instruction lines into L2) without touching this cache's KV
cache_b = P.KvCache(P.CacheConfig(1, 32, 8, 128, L))
WorkloadSpec(length=L, sink_fraction=0.625, seed=7).fill(cache_b)
P.set_timing(cache_b, False)
out_b = torch.empty_like(q)
st_b = torch.cuda.ExternalStream(cache_b.stream)
cols = {"route_end": 0, "producer_done": 7, "stream_end": 1, "merge_wait": 3, "exit": 2}
for cold in (0, 1, 2):
    acc = {k: [] for k in cols}
    for _ in range(9):
        for _ in range(3):
            P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())
        if cold:
            with torch.cuda.stream(st):
                flush.sum()
        torch.cuda.synchronize()
        if cold == 2:
            P.routed_decode_async(q.data_ptr(), 0, cache_b, cfg, d_outputs=out_b.data_ptr())
            torch.cuda.synchronize()
        buf = (C.c_ulonglong * (G * 8))()
        P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())
        torch.cuda.synchronize()
        _abi.lib().sinkr_debug_trace(cache.handle, buf)
        a = np.array(buf, dtype=np.float64).reshape(G, 8)
        t0 = a[:, 4].min()
        if os.environ.get("SHOW_LATE"):
            ex = a[:, 2]
            late = np.argsort(ex)[-3:]
            print("   latest exits:", [(int(b), round((a[b, 0] - t0) / 1e3, 2), round((a[b, 1] - t0) / 1e3, 2),
                                        round((ex[b] - t0) / 1e3, 2)) for b in late])
        for k, c in cols.items():
            x = a[:, c]
            x = x[x > t0 - 1]
            if len(x):
                acc[k].append(np.percentile((x - t0) / 1e3, [0, 50, 100]))
    print(f"L={L} tau={tau} {['warm', 'cold', 'cold KV, code warm'][cold]} (min / median / max over CTAs, us):")
    for k, v in acc.items():
        if v:
            m = np.median(np.array(v), axis=0)
            print(f"   {k:14s} {m[0]:7.2f} {m[1]:7.2f} {m[2]:7.2f}")
cache.close()
cache_b.close()
