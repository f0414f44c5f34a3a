"""Dev tool: lead-CTA cycle stamps (STAMP(i) in step.cuh) and per-CTA phase
trace of the fused step kernel at several contexts, to attribute fixed costs.
Usage: python scripts/phase_probe.py [L ...]"""
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

NAMES = {0: "start", 1: "mbar-init", 13: "loads-issued", 15: "estimate+sync", 14: "decide",
         16: "sync", 3: "exact-fallback", 7: "sync", 8: "zero-rows+sync",
         9: "stream-end", 10: "merge-end", 11: "exit-count"}
ORDER = [0, 1, 13, 15, 14, 16, 3, 7, 8, 9, 10, 11]
if os.environ.get("DIST"):
    NAMES.update({17: "flags", 18: "reduce", 19: "scan", 20: "actlist", 21: "flatscan"})
    ORDER = [0, 1, 15, 14, 16, 17, 18, 19, 20, 21, 7, 8, 9, 10, 11]

Ls = [int(x) for x in sys.argv[1:]] or [32768, 524288]
HQ, HKV, B = (int(os.environ.get(k, d)) for k, d in (("HQ", 32), ("HKV", 8), ("B", 1)))
IMG = int(os.environ.get("IMG", 0))
for L in Ls:
    spec = WorkloadSpec(num_q_heads=HQ, num_kv_heads=HKV, num_seqs=B, length=L, sink_fraction=0.625,
                        image_tokens=IMG)
    cache = P.KvCache(P.CacheConfig(1, HQ, HKV, 128, L, B))
    spec.fill(cache)
    q = torch.from_numpy(spec.queries().reshape(B * HQ, 128)).cuda()
    out = torch.zeros_like(q)
    P.set_timing(cache, False)
    G = cache.decode_grid()
    st = torch.cuda.ExternalStream(cache.stream)
    for tau in (2.0, 0.5):
        cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(tau), excluded_layers=())
        for _ in range(5):
            P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(40):
            P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())
        e1.record(st)
        torch.cuda.synchronize()
        b2b = e0.elapsed_time(e1) / 40 * 1e3
        buf = (C.c_ulonglong * (G * 8))()
        _abi.lib().sinkr_debug_trace(cache.handle, buf)  # clear
        P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())
        res = P.fetch_step_info(cache) if hasattr(P, "fetch_step_info") else None
        _abi.lib().sinkr_debug_trace(cache.handle, buf)
        stamps = (C.c_ulonglong * 24)()
        _abi.lib().sinkr_debug_stamps(cache.handle, stamps, 24)
        s = np.array(stamps, dtype=np.int64)
        a = np.array(buf, dtype=np.float64).reshape(G, 8)
        t0 = a[:, 4].min()
        rel = lambda x: (x - t0) / 1e3
        print(f"L={L} tau={tau}: back-to-back {b2b:.2f} us/step")
        print(f"  CTA start spread {rel(a[:, 4]).max():.2f} us; routing end min/med/max "
              f"{rel(a[:, 0]).min():.2f}/{np.median(rel(a[:, 0])):.2f}/{rel(a[:, 0]).max():.2f}")
        se = rel(a[:, 1])
        print(f"  stream end min/med/max {se.min():.2f}/{np.median(se):.2f}/{se.max():.2f}; "
              f"merge end max {rel(a[:, 2]).max():.2f}; last-CTA stamp {(rel(a[:, 5][a[:, 5] > 0]).max() if (a[:, 5] > 0).any() else float('nan')):.2f}")
        lc = a[G - 1]
        print(f"  CTA G-1 (prewarm): start {rel(lc[4]):.2f}, dry stream pass end {rel(lc[3]):.2f}, "
              f"dry merge end {rel(lc[5]):.2f}, routing end {rel(lc[0]):.2f}, stream end {rel(lc[1]):.2f} us")
        ne = (a[:, 6].astype(np.uint64) >> np.uint64(32)).astype(np.int64)
        te = (a[:, 6].astype(np.uint64) & np.uint64(0xffffffff)).astype(np.int64)
        pe = rel(a[:, 7])
        late = np.argsort(se)[-6:]
        print("  latest CTAs (id: stream_end, producer_end, claims, tokens):",
              [(int(c), round(se[c], 2), round(pe[c], 2), int(ne[c]), int(te[c])) for c in late])
        print(f"  tokens/CTA min/med/max {te.min()}/{int(np.median(te))}/{te.max()}; "
              f"producer end min/med/max {pe.min():.2f}/{np.median(pe):.2f}/{pe.max():.2f}")
        if s[0]:
            prev = s[0]
            line = []
            for i in ORDER:
                line.append(f"{NAMES[i]}:{(s[i] - prev)}")
                prev = s[i]
            print("  lead cycles:", " ".join(line))
    import time
    runner = P.StepRunner(cache, P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=()))
    qh = spec.queries() if B > 1 else spec.queries()[0]
    for _ in range(10):
        runner(qh)
    t = time.perf_counter()
    for _ in range(50):
        runner(qh)
    print(f"  e2e StepRunner {(time.perf_counter() - t) / 50 * 1e6:.2f} us/step")
    cache.close()
