"""Dev tool: per-CTA timeline of ONE step (warm = back to back, cold = after a
256 MB L2 flush): quantiles over CTAs of stream start, producer end, stream
end, merge end, exit, and the tokens/claims each CTA streamed.

    python scripts/cta_profile.py [L] [tau]
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
hq = int(os.environ.get("HQ", 32))
spec = WorkloadSpec(num_q_heads=hq, num_kv_heads=8, head_dim=128, length=L, sink_fraction=0.625)
cache = P.KvCache(P.CacheConfig(1, hq, 8, 128, L))
spec.fill(cache)
P.set_timing(cache, False)
q = torch.from_numpy(spec.queries()[0]).cuda()
out = torch.empty_like(q)
G = cache.decode_grid()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
st = torch.cuda.ExternalStream(cache.stream)
cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(tau), excluded_layers=())
buf = (C.c_ulonglong * (G * 8))()


def step():
    P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())


for _ in range(5):
    step()
torch.cuda.synchronize()
qs = (0, 10, 50, 90, 100)
for cold in (False, True):
    rows = []
    for it in range(8):
        if cold:
            with torch.cuda.stream(st):
                flush.sum()  # read-only: evicts L2 without leaving dirty lines
        else:
            step()
        _abi.lib().sinkr_debug_trace(cache.handle, buf)  # clears
        step()
        torch.cuda.synchronize()
        _abi.lib().sinkr_debug_trace(cache.handle, buf)
        a = np.array(buf, dtype=np.uint64).reshape(G, 8)
        rows.append(a)
    a = rows[-1].astype(np.float64)
    t0 = a[:, 4].min()
    rel = lambda c: (a[:, c] - t0) / 1e3  # noqa: E731
    emits = (rows[-1][:, 6] >> np.uint64(32)).astype(np.int64)
    toks = (rows[-1][:, 6] & np.uint64(0xFFFFFFFF)).astype(np.int64)
    print(f"== L={L} tau={tau} {'cold' if cold else 'warm'}  (us from first CTA start; "
          f"quantiles over {G} CTAs: {qs})")
    for name, c in (("kernel start", 4), ("stream start", 0), ("producer end", 7),
                    ("stream end", 1), ("merge end", 3), ("exit", 2)):
        v = rel(c)
        v = v[a[:, c] > 0]
        if len(v):
            print(f"  {name:13s} " + " ".join(f"{np.percentile(v, p):7.2f}" for p in qs))
    print(f"  reset (last CTA) {(a[:, 5].max() - t0) / 1e3:7.2f}")
    print(f"  claims/CTA {np.percentile(emits, qs)}  tokens/CTA {np.percentile(toks, qs)}  "
          f"total tokens {toks.sum()}")
    # per-CTA streamed bytes vs its stream time
    dur = (a[:, 1] - a[:, 0]) / 1e3
    gbs = toks * 512 / np.maximum(dur, 1e-3) / 1e3
    print(f"  per-CTA stream GB/s quantiles {np.percentile(gbs, qs).round(1)}")
    for b in list(np.argsort(-a[:, 2])[:3]) + [0]:
        print(f"  cta {b:3d}: start {rel(4)[b]:6.2f} stream {rel(0)[b]:6.2f} prod_end {rel(7)[b]:6.2f} "
              f"stream_end {rel(1)[b]:6.2f} merge {rel(3)[b] if a[b, 3] else float('nan'):6.2f} "
              f"exit {rel(2)[b]:6.2f} claims {emits[b]} tokens {toks[b]} t6 {(a[b, 6] - t0) / 1e3:9.2f}")
cache.close()
