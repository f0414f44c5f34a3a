"""Dev tool: per-phase timing of ONE step after an L2 flush (bench's
other_configs condition) vs back to back: where the cold-L2 penalty lands
(routing end, stream end, merge end, reset; per-CTA %globaltimer trace)."""
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
spec = WorkloadSpec(length=L, sink_fraction=0.625)
cache = P.KvCache(P.CacheConfig(1, 32, 8, 128, L))
spec.fill(cache)
P.set_timing(cache, False)
q = torch.from_numpy(spec.queries()[0]).cuda()
out = torch.empty_like(q)
G = cache.decode_grid()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
st = torch.cuda.ExternalStream(cache.stream)
for tau in (0.5, 2.0):
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(tau), excluded_layers=())
    for cold in (False, True):
        rows = []
        for _ in range(8):
            for _ in range(3):
                P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())
            if cold:
                with torch.cuda.stream(st):
                    flush.sum()
            torch.cuda.synchronize()
            buf = (C.c_ulonglong * (G * 8))()
            _abi.lib().sinkr_debug_trace(cache.handle, buf)
            P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())
            torch.cuda.synchronize()
            _abi.lib().sinkr_debug_trace(cache.handle, buf)
            a = np.array(buf, dtype=np.float64).reshape(G, 8)
            t0 = a[:, 4].min()
            rel = lambda x: (x - t0) / 1e3
            x5 = a[:, 5][a[:, 5] > 0]
            rows.append((rel(a[:, 4]).max(), rel(a[:, 0]).max(), rel(a[:, 1]).max(), rel(a[:, 2]).max(),
                         rel(x5).max() if len(x5) else float("nan")))
        m = np.median(np.array(rows), axis=0)
        print(f"L={L} tau={tau} {'cold' if cold else 'warm'}: CTA start spread {m[0]:.2f}, routing end {m[1]:.2f}, "
              f"stream end {m[2]:.2f}, merge end {m[3]:.2f}, last-CTA stamp {m[4]:.2f} us")
