"""Dev tool: graph-replayed steps back-to-back with per-CTA trace of one step in
the middle, to see inter-kernel gaps (SINKR_TRACE=1)."""
import os, sys, ctypes as C
os.environ["SINKR_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2604_16883_b200 as P
from paper_2604_16883_b200 import _abi
from paper_2604_16883_b200.workload import WorkloadSpec
L = 524288
spec = WorkloadSpec(length=L, sink_fraction=0.625)
cache = P.KvCache(P.CacheConfig(1, 32, 8, 128, L)); spec.fill(cache)
q = torch.from_numpy(spec.queries()[0]).cuda(); out = torch.zeros_like(q)
P.set_timing(cache, False)
cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
G = cache.decode_grid()
for _ in range(5): P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())
torch.cuda.synchronize()
buf = (C.c_ulonglong * (G * 8))()
# trace buffer keeps the LAST writer: run 3 steps back to back, read after each pair
starts, ends = [], []
for it in range(4):
    _abi.lib().sinkr_debug_trace(cache.handle, buf)  # clears
    P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())
    torch.cuda.synchronize()
    _abi.lib().sinkr_debug_trace(cache.handle, buf)
    a = np.array(buf, dtype=np.float64).reshape(G, 8)
    starts.append(a[:, 4].min()); ends.append(max(a[:, 5].max(), a[:, 2].max()))
    print(f"step {it}: cta-start spread {(a[:,4].max()-a[:,4].min())/1e3:.2f} us, first start -> last reset {(ends[-1]-starts[-1])/1e3:.1f} us")
st = torch.cuda.ExternalStream(cache.stream)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(50): P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())
e1.record(st); torch.cuda.synchronize()
print("back-to-back graph step us", e0.elapsed_time(e1) / 50 * 1e3)
