"""Dev tool: per-CTA phase stamps of the fused step kernel (SINKR_TRACE=1)."""
import os, sys, ctypes as C
os.environ["SINKR_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2604_16883_b200 as P
from paper_2604_16883_b200 import _abi
from paper_2604_16883_b200.workload import WorkloadSpec
L = int(sys.argv[1]) if len(sys.argv) > 1 else 524288
spec = WorkloadSpec(length=L, sink_fraction=float(sys.argv[2]) if len(sys.argv) > 2 else 0.625)
cache = P.KvCache(P.CacheConfig(1, 32, 8, 128, L)); spec.fill(cache)
q = torch.from_numpy(spec.queries()[0]).cuda(); out = torch.zeros_like(q)
P.set_timing(cache, False)
for tau in (2.0, 0.5):
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(tau), excluded_layers=())
    for _ in range(5): P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())
    torch.cuda.synchronize()
    G = cache.decode_grid()
    import ctypes as CC
    _abi.lib().sinkr_debug_trace(cache.handle, (CC.c_ulonglong * (G * 8))())
    P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * (G * 8))()
    _abi.lib().sinkr_debug_trace(cache.handle, buf)
    a = np.array(buf, dtype=np.float64).reshape(G, 8)
    t0 = a[:, 0].min()
    rs, se, me = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3, (a[:, 2] - t0) / 1e3
    st = (a[:, 4] - t0) / 1e3
    print(f"tau={tau}: start us min {st.min():.1f} max {st.max():.1f}; routing-end us  min {rs.min():.1f} max {rs.max():.1f}")
    ex = a[:, 5][a[:, 5] > 0]
    if len(ex): print(f"   last-CTA reset done us {(ex.max() - t0) / 1e3:.1f}")
    print(f"   stream-end us  min {se.min():.1f} p10 {np.percentile(se,10):.1f} med {np.median(se):.1f} p90 {np.percentile(se,90):.1f} max {se.max():.1f}")
    print(f"   merge-end  us  min {me.min():.1f} med {np.median(me):.1f} max {me.max():.1f}")
    sp = a[:, 3]
    has = sp > 0
    if has.any():
        spd = (sp[has] - t0) / 1e3
        print(f"   spin-done  us  min {spd.min():.1f} med {np.median(spd):.1f} max {spd.max():.1f} (n={has.sum()})")
    print("   earliest stream-end CTAs:", np.argsort(se)[:8].tolist(), np.sort(se)[:8].round(1).tolist())
