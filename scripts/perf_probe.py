"""Dev tool: time routed vs dense decode at one context length (device-resident)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2604_16883_b200 as P
from paper_2604_16883_b200.workload import WorkloadSpec

L = int(sys.argv[1]) if len(sys.argv) > 1 else 524288
p = float(sys.argv[2]) if len(sys.argv) > 2 else 0.625
spec = WorkloadSpec(length=L, sink_fraction=p)
cache = P.KvCache(P.CacheConfig(1, 32, 8, 128, L))
t0 = time.time(); spec.fill(cache); print("fill s", time.time() - t0, flush=True)
q = torch.from_numpy(spec.queries()[0]).cuda()
out = torch.zeros_like(q)
stream = torch.cuda.ExternalStream(cache.stream)
for tau, name in ((2.0, "dense"), (0.5, "routed"), (-2.0, "allsink")):
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(tau), excluded_layers=())
    for _ in range(5):
        P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())
    torch.cuda.synchronize()
    dec = []
    for _ in range(20):
        P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())
        n, dms, sms = P.last_step_stats(cache)
        dec.append((dms, sms))
    dec = np.array(dec)
    info = P.fetch_step_info(cache)
    import ctypes as C
    from paper_2604_16883_b200 import _abi
    st = (C.c_ulonglong * 13)()
    if hasattr(_abi.lib(), "sinkr_debug_stamps"):
        _abi.lib().sinkr_debug_stamps(cache.handle, st, 13)
        d = [int(st[i + 1]) - int(st[i]) for i in range(11)]
        print("  stamp deltas (cycles):", d, "loads+products(thread0):", int(st[12]) - int(st[1]))
    hq = spec.queries()[0]
    res = P.routed_decode_step(hq, 0, cache, cfg)
    c = res.counters
    print(f"  phases us: routing={c.routing_seconds*1e6:.1f} attention={c.attention_seconds*1e6:.1f} merge={c.merge_seconds*1e6:.1f}")
    P.set_timing(cache, False)
    for _ in range(3):
        P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(20):
            P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())
        e1.record(stream)
    torch.cuda.synchronize()
    P.set_timing(cache, True)
    step_us = e0.elapsed_time(e1) / 20 * 1e3
    nact = info.counters.groups_active
    bytes_ = nact * 2 * L * 128 * 2
    dmed = max(np.median(dec[:, 0]) * 1e3, 1e-3)
    print(f"{name}: active={nact} step_us={step_us:.1f} decode_us_med={dmed:.1f} stepev_us={np.median(dec[:,1])*1e3:.1f} "
          f"GB/s(decode)={bytes_/dmed/1e3:.0f} GB/s(step)={bytes_/step_us/1e3:.0f}", flush=True)
