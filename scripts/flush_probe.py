"""Dev tool: C1 (32K) step time under different cache conditions: back-to-back
replays, after a 256 MB read flush (bench.py's method), after a 256 MB write
flush, and after a flush of only the KV-sized footprint."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_16883_b200 as P
from paper_2604_16883_b200.workload import WorkloadSpec

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
spec = WorkloadSpec(length=L, sink_fraction=0.625)
cache = P.KvCache(P.CacheConfig(1, 32, 8, 128, L)); spec.fill(cache)
P.set_timing(cache, False)
q = torch.from_numpy(spec.queries()[0]).cuda(); out = torch.empty_like(q)
st = torch.cuda.ExternalStream(cache.stream)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for tau in (-2.0, 0.5, 2.0):
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(tau), excluded_layers=())
    for _ in range(5):
        P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())
    torch.cuda.synchronize()
    res = {}
    for mode in ("b2b", "read-flush", "write-flush", "read-flush+gap"):
        ts = []
        with torch.cuda.stream(st):
            for _ in range(10):
                if mode.startswith("read"):
                    flush.sum()
                elif mode == "write-flush":
                    flush.fill_(1)
                if mode.endswith("gap"):
                    torch.cuda._sleep(20000)
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record(st)
                P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())
                e1.record(st)
                ts.append((e0, e1))
        torch.cuda.synchronize()
        res[mode] = statistics.median(a.elapsed_time(b) * 1e3 for a, b in ts)
    print(f"L={L} tau={tau}: " + "  ".join(f"{k} {v:.2f} us" for k, v in res.items()))
