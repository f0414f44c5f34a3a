"""Dev tool: step time at several contexts, back to back (graph replays, CUDA
events over the sequence) and L2-flushed (read-only 256 MiB flush before each
step, median of per-step events) -- for A/B runs of scheduler knobs set by env
(e.g. SINKR_STATIC_PCT).  Prints one JSON line.

    SINKR_STATIC_PCT=70 python scripts/sched_ab.py [L ...]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_16883_b200 as P
from paper_2604_16883_b200.workload import WorkloadSpec

Ls = [int(x) for x in sys.argv[1:]] or [32768, 65536, 524288]
hq = int(os.environ.get("HQ", 32))
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
res = {"env": {k: v for k, v in os.environ.items() if k.startswith("SINKR_")}}
for L in Ls:
    spec = WorkloadSpec(num_q_heads=hq, num_kv_heads=8, head_dim=128, length=L, sink_fraction=0.625)
    with P.KvCache(P.CacheConfig(1, hq, 8, 128, L)) as cache:
        spec.fill(cache)
        P.set_timing(cache, False)
        q = torch.from_numpy(spec.queries()[0]).cuda()
        out = torch.empty_like(q)
        st = torch.cuda.ExternalStream(cache.stream)
        for name, tau in (("routed", 0.5), ("dense", 2.0))[:int(os.environ.get("AB_CASES", 2))]:
            cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(tau), excluded_layers=())

            def step():
                P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=out.data_ptr())

            for _ in range(5):
                step()
            torch.cuda.synchronize()
            with torch.cuda.stream(st):
                torch.cuda._sleep(4_000_000)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            nb = int(os.environ.get("AB_STEPS", 40))
            for _ in range(nb):
                step()
            e1.record(st)
            torch.cuda.synchronize()
            b2b = e0.elapsed_time(e1) / nb * 1e3
            evs = []
            with torch.cuda.stream(st):
                torch.cuda._sleep(8_000_000)
                for _ in range(int(os.environ.get("AB_COLD", 20))):
                    flush.sum()
                    a = torch.cuda.Event(enable_timing=True)
                    b = torch.cuda.Event(enable_timing=True)
                    a.record(st)
                    step()
                    b.record(st)
                    evs.append((a, b))
            torch.cuda.synchronize()
            ts = sorted(x.elapsed_time(y) * 1e3 for x, y in evs)
            cold = statistics.median(ts)
            k = len(ts) // 10
            cold_mean = statistics.fmean(ts[k:len(ts) - k])  # 10 % trimmed: event ticks are ~1 us
            P.fetch_step_info(cache)  # raises on a step-kernel error
            res[f"{L}_{name}"] = {"b2b_us": round(b2b, 2), "flushed_us": round(cold, 2),
                                  "flushed_mean_us": round(cold_mean, 2)}
print(json.dumps(res), flush=True)
