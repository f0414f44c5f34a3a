"""Dev tool: back-to-back and L2-flushed step times of the batched BASELINE
configs (C3 Yi-9B B=16 at 200K, C5 LLaVA-13B B=32 at 8K), routed and dense,
one `LABEL {json}` line (scripts/ab_summary.py reads it)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_16883_b200 as P
from paper_2604_16883_b200.workload import WorkloadSpec

CASES = {"C3": dict(num_q_heads=32, num_kv_heads=4, length=204800, num_seqs=16),
         "C5": dict(num_q_heads=40, num_kv_heads=40, length=8192, num_seqs=32, image_tokens=576)}
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
res = {}
for name, kw in CASES.items():
    spec = WorkloadSpec(**kw, sink_fraction=0.625, seed=42)
    with P.KvCache(P.CacheConfig(1, spec.num_q_heads, spec.num_kv_heads, 128, spec.length,
                                 spec.num_seqs)) as cache:
        spec.fill(cache)
        P.set_timing(cache, False)
        dq = torch.from_numpy(spec.queries()).cuda()
        dout = torch.empty_like(dq)
        st = torch.cuda.ExternalStream(cache.stream)
        for cname, tau in (("routed", 0.5), ("dense", 2.0)):
            cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(tau), excluded_layers=())

            def step():
                P.routed_decode_async(dq.data_ptr(), 0, cache, cfg, d_outputs=dout.data_ptr())

            for _ in range(5):
                step()
            torch.cuda.synchronize()
            with torch.cuda.stream(st):
                torch.cuda._sleep(20_000_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(30):
                step()
            e1.record(st)
            torch.cuda.synchronize()
            b2b = e0.elapsed_time(e1) / 30 * 1e3
            evs = []
            with torch.cuda.stream(st):
                torch.cuda._sleep(20_000_000)
                for _ in range(20):
                    flush.sum()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(st)
                    step()
                    b.record(st)
                    evs.append((a, b))
            torch.cuda.synchronize()
            ts = sorted(x.elapsed_time(y) * 1e3 for x, y in evs)
            P.fetch_step_info(cache)
            res[f"{name}_{cname}"] = {"b2b_us": round(b2b, 2), "flushed_us": round(statistics.median(ts), 2),
                                      "flushed_mean_us": round(statistics.fmean(ts[2:-2]), 2)}
print(json.dumps(res))
