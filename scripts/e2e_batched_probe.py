"""Dev tool: e2e (host in, host out) StepRunner latency of a batched step,
copying form vs the engine's pinned step buffers (sinkr_step_io_buffers)."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_16883_b200 as P
from paper_2604_16883_b200.workload import WorkloadSpec

HQ, HKV, B, L, IMG = (int(os.environ.get(k, d)) for k, d in
                      (("HQ", 40), ("HKV", 40), ("B", 32), ("LEN", 8192), ("IMG", 576)))
spec = WorkloadSpec(num_q_heads=HQ, num_kv_heads=HKV, num_seqs=B, length=L, sink_fraction=0.625,
                    image_tokens=IMG)
cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
with P.KvCache(P.CacheConfig(1, HQ, HKV, 128, L, B)) as cache:
    spec.fill(cache)
    q = spec.queries()
    P.set_timing(cache, False)
    dq = torch.from_numpy(q.reshape(B * HQ, 128)).cuda()
    dout = torch.empty_like(dq)
    st = torch.cuda.ExternalStream(cache.stream)
    for _ in range(5):
        P.routed_decode_async(dq.data_ptr(), 0, cache, cfg, d_outputs=dout.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(30):
        P.routed_decode_async(dq.data_ptr(), 0, cache, cfg, d_outputs=dout.data_ptr())
    e1.record(st)
    torch.cuda.synchronize()
    print(f"B={B} Hq={HQ} Hkv={HKV} L={L}: device back-to-back {e0.elapsed_time(e1) / 30 * 1e3:.1f} us")
    for name, pinned in (("copying", False), ("pinned", True)):
        r = P.StepRunner(cache, cfg, pinned_io=pinned)
        if pinned:
            r.queries[...] = q
        call = (lambda: r()) if pinned else (lambda: r(q))
        for _ in range(10):
            call()
        ts = []
        for _ in range(100):
            t0 = time.perf_counter()
            call()
            ts.append((time.perf_counter() - t0) * 1e6)
        print(f"  e2e StepRunner ({name}): median {statistics.median(ts):.1f} us")
