"""Time attention_bos_mass alone at the headline shape.

Run under ncu for the kernel launch list:
  ncu --metrics gpu__time_duration.sum --clock-control none python scripts/bos_probe.py
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_16883_b200 as P  # noqa: E402
from paper_2604_16883_b200 import analysis as A  # noqa: E402
from bench import SHAPE  # noqa: E402
from paper_2604_16883_b200.workload import WorkloadSpec  # noqa: E402

L = int(os.environ.get("LEN", 524288))
N = int(os.environ.get("ITERS", 10))
spec = WorkloadSpec(**SHAPE, length=L, sink_fraction=0.75, seed=0)
with P.KvCache(P.CacheConfig(1, 32, 8, 128, L)) as cache:
    spec.fill(cache)
    q = spec.queries()[0]
    st = torch.cuda.ExternalStream(cache.stream)
    ts, ks = [], []
    for _ in range(N):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        A.attention_bos_mass(cache, q, 0)
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
        ks.append(A.last_kernel_seconds(cache) * 1e6)
    us, kus = statistics.median(ts[2:] or ts), statistics.median(ks[2:] or ks)
    kb = 8 * L * 128 * 2
    print(f"bos_mass L={L}: call {us:.1f} us, kernels {kus:.1f} us = {kb / kus / 1e3:.1f} GB/s")
