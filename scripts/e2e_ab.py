"""Dev tool: the C-ABI host-buffer step from a C++ loop (bench-support
timer), median of 400 calls, headline shape at L (default 32K: host costs
dominate).  Run under scripts/ab_libs.sh-style library swaps."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2604_16883_b200 as P
from paper_2604_16883_b200 import build
from paper_2604_16883_b200.workload import WorkloadSpec

L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
spec = WorkloadSpec(length=L, sink_fraction=0.625)
with P.KvCache(P.CacheConfig(1, 32, 8, 128, L)) as cache:
    spec.fill(cache)
    P.set_timing(cache, False)
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
    run = P.StepRunner(cache, cfg, pinned_io=True)
    run.queries[...] = spec.queries()[0]
    timer = C.CDLL(build.BENCH_LIB).sinkr_bench_time_steps
    timer.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t] + [C.c_void_p] * 6 + [C.c_size_t, C.c_void_p]
    h, _, layer, c, o, out, g, hs, ctr = run._args
    us = np.zeros(400)
    timer(h, run.queries.ctypes.data, 0, c, o, out, g, hs, ctr, 50, us.ctypes.data)
    timer(h, run.queries.ctypes.data, 0, c, o, out, g, hs, ctr, 400, us.ctypes.data)
    print(f"L={L} e2e C-ABI median {np.median(us):.2f} us, p10 {np.percentile(us, 10):.2f}")
