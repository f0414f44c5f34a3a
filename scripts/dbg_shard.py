import os, sys, faulthandler
faulthandler.enable()
sys.path.insert(0, os.getcwd())
import torch, torch.distributed as dist
import paper_2604_16883_b200 as P
from paper_2604_16883_b200 import sharding
from paper_2604_16883_b200.workload import WorkloadSpec
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
spec = WorkloadSpec(num_q_heads=32, num_kv_heads=8, head_dim=128, length=int(os.environ.get("LEN", 65536)), sink_fraction=0.625)
print("build", flush=True)
cache, (lo, hi) = sharding.build_sequence_shard(P, spec, 0, 1, 0)
print("built", lo, hi, flush=True)
P.set_timing(cache, False)
opts = P.EngineOptions(global_context_len=spec.length)
q = torch.from_numpy(spec.queries()[0]).pin_memory()
print("pinned", flush=True)
dq = q.cuda(); dout = torch.empty_like(dq)
nf = P.rank_partial_floats(cache)
print("nf", nf, flush=True)
partial = torch.empty(nf, dtype=torch.float32, device="cuda")
gathered = torch.empty(nf, dtype=torch.float32, device="cuda")
cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
P.decode_rank_partial_async(dq.data_ptr(), 0, cache, cfg, opts, partial.data_ptr())
torch.cuda.synchronize(); print("partial ok", flush=True)
sharding.sharded_step(P, torch, dist, cache, cfg, opts, dq, partial, gathered, dout, 1)
torch.cuda.synchronize(); print("step ok", flush=True)
import argparse, bench
args = argparse.Namespace(steps=5, warmup=3)
print("bench fn", flush=True)
res = sharding.bench_sequence_sharded(P, torch, dist, spec, cfg, P.RoutingConfig(profile=P.ThresholdProfile.constant(2.0), excluded_layers=()),
                                      args, 0, 1, 0, peak_gbs=6500.0, peak_src="x",
                                      clock_sampler=bench.ClockSampler if os.environ.get("CLK") else None)
print(res, flush=True)
dist.destroy_process_group()
