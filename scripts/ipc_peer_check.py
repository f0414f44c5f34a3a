"""Dev check: the fused peer merge across PROCESSES (CUDA IPC mappings), two
ranks on one GPU (gloo for the handle exchange, SINKR_DEBUG_GRID=74 so both
cooperative kernels fit side by side).  Run:
  SINKR_DEBUG_GRID=74 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/ipc_peer_check.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
import paper_2604_16883_b200 as P
from paper_2604_16883_b200 import sharding
from paper_2604_16883_b200.workload import WorkloadSpec

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
L = 65536
spec = WorkloadSpec(length=L, sink_fraction=0.625, seed=8)
cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
q = torch.from_numpy(spec.queries()[0]).cuda()
ref = None
if rank == 0:
    os.environ.pop("SINKR_DEBUG_GRID", None)
    with P.KvCache(P.CacheConfig(1, 32, 8, 128, L)) as full:
        spec.fill(full)
        ref = torch.empty_like(q)
        P.routed_decode_async(q.data_ptr(), 0, full, cfg, d_outputs=ref.data_ptr())
        torch.cuda.synchronize()
    os.environ["SINKR_DEBUG_GRID"] = "74"
# every rank checks against the unsharded step (computed once, broadcast)
ref_host = ref.cpu() if rank == 0 else torch.empty(q.shape, dtype=torch.float32)
dist.broadcast(ref_host, 0)
ref = ref_host.cuda()
cache, _ = sharding.build_sequence_shard(P, spec, rank, world, 0)
pm = sharding.PeerMerge(P, cache, world, rank, dist, torch)
dist.barrier()
out = torch.empty_like(q)
opts = P.EngineOptions(global_context_len=L)
for it in range(3):
    out.fill_(float("nan"))
    pm.step(q, out, cfg, opts)
    torch.cuda.synchronize()
    info = P.fetch_step_info(cache)  # raises on a step-kernel error (e.g. the 2 s watchdog)
    dist.barrier()
    err = (out - ref).abs().max().item()
    rel = (torch.linalg.norm(out - ref) / torch.linalg.norm(ref)).item()
    print(f"rank {rank} step {it}: max|out-ref| = {err:.3e} rel-L2 = {rel:.3e}", flush=True)
    assert err <= 2e-3 and rel <= 1e-3
print(f"rank {rank} ok", flush=True)
cache.close()
dist.destroy_process_group()
