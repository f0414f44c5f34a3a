"""Multi-GPU partitioning of the decode step.

Two ways to use N GPUs of one node, one process per GPU:

* KV-head (unit) sharding — units (seq, kv_head) are independent
  (SPEC.md:336): rank k owns a contiguous range of units and the query heads
  that read them.  No collective on the step path.  `unit_shard` gives the
  range; each rank simply builds its engine over its own heads.

* Sequence sharding — for 512K+ contexts every rank owns the token range
  `split_ranges(L, N)[rank]` (the reference's even-remainder rule,
  attention.cpp:185-202) of every KV group.  Anchors (token 0's key and norm)
  are replicated to every rank, so each rank computes the identical route
  bitmap with tau(L_global).  A rank's engine writes one un-normalised LSE
  partial per (unit, head); the N partials are all-gathered (NCCL over NVLink,
  33 KB per rank for the 70B shape) and LSE-merged on device
  (merge_partials, attention.cpp:159-183).

torch.distributed is the plumbing (process group, NCCL all-gather on the
engine's stream); the math runs in the engine's CUDA kernels.
"""
from __future__ import annotations

from typing import List, Tuple


def split_ranges(length: int, n: int) -> List[Tuple[int, int]]:
    """attention.cpp:185-202 (host integer logic, also usable without a GPU)."""
    if n <= 0 or n > length:
        raise ValueError(f"num_splits must be in [1, len], got {n} for len {length}")
    base, rem = divmod(length, n)
    out, start = [], 0
    for c in range(n):
        sz = base + (1 if c < rem else 0)
        out.append((start, start + sz))
        start += sz
    return out


def sequence_shard(length: int, world: int, rank: int) -> Tuple[int, int]:
    return split_ranges(length, world)[rank]


def unit_shard(num_units: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous (seq, kv_head) unit range owned by `rank` (KV-head sharding)."""
    return split_ranges(num_units, world)[rank] if num_units >= world else (
        (rank, rank + 1) if rank < num_units else (num_units, num_units))


def build_sequence_shard(P, spec, rank: int, world: int, device: int):
    """Engine holding this rank's token slice of every (layer, kv_head) slot,
    with the global token-0 anchor installed (replicated metadata)."""
    lo, hi = sequence_shard(spec.length, world, rank)
    cache = P.KvCache(P.CacheConfig(spec.num_layers, spec.num_q_heads, spec.num_kv_heads,
                                    spec.head_dim, hi - lo, spec.num_seqs), device=device)
    for s in range(spec.num_seqs):
        for g in range(spec.num_kv_heads):
            k0, v0 = spec.first_rows(s, g)
            kk, kv = spec.slot_keys(s, g)
            if lo == 0:
                cache.append(spec.layer, g, k0, v0, seq=s)
                if hi > 1:
                    cache.append_synthetic(spec.layer, g, kk, kv, hi - 1, seq=s, global_row0=1)
            else:
                cache.append_synthetic(spec.layer, g, kk, kv, hi - lo, seq=s, global_row0=lo)
                cache.set_anchor(spec.layer, g, k0, anchor_norm(k0), seq=s)
    return cache, (lo, hi)


def anchor_norm(k0) -> float:
    """kv_cache.cpp:19-23,76: (float) sqrt(sum (double) k^2), index order."""
    import math

    import numpy as np

    s = 0.0
    for x in np.asarray(k0, dtype=np.float32).tolist():
        s += x * x
    return float(np.float32(math.sqrt(s)))


class PeerMerge:
    """The fused alternative to all-gather + combine: each rank's step kernel
    writes its LSE partials straight into every rank's exchange block (CUDA IPC
    mappings over NVLink) and merges all ranks' partials itself.  Set up once
    per engine; then `step` is one kernel launch per rank per step.

    One process per rank: PeerMerge(P, cache, world, rank, dist, torch) exchanges
    the blocks' CUDA IPC handles over the process group.  Ranks in one process
    (tests): peer_merge_in_process(P, caches)."""

    def __init__(self, P, cache, world: int, rank: int, dist=None, torch=None):
        import ctypes as C

        from ._abi import check, lib

        self.P, self.cache, self.world = P, cache, world
        nbytes = C.c_size_t()
        check(lib().sinkr_peer_setup(cache.handle, world, rank, C.byref(nbytes)))
        self.block = lib().sinkr_peer_block(cache.handle)
        if dist is not None:
            h = (C.c_uint8 * 64)()
            check(lib().sinkr_peer_ipc_handle(cache.handle, h))
            dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
            mine = torch.tensor(list(bytes(h)), dtype=torch.uint8, device=dev)
            parts = [torch.empty(64, dtype=torch.uint8, device=dev) for _ in range(world)]
            dist.all_gather(parts, mine)
            allh = torch.cat(parts)
            buf = (C.c_uint8 * (world * 64))(*allh.cpu().tolist())
            check(lib().sinkr_peer_open(cache.handle, buf))

    def connect_local(self, blocks) -> None:
        import ctypes as C

        from ._abi import check, lib

        arr = (C.c_void_p * self.world)(*blocks)
        check(lib().sinkr_peer_set_blocks(self.cache.handle, arr))

    def step(self, dq, dout, cfg, opts, layer: int = 0):
        self.P.routed_decode_peer_async(dq.data_ptr(), layer, self.cache, cfg, opts, dout.data_ptr())

    def host_runner(self, cfg, opts, layer: int = 0):
        """Blocking host-buffer form (sinkr_routed_decode_peer) over the
        engine's pinned step buffers: fill `.queries`, call, read `.out`."""
        import ctypes as C

        from ._abi import check, lib

        r = self.P.StepRunner(self.cache, cfg, opts, layer, pinned_io=True)
        fn = lib().sinkr_routed_decode_peer
        h, _, lay, c, o, out, groups, hs, ctr = r._args

        def call():
            rc = fn(h, r.queries.ctypes.data, lay, c, o, out, groups, hs, ctr)
            if rc:
                check(rc)
            return r.out

        r.call = call
        return r


def peer_merge_in_process(P, caches):
    """Peer merge between engines of one process (same or different GPUs)."""
    world = len(caches)
    pms = [PeerMerge(P, c, world, k) for k, c in enumerate(caches)]
    for pm in pms:
        pm.connect_local([x.block for x in pms])
    return pms


def sharded_step(P, torch, dist, cache, cfg, opts, dq, partial, gathered, dout, world: int):
    """One sequence-sharded decode step on this rank's engine stream."""
    P.decode_rank_partial_async(dq.data_ptr(), 0, cache, cfg, opts, partial.data_ptr())
    stream = torch.cuda.ExternalStream(cache.stream)
    with torch.cuda.stream(stream):
        dist.all_gather_into_tensor(gathered, partial)
    P.merge_rank_partials_async(cache, gathered.data_ptr(), world, dout.data_ptr())


def _gate(torch, stream, ms: float = 2.0):
    """Hold the stream in a short spin kernel while the host enqueues a timed
    sequence (host launch latency then never lands inside a timed step)."""
    with torch.cuda.stream(stream):
        torch.cuda._sleep(int(ms * 2.0e6))


def _peer_self_check(P, torch, dist, pm, cache, cfg, opts, dq, partial, gathered, world):
    """One fused peer-merge step against one all-gather + combine step on the
    same inputs, on every rank: the fused path is used only if every rank
    agrees (outputs within 1e-5, no step-kernel error such as the peer
    watchdog).  Returns None when it passed, else the reason."""
    why = None
    try:
        a = torch.empty_like(dq)
        b = torch.empty_like(dq)
        a.fill_(float("nan"))
        pm.step(dq, a, cfg, opts)
        torch.cuda.synchronize()
        P.fetch_step_info(cache)  # raises on a step-kernel error (peer watchdog)
        sharded_step(P, torch, dist, cache, cfg, opts, dq, partial, gathered, b, world)
        torch.cuda.synchronize()
        err = (a - b).abs().max().item()
        if not err <= 1e-5:  # NaN fails too
            why = f"self-check: fused peer merge differs from all-gather + combine by {err:.3e}"
    except Exception as ex:  # noqa: BLE001 -- reported in the bench line
        why = f"self-check: {type(ex).__name__}: {ex}"
    ok = torch.tensor([0 if why else 1], device="cuda")
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if why is None and int(ok.item()) == 0:
        why = "self-check failed on another rank"
    return why


def time_sequence_sharded(P, torch, dist, spec, routed_cfg, dense_cfg, args, rank, world, dev,
                          clock_sampler=None, e2e=True):
    """Strong-scaling timing of one sequence-sharded workload: routed and dense
    back-to-back steps on the product path (fused peer merge when every rank
    passes the self-check, else NCCL all-gather + combine), the all-gather path
    beside it, and the host-buffer e2e.  Every number is the max over ranks."""
    import statistics
    import time

    cache, (lo, hi) = build_sequence_shard(P, spec, rank, world, dev)
    P.set_timing(cache, False)
    opts = P.EngineOptions(global_context_len=spec.length)
    q_host = torch.from_numpy(spec.queries()[0]).pin_memory()
    dq = q_host.cuda()
    dout = torch.empty_like(dq)
    out_host = torch.empty_like(q_host).pin_memory()
    nf = P.rank_partial_floats(cache)
    partial = torch.empty(nf, dtype=torch.float32, device="cuda")
    gathered = torch.empty(world * nf, dtype=torch.float32, device="cuda")
    stream = torch.cuda.ExternalStream(cache.stream)
    # the merge fused into the step kernel over peer memory; NCCL all-gather +
    # combine kernel when peer mappings are unavailable or the self-check fails
    pm, peer_err = None, None
    try:
        pm = PeerMerge(P, cache, world, rank, dist, torch)
    except Exception as ex:  # no P2P / IPC on this node
        peer_err = f"{type(ex).__name__}: {ex}"
    ok = torch.tensor([0 if pm is None else 1], device="cuda")
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if int(ok.item()) == 0:
        pm = None
        peer_err = peer_err or "peer mapping failed on another rank"
    if pm is not None:
        peer_err = _peer_self_check(P, torch, dist, pm, cache, routed_cfg, opts, dq, partial,
                                    gathered, world)
        if peer_err:
            pm = None

    def step(cfg):
        if pm is not None:
            pm.step(dq, dout, cfg, opts)
        else:
            sharded_step(P, torch, dist, cache, cfg, opts, dq, partial, gathered, dout, world)

    def maxed(x: float) -> float:
        t = torch.tensor([x], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    res = {}
    clocks = None
    n_act = 0
    for name, cfg in (("routed", routed_cfg), ("dense", dense_cfg)):
        for _ in range(max(3, args.warmup)):
            step(cfg)
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        sampler = clock_sampler(dev) if (clock_sampler and name == "routed") else None
        if sampler:
            sampler.__enter__()
        _gate(torch, stream)
        e0.record(stream)
        for _ in range(args.steps):
            step(cfg)
        e1.record(stream)
        torch.cuda.synchronize()
        if sampler:
            sampler.__exit__(None, None, None)
            clocks = sampler.summary()
        dist.barrier()
        res[name] = maxed(e0.elapsed_time(e1) / args.steps)
        if name == "routed":
            n_act = P.fetch_step_info(cache).counters.groups_active

    # a rank's Active KV fits in L2 at high N (8-way at 512K: 96 MiB of the
    # 126 MB L2): then back-to-back steps could re-read it from L2, so each
    # step is timed alone behind a 256 MiB L2 flush (median of per-step event
    # pairs, max over ranks) and that is the reported value
    kv_rank_routed = n_act * 2 * (hi - lo) * spec.head_dim * 2
    flushed = None
    if kv_rank_routed < 2 * 126 * 1024 * 1024:
        flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
        flushed = {}
        for name, cfg in (("routed", routed_cfg), ("dense", dense_cfg)):
            step(cfg)
            torch.cuda.synchronize()
            dist.barrier()
            evs = []
            for _ in range(max(args.steps, 10)):
                with torch.cuda.stream(stream):
                    flush.sum()  # read-only flush: evicts L2 without dirty write-backs
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                step(cfg)
                e1.record(stream)
                evs.append((e0, e1))
            torch.cuda.synchronize()
            flushed[name] = maxed(statistics.median(a.elapsed_time(b) for a, b in evs))
        del flush
        res["back_to_back_routed"], res["back_to_back_dense"] = res["routed"], res["dense"]
        res["routed"], res["dense"] = flushed["routed"], flushed["dense"]

    # the all-gather + combine path beside it (same steps, same clock)
    nccl_us = None
    if pm is not None:
        for _ in range(3):
            sharded_step(P, torch, dist, cache, routed_cfg, opts, dq, partial, gathered, dout, world)
        torch.cuda.synchronize()
        dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        _gate(torch, stream)
        e0.record(stream)
        for _ in range(args.steps):
            sharded_step(P, torch, dist, cache, routed_cfg, opts, dq, partial, gathered, dout, world)
        e1.record(stream)
        torch.cuda.synchronize()
        nccl_us = maxed(e0.elapsed_time(e1) / args.steps) * 1e3

    out = {"routed_ms": res["routed"], "dense_ms": res["dense"], "groups_active": n_act,
           "l2_flushed": flushed is not None,
           "back_to_back_ms": ({"routed": res["back_to_back_routed"],
                                "dense": res["back_to_back_dense"]} if flushed else None),
           "lo": lo, "hi": hi, "peer": pm is not None, "peer_err": peer_err, "clocks": clocks,
           "allgather_us": nccl_us, "partial_bytes_per_rank": nf * 4}
    if e2e:
        # e2e: host queries in (pinned H2D), sharded step, host outputs out, per
        # step; with the fused peer merge, the blocking host-buffer call over the
        # engine's pinned step buffers (one graph: upload + step, outputs
        # zero-copy, completion word)
        e2e_peer_us = None
        if pm is not None:
            hr = pm.host_runner(routed_cfg, opts)
            hr.queries[...] = q_host.numpy().reshape(hr.queries.shape)
            for _ in range(3):
                hr.call()
            dist.barrier()
            ts = []
            for _ in range(max(args.steps, 50)):
                t0 = time.perf_counter()
                hr.call()
                ts.append((time.perf_counter() - t0) * 1e6)
            e2e_peer_us = maxed(statistics.median(ts))
        for _ in range(2):
            with torch.cuda.stream(stream):
                dq.copy_(q_host, non_blocking=True)
            step(routed_cfg)
            with torch.cuda.stream(stream):
                out_host.copy_(dout, non_blocking=True)
            stream.synchronize()
        dist.barrier()
        ts = []
        for _ in range(max(args.steps, 50)):  # each step timed alone, median
            t0 = time.perf_counter()
            with torch.cuda.stream(stream):
                dq.copy_(q_host, non_blocking=True)
            step(routed_cfg)
            with torch.cuda.stream(stream):
                out_host.copy_(dout, non_blocking=True)
            stream.synchronize()
            ts.append((time.perf_counter() - t0) * 1e6)
        e2e_copy_us = maxed(statistics.median(ts))
        h2d_bytes, d2h_bytes = int(q_host.numel() * 4), int(out_host.numel() * 4)
        if pm is not None:  # the peer call moves the staged input block and the result block
            h2d_bytes, d2h_bytes = cache.step_io_bytes()
        out.update(e2e_us=e2e_peer_us if pm is not None else e2e_copy_us, e2e_copy_us=e2e_copy_us,
                   h2d_bytes=h2d_bytes, d2h_bytes=d2h_bytes)
    # pinned host blocks record an event on the engine stream when freed: free
    # them while the engine (and its stream) is alive
    stream.synchronize()
    del q_host, out_host
    cache.close()
    return out


def bench_sequence_sharded(P, torch, dist, spec, routed_cfg, dense_cfg, args, rank, world, dev,
                           peak_gbs=None, peak_src="", clock_sampler=None, config=None):
    """bench.py's N>1 path (and --force-sharded at N=1): strong scaling of the
    headline workload, every number the max over ranks; other_configs adds
    BASELINE configs[3] (Llama-3.1-70B shape, 512K, sequence-sharded -- the
    north star's 8-way case) and configs[2] (Yi-9B, B=16, unit-sharded)."""
    import json

    t = time_sequence_sharded(P, torch, dist, spec, routed_cfg, dense_cfg, args, rank, world, dev,
                              clock_sampler=clock_sampler)
    pm = t["peer"]
    n_act, lo, hi = t["groups_active"], t["lo"], t["hi"]
    kv_total = n_act * 2 * spec.length * spec.head_dim * 2          # all ranks
    kv_rank = n_act * 2 * (hi - lo) * spec.head_dim * 2             # this rank
    routed_ms, dense_ms = t["routed_ms"], t["dense_ms"]
    per_gpu_gbs = kv_rank / (routed_ms * 1e-3) / 1e9  # the step time is already max-over-ranks
    # `config` is bench.py's workload dict, printed identically by the
    # reference arm; how this arm shards it goes under "sharding"
    cfg_dict = dict(config or {
        "workload": f"llama3.1-8b-attn L={spec.length} B=1 routed={spec.sink_fraction}",
        "parallelism": f"sequence-shard x{world}"})
    shard_info = {
        "merge": ("LSE merge fused into the step kernel over peer memory (NVLink)" if pm else
                  "NCCL all-gather + combine kernel"),
        "tokens_per_rank": hi - lo,
        "l2": ("a rank's Active KV fits in 2x L2: every step timed alone behind a 256 MiB "
               "L2 flush (median, max over ranks); back_to_back_us beside it"
               if t["l2_flushed"] else
               "a rank's Active KV is larger than 2x L2: back-to-back steps, no flush"),
        "back_to_back_us": ({k: round(v * 1e3, 2) for k, v in t["back_to_back_ms"].items()}
                            if t["back_to_back_ms"] else None)}
    line = {
        "metric": ("decode-attn \u00b5s/step & KV GB/s (% HBM peak) at 512K; "
                   "speedup vs own dense path"),
        "value": round(routed_ms * 1e3, 2), "unit": "us/step", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(routed_ms, 5),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic planted-sink KV (device generator, seeded); fp32 queries",
        "config": cfg_dict,
        "sharding": shard_info,
        "dense_us_per_step": round(dense_ms * 1e3, 2),
        "speedup_vs_dense": round(dense_ms / routed_ms, 3),
        "kv_gbs_routed_step": round(kv_total / (routed_ms * 1e-3) / 1e9, 1),
        "roofline": {"bound": "hbm", "achieved": round(per_gpu_gbs, 1),
                     "peak": peak_gbs, "unit": "GB/s",
                     "frac": round(per_gpu_gbs / peak_gbs, 4) if peak_gbs else None,
                     "traffic": None,
                     "kernel": ("step_kernel<128> with the rank merge fused over peer memory (mode 3)"
                                if pm else
                                "step_kernel<128> rank partial (per GPU) + NCCL all-gather + combine_kernel"),
                     "achieved_def": "this rank's Active K+V bytes / max-over-ranks step time",
                     "peak_source": peak_src},
        "e2e": {"value": round(t["e2e_us"], 2), "unit": "us/step",
                "h2d_bytes_per_step": t["h2d_bytes"],
                "d2h_bytes_per_step": t["d2h_bytes"],
                "method": ("blocking sinkr_routed_decode_peer over the engine's pinned step "
                           "buffers, per-step median, max over ranks" if pm else
                           "torch pinned copies around the all-gather step, per-step median, "
                           "max over ranks"),
                "torch_copies_us": round(t["e2e_copy_us"], 2)},
        "gpu_launches": (1 if pm else 2) * args.steps,  # ours only (NCCL's not counted)
        "allgather_combine_us_per_step": (round(t["allgather_us"], 2)
                                          if t["allgather_us"] is not None else None),
        "peer_merge_unavailable": t["peer_err"],
        "clocks": t["clocks"],
        "note": json.dumps({"partial_bytes_per_rank": t["partial_bytes_per_rank"]}),
    }
    line["other_configs"] = [
        bench_c4_sequence_sharded(P, torch, dist, spec_cls=type(spec), args=args, rank=rank,
                                  world=world, dev=dev, routed_cfg=routed_cfg, dense_cfg=dense_cfg,
                                  peak_gbs=peak_gbs),
        bench_unit_sharded(P, torch, dist, spec_cls=type(spec), args=args, rank=rank, world=world,
                           dev=dev, routed_cfg=routed_cfg, dense_cfg=dense_cfg)]
    return line


def bench_c4_sequence_sharded(P, torch, dist, spec_cls, args, rank, world, dev, routed_cfg,
                              dense_cfg, peak_gbs=None):
    """BASELINE configs[3]: Llama-3.1-70B attention shape (64 q / 8 KV heads,
    r = 8) at L = 524,288, sequence-sharded over the ranks with the product
    merge path; per-GPU roofline fraction of this rank's Active K+V stream."""
    spec = spec_cls(num_q_heads=64, num_kv_heads=8, head_dim=128, length=524288,
                    sink_fraction=args.sink_fraction, seed=args.seed + 70)
    t = time_sequence_sharded(P, torch, dist, spec, routed_cfg, dense_cfg, args, rank, world, dev,
                              e2e=False)
    n_act, lo, hi = t["groups_active"], t["lo"], t["hi"]
    kv_rank = n_act * 2 * (hi - lo) * 128 * 2
    gbs = kv_rank / (t["routed_ms"] * 1e-3) / 1e9
    return {"config": f"C4 llama3.1-70b-attn L=524288 B=1, sequence-sharded x{world}",
            "merge": "fused peer merge (mode 3)" if t["peer"] else "NCCL all-gather + combine",
            "peer_merge_unavailable": t["peer_err"],
            "groups_active": n_act, "groups_total": 8, "tokens_per_rank": hi - lo,
            "routed_us": round(t["routed_ms"] * 1e3, 2), "dense_us": round(t["dense_ms"] * 1e3, 2),
            "speedup_vs_dense": round(t["dense_ms"] / t["routed_ms"], 3),
            "per_gpu_kv_gbs_routed": round(gbs, 1),
            "per_gpu_roofline_frac": round(gbs / peak_gbs, 4) if peak_gbs else None,
            "allgather_combine_us": (round(t["allgather_us"], 2)
                                     if t["allgather_us"] is not None else None)}


def bench_unit_sharded(P, torch, dist, spec_cls, args, rank, world, dev, routed_cfg, dense_cfg):
    """BASELINE config 3 (Yi-9B-200K shape, 32 q / 4 KV heads, L = 204,800,
    B = 16) with (seq, kv_head) units sharded across the ranks: rank k owns
    sequences [k*B/N, (k+1)*B/N) -- all their units -- and steps them with no
    collective at all.  Back-to-back steps, max over ranks."""
    B = 16
    if B % world:
        return {"config": "C3 yi-9b-200k unit-sharded", "skipped": f"B={B} not divisible by {world}"}
    nb = B // world
    spec = spec_cls(num_q_heads=32, num_kv_heads=4, head_dim=128, length=204800, num_seqs=nb,
                    sink_fraction=args.sink_fraction, seed=args.seed + 1000 + rank)
    cache = P.KvCache(P.CacheConfig(1, 32, 4, 128, spec.length, nb), device=dev)
    spec.fill(cache)
    P.set_timing(cache, False)
    dq = torch.from_numpy(spec.queries()).cuda()
    dout = torch.empty_like(dq)
    stream = torch.cuda.ExternalStream(cache.stream)
    res = {}
    for name, cfg in (("routed", routed_cfg), ("dense", dense_cfg)):
        for _ in range(max(3, args.warmup)):
            P.routed_decode_async(dq.data_ptr(), 0, cache, cfg, d_outputs=dout.data_ptr())
        torch.cuda.synchronize()
        dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        _gate(torch, stream)
        e0.record(stream)
        for _ in range(args.steps):
            P.routed_decode_async(dq.data_ptr(), 0, cache, cfg, d_outputs=dout.data_ptr())
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res[name] = float(t.item()) * 1e3
        if name == "routed":
            n_act = torch.tensor([P.fetch_step_info(cache).counters.groups_active], device="cuda")
            dist.all_reduce(n_act)
    cache.close()
    kv = int(n_act.item()) * 2 * spec.length * 128 * 2
    return {"config": f"C3 yi-9b-200k-attn L=204800 B={B}, (seq, kv_head) units sharded x{world}, "
                      "no collective",
            "groups_active": int(n_act.item()), "groups_total": B * 4,
            "routed_us": round(res["routed"], 2), "dense_us": round(res["dense"], 2),
            "speedup_vs_dense": round(res["dense"] / res["routed"], 3),
            "kv_gbs_routed": round(kv / (res["routed"] * 1e-6) / 1e9, 1),
            "sequences_per_s_routed": round(B / (res["routed"] * 1e-6), 1)}
