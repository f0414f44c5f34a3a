"""Sequence-sharded decode, N shards simulated on one GPU: each shard engine
holds its token slice + the replicated anchor, writes its LSE partial, the
partials are concatenated (what NCCL all-gather produces) and merged on device.
Must equal the single-engine step: bitmap identical, outputs within tolerance.
Also KV-head (unit) sharding: disjoint head ranges reproduce the full step."""
import numpy as np
import pytest
import torch

import oracle
import paper_2604_16883_b200 as P
from paper_2604_16883_b200 import sharding
from paper_2604_16883_b200.workload import WorkloadSpec

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,L,hq,hkv", [(2, 4096, 32, 8), (4, 10001, 64, 8), (8, 65536, 64, 8)])
def test_sequence_shards_match_single(world, L, hq, hkv):
    spec = WorkloadSpec(num_q_heads=hq, num_kv_heads=hkv, head_dim=128, length=L,
                        sink_fraction=0.625, seed=world)
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
    q = spec.queries()[0]
    with P.KvCache(P.CacheConfig(1, hq, hkv, 128, L)) as full:
        spec.fill(full)
        ref = P.routed_decode_step(q, 0, full, cfg)
    dq = torch.from_numpy(q).cuda()
    parts, caches = [], []
    opts = P.EngineOptions(global_context_len=L)
    for rank in range(world):
        cache, (lo, hi) = sharding.build_sequence_shard(P, spec, rank, world, 0)
        caches.append(cache)
        part = torch.empty(cache.rank_partial_floats(), dtype=torch.float32, device="cuda")
        P.decode_rank_partial_async(dq.data_ptr(), 0, cache, cfg, opts, part.data_ptr())
        torch.cuda.synchronize()
        info = P.fetch_step_info(cache)
        assert np.array_equal(info.route_bitmap, ref.route_bitmap)
        for g, gr in zip(info.groups, ref.groups):
            assert g.decision.group_score == gr.decision.group_score
            assert g.tokens_loaded == (0 if gr.decision.sink else hi - lo)
        parts.append(part)
    gathered = torch.cat(parts)
    out = torch.zeros_like(dq)
    P.merge_rank_partials_async(caches[0], gathered.data_ptr(), world, out.data_ptr())
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    assert np.abs(o - ref.outputs).max() <= 2e-3
    assert np.linalg.norm(o - ref.outputs) <= 1e-3 * np.linalg.norm(ref.outputs)
    r = hq // hkv
    for gi, g in enumerate(ref.groups):
        if g.decision.sink:
            assert not np.any(o[gi * r:(gi + 1) * r].view(np.uint32))
    for c in caches:
        c.close()


def test_unit_shards_match_single():
    """KV-head sharding: rank k owns kv heads [a, b) and their query heads."""
    hq, hkv, L, world = 32, 8, 3000, 4
    spec = WorkloadSpec(num_q_heads=hq, num_kv_heads=hkv, head_dim=128, length=L,
                        sink_fraction=0.5, seed=9)
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
    q = spec.queries()[0]
    with P.KvCache(P.CacheConfig(1, hq, hkv, 128, L)) as full:
        spec.fill(full)
        ref = P.routed_decode_step(q, 0, full, cfg)
        r = hq // hkv
        for rank in range(world):
            a, b = sharding.unit_shard(hkv, world, rank)
            with P.KvCache(P.CacheConfig(1, (b - a) * r, b - a, 128, L)) as part:
                for g in range(a, b):
                    k, v = full.historical(0, g, 0, L)
                    part.append(0, g - a, k, v)
                res = P.routed_decode_step(q[a * r:b * r], 0, part, cfg)
                assert np.array_equal(res.route_bitmap, ref.route_bitmap[a:b])
                np.testing.assert_allclose(res.outputs, ref.outputs[a * r:b * r], atol=1e-6)


def _one_gpu_peer_setup(P, caches):
    return sharding.peer_merge_in_process(P, caches)


def test_peer_merge_world1_matches_fused_step():
    """The fused peer-merge step at world 1 (the kernel writes its partial into
    its own exchange block as tagged LL words, merges) equals the plain step,
    over several steps (step-parity buffers, step tags advancing)."""
    spec = WorkloadSpec(length=40000, sink_fraction=0.5, seed=3)
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
    with P.KvCache(P.CacheConfig(1, 32, 8, 128, spec.length)) as cache:
        spec.fill(cache)
        q = torch.from_numpy(spec.queries()[0]).cuda()
        ref = torch.empty_like(q)
        P.routed_decode_async(q.data_ptr(), 0, cache, cfg, d_outputs=ref.data_ptr())
        torch.cuda.synchronize()
        (pm,) = _one_gpu_peer_setup(P, [cache])
        out = torch.empty_like(q)
        for _ in range(5):
            out.fill_(float("nan"))
            pm.step(q, out, cfg, P.EngineOptions())
            torch.cuda.synchronize()
            assert torch.equal(out, ref) or (out - ref).abs().max().item() <= 1e-6
        info = P.fetch_step_info(cache)
        assert info.counters.groups_skipped == 4


@pytest.mark.parametrize("world", [2])
def test_peer_merge_two_ranks_on_one_gpu(world, monkeypatch):
    """Two sequence-shard engines on one GPU, each with half the SMs
    (SINKR_DEBUG_GRID), exchanging partials through each other's blocks inside
    their step kernels: both produce the single-engine step's outputs."""
    from paper_2604_16883_b200 import sharding

    monkeypatch.setenv("SINKR_DEBUG_GRID", "74")
    L = 65536
    spec = WorkloadSpec(length=L, sink_fraction=0.625, seed=8)
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
    q = torch.from_numpy(spec.queries()[0]).cuda()
    with P.KvCache(P.CacheConfig(1, 32, 8, 128, L)) as full:
        spec.fill(full)
        ref = torch.empty_like(q)
        P.routed_decode_async(q.data_ptr(), 0, full, cfg, d_outputs=ref.data_ptr())
        torch.cuda.synchronize()
    shards = [sharding.build_sequence_shard(P, spec, k, world, 0)[0] for k in range(world)]
    pms = _one_gpu_peer_setup(P, shards)
    opts = P.EngineOptions(global_context_len=L)
    outs = [torch.empty_like(q) for _ in range(world)]
    for _ in range(3):
        for pm, o in zip(pms, outs):
            o.fill_(float("nan"))
            pm.step(q, o, cfg, opts)
        torch.cuda.synchronize()
        for o in outs:
            assert (o - ref).abs().max().item() <= 2e-3
            assert torch.linalg.norm(o - ref).item() <= 1e-3 * torch.linalg.norm(ref).item()
    for s_ in shards:
        info = P.fetch_step_info(s_)
        assert info.counters.groups_skipped == 5
        s_.close()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_peer_merge_world_n_vs_reference(world, monkeypatch, oracle_libs):
    """The DEFAULT multi-GPU product path -- the rank merge fused into the step
    kernel over peer memory (mode 3) -- at world 2/4/8, against the COMPILED
    REFERENCE's unsharded routed_decode_step.  BASELINE configs[3] shape
    (Llama-3.1-70B: 64 q / 8 KV heads, r = 8), 65,536 tokens per rank (world 8
    = the 512K config); the ranks are `world` engines on one GPU, each with
    floor(#SMs / world) CTAs, so their cooperative step kernels run side by
    side and exchange partials through each other's blocks.  Three steps
    (both parities of the exchange slots).  Bar: bitmap and group-score bytes
    equal, per-group rows summed over ranks equal to the reference's
    kv_floats, max-abs <= 2e-3 AND rel-L2 <= 1e-3 on every rank, Sink rows
    bitwise zero."""
    ref_lib, orc = oracle_libs
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    monkeypatch.setenv("SINKR_DEBUG_GRID", str(sms // world))
    per_rank = 65536
    L = per_rank * world
    spec = WorkloadSpec(num_q_heads=64, num_kv_heads=8, head_dim=128, length=L,
                        sink_fraction=0.625, seed=300 + world)
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
    q = spec.queries()[0]
    dq = torch.from_numpy(q).cuda()
    shards = [sharding.build_sequence_shard(P, spec, k, world, 0) for k in range(world)]
    caches = [c for c, _ in shards]
    pms = _one_gpu_peer_setup(P, caches)
    opts = P.EngineOptions(global_context_len=L)
    outs = [torch.empty_like(dq) for _ in range(world)]
    got = []
    for _ in range(3):
        for pm, o in zip(pms, outs):
            o.fill_(float("nan"))
            pm.step(dq, o, cfg, opts)
        torch.cuda.synchronize()
        got.append([o.cpu().numpy() for o in outs])
    infos = [P.fetch_step_info(c) for c in caches]
    kv_sum = np.zeros(spec.num_kv_heads, dtype=np.uint64)
    for info, (_, (lo, hi)) in zip(infos, shards):
        assert np.array_equal(info.route_bitmap, infos[0].route_bitmap)
        kv_sum += np.array([g.kv_floats_loaded for g in info.groups], dtype=np.uint64)
        for g in info.groups:
            assert g.tokens_loaded == (0 if g.decision.sink else hi - lo)
    # the unsharded reference over exactly the tokens the shards hold
    r = spec.r
    if ref_lib is not None:
        rc = oracle.RefCache(ref_lib, 1, 64, 8, 128, L)
        for g in range(spec.num_kv_heads):
            ks, vs = [], []
            for c, (lo, hi) in shards:
                k, v = c.historical(0, g, 0, hi - lo)
                ks.append(k)
                vs.append(v)
            rc.append_rows(0, g, np.concatenate(ks), np.concatenate(vs))
            del ks, vs
        ref = rc.routed_decode_step(q, 0, oracle.Profile.constant(0.5), excluded=(), workers=16)
        rc.close()
    else:  # no compiled reference on this host: the pinned C restatement
        k = np.stack([np.concatenate([c.historical(0, g, 0, hi - lo)[0] for c, (lo, hi) in shards])
                      for g in range(8)])
        v = np.stack([np.concatenate([c.historical(0, g, 0, hi - lo)[1] for c, (lo, hi) in shards])
                      for g in range(8)])
        k0 = np.ascontiguousarray(k[:, 0])
        ref = orc.routed_decode_step(k, v, k0, [orc.anchor_norm(x) for x in k0], q, 0,
                                     oracle.Profile.constant(0.5), excluded=(), threads=16)
        del k, v
    assert np.array_equal(infos[0].route_bitmap.astype(np.int32), ref.sink.astype(np.int32))
    gs = np.array([g.decision.group_score for g in infos[0].groups])
    assert gs.tobytes() == np.asarray(ref.group_scores).tobytes()
    assert list(kv_sum) == [int(x) for x in ref.group_kv_floats]
    ro = np.asarray(ref.outputs).reshape(64, 128)
    for step_outs in got:
        for o in step_outs:
            assert np.abs(o - ro).max() <= 2e-3
            assert np.linalg.norm(o - ro) <= 1e-3 * np.linalg.norm(ro)
            for gi in range(8):
                if ref.sink[gi]:
                    assert not np.any(o[gi * r:(gi + 1) * r].view(np.uint32))
    for c in caches:
        c.close()


def test_peer_merge_across_processes_ipc():
    """The fused peer merge between two PROCESSES (one engine each, CUDA IPC
    mappings of each other's exchange blocks, gloo for the handle exchange), on
    one GPU with half the SMs each: both ranks reproduce the unsharded step."""
    import os
    import socket
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    env = dict(os.environ, SINKR_DEBUG_GRID="74")
    res = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                          "--master-port", str(port), os.path.join(root, "scripts", "ipc_peer_check.py")],
                         capture_output=True, text=True, timeout=240, env=env, cwd=root)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]
    assert "rank 0 ok" in res.stdout and "rank 1 ok" in res.stdout


@pytest.mark.parametrize("timing", [False, True])
def test_peer_host_buffer_step_world1(timing):
    """sinkr_routed_decode_peer (host buffers, zero-copy outputs) at world 1
    returns the plain step's outputs and routing record, repeatedly.  With
    timing off the call is the single captured graph (H2D + mode-3 step,
    outputs into mapped host memory) that the sharded bench's e2e measures;
    plain steps and device-buffer peer steps are interleaved between host
    calls, so graph keying and the device-side peer epoch / arrival base are
    exercised across all three entry points."""
    spec = WorkloadSpec(length=30000, sink_fraction=0.5, seed=8)
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
    with P.KvCache(P.CacheConfig(1, 32, 8, 128, spec.length)) as cache:
        spec.fill(cache)
        P.set_timing(cache, timing)
        q = spec.queries()[0]
        ref = P.routed_decode_step(q, 0, cache, cfg)
        (pm,) = _one_gpu_peer_setup(P, [cache])
        hr = pm.host_runner(cfg, P.EngineOptions())
        hr.queries[...] = q.reshape(hr.queries.shape)
        dq = torch.from_numpy(q).cuda()
        dout = torch.empty_like(dq)
        for it in range(6):
            out = hr.call()
            assert np.abs(out.reshape(ref.outputs.shape) - ref.outputs).max() <= 1e-6, it
            res = hr.result()
            assert [g.decision.sink for g in res.groups] == [g.decision.sink for g in ref.groups]
            assert res.counters.kv_floats_loaded == ref.counters.kv_floats_loaded
            if it % 2 == 0:  # a plain host step between peer calls
                again = P.routed_decode_step(q, 0, cache, cfg)
                assert np.abs(again.outputs - ref.outputs).max() <= 1e-6
            else:  # a device-buffer peer step between host peer calls
                dout.fill_(float("nan"))
                pm.step(dq, dout, cfg, P.EngineOptions())
                torch.cuda.synchronize()
                assert (dout.cpu().numpy() - ref.outputs).__abs__().max() <= 1e-6


def test_peer_merge_watchdog_and_reconnect(monkeypatch):
    """A rank that never delivers: the other rank's fused-merge step ends with
    the peer-merge watchdog error after ~2 s (NaN in the outputs it owns,
    never a hang), the exchange then refuses steps, and after every rank sets
    it up again and reconnects a two-rank step matches the unsharded step."""
    import time

    from paper_2604_16883_b200 import sharding
    from paper_2604_16883_b200._abi import LogicError

    monkeypatch.setenv("SINKR_DEBUG_GRID", "74")
    L = 16384
    spec = WorkloadSpec(length=L, sink_fraction=0.5, seed=9)
    cfg = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())
    q = torch.from_numpy(spec.queries()[0]).cuda()
    with P.KvCache(P.CacheConfig(1, 32, 8, 128, L)) as full:
        spec.fill(full)
        ref = torch.empty_like(q)
        P.routed_decode_async(q.data_ptr(), 0, full, cfg, d_outputs=ref.data_ptr())
        torch.cuda.synchronize()
    shards = [sharding.build_sequence_shard(P, spec, k, 2, 0)[0] for k in range(2)]
    try:
        pms = sharding.peer_merge_in_process(P, shards)
        opts = P.EngineOptions(global_context_len=L)
        out = torch.zeros_like(q)
        t0 = time.time()
        pms[0].step(q, out, cfg, opts)  # rank 1 never steps
        torch.cuda.synchronize()
        assert 1.5 < time.time() - t0 < 60
        with pytest.raises(RuntimeError, match="peer merge watchdog"):
            P.fetch_step_info(shards[0])
        assert torch.isnan(out).any()
        with pytest.raises(LogicError):
            pms[0].step(q, out, cfg, opts)
        pms = sharding.peer_merge_in_process(P, shards)  # every rank: set up again, reconnect
        outs = [torch.empty_like(q) for _ in range(2)]
        for _ in range(2):
            for pm, o in zip(pms, outs):
                pm.step(q, o, cfg, opts)
            torch.cuda.synchronize()
            for o in outs:
                assert (o - ref).abs().max().item() <= 2e-3
    finally:
        for s_ in shards:
            s_.close()
