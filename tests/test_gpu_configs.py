"""Full-size parity for every BASELINE.json config shape (GPU).

The engine's cache is read back (exact f32 upcast of the stored bf16) and fed to
the C restatement / the compiled reference, so both sides see identical tokens.
Bar: route bitmap, group scores and per-group loaded rows bit-exact; outputs
within max-abs 2e-3, rel-L2 1e-3; Sink rows bitwise zero."""
import zlib

import numpy as np
import pytest
import torch

import oracle
import paper_2604_16883_b200 as P
from paper_2604_16883_b200 import sharding
from paper_2604_16883_b200.workload import WorkloadSpec

pytestmark = pytest.mark.gpu

CFG = P.RoutingConfig(profile=P.ThresholdProfile.constant(0.5), excluded_layers=())


def read_back(cache, spec, seq):
    ks, vs = [], []
    for g in range(spec.num_kv_heads):
        k, v = cache.historical(spec.layer, g, 0, spec.length, seq=seq)
        ks.append(k)
        vs.append(v)
    return np.stack(ks), np.stack(vs)


def check_seq(orc, res_out, groups, spec, seq, q, k, v, kv_floats=None):
    k0 = np.ascontiguousarray(k[:, 0])
    kn = [orc.anchor_norm(k0[g]) for g in range(spec.num_kv_heads)]
    ref = orc.routed_decode_step(k, v, k0, kn, q, spec.layer, oracle.Profile.constant(0.5),
                                 excluded=(), threads=16)
    sink = np.array([g.decision.sink for g in groups], dtype=np.int32)
    assert np.array_equal(sink, ref.sink)
    gs = np.array([g.decision.group_score for g in groups])
    assert gs.tobytes() == ref.group_scores.tobytes()
    if kv_floats is None:
        kv_floats = [g.kv_floats_loaded for g in groups]
    assert list(kv_floats) == list(ref.group_kv_floats)
    out = np.asarray(res_out)
    r = spec.r
    for gi in range(spec.num_kv_heads):
        if ref.sink[gi]:
            assert not np.any(out[gi * r:(gi + 1) * r].view(np.uint32))
    assert np.abs(out - ref.outputs).max() <= 2e-3
    assert np.linalg.norm(out - ref.outputs) <= 1e-3 * np.linalg.norm(ref.outputs)
    return ref


@pytest.mark.parametrize("name,kw", [
    ("C1-llama8b-32K", dict(num_q_heads=32, num_kv_heads=8, length=32768)),
    ("C3-yi9b-200K-B2", dict(num_q_heads=32, num_kv_heads=4, length=204800, num_seqs=2)),
    # the BASELINE batch: 32 Active groups -> distributed routing, global
    # token-space scheduler, warp-claimed queue merge over many partials
    ("C3-yi9b-200K-B16", dict(num_q_heads=32, num_kv_heads=4, length=204800, num_seqs=16)),
    ("C5-llava13b-8K-B8-image", dict(num_q_heads=40, num_kv_heads=40, length=8192, num_seqs=8,
                                      image_tokens=576)),
    # the BASELINE batch: 480 Active groups > 148 SMs -> the global token-space scheduler
    ("C5-llava13b-8K-B32-image", dict(num_q_heads=40, num_kv_heads=40, length=8192, num_seqs=32,
                                       image_tokens=576)),
])
def test_config_parity(oracle_libs, name, kw):
    _, orc = oracle_libs
    spec = WorkloadSpec(**kw, sink_fraction=0.625, seed=zlib.crc32(name.encode()) % 1000)
    cc = P.CacheConfig(1, spec.num_q_heads, spec.num_kv_heads, 128, spec.length, spec.num_seqs)
    q = spec.queries()
    with P.KvCache(cc) as cache:
        spec.fill(cache)
        res = P.routed_decode_step(q if spec.num_seqs > 1 else q[0], 0, cache, CFG)
        outs = res.outputs if spec.num_seqs > 1 else res.outputs[None]
        H = spec.num_kv_heads
        for s in range(spec.num_seqs):
            k, v = read_back(cache, spec, s)
            check_seq(orc, outs[s], res.groups[s * H:(s + 1) * H], spec, s, q[s], k, v)
        assert res.counters.groups_skipped == spec.num_seqs * spec.n_sink()


def test_headline_512k_vs_compiled_reference(oracle_libs):
    """BASELINE.json configs[1] at 512K, against the reference's own
    routed_decode_step (oracle/_ref, ThreadPool(16))."""
    ref_lib, _ = oracle_libs
    if ref_lib is None:
        pytest.skip("oracle/_ref not built")
    spec = WorkloadSpec(length=524288, sink_fraction=0.625, seed=42)
    q = spec.queries()[0]
    with P.KvCache(P.CacheConfig(1, 32, 8, 128, spec.length)) as cache:
        spec.fill(cache)
        res = P.routed_decode_step(q, 0, cache, CFG)
        rc = oracle.RefCache(ref_lib, 1, 32, 8, 128, spec.length)
        for g in range(8):
            k, v = cache.historical(0, g, 0, spec.length)
            rc.append_rows(0, g, k, v)
            del k, v
    ref = rc.routed_decode_step(q, 0, oracle.Profile.constant(0.5), excluded=(), workers=16)
    rc.close()
    assert np.array_equal(res.route_bitmap.astype(np.int32), ref.sink)
    assert np.array([g.decision.group_score for g in res.groups]).tobytes() == \
        ref.group_scores.tobytes()
    assert res.counters.kv_floats_loaded == ref.counters["kv_floats_loaded"]
    assert np.abs(res.outputs - ref.outputs).max() <= 2e-3
    assert np.linalg.norm(res.outputs - ref.outputs) <= 1e-3 * np.linalg.norm(ref.outputs)


def test_c4_70b_512k_sequence_sharded(oracle_libs):
    """BASELINE.json configs[3]: Llama-3.1-70B shape at 512K, sequence-sharded
    8 ways (simulated on one GPU: 8 shard engines + device LSE merge of their
    all-gathered partials) == the unsharded oracle."""
    _, orc = oracle_libs
    spec = WorkloadSpec(num_q_heads=64, num_kv_heads=8, length=524288, sink_fraction=0.625,
                        seed=70)
    q = spec.queries()[0]
    dq = torch.from_numpy(q).cuda()
    opts = P.EngineOptions(global_context_len=spec.length)
    parts, caches, ks, vs = [], [], [], []
    kv_sum = np.zeros(spec.num_kv_heads, dtype=np.uint64)
    for rank in range(8):
        cache, (lo, hi) = sharding.build_sequence_shard(P, spec, rank, 8, 0)
        part = torch.empty(cache.rank_partial_floats(), dtype=torch.float32, device="cuda")
        P.decode_rank_partial_async(dq.data_ptr(), 0, cache, CFG, opts, part.data_ptr())
        torch.cuda.synchronize()
        info = P.fetch_step_info(cache)
        kv_sum += np.array([g.kv_floats_loaded for g in info.groups], dtype=np.uint64)
        parts.append(part)
        caches.append(cache)
        kk, vv = read_back_shard(cache, spec, hi - lo)
        ks.append(kk)
        vs.append(vv)
    out = torch.zeros_like(dq)
    P.merge_rank_partials_async(caches[0], torch.cat(parts).data_ptr(), 8, out.data_ptr())
    torch.cuda.synchronize()
    k = np.concatenate(ks, axis=1)
    v = np.concatenate(vs, axis=1)
    del ks, vs
    check_seq(orc, out.cpu().numpy(), info.groups, spec, 0, q, k, v, kv_floats=kv_sum)
    for c in caches:
        c.close()


def read_back_shard(cache, spec, rows):
    ks, vs = [], []
    for g in range(spec.num_kv_heads):
        k, v = cache.historical(spec.layer, g, 0, rows)
        ks.append(k)
        vs.append(v)
    return np.stack(ks), np.stack(vs)


def test_wide_gqa_405b_shape_vs_compiled_reference(oracle_libs):
    """GQA width 16 (Llama-3.1-405B attention: 128 q / 8 KV heads, D = 128) at
    64K on the WIDE step kernel, against the reference's own routed_decode_step
    (oracle/_ref): bitmap and group scores bit-exact, loaded floats equal,
    outputs within the bar."""
    ref_lib, _ = oracle_libs
    if ref_lib is None:
        pytest.skip("oracle/_ref not built")
    spec = WorkloadSpec(num_q_heads=128, num_kv_heads=8, length=65536, sink_fraction=0.5, seed=405)
    q = spec.queries()[0]
    with P.KvCache(P.CacheConfig(1, 128, 8, 128, spec.length)) as cache:
        spec.fill(cache)
        res = P.routed_decode_step(q, 0, cache, CFG)
        rc = oracle.RefCache(ref_lib, 1, 128, 8, 128, spec.length)
        for g in range(8):
            k, v = cache.historical(0, g, 0, spec.length)
            rc.append_rows(0, g, k, v)
            del k, v
    ref = rc.routed_decode_step(q, 0, oracle.Profile.constant(0.5), excluded=(), workers=16)
    rc.close()
    assert np.array_equal(res.route_bitmap.astype(np.int32), ref.sink) and ref.sink.sum() == 4
    assert np.array([g.decision.group_score for g in res.groups]).tobytes() == ref.group_scores.tobytes()
    assert res.counters.kv_floats_loaded == ref.counters["kv_floats_loaded"]
    assert np.abs(res.outputs - ref.outputs).max() <= 2e-3
    assert np.linalg.norm(res.outputs - ref.outputs) <= 1e-3 * np.linalg.norm(ref.outputs)
