"""CPU, world_size 2 over gloo: the sequence-sharded split of the decode step.

Each rank owns split_ranges(L, 2)[rank] of every KV group, holds the
replicated token-0 anchor, routes with tau(L_global) (so both ranks produce
the identical bitmap), and computes one LSE partial per (group, head) for its
slice with the oracle's attend_chunk.  The partials are all-gathered (gloo
here, NCCL on the GPUs) and merged with merge_partials; the result must match
the unsharded routed_decode_step of the compiled reference.  The device-side
math is covered by tests/test_gpu_sharding.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_16883_b200 import sharding


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    from paper_2604_16883_b200.workload import WorkloadSpec

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = oracle.orc()
        spec = WorkloadSpec(num_q_heads=16, num_kv_heads=4, head_dim=64, length=1001,
                            sink_fraction=0.5, seed=3)
        k, v = spec.host_cache(0)
        q = spec.queries()[0]
        lo, hi = sharding.sequence_shard(spec.length, world, rank)
        r, D = spec.r, spec.head_dim
        # routing from the replicated anchor with the GLOBAL length
        prof = oracle.Profile.constant(0.5)
        kn = [orc.anchor_norm(k[g, 0]) for g in range(4)]
        sinks, scores = [], []
        for g in range(4):
            hs = [orc.proxy_score(q[g * r + i], k[g, 0], kn[g])[0] for i in range(r)]
            s = orc.group_score(hs, r)
            sk, _ = orc.route(0, s, spec.length, prof, excluded=())
            sinks.append(sk)
            scores.append(s)
        # this rank's partials: [group][m(r), l(r), acc(r*D)]
        part = np.zeros((4, r * (D + 2)), np.float64)
        for g in range(4):
            if sinks[g]:
                continue
            m, lsum, acc = orc.attend_chunk(q[g * r:(g + 1) * r], k[g, lo:hi], v[g, lo:hi])
            part[g, :r], part[g, r:2 * r], part[g, 2 * r:] = m, lsum, acc.reshape(-1)
        t = torch.from_numpy(part)
        gathered = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(gathered, t)
        bits = torch.tensor(sinks, dtype=torch.int32)
        all_bits = [torch.zeros_like(bits) for _ in range(world)]
        dist.all_gather(all_bits, bits)
        if rank == 0:
            out = np.zeros((16, D), np.float32)
            for g in range(4):
                if sinks[g]:
                    continue
                parts = []
                for w, (a, b) in enumerate(sharding.split_ranges(spec.length, world)):
                    p = gathered[w].numpy()[g]
                    parts.append((p[:r], p[r:2 * r], p[2 * r:].reshape(r, D), b - a))
                out[g * r:(g + 1) * r] = orc.merge_partials(parts, r, D)
            ref = orc.routed_decode_step(k, v, k[:, 0].copy(), kn, q, 0, prof, excluded=(),
                                         threads=2)
            result_q.put(dict(
                same_bits=all(torch.equal(all_bits[0], b) for b in all_bits),
                bits_match_ref=list(map(bool, ref.sink)) == list(map(bool, sinks)),
                max_abs=float(np.abs(out - ref.outputs).max()),
                zero_rows=all(not np.any(out[g * r:(g + 1) * r]) for g in range(4) if sinks[g])))
    finally:
        dist.destroy_process_group()


def test_sequence_sharded_merge_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res["same_bits"] and res["bits_match_ref"] and res["zero_rows"]
    assert res["max_abs"] <= 1e-6


@pytest.mark.parametrize("L,world", [(1, 1), (10, 3), (524288, 8), (1001, 2), (7, 7)])
def test_sequence_shards_partition(L, world):
    rs = [sharding.sequence_shard(L, world, k) for k in range(world)]
    assert rs[0][0] == 0 and rs[-1][1] == L
    assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
    assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


@pytest.mark.parametrize("units,world", [(8, 2), (8, 8), (4, 8), (1280, 8), (5, 3)])
def test_unit_shards_partition(units, world):
    covered = []
    for k in range(world):
        a, b = sharding.unit_shard(units, world, k)
        covered.extend(range(a, b))
    assert covered == list(range(units))


def test_anchor_norm_matches_reference(oracle_libs):
    _, orc = oracle_libs
    rng = np.random.default_rng(2)
    for _ in range(50):
        k0 = (rng.standard_normal(128) * rng.uniform(0.01, 40)).astype(np.float32)
        assert sharding.anchor_norm(k0) == orc.anchor_norm(k0)
