"""Generate tests/golden/*.npz from the COMPILED REFERENCE (oracle/_ref).

Run here (the reference sources exist only in this container):
    python tests/golden/make_golden.py

Each fixture holds the inputs that are not reproducible from our own
counter-based generator (queries, planted token-0 rows, explicit K/V for the
hand-built cases), the WorkloadSpec parameters for the rest, and the
reference's routed_decode_step results.  tests/test_oracle.py pins the C
restatement to these bit-exactly; tests/test_gpu_parity.py checks the engine.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2604_16883_b200.workload import WorkloadSpec, round_bf16  # noqa: E402


def planted(name, prof, excluded=(), sink_on_tie=False, observe_only=False, layer=0,
            num_splits=0, **spec_kw):
    spec = WorkloadSpec(**spec_kw)
    k, v = spec.host_cache(0)
    q = spec.queries()[0]
    return dict(name=name, kind="planted", spec=spec_kw, prof=prof, excluded=list(excluded),
                sink_on_tie=sink_on_tie, observe_only=observe_only, layer=layer,
                num_splits=num_splits), k, v, q


def explicit(name, k, v, q, prof, excluded=(), sink_on_tie=False, observe_only=False, layer=0,
             num_splits=0):
    return dict(name=name, kind="explicit", prof=prof, excluded=list(excluded),
                sink_on_tie=sink_on_tie, observe_only=observe_only, layer=layer,
                num_splits=num_splits), k, v, q


def cases():
    const = lambda t: [[0.0, 0.0, 0.0, t], 1.0, min(t, 0.0), max(t, 1.0)]
    yield planted("llama8b_L300_p50", const(0.5), num_q_heads=32, num_kv_heads=8, head_dim=128,
                  length=300, sink_fraction=0.5, seed=101)
    yield planted("mha_L64_p25_observe", const(0.5), observe_only=True, num_q_heads=8,
                  num_kv_heads=8, head_dim=64, length=64, sink_fraction=0.25, seed=102)
    cubic = [[0.2, -0.3, 0.1, 0.45], 1000.0, 0.35, 0.75]
    yield planted("gqa_D32_L1000_cubic_tie", cubic, sink_on_tie=True, num_q_heads=16,
                  num_kv_heads=4, head_dim=32, length=1000, sink_fraction=0.5, seed=103)
    yield planted("excluded_layer0", const(0.5), excluded=(0, 1), num_q_heads=32, num_kv_heads=8,
                  head_dim=128, length=200, sink_fraction=0.5, seed=104)
    yield planted("yi_r8_L777_splits3", const(0.5), num_splits=3, num_q_heads=32, num_kv_heads=4,
                  head_dim=128, length=777, sink_fraction=0.5, seed=105)
    yield planted("single_token", const(0.5), num_q_heads=32, num_kv_heads=8, head_dim=128,
                  length=1, sink_fraction=0.5, seed=106)
    # exact tie: q = [3, 4, 0...], k0 = [1, 0...] -> S == 0.6 == tau
    D, L = 64, 80
    rng = np.random.default_rng(107)
    k = np.vstack([np.eye(1, D, dtype=np.float32), rng.standard_normal((L - 1, D))])
    v = rng.standard_normal((L, D))
    k = round_bf16(k.astype(np.float32)).reshape(1, L, D)
    v = round_bf16(v.astype(np.float32)).reshape(1, L, D)
    q = np.zeros((4, D), np.float32)
    q[:, 0], q[:, 1] = 3.0, 4.0
    yield explicit("tie_active", k, v, q, const(0.6))
    yield explicit("tie_sink_on_tie", k, v, q, const(0.6), sink_on_tie=True)
    # degenerate query in group 0, diffuse random cache, tau < -1 (all sink otherwise)
    rng = np.random.default_rng(108)
    k = round_bf16(rng.standard_normal((2, 50, 128)).astype(np.float32)).reshape(2, 50, 128)
    v = round_bf16(rng.standard_normal((2, 50, 128)).astype(np.float32)).reshape(2, 50, 128)
    q = rng.standard_normal((8, 128)).astype(np.float32)
    q[1] = 0.0
    yield explicit("degenerate_full_skip", k, v, q, const(-2.0))


def run_ref(ref, meta, k, v, q):
    hkv, L, D = k.shape
    hq = q.shape[0]
    rc = oracle.RefCache(ref, max(2, meta["layer"] + 1), hq, hkv, D, L)
    for layer in range(max(2, meta["layer"] + 1)):
        for g in range(hkv):
            rc.append_rows(layer, g, k[g], v[g])
    c, n, lo, hi = meta["prof"]
    res = rc.routed_decode_step(q, meta["layer"], oracle.Profile(tuple(c), n, lo, hi),
                                excluded=tuple(meta["excluded"]),
                                sink_on_tie=meta["sink_on_tie"], num_splits=meta["num_splits"],
                                observe_only=meta["observe_only"], workers=4)
    rc.close()
    return res


def main():
    ref = oracle.ref()
    index = []
    for meta, k, v, q in cases():
        res = run_ref(ref, meta, k, v, q)
        arrays = dict(q=q, outputs=res.outputs, group_scores=res.group_scores,
                      thresholds=res.thresholds, sink=res.sink, degenerate=res.degenerate,
                      group_kv_floats=res.group_kv_floats, head_scores=res.head_scores,
                      counters=np.array([res.counters[key] for key in (
                          "kv_floats_loaded", "anchor_floats_loaded", "groups_active",
                          "groups_skipped")], dtype=np.uint64))
        if meta["kind"] == "explicit":
            arrays.update(k=k, v=v)
        np.savez_compressed(os.path.join(HERE, meta["name"] + ".npz"), **arrays)
        index.append(meta)
        print(meta["name"], "sinks", res.sink.tolist(), "kv", res.counters["kv_floats_loaded"])
    with open(os.path.join(HERE, "index.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py (compiled reference, oracle/_ref)",
                   "cases": index}, f, indent=1)


if __name__ == "__main__":
    main()
