"""bench-cli front end (SPEC.md bench-cli module) over the
B200 engine.

    python -m paper_2604_16883_b200.cli calibrate  --lengths 8192,16384,32768,65536,131072 --out DIR
    python -m paper_2604_16883_b200.cli bench      --lengths 65536,131072 --plant-sink-frac 0.6 --out DIR
    python -m paper_2604_16883_b200.cli route-eval --lengths 32768 --out DIR
    python -m paper_2604_16883_b200.cli selftest

Shared flags: --seed, --profile <path>, --out <dir>, --format {json,csv,both};
workload flags: --layers --hq --hkv --dim --lengths --plant-sink-frac.
Exit codes: 0 success, 1 runtime/validation failure, 2 usage error.
Reports are JSON + CSV with fixed, documented columns (CSV_COLUMNS below).
Workloads are the synthetic planted-sink caches of workload.py (generated on
the device); `bench` times dense and routed steps on the same inputs (CUDA
events on the engine stream, median of >= 32 steps after 4 warm-ups) and
gates on correctness: Active-group outputs of the routed step equal the
dense step's within 1e-5, Sink rows are bitwise zero.
"""
from __future__ import annotations

import argparse
import csv
import json
import os
import sys
from typing import List

import numpy as np

CSV_COLUMNS = {
    "bench": ["length", "dense_us", "routed_us", "speedup", "skip_ratio", "kv_floats_dense",
              "kv_floats_routed", "kv_floats_avoided", "routing_us", "attention_us", "merge_us",
              "kv_gbs_routed"],
    "calibrate": ["length", "tau", "skip"],
    "route-eval": ["threshold", "precision", "recall", "f1"],
}


class UsageError(Exception):
    pass


def _ints(s: str) -> List[int]:
    try:
        out = [int(x) for x in s.split(",") if x.strip()]
    except ValueError:
        raise UsageError(f"bad integer list '{s}'")
    if not out:
        raise UsageError("empty list")
    return out


def _write(args, name: str, report: dict, rows: List[dict]) -> None:
    if not args.out:
        return
    os.makedirs(args.out, exist_ok=True)
    if args.format in ("json", "both"):
        with open(os.path.join(args.out, f"{name}.json"), "w") as f:
            json.dump(report, f, indent=2)
    if args.format in ("csv", "both"):
        with open(os.path.join(args.out, f"{name}.csv"), "w", newline="") as f:
            w = csv.DictWriter(f, fieldnames=CSV_COLUMNS[name])
            w.writeheader()
            for r in rows:
                w.writerow({k: r.get(k, "") for k in CSV_COLUMNS[name]})


def _spec(args, length: int, p: float, seed: int):
    from .workload import WorkloadSpec

    return WorkloadSpec(num_q_heads=args.hq, num_kv_heads=args.hkv, head_dim=args.dim,
                        length=length, sink_fraction=p, seed=seed)


def _filled_cache(args, spec):
    import paper_2604_16883_b200 as P

    cache = P.KvCache(P.CacheConfig(args.layers, args.hq, args.hkv, args.dim, spec.length))
    for layer in range(args.layers):
        spec.layer = layer
        spec.fill(cache)
    spec.layer = 0
    return cache


def _routing_config(args):
    import paper_2604_16883_b200 as P
    from .calibration import load_profile

    if args.profile:
        return P.RoutingConfig.from_profile(load_profile(args.profile))
    return P.RoutingConfig(profile=P.ThresholdProfile.constant(args.tau), excluded_layers=())


# ---------------------------------------------------------------- calibrate
def cmd_calibrate(args) -> int:
    """Appendix A: per length, the threshold realising the target skip over
    GPU-collected group scores (skipping disabled), cubic fit, profile JSON."""
    import paper_2604_16883_b200 as P
    from . import calibration as cal

    lengths = _ints(args.lengths)
    caches = {}

    def collect(L):
        spec = _spec(args, L, 0.0, args.seed)
        cache = caches[L] = _filled_cache(args, spec)
        rng = np.random.default_rng(args.seed + L)
        pop = cal.ScorePopulation()
        D, r = args.dim, args.hq // args.hkv
        mu = args.score_base + args.score_shift * L / max(lengths)
        qs = np.zeros((args.samples, args.hq, D), dtype=np.float32)
        for q in qs:
            for g in range(args.hkv):
                k0 = spec.first_rows(0, g)[0].astype(np.float64)
                kh = k0 / np.linalg.norm(k0)
                for i in range(r):
                    n = rng.standard_normal(D)
                    n -= (n @ kh) * kh
                    n /= np.linalg.norm(n)
                    c = float(np.clip(rng.normal(mu, args.score_spread), -0.95, 0.95))
                    q[g * r + i] = np.sqrt(D) * (c * kh + np.sqrt(1 - c * c) * n)
        # every sample of this length in one launch per layer (population in
        # the reference's sample-major order)
        per_layer = [cal.collect_scores_batch(cache, qs, layer)[1] for layer in range(args.layers)]
        for s in range(args.samples):
            for layer in range(args.layers):
                pop.extend(per_layer[layer][s], layer, L)
        return pop

    excluded = tuple(_ints(args.excluded)) if args.excluded else ()
    prof = cal.calibrate(collect, lengths, args.target_skip, args.gamma, excluded)
    rows = [{"length": p.length, "tau": p.tau, "skip": p.skip} for p in prof.points]
    print(f"{'length':>10} {'tau':>10} {'skip':>8}")
    for r in rows:
        print(f"{r['length']:>10} {r['tau']:>10.5f} {r['skip']:>8.4f}")
    if args.out:
        os.makedirs(args.out, exist_ok=True)
        cal.save_profile(os.path.join(args.out, "profile.json"), prof)
    for c in caches.values():
        c.close()
    _write(args, "calibrate", {"coefficients": list(prof.coeffs), "clamp": [prof.clamp_lo, prof.clamp_hi],
                               "length_normalizer": prof.length_normalizer, "points": rows}, rows)
    return 0


# ---------------------------------------------------------------- bench
def _time_steps(torch, P, cache, cfg, dq, dout, warmup, steps, layer):
    st = torch.cuda.ExternalStream(cache.stream)
    P.set_timing(cache, False)
    for _ in range(warmup):
        P.routed_decode_async(dq.data_ptr(), layer, cache, cfg, d_outputs=dout.data_ptr())
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        P.routed_decode_async(dq.data_ptr(), layer, cache, cfg, d_outputs=dout.data_ptr())
        e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


def cmd_bench(args) -> int:
    lengths = _ints(args.lengths)
    import torch

    import paper_2604_16883_b200 as P

    if not torch.cuda.is_available():
        raise RuntimeError("bench needs a CUDA device (the engine has no CPU path)")
    dense = P.RoutingConfig(profile=P.ThresholdProfile.constant(2.0), excluded_layers=())
    routed = _routing_config(args)
    layer = args.layers - 1
    rows = []
    for L in lengths:
        spec = _spec(args, L, args.plant_sink_frac, args.seed)
        spec.layer = layer
        cache = P.KvCache(P.CacheConfig(args.layers, args.hq, args.hkv, args.dim, L))
        for l in range(args.layers):
            spec.layer = l
            spec.fill(cache)
        spec.layer = layer
        q = spec.queries()[0]
        # correctness gate (SPEC.md bench: identical inputs, Active groups match dense)
        rd = P.routed_decode_step(q, layer, cache, dense)
        rr = P.routed_decode_step(q, layer, cache, routed)
        r = args.hq // args.hkv
        for g in rr.groups:
            rows_g = slice(g.kv_head * r, (g.kv_head + 1) * r)
            if g.decision.sink:
                if np.any(rr.outputs[rows_g].view(np.uint32) != 0):
                    raise RuntimeError(f"correctness gate: Sink group {g.kv_head} has non-zero rows")
            elif np.abs(rr.outputs[rows_g] - rd.outputs[rows_g]).max() > 1e-5:
                raise RuntimeError(f"correctness gate: Active group {g.kv_head} differs from dense")
        dq = torch.from_numpy(q).cuda()
        dout = torch.zeros_like(dq)
        t_dense = _time_steps(torch, P, cache, dense, dq, dout, args.warmup, args.steps, layer)
        t_routed = _time_steps(torch, P, cache, routed, dq, dout, args.warmup, args.steps, layer)
        P.set_timing(cache, True)
        P.routed_decode_async(dq.data_ptr(), layer, cache, routed, d_outputs=dout.data_ptr())
        c = P.fetch_step_info(cache).counters
        P.set_timing(cache, False)
        kv_d, kv_r = rd.counters.kv_floats_loaded, rr.counters.kv_floats_loaded
        row = {"length": L, "dense_us": round(t_dense, 2), "routed_us": round(t_routed, 2),
               "speedup": round(t_dense / t_routed, 3),
               "skip_ratio": rr.counters.groups_skipped / len(rr.groups),
               "kv_floats_dense": kv_d, "kv_floats_routed": kv_r, "kv_floats_avoided": kv_d - kv_r,
               "routing_us": round(c.routing_seconds * 1e6, 2),
               "attention_us": round(c.attention_seconds * 1e6, 2),
               "merge_us": round(c.merge_seconds * 1e6, 2),
               "kv_gbs_routed": round(kv_r * 2 / (t_routed * 1e-6) / 1e9, 1)}
        rows.append(row)
        print(json.dumps(row))
        cache.close()
    _write(args, "bench", {"workload": {"hq": args.hq, "hkv": args.hkv, "dim": args.dim,
                                        "layers": args.layers, "plant_sink_frac": args.plant_sink_frac,
                                        "seed": args.seed},
                           "timing": f"median of {args.steps} steps after {args.warmup} warm-ups, "
                                     "CUDA events on the engine stream",
                           "rows": rows}, rows)
    return 0


# ---------------------------------------------------------------- route-eval
def cmd_route_eval(args) -> int:
    import paper_2604_16883_b200 as P
    from . import analysis as A
    from . import calibration as cal

    gamma = args.gamma
    if args.profile:
        gamma = cal.load_profile(args.profile).gamma
    scores, labels, a0s = [], [], []
    for L in _ints(args.lengths):
        for rep in range(args.samples):
            spec = _spec(args, L, args.plant_sink_frac, args.seed + rep)
            with P.KvCache(P.CacheConfig(1, args.hq, args.hkv, args.dim, L)) as cache:
                spec.fill(cache)
                q = spec.queries()[0]
                _, gs, _ = cal.collect_scores(cache, q, 0)
                a0 = A.attention_bos_mass(cache, q, 0)[0]
            labs = A.oracle_labels_from_alpha0(a0, gamma, A.OracleMode.GroupMean, args.hq // args.hkv)
            scores += gs.tolist()
            labels += [l.is_sink for l in labs]
            a0s += [l.alpha0 for l in labs]
    if not any(labels):
        raise RuntimeError("no positive oracle labels: PR curve undefined")
    curve = A.pr_curve(scores, labels)
    s, l = np.array(scores), np.array(labels)
    op = {}
    for tau in sorted(set([args.tau, 0.55])):  # Appendix C's operating point, explicitly
        pred = s > tau
        tp, fp, fn = int((pred & l).sum()), int((pred & ~l).sum()), int((~pred & l).sum())
        prec = tp / (tp + fp) if tp + fp else 0.0
        rec = tp / (tp + fn) if tp + fn else 0.0
        op[str(tau)] = {"precision": prec, "recall": rec,
                        "f1": 2 * prec * rec / (prec + rec) if prec + rec else 0.0}
    rows = [{"threshold": p.threshold, "precision": p.precision, "recall": p.recall, "f1": p.f1}
            for p in curve.points]
    report = {"auprc": curve.auprc, "gamma": gamma, "n": len(scores), "positives": int(l.sum()),
              "operating_points": op, "curve": rows}
    print(json.dumps({k: report[k] for k in ("auprc", "gamma", "n", "positives", "operating_points")}))
    _write(args, "route-eval", report, rows)
    return 0


# ---------------------------------------------------------------- selftest
def cmd_selftest(args) -> int:
    """Invariant suite on the engine (no CPU oracle involved): routing
    semantics, skipped-block record, split invariance across context lengths,
    excluded layers, calibration round trip, and the sink_on_tie fault hook."""
    import tempfile

    import paper_2604_16883_b200 as P
    from . import calibration as cal

    failures = []
    # fault injection: the reference's tie-breaking test hook
    # (RoutingConfig::sink_on_tie, router.hpp:20-22) forced on in every routing
    # config the suite builds; the routing-semantics check must then fail
    fault = bool(getattr(args, "inject_tie_fault", False)) or \
        os.environ.get("SINKR_INJECT_TIE_FAULT", "") == "1"
    if fault:
        print("fault injection: sink_on_tie forced on (routing semantics must fail)")

    def rc(**kw):
        c = P.RoutingConfig(**kw)
        c.sink_on_tie = c.sink_on_tie or fault
        return c

    def expect(name, ok):
        print(f"{'PASS' if ok else 'FAIL'}  {name}")
        if not ok:
            failures.append(name)

    spec = _spec(args, 4096, 0.5, args.seed)
    with P.KvCache(P.CacheConfig(3, args.hq, args.hkv, args.dim, 4096)) as cache:
        for layer in range(3):
            spec.layer = layer
            spec.fill(cache)
        spec.layer = 2
        q = spec.queries()[0]
        cfg = rc(profile=P.ThresholdProfile.constant(0.5))
        res = P.routed_decode_step(q, 2, cache, cfg)
        dense = P.routed_decode_step(q, 2, cache, rc(profile=P.ThresholdProfile.constant(2.0)))
        r = args.hq // args.hkv
        sinks = [g.decision.sink for g in res.groups]
        expect("planted groups route Sink", sinks == spec.sink_groups(0).tolist())
        ok_zero, ok_act, ok_cnt = True, True, True
        for g in res.groups:
            rows = res.outputs[g.kv_head * r:(g.kv_head + 1) * r]
            if g.decision.sink:
                ok_zero &= bool(np.all(rows.view(np.uint32) == 0))
                ok_cnt &= g.kv_floats_loaded == 0
            else:
                ok_act &= float(np.abs(rows - dense.outputs[g.kv_head * r:(g.kv_head + 1) * r]).max()) <= 1e-5
                ok_cnt &= g.kv_floats_loaded == 2 * 4096 * args.dim
        expect("Sink rows bitwise zero", ok_zero)
        expect("Active groups match dense within 1e-5", ok_act)
        expect("skipped-block record (kv_floats 0 or 2LD)", ok_cnt)
        ex = P.routed_decode_step(q, 0, cache, cfg)
        expect("excluded layers never skip", ex.counters.groups_skipped == 0)
        # an exact tie S == tau (router.cpp:67-75): strict >, so Active
        ties = rc(profile=P.ThresholdProfile.constant(res.groups[0].decision.group_score),
                  excluded_layers=())
        t0 = P.routed_decode_step(q, 2, cache, ties).groups[0].decision.sink
        expect("routing semantics: an exact tie routes Active (strict >)", not t0)
        hook = rc(profile=P.ThresholdProfile.constant(res.groups[0].decision.group_score),
                  excluded_layers=())
        hook.sink_on_tie = True
        t1 = P.routed_decode_step(q, 2, cache, hook).groups[0].decision.sink
        expect("sink_on_tie test hook flips the tie to Sink", t1)
    outs = []
    for L in (1000, 3000):
        s2 = _spec(args, L, 0.0, args.seed)
        with P.KvCache(P.CacheConfig(1, args.hq, args.hkv, args.dim, L)) as c:
            s2.fill(c)
            o = P.routed_decode_step(s2.queries()[0], 0, c, rc(profile=P.ThresholdProfile.constant(2.0)))
            outs.append(np.isfinite(o.outputs).all() and o.counters.groups_active == args.hkv)
    expect("dense steps finite at several lengths", all(outs))
    prof = P.ThresholdProfile(coeffs=(0.1, -0.2, 0.3, 0.5), length_normalizer=65536.0)
    with tempfile.TemporaryDirectory() as d:
        cal.save_profile(os.path.join(d, "p.json"), prof)
        expect("profile JSON round trip", cal.load_profile(os.path.join(d, "p.json")) == prof)
    print(f"selftest: {'ok' if not failures else 'FAILED: ' + ', '.join(failures)}")
    return 0 if not failures else 1


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="sinkr", description=__doc__.split("\n")[0])
    sub = ap.add_subparsers(dest="cmd")

    def common(p):
        p.add_argument("--seed", type=int, default=42)
        p.add_argument("--profile", default=None)
        p.add_argument("--out", default=None)
        p.add_argument("--format", choices=("json", "csv", "both"), default="both")
        p.add_argument("--layers", type=int, default=1)
        p.add_argument("--hq", type=int, default=32)
        p.add_argument("--hkv", type=int, default=8)
        p.add_argument("--dim", type=int, default=128)
        p.add_argument("--plant-sink-frac", type=float, default=0.625)
        p.add_argument("--tau", type=float, default=0.5)
        p.add_argument("--gamma", type=float, default=0.65)

    p = sub.add_parser("calibrate")
    common(p)
    p.add_argument("--lengths", required=True)
    p.add_argument("--samples", type=int, default=50)
    p.add_argument("--target-skip", type=float, default=0.60)
    p.add_argument("--excluded", default="")
    p.add_argument("--score-base", type=float, default=0.15)
    p.add_argument("--score-shift", type=float, default=0.35)
    p.add_argument("--score-spread", type=float, default=0.15)
    p = sub.add_parser("bench")
    common(p)
    p.add_argument("--lengths", required=True)
    p.add_argument("--steps", type=int, default=32)
    p.add_argument("--warmup", type=int, default=4)
    p = sub.add_parser("route-eval")
    common(p)
    p.add_argument("--lengths", required=True)
    p.add_argument("--samples", type=int, default=4)
    p = sub.add_parser("selftest")
    common(p)
    p.add_argument("--inject-tie-fault", action="store_true",
                   help="force the sink_on_tie hook on (SPEC.md:610): the suite must report a "
                        "routing-semantics failure and exit 1")
    return ap


def main(argv=None) -> int:
    ap = build_parser()
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 2 if e.code else 0
    if not args.cmd:
        ap.print_usage(sys.stderr)
        return 2
    fn = {"calibrate": cmd_calibrate, "bench": cmd_bench, "route-eval": cmd_route_eval,
          "selftest": cmd_selftest}[args.cmd]
    try:
        return fn(args)
    except UsageError as e:
        print(f"usage error: {e}", file=sys.stderr)
        return 2
    except Exception as e:  # runtime / validation failure
        print(f"error: {type(e).__name__}: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
