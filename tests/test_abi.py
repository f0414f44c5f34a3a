"""CPU: the C-ABI library (built for sm_100a) loads, exports exactly what
include/sinkr_cuda.h declares, its host-side control logic matches the
compiled reference bit for bit, and it refuses to run without a GPU (no CPU
fallback).  No compute call is made here."""
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
from paper_2604_16883_b200 import _abi, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sinkr_cuda.h")


@pytest.fixture(scope="module")
def L(built_lib):
    return _abi.lib()


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(sinkr_[a-z0-9_]+)\s*\(", src))


def test_header_matches_exports(L):
    decl = declared()
    assert decl == set(_abi.EXPORTS), decl ^ set(_abi.EXPORTS)
    nm = subprocess.run(["nm", "-D", "--defined-only", build.LIB], capture_output=True, text=True)
    exported = set(re.findall(r"\bT (sinkr_[a-z0-9_]+)\b", nm.stdout))
    assert decl <= exported, decl - exported
    for name in decl:
        assert hasattr(L, name)


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", build.LIB], capture_output=True, text=True)
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_sass_uses_tma_and_tensor_cores():
    out = subprocess.run(["cuobjdump", "-sass", build.LIB], capture_output=True, text=True).stdout
    assert "UTMALDG" in out           # cp.async.bulk.tensor
    assert "HMMA.16816.F32.BF16" in out
    assert "LDSM" in out
    assert "SYNCS" in out             # mbarrier


def test_host_helpers_match_reference(L, oracle_libs):
    ref, _ = oracle_libs
    if ref is None:
        pytest.skip("reference not built")
    import paper_2604_16883_b200 as P

    rng = np.random.default_rng(0)
    for _ in range(300):
        coeffs = tuple(rng.standard_normal(4))
        norm = float(rng.integers(1, 10 ** 6))
        lo, hi = sorted(rng.uniform(-1, 1, 2))
        length = int(rng.integers(1, 10 ** 6))
        prof = P.ThresholdProfile(coeffs=coeffs, length_normalizer=norm, clamp_lo=lo, clamp_hi=hi)
        t_ours = P.threshold_for_length(length, prof)
        t_ref = ref.threshold_for_length(length, oracle.Profile(coeffs, norm, lo, hi))
        assert t_ours == t_ref  # bit-exact (no FMA contraction on the host)
        score = float(rng.uniform(-1, 1))
        layer = int(rng.integers(0, 4))
        cfg = P.RoutingConfig(profile=prof, sink_on_tie=bool(rng.integers(0, 2)))
        d = P.route(layer, score, length, cfg)
        assert (d.sink, d.threshold) == ref.route(layer, score, length,
                                                  oracle.Profile(coeffs, norm, lo, hi),
                                                  sink_on_tie=cfg.sink_on_tie)
    for n in (1, 7, 8191, 8192, 8193, 65536, 10 ** 7):
        assert P.auto_num_splits(n) == ref.auto_num_splits(n)
    for length, n in ((10, 3), (7, 7), (1, 1), (100, 16)):
        assert P.split_ranges(length, n) == ref.split_ranges(length, n)
    with pytest.raises(ValueError):
        P.split_ranges(3, 4)
    with pytest.raises(ValueError):
        P.threshold_for_length(0, P.ThresholdProfile.constant(0.5))


def test_profile_constant_matches_reference(oracle_libs):
    import paper_2604_16883_b200 as P

    for tau in (-2.0, -0.3, 0.0, 0.55, 1.0, 2.0):
        p = P.ThresholdProfile.constant(tau)
        o = oracle.Profile.constant(tau)
        assert (tuple(p.coeffs), p.clamp_lo, p.clamp_hi) == (o.coeffs, o.lo, o.hi)


def test_no_cpu_fallback_without_gpu(L):
    """The engine refuses to run without an sm_100 device instead of silently
    computing on the CPU."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2604_16883_b200 as P

    with pytest.raises(_abi.SinkrCudaError, match="no CUDA device"):
        P.KvCache(P.CacheConfig(1, 32, 8, 128, 1024))


def test_config_validation_mirrors_reference(L):
    """CacheConfig::validate (kv_cache.cpp:32-39) errors come before any device work."""
    import paper_2604_16883_b200 as P

    bad = [P.CacheConfig(0, 32, 8, 128, 16), P.CacheConfig(1, 32, 0, 128, 16),
           P.CacheConfig(1, 30, 8, 128, 16), P.CacheConfig(1, 32, 8, 0, 16),
           P.CacheConfig(1, 32, 8, 128, 0), P.CacheConfig(1, 32, 8, 96, 16),
           P.CacheConfig(1, 34, 2, 128, 16)]  # GQA width 17 > 16
    for cfg in bad:
        with pytest.raises(ValueError):
            P.KvCache(cfg)


def test_bench_support_library(L):
    """The bench's C++ decode-loop timer (tools/e2e_timer.cpp) is built beside
    the product library, links against it and exports its one entry point;
    the product library does not carry it."""
    build.build_bench_lib()
    nm = subprocess.run(["nm", "-D", "--defined-only", build.BENCH_LIB], capture_output=True, text=True)
    assert re.search(r"\bT sinkr_bench_time_steps\b", nm.stdout)
    ldd = subprocess.run(["ldd", build.BENCH_LIB], capture_output=True, text=True).stdout
    assert "libsinkr_cuda.so" in ldd
    prod = subprocess.run(["nm", "-D", "--defined-only", build.LIB], capture_output=True, text=True).stdout
    assert "sinkr_bench_time_steps" not in prod
