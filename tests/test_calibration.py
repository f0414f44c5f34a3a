"""CPU: the calibration host logic of the library against the
compiled reference, bit for bit — sweep / skip_ratio_at / solve_threshold,
fit_cubic, calibrate and the profile JSON both ways — plus the SPEC.md
known-answer examples and error behaviour.  No GPU call is made here."""
import json

import numpy as np
import pytest

import paper_2604_16883_b200 as P
from paper_2604_16883_b200 import calibration as cal


@pytest.fixture(scope="module")
def ref(oracle_libs):
    r, _ = oracle_libs
    if r is None:
        pytest.skip("reference not built")
    return r


def test_spec_examples(built_lib):
    pop = np.arange(1, 11) / 10.0
    # target 0.6 -> tau 0.4, realised skip exactly 0.6
    tau = cal.solve_threshold(pop, 0.6)
    assert tau == 0.4
    assert cal.skip_ratio_at(pop, tau) == 0.6
    assert cal.solve_threshold(pop, 0.0) == 1.0
    assert cal.skip_ratio_at(pop, 1.0) == 0.0
    # sweep is non-increasing in the threshold
    sw = cal.sweep(pop, np.linspace(0, 1.1, 23))
    skips = [s for _, s in sw]
    assert all(a >= b for a, b in zip(skips, skips[1:]))
    # exact cubic recovery and the constant fit
    xs = [0.1, 0.35, 0.6, 0.8, 1.0]
    f = cal.fit_cubic([(x, ((1 * x - 2) * x + 0.5) * x + 0.3) for x in xs])
    assert np.allclose(f.coeffs, (1, -2, 0.5, 0.3), atol=1e-6)
    f = cal.fit_cubic([(x, 0.55) for x in xs])
    assert np.allclose(f.coeffs, (0, 0, 0, 0.55), atol=1e-8)


def test_errors(built_lib):
    with pytest.raises(ValueError, match="empty score population"):
        cal.solve_threshold([], 0.5)
    with pytest.raises(ValueError, match="target_skip"):
        cal.solve_threshold([0.1, 0.2], 1.0)
    with pytest.raises(ValueError, match="4 distinct x"):
        cal.fit_cubic([(0, 1), (1, 2), (2, 3), (2, 4)])
    with pytest.raises(ValueError, match="4 distinct lengths"):
        cal.calibrate(lambda L: cal.ScorePopulation(), [8, 16, 32, 32], 0.6, 0.65)


@pytest.mark.parametrize("seed", range(6))
def test_statistics_bit_exact(built_lib, ref, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 400))
    s = rng.normal(0.3, 0.3, n)
    if seed % 2:
        s = np.round(s, 2)  # ties
    t = np.concatenate([rng.uniform(-1, 1.5, 20), s[:5]])
    assert np.array_equal(np.array([x for _, x in cal.sweep(s, t)]), ref.sweep(s, t))
    for target in (0.0, 0.3, 0.6, 0.95, rng.uniform(0, 0.999)):
        a, b = cal.solve_threshold(s, target), ref.solve_threshold(s, target)
        assert a == b
        assert cal.skip_ratio_at(s, a) == ref.skip_ratio_at(s, b)


@pytest.mark.parametrize("seed", range(8))
def test_fit_cubic_bit_exact(built_lib, ref, seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(4, 40))
    x = rng.uniform(0, 1, n)
    x[:4] = [0.1, 0.4, 0.7, 1.0]
    y = rng.normal(0.5, 0.2, n)
    ours = cal.fit_cubic(list(zip(x, y)))
    co, res = ref.fit_cubic(x, y)
    assert np.array_equal(np.array(ours.coeffs), co), (ours.coeffs, co)
    assert ours.residual == res


@pytest.mark.parametrize("seed", range(5))
def test_calibrate_bit_exact(built_lib, ref, seed):
    rng = np.random.default_rng(200 + seed)
    lengths = [8192, 16384, 32768, 65536, 131072]
    if seed == 3:
        lengths = lengths + [16384]  # duplicates: collected once
    pops = []
    for i, L in enumerate(lengths):
        n = int(rng.integers(20, 300))
        scores = rng.normal(0.3 + 0.05 * i, 0.2, n)
        layers = rng.integers(0, 6, n)
        pops.append((scores, layers))
    excluded = (0, 1) if seed != 4 else ()
    calls = []

    def collect(L):
        calls.append(L)
        i = lengths.index(L)
        pop = cal.ScorePopulation()
        for s, l in zip(*pops[i]):
            pop.add(s, int(l), L)
        return pop

    prof = cal.calibrate(collect, lengths, 0.6, 0.65, excluded)
    r = ref.calibrate(lengths, pops, 0.6, 0.65, excluded)
    assert sorted(calls) == sorted(set(lengths)) and r["collector_calls"] == len(set(lengths))
    assert np.array_equal(np.array(prof.coeffs), r["coeffs"])
    assert prof.length_normalizer == r["normalizer"]
    assert (prof.clamp_lo, prof.clamp_hi) == (r["lo"], r["hi"])
    assert (prof.target_skip, prof.gamma) == (r["target_skip"], r["gamma"])
    assert list(prof.excluded_layers) == r["excluded"]
    assert [(p.length, p.tau, p.skip) for p in prof.points] == r["points"]


def test_profile_json_interop(built_lib, ref, tmp_path):
    rng = np.random.default_rng(7)
    prof = P.ThresholdProfile(coeffs=tuple(rng.normal(size=4)), length_normalizer=131072.0,
                              clamp_lo=-0.25, clamp_hi=0.9, target_skip=0.6, gamma=0.65,
                              excluded_layers=(0, 1, 5),
                              points=[cal.CalibrationPoint(8192 * (i + 1), float(rng.uniform()),
                                                           float(rng.uniform())) for i in range(5)])
    ours = tmp_path / "ours.json"
    cal.save_profile(ours, prof)
    back = cal.load_profile(ours)
    assert back == prof  # field-wise round trip (SPEC.md profile round-trip identity)
    r = ref.load_profile(ours)  # the reference reads our file ...
    assert np.array_equal(r["coeffs"], np.array(prof.coeffs))
    assert r["points"] == [(p.length, p.tau, p.skip) for p in prof.points]
    theirs = tmp_path / "theirs.json"
    ref.save_profile(theirs, r)  # ... and we read the reference's
    assert cal.load_profile(theirs) == prof
    assert json.load(open(ours)).keys() == json.load(open(theirs)).keys()


def test_profile_json_errors(built_lib, tmp_path, capfd):
    p = tmp_path / "p.json"
    good = {"version": 1, "gamma": 0.65, "target_skip": 0.6, "length_normalizer": 1.0,
            "coefficients": [0, 0, 0, 0.5], "clamp": [0, 1], "excluded_layers": [0, 1],
            "calibration_points": []}
    bad = dict(good)
    del bad["coefficients"]
    p.write_text(json.dumps(bad))
    with pytest.raises(RuntimeError, match='missing key "coefficients"'):
        cal.load_profile(p)
    p.write_text(json.dumps(dict(good, version=2)))
    with pytest.raises(RuntimeError, match="unsupported profile version"):
        cal.load_profile(p)
    p.write_text(json.dumps(dict(good, coefficients=[1, 2])))
    with pytest.raises(RuntimeError, match="4-element array"):
        cal.load_profile(p)
    p.write_text("{ not json")
    with pytest.raises(RuntimeError, match="parse error"):
        cal.load_profile(p)
    p.write_text(json.dumps(dict(good, extra_key=3)))
    assert cal.load_profile(p).coeffs == (0.0, 0.0, 0.0, 0.5)
    assert 'ignoring unknown key "extra_key"' in capfd.readouterr().err
