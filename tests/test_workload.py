"""CPU: the synthetic planted-sink workload is reproducible and does what it
claims (checked with the compiled reference)."""
import numpy as np
import pytest

import oracle
from paper_2604_16883_b200.workload import WorkloadSpec, host_rows, mix_seed


def test_generator_matches_c_restatement(oracle_libs):
    _, orc = oracle_libs
    for seed, tags in ((42, (0, 0, 3, 1)), (7, (2, 5, 1, 2)), (0, ())):
        assert mix_seed(seed, tags) == orc.mix_seed(seed, list(tags))
    key = mix_seed(1, (0, 0, 0, 1))
    for row0, rows, d in ((1, 40, 128), (1000, 3, 64), (0, 5, 32)):
        assert host_rows(key, row0, rows, d).tobytes() == orc.fill_rows(key, row0, rows, d).tobytes()


def test_generator_statistics():
    x = host_rows(mix_seed(3, (1,)), 0, 2000, 128)
    assert abs(x.mean()) < 0.02 and abs(x.std() - 1.0) < 0.02
    assert np.all(x.view(np.uint32) & 0xFFFF == 0)  # bf16-representable


@pytest.mark.parametrize("p,expect", [(0.0, 0), (0.125, 1), (0.5, 4), (0.625, 5), (0.875, 7),
                                      (1.0, 8)])
def test_planted_fraction(p, expect):
    spec = WorkloadSpec(sink_fraction=p, length=8)
    assert spec.n_sink() == expect
    assert spec.sink_groups(0).sum() == expect


def test_planted_sink_routes_and_dominates(oracle_libs):
    """Sink-planted groups score ~rho and have alpha0 > 0.99;
    the others score ~0 and alpha0 < 0.1."""
    ref, orc = oracle_libs
    if ref is None:
        pytest.skip("reference not built")
    spec = WorkloadSpec(length=4096, sink_fraction=0.5, seed=5)
    k, v = spec.host_cache(0)
    q = spec.queries()[0]
    r = spec.r
    kn = [orc.anchor_norm(k[g, 0]) for g in range(8)]
    res = orc.routed_decode_step(k, v, k[:, 0].copy(), kn, q, 0, oracle.Profile.constant(0.5),
                                 excluded=(), threads=4)
    planted = spec.sink_groups(0)
    assert np.array_equal(res.sink.astype(bool), planted)
    for g in range(8):
        w = ref.attention_weights(q[g * r:(g + 1) * r], k[g])
        a0 = w[:, 0].mean()
        if planted[g]:
            assert abs(res.group_scores[g] - spec.rho_sink) < 1e-3 and a0 > 0.99
        else:
            assert abs(res.group_scores[g]) < 1e-5 and a0 < 0.1
    # traffic accounting (SPEC.md acceptance 6): kv_floats == (1 - s) * dense exactly
    dense = 8 * 2 * 4096 * 128
    s = planted.mean()
    assert res.counters["kv_floats_loaded"] == int((1 - s) * dense)


def test_queries_deterministic():
    a = WorkloadSpec(length=16, sink_fraction=0.5, seed=9).queries()
    b = WorkloadSpec(length=16, sink_fraction=0.5, seed=9).queries()
    assert a.tobytes() == b.tobytes()
