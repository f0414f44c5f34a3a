"""CPU: SNKT files byte-identical to the reference's and
read with its error semantics; oracle labels and the PR curve (§8 f4) on the
SPEC.md known answers and against a brute-force confusion-matrix oracle.
No GPU call is made here."""
import numpy as np
import pytest

from paper_2604_16883_b200 import analysis as A
from paper_2604_16883_b200 import snapshot as S


@pytest.fixture(scope="module")
def ref(oracle_libs):
    r, _ = oracle_libs
    if r is None:
        pytest.skip("reference not built")
    return r


@pytest.mark.parametrize("shape", [(1,), (7,), (3, 5), (2, 3, 4), (17, 128)])
def test_snkt_byte_identical(built_lib, ref, tmp_path, shape):
    rng = np.random.default_rng(sum(shape))
    a = rng.normal(size=shape).astype(np.float32)
    ours, theirs = tmp_path / "o.snkt", tmp_path / "t.snkt"
    S.write_tensor(ours, a)
    ref.write_tensor(theirs, a)
    assert ours.read_bytes() == theirs.read_bytes()
    assert ours.stat().st_size == S.snkt_file_size(shape) == ref.snkt_file_size(shape)
    assert np.array_equal(S.read_tensor(theirs), a)
    assert np.array_equal(ref.read_tensor(ours), a)


def test_snkt_file_size_kat(built_lib):
    assert S.snkt_file_size([1]) == 28  # SURVEY.md §8c (SPEC.md's guess was 29)


def test_snkt_errors(built_lib, tmp_path):
    p = tmp_path / "x.snkt"
    S.write_tensor(p, np.ones((2, 3), dtype=np.float32))
    raw = p.read_bytes()
    cases = {
        b"SNKX" + raw[4:]: "bad magic",
        raw[:6]: r"truncated header \(version\)",
        raw[:4] + (2).to_bytes(4, "little") + raw[8:]: "unsupported version 2",
        raw[:8] + (2).to_bytes(4, "little") + raw[12:]: "unsupported dtype 2",
        raw[:12] + (0).to_bytes(4, "little") + raw[16:]: "bad ndim 0",
        raw[:20]: "truncated dims",
        raw[:16] + (0).to_bytes(8, "little") + raw[24:]: "zero dim 0",
        raw[:-4]: "short payload",
        raw + b"\0": "trailing bytes",
    }
    for blob, msg in cases.items():
        p.write_bytes(blob)
        with pytest.raises(RuntimeError, match="SNKT parse error.*" + msg):
            S.read_tensor(p)
    with pytest.raises(RuntimeError, match="cannot open"):
        S.read_tensor(tmp_path / "missing.snkt")


def test_oracle_label_kats(built_lib):
    # SPEC.md oracle_labels examples (Table 1 regimes, strict tie rule)
    assert A.oracle_labels_from_alpha0([0.803], 0.65)[0].is_sink
    assert not A.oracle_labels_from_alpha0([0.410], 0.65)[0].is_sink
    g = A.oracle_labels_from_alpha0([0.7, 0.7, 0.6, 0.6], 0.65, A.OracleMode.GroupMean, 4)
    assert len(g) == 1 and abs(g[0].alpha0 - 0.65) < 1e-15 and not g[0].is_sink
    w = np.full((2, 4), 0.25)
    w[0] = [0.85, 0.05, 0.05, 0.05]
    labs = A.oracle_labels(w, 2, 4, 0.65, A.OracleMode.Head)
    assert [l.is_sink for l in labs] == [True, False]
    with pytest.raises(ValueError, match="sum to 1"):
        A.oracle_labels(np.full((1, 4), 0.3), 1, 4, 0.65, A.OracleMode.Head)


def brute_force_ap(scores, labels):
    """O(n^2) confusion-matrix recomputation at every distinct threshold."""
    pos = labels.sum()
    pts, ap, prev_r = [], 0.0, 0.0
    for t in sorted(set(scores.tolist()), reverse=True):
        pred = scores >= t
        tp = int((pred & labels).sum())
        fp = int((pred & ~labels).sum())
        p, r = tp / (tp + fp), tp / pos
        ap += (r - prev_r) * p
        prev_r = r
        pts.append((t, p, r))
    return pts, ap


def test_pr_curve(built_lib):
    # perfect separation -> 1.0; all scores equal -> one point at the prevalence
    c = A.pr_curve([0.9, 0.8, 0.2, 0.1], [1, 1, 0, 0])
    assert c.auprc == 1.0
    c = A.pr_curve([0.5] * 10, [1, 0, 0, 1, 0, 0, 0, 0, 0, 0])
    assert len(c.points) == 1 and c.points[0].precision == pytest.approx(0.2)
    with pytest.raises(ValueError, match="positive"):
        A.pr_curve([0.1, 0.2], [0, 0])
    rng = np.random.default_rng(3)
    for _ in range(10):
        s = np.round(rng.uniform(size=200), 2)
        l = rng.uniform(size=200) < 0.3
        c = A.pr_curve(s, l)
        pts, ap = brute_force_ap(s, l)
        assert abs(c.auprc - ap) < 1e-9
        assert [(p.threshold, p.precision, p.recall) for p in c.points] == pytest.approx(pts)
        recalls = [p.recall for p in c.points]
        assert all(a <= b for a, b in zip(recalls, recalls[1:]))
        # invariant under a strictly increasing transform of the scores
        assert abs(A.pr_curve(np.exp(3 * s), l).auprc - c.auprc) < 1e-12
