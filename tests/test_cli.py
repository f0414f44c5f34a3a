"""bench-cli front end (SPEC.md bench-cli): exit codes and
usage on CPU, the four subcommands end to end on the GPU."""
import csv
import json
import os

import pytest

from paper_2604_16883_b200 import cli


def test_usage_errors(capsys):
    assert cli.main([]) == 2
    assert cli.main(["bench"]) == 2                      # missing --lengths
    assert cli.main(["bench", "--lengths", "x,y"]) == 2  # bad list
    assert cli.main(["no-such-command"]) == 2


def test_calibrate_rank_error_exit_1(built_lib, capsys):
    rc = cli.main(["calibrate", "--lengths", "1024,2048,2048,4096"])
    assert rc == 1
    assert "4 distinct lengths" in capsys.readouterr().err


@pytest.mark.gpu
def test_cli_end_to_end(tmp_path, capsys):
    out = str(tmp_path)
    assert cli.main(["calibrate", "--lengths", "2048,4096,8192,16384,32768", "--samples", "60",
                     "--out", out]) == 0
    prof = json.load(open(os.path.join(out, "profile.json")))
    assert len(prof["calibration_points"]) == 5
    rows = list(csv.DictReader(open(os.path.join(out, "calibrate.csv"))))
    assert all(abs(float(r["skip"]) - 0.6) <= 0.03 for r in rows)
    assert cli.main(["bench", "--lengths", "16384,65536", "--plant-sink-frac", "0.625",
                     "--steps", "32", "--out", out]) == 0
    b = json.load(open(os.path.join(out, "bench.json")))
    for row in b["rows"]:
        assert row["skip_ratio"] == 0.625
        assert row["kv_floats_routed"] * 8 == row["kv_floats_dense"] * 3  # counter coherence
        assert row["speedup"] > 1.0
    assert list(csv.DictReader(open(os.path.join(out, "bench.csv"))))[0].keys() == \
        set(cli.CSV_COLUMNS["bench"])
    assert cli.main(["route-eval", "--lengths", "8192", "--samples", "2", "--out", out]) == 0
    r = json.load(open(os.path.join(out, "route-eval.json")))
    assert r["auprc"] == 1.0 and "0.55" in r["operating_points"]
    assert cli.main(["selftest"]) == 0
    assert "selftest: ok" in capsys.readouterr().out


@pytest.mark.gpu
def test_selftest_reports_injected_tie_fault(capsys, monkeypatch):
    """with the tie-breaking test hook forced on, selftest
    reports the routing-semantics failure and exits 1 (flag or env var)."""
    assert cli.main(["selftest", "--inject-tie-fault"]) == 1
    out = capsys.readouterr().out
    assert "FAIL  routing semantics: an exact tie routes Active (strict >)" in out
    assert "selftest: FAILED" in out
    monkeypatch.setenv("SINKR_INJECT_TIE_FAULT", "1")
    assert cli.main(["selftest"]) == 1
    assert "routing semantics" in capsys.readouterr().out.split("FAILED:")[1]
