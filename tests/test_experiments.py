"""trunkctl-compatible scaling report: experiments.py
mirrors gnnmpc.experiments.run_scaling_sweep / loglog_slope and
gnnmpc.cli.cmd_scaling / _write_summary (cli.py:263-299, :31-46)."""

import csv
import json

import numpy as np
import pytest

from paper_2602_17601_b200 import experiments as ex

REF_HEADER = "node_count,threads,linearize_ms,condense_ms,solve_ms,condense_peak_mb"  # cli.py:276


def test_loglog_slope_known_answers():
    x = [16, 32, 64, 128]
    assert ex.loglog_slope(x, [3.0 * v ** 1.5 for v in x]) == pytest.approx(1.5, abs=1e-12)
    assert ex.loglog_slope(x, [7.0] * 4) == pytest.approx(0.0, abs=1e-12)


def test_config_hash_is_canonical_sha256():
    a = ex.config_hash({"m_list": [16, 32], "reps": 3})
    b = ex.config_hash({"reps": 3, "m_list": [16, 32]})
    assert a == b and len(a) == 16
    import hashlib

    assert a == hashlib.sha256(b'{"m_list":[16,32],"reps":3}').hexdigest()[:16]


def test_report_files_in_reference_format(tmp_path):
    rows = [ex.ScalingRow(16, 1.0, 2.0, 3.0, 4.0), ex.ScalingRow(32, 1.5, 4.1, 3.2, 8.0)]
    ex.write_scaling_csv(tmp_path / "scaling.csv", [(rows, 1), (None, 8)])
    lines = (tmp_path / "scaling.csv").read_text().splitlines()
    assert lines[0] == REF_HEADER
    assert lines[1] == "16,1,1,2,3,4" and lines[2] == "32,1,1.5,4.1,3.2,8"
    m = ex.scaling_metrics(rows)
    assert set(m) == {"m_list", "condense_ms_single", "condense_time_slope_single", "condense_memory_slope",
                      "linearize_ms_single", "solve_ms_single"}
    assert m["condense_memory_slope"] == pytest.approx(1.0)
    s = ex.write_summary(tmp_path, "scaling", {"reps": 1}, 0, m, ["scaling.csv"])
    on_disk = json.loads((tmp_path / "summary.json").read_text())
    assert on_disk == s and list(on_disk) == ["command", "config_hash", "seed", "metrics", "artifacts"]


@pytest.mark.gpu
def test_scaling_report_on_gpu(tmp_path):
    metrics = ex.cmd_scaling({"m_list": [16, 32], "reps": 1, "horizon": 5}, tmp_path, seed=0)
    rows = list(csv.DictReader(open(tmp_path / "scaling.csv")))
    assert [int(r["node_count"]) for r in rows] == [16, 32]
    assert all(float(r["condense_ms"]) > 0 and float(r["solve_ms"]) > 0 for r in rows)
    dev = list(csv.DictReader(open(tmp_path / "scaling_device.csv")))
    assert all(r["status"] == "optimal" for r in dev)
    assert np.isfinite(metrics["condense_time_slope_single"])
    assert np.isfinite(metrics["device"]["step_time_slope"])
    summ = json.loads((tmp_path / "summary.json").read_text())
    assert summ["command"] == "scaling" and summ["artifacts"] == ["scaling.csv", "scaling_device.csv"]
