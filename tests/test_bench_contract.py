"""CPU: the bench line contract, checked on the committed GPU evidence
(profiles/bench_r02j.json, written by `python bench.py` on a B200) and on
bench.py's reference arm entry point -- the keys the driver and the judge
read, their units and their internal consistency."""
from __future__ import annotations

import json
import os

from conftest import ROOT

LINE = os.path.join(ROOT, "profiles", "bench_r02j.json")


def _line():
    with open(LINE) as fh:
        return json.loads(fh.read().strip().splitlines()[-1])


def test_bench_line_has_the_contract_keys():
    d = _line()
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "clocks", "e2e", "gpu_launches", "roofline", "cpu_baseline"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["warmup"] >= 3 and d["higher_is_better"] is True
    assert d["unit"] == "evals/s" and d["dtype"] == "f64" and d["vs_baseline"] is None
    assert d["gpu_launches"] > 0
    assert "workload" in d["config"] and "l2" in d["config"]
    assert set(d["e2e"]) >= {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"}
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}


def test_bench_line_is_consistent():
    d = _line()
    evals = d["config"]["evals_per_step"]
    assert evals == d["config"]["m"] * d["config"]["p"]
    # value = evals per step / step time; the e2e rate cannot exceed the device-timed one by more than noise
    assert abs(d["value"] - evals / (d["ms_per_step"] * 1e-3)) <= 1e-6 * d["value"]
    assert d["e2e"]["value"] <= 1.01 * d["value"]
    r = d["roofline"]
    assert r["unit"] == "TFLOP/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12
    # achieved = ops per eval x evals per second of the kernel alone
    assert abs(r["achieved"] - r["ops_per_eval"] * evals / (r["kernel_ms"] * 1e-3) / 1e12) <= 1e-9 * r["achieved"]
    assert 0.0 < r["share_of_step"] <= 1.0
    c = d["cpu_baseline"]
    assert c["kind"] == "reference" and c["cores"] >= 1 and c["unit"] == d["unit"]
    assert d["time_to_epsrel_headline"]["cpu_reference"]["iterations"] == \
        d["time_to_epsrel_headline"]["gpu_compat"]["iterations"]


def test_reference_arm_prints_the_same_workload(monkeypatch, capsys):
    """bench.py --impl reference on rank 1 of a multi-rank launch does no
    work (rank 0 alone times the reference)."""
    import sys

    sys.path.insert(0, ROOT)
    import bench

    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--impl", "reference", "--gpus", "2"])
    assert bench.main() == 0
    assert capsys.readouterr().out == ""
