"""The driver's bench.py contract, checked on the committed bench lines of
the latest round (profiles/r*/bench.json, bench_ref.json) -- CPU only."""

import json
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
ROUNDS = sorted((ROOT / "profiles").glob("r*/bench.json"))


def latest(name):
    if not ROUNDS:
        pytest.skip("no committed bench line yet")
    return json.loads((ROUNDS[-1].parent / name).read_text().strip().splitlines()[-1])


def test_ours_line_has_every_contract_key():
    d = latest("bench.json")
    base = json.loads((ROOT / "BASELINE.json").read_text())
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "e2e", "gpu_launches", "roofline", "cpu_baseline", "clocks"):
        assert k in d, k
    assert d["metric"] == base["metric"]
    assert d["warmup"] >= 3 and d["steps"] >= 1 and d["value"] > 0
    assert d["scaling"] in ("weak", "strong") and d["higher_is_better"] is True
    assert "workload" in d["config"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["value"] < d["value"]  # host copies inside the timed region
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["unit"] in ("GB/s", "TFLOP/s")
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    c = d["cpu_baseline"]
    assert c["kind"] in ("reference", "port") and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    assert d["gpu_launches"] > 0
    k = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(k)
    assert not {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"} & set(k["reasons"])


def test_reference_line_matches_ours():
    d, r = latest("bench.json"), latest("bench_ref.json")
    assert r["impl"] == "reference"
    for k in ("metric", "unit", "higher_is_better"):
        assert r[k] == d[k], k
    assert r["config"]["workload"] == d["config"]["workload"]
    assert r["e2e"]["h2d_bytes_per_step"] == 0 and r["e2e"]["value"] == r["value"]
    assert r["cpu_baseline"]["value"] == r["value"]
