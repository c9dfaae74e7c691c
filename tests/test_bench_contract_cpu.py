"""The bench line contract (keys the driver and the judge read), checked on the committed final
bench lines (profiles/r02_bench_repeats.jsonl, profiles/r02_bench_reference_arm.json) so a change to
bench.py's JSON assembly that drops a key shows up here, without a GPU."""

import json
from pathlib import Path

import pytest

PROF = Path(__file__).resolve().parents[1] / "profiles"


def _lines():
    return [json.loads(l) for l in (PROF / "r02_bench_repeats.jsonl").read_text().splitlines() if l.strip()]


def test_device_line_keys_and_sanity():
    for d in _lines():
        for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                  "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
            assert k in d, k
        assert d["metric"] == "refined seed trajectories/sec" and d["higher_is_better"] is True
        assert d["scaling"] in ("weak", "strong") and d["warmup"] >= 3 and d["steps"] >= 1
        assert "workload" in d["config"]
        r = d["roofline"]
        for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
            assert k in r, k
        assert abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-9
        e = d["e2e"]
        assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and e["value"] > 0
        assert d["gpu_launches"] > 0
        c = d["clocks"]
        assert "sm_mhz" in c and "reasons" in c
        assert not {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"} & set(c["reasons"])
        # value = trajectories of the job / time of a step
        P, S = d["config"]["problems"], d["config"]["seeds"]
        assert d["value"] == pytest.approx(P * S / (d["ms_per_step"] / 1e3), rel=1e-6)
    assert _lines()[0]["cpu_baseline"]["cores"] >= 1


def test_reference_arm_line():
    d = json.loads((PROF / "r02_bench_reference_arm.json").read_text())
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["metric"] == _lines()[0]["metric"] and d["unit"] == _lines()[0]["unit"]
