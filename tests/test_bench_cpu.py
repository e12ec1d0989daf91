"""bench.py's roofline accounting on CPU: the pipe that
bounds each kernel, per-mode sums for the small-mode precontraction, frac <= 1 for a
measured time at or above the roof."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_tc_path_is_fp64_bound(bench):
    info = {"tensor_cores": True, "modes": [{"smp": 0}] * 3}
    r = bench.roofline(3, 10, "F32-B", info, 1, 148, 1965.0, 1e8, 4.2e-3, "f32", "c5")
    assert r["pipe"] == "fp64" and r["work_per_entry"]["fp64_fma"] == 100 + 66
    # 166 fp64 FMAs x 1e8 entries at 148 x 64 x 2 x 1.965 GHz = 0.892 ms
    assert abs(r["roof_ms"] - 0.8919) < 1e-3
    assert abs(r["frac"] - r["roof_ms"] / 4.2) < 1e-9


def test_alu_path_counts_ttv_chain(bench):
    info = {"tensor_cores": False, "modes": [{"smp": 0}] * 5}
    r = bench.roofline(5, 5, "F32-C", info, 1, 148, 1965.0, 1e7, 6e-3, "f32", "c4")
    # inner J^N = 3125 fp32; the outer levels 25 + 125 + 625 in fp64 (F32-C) + 21 (B, c, x^2)
    assert r["work_per_entry"]["fp32_fma"] == 3125
    assert r["work_per_entry"]["fp64_fma"] == 25 + 125 + 625 + 21
    assert r["pipe"] == "fp32"


def test_smp_modes_use_the_shipped_work(bench):
    info = {"tensor_cores": False, "modes": [{"smp": 2}, {"smp": 2}, {"smp": 1}, {"smp": 1}]}
    mode_s = [1.9e-3, 1.7e-3, 3.2e-3, 3.2e-3]
    r = bench.roofline(4, 10, "F32-C", info, 1, 148, 1965.0, 2e7, sum(mode_s) / 4, "f32", "c3", mode_s)
    kinds = [m["smp"] for m in r["per_mode"]]
    assert kinds == [2, 2, 1, 1]
    assert r["per_mode"][0]["fp64_fma"] == 100 + 66 and r["per_mode"][2]["fp32_fma"] == 1000
    assert 0 < r["frac"] <= 1.0
    assert abs(r["frac"] - r["roof_ms"] / (sum(mode_s) * 1e3)) < 1e-9


def test_smp_table_mode_on_tensor_cores(bench):
    info = {"tensor_cores": False, "modes": [{"smp": 2}, {"smp": 2}, {"smp": 1, "tc_table": True},
                                             {"smp": 1, "tc_table": True}]}
    mode_s = [1.9e-3, 1.7e-3, 2.4e-3, 2.4e-3]
    r = bench.roofline(4, 10, "F32-C", info, 1, 148, 1965.0, 2e7, sum(mode_s) / 4, "f32", "c3", mode_s)
    m2 = r["per_mode"][2]
    assert m2["fp32_fma"] == 0 and m2["tc_mac"] == 1000 and m2["fp64_fma"] == 166 and m2["pipe"] == "fp64"
    assert 0 < r["frac"] <= 1.0


def test_reference_arm_json_line():
    """`bench.py --impl reference` (the oracle arm, CPU only) prints one JSON line with the
    contract's keys; its e2e and cpu_baseline describe the same run."""
    import json
    import subprocess
    import sys
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                        "--steps", "1", "--warmup", "1", "--ref-seconds", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    d = json.loads(line)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    # every step is one sampled iteration: ms_per_step is what ran, and the sample says how much
    assert d["sample"]["steps_timed"] == 1 and 0 < d["sample"]["fraction_of_full_iteration"] <= 1
    assert d["ms_per_step"] * d["steps"] / 1e3 <= d["sample"]["timed_wall_s"] + 1e-6
