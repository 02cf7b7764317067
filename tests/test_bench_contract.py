"""The bench.py JSON contract (the driver parses it): the reference arm on CPU,
and the GPU arm on the small config (gpu marker)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def run_bench(*args, timeout=900):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--config", "dd", "--steps", "2", "--warmup", "1")
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 1
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    # the driver divides the two arms: same metric, unit, direction and config
    assert d["metric"] == bench.METRIC and d["unit"] == "products/s" and d["higher_is_better"] is True
    assert d["config"] == bench.bench_config(bench.workload("dd"), "dd", 1)


@pytest.mark.gpu
def test_gpu_arm_line():
    d = run_bench("--config", "dd", "--steps", "3", "--warmup", "3")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks", "next_rows"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] >= 3 and d["higher_is_better"] is True
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["gpu_launches"] > 0
    assert d["metric"] == bench.METRIC and d["config"] == bench.bench_config(bench.workload("dd"), "dd", 1)
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert 0 < r["frac"] < 1 and abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-9
    assert 0 < d["ms_min"] <= d["ms_median"] and r["compulsory_gbs"] > 0 and r["fma_as_2_peak_tflops"] > r["peak"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    n = d["next_rows"]
    assert n["toeplitz_solve"]["ms"] > 0 and n["newton_step"]["ms"] > 0


def test_table1_equivalent_ops():
    """The paper-equivalent op count of one series product (PAPER.md:109-147
    Table 1 x the 2D(D+1) md mul + 2D^2 md add of SURVEY §8(a) a7) against
    SURVEY §8(a)'s per-config figures and BASELINE.md's totals."""
    # Table-1 ops per product dd 22,752; qd 891,904; od 16.70 M; deca 28.95 M
    assert bench.table1_ops_per_product(16, 2) == 22752
    assert bench.table1_ops_per_product(32, 4) == 891904
    assert round(bench.table1_ops_per_product(64, 8) / 1e6, 2) == 16.70
    assert round(bench.table1_ops_per_product(64, 10) / 1e6, 2) == 28.95
    # md add / mul totals per limb count (dd 20 / 23 ... deca 397 / 3,089)
    assert [bench.TABLE1_ADD[L] for L in (2, 3, 4, 5, 8, 10)] == [20, 35, 89, 122, 269, 397]
    assert [bench.TABLE1_MUL[L] for L in (2, 3, 4, 5, 8, 10)] == [23, 209, 336, 554, 1742, 3089]
    # 2D(D+1) real md mul + 2D^2 real md add, any D
    for D in (1, 9, 33, 128):
        for L in (2, 3, 4, 5, 8, 10):
            assert bench.table1_ops_per_product(D, L) == 2 * D * (D + 1) * bench.TABLE1_MUL[L] + \
                2 * D * D * bench.TABLE1_ADD[L]
