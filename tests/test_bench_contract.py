"""The bench.py JSON contract the driver depends on: one line, the required keys, both arms.
The reference arm runs on CPU (bounded sample); the b200 arm needs the GPU."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
             "cpu_baseline", "gpu_launches"}


def run_bench(*flags):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *flags],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    from oracle import oracle
    oracle.build()
    d = run_bench("--impl", "reference", "--scale", "12", "--steps", "1", "--warmup", "0",
                  "--cpu-target", "2000")
    assert d["impl"] == "reference" and BASE_KEYS <= set(d)
    assert d["metric"] == "hsaw_per_sec" and d["unit"] == "HSAW/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"] == d["e2e"]["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["gpu_launches"] == 0 and "workload" in d["config"]


@pytest.mark.gpu
def test_b200_arm_line():
    d = run_bench("--scale", "14", "--batches", "16384", "--steps", "3", "--warmup", "3",
                  "--cpu-target", "20000")
    assert "impl" not in d and BASE_KEYS <= set(d)
    assert d["metric"] == "hsaw_per_sec" and d["value"] > 0 and d["n_gpus"] == 1
    assert d["higher_is_better"] is True and d["scaling"] == "weak" and d["vs_baseline"] is None
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["achieved"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["value"] != d["value"]
    c = d["cpu_baseline"]
    assert c["value"] > 0 and c["cores"] >= 1 and c["kind"] in ("reference", "port") and c["sample"]
    assert d["gpu_launches"] > 0 and {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert "workload" in d["config"] and "model" not in d["config"]
    assert d["esia"]["passed_check"] in (True, False) and d["esia"]["same_result_e2e"] is True
    # the legs either side of the path: forward simulation of the solution, the k = 1000 solve
    s = d["suspension"]
    assert "error" not in s and s["paired_runs_per_sec"] > 0 and s["mean_residual"] <= s["mean_full"]
    assert s["estimate"]["runs"] >= 1 and s["cpu_baseline"]["runs_per_sec"] > 0
    assert d["esia_k1000"]["k"] == 1000 and d["esia_k1000"]["seconds_to_solution"] > 0
