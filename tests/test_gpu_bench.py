"""bench.py's JSON line on a real GPU: the contract keys (metric, value, roofline, cpu_baseline,
e2e, gpu_launches, clocks, ...) on a small config, for the default (replicas) and --sharded
modes."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)


def run_bench(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    return json.loads(lines[0])


def test_bench_line_contract():
    d = run_bench("--config", "2", "--steps", "5", "--warmup", "3", "--cpu-sample", "200000",
                  "--full-key-steps", "1", "--e2e-steps", "1")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] >= 3 and d["value"] > 0
    assert d["config"]["workload"] == "cfg2_uint64_clusters"
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and rf["achieved"] > 0 and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] > 0 and cb["cores"] >= 1 and cb["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 16_000_000 * 8 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}


def test_bench_line_paths_and_ratios():
    d = run_bench("--config", "5", "--steps", "4", "--warmup", "3", "--no-cpu-baseline", "--no-e2e",
                  "--full-key-steps", "1")
    pr = d["path_roofline"]
    # the whole path on the work actually run: between the dominant kernel's bytes and the
    # full-width formula's
    assert 0 < pr["actual_bytes_per_key"] < sum(pr["formula_bytes_per_key"].values())
    assert 0 < pr["actual_frac_of_peak"] < 1.0
    ps = d["paper_stats"]
    for mode in ("single_sort", "by_prefixes"):
        assert ps[mode]["total_ratio"] > 1.0 and ps[mode]["full_key_passes"] > ps[mode]["compressed_passes"]
    assert d["rebuild"]["verified_ms_per_step"] >= d["rebuild"]["ms_per_step"] * 0.9


def test_bench_sharded_line():
    d = run_bench("--config", "2", "--steps", "3", "--warmup", "3", "--sharded", "--e2e-steps", "1")
    assert d["value"] > 0 and d["config"]["n_total"] == d["config"]["n_per_rank"] and d["gpu_launches"] > 0
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 16_000_000 * 8
