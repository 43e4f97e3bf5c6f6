"""bench.py: the algorithmic byte counts behind `roofline` (CPU) and the JSON line contract (GPU)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_algorithmic_bytes_per_token():
    """per compressed token and side 4D (f32 mean) + H*D*b/8 (codes) + 8H (scale, min)."""
    import bench

    assert bench.tok_bytes(4) == 4 * 128 + 8 * 64 + 64 == 1088
    assert bench.tok_bytes(2) == 4 * 128 + 8 * 32 + 64 == 832
    assert bench.tok_bytes(8) == 4 * 128 + 8 * 128 + 64 == 1600
    # one launch: both sides of every compressed token, residual rows as bf16, q and out
    bench.use_config(2)
    assert bench.attn_alg_bytes(4, 16, 32768, 0) == 16 * (2 * 32768 * 1088 + 2 * 32 * 128 * 2)
    assert bench.attn_alg_bytes(4, 16, 32768, 10) - bench.attn_alg_bytes(4, 16, 32768, 0) == 16 * 2 * 10 * 8 * 128 * 2


def test_configs_match_baseline():
    import bench

    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert base["metric"]
    assert set(bench.CONFIGS) == {2, 4, 5}
    assert bench.CONFIGS[2]["plan"] == [8] * 2 + [4] * 22 + [2] * 8
    assert all(len(c["plan"]) == c["L"] for c in bench.CONFIGS.values())


@pytest.mark.gpu
def test_bench_json_line():
    """A short run of config 4 prints one JSON line with every key the driver reads."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "4", "--steps", "3", "--warmup", "3",
                        "--no-cpu"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert r.returncode == 0 and len(lines) == 1, r.stderr[-2000:]
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "clocks", "roofline", "cpu_baseline"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["gpu_launches"] > 0
    assert "workload" in d["config"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] < 1.2
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
