"""The bench.py contract on the GPU: one JSON line with every key the driver reads,
the timing rules (warm-up >= 3, device timing, L2 flush named in config), the
roofline / cpu_baseline / e2e / clocks / gpu_launches objects, and the oracle arm."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("cfg", ["c1", "c3", "c4"])
def test_bench_line_keys(cfg):
    d = _line("--config", cfg, "--steps", "2", "--warmup", "3")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks",
              "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["config"]["workload"] == cfg
    assert "l2" in d["config"]
    r = d["roofline"]
    if cfg == "c1":   # one pair on one SM: latency-bound, reported per iteration
        assert r["bound"] == "latency" and r["unit"] == "us/iteration" and r["achieved"] > 0
    else:             # the streaming kernels: HBM roofline, both denominators
        assert r["bound"] == "hbm" and 0 < r["frac"] < 1 and r["peak"] > 0
        assert abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-9
        assert abs(r["achieved"] / 8000.0 - r["frac_nominal"]) < 1e-9
        assert d["hbm_gbs"] == pytest.approx(r["achieved"])
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] > 0 and cb["cores"] >= 1 and cb["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= d["steps"]
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}


def test_bench_default_is_c3():
    """The driver's line (no --config) is the largest single-GPU config, C3."""
    d = _line("--steps", "1", "--warmup", "3", "--no-cpu-baseline", "--no-e2e")
    assert d["config"]["workload"] == "c3" and d["roofline"]["bound"] == "hbm"


def test_bench_reference_arm():
    d = _line("--impl", "reference", "--steps", "1", "--warmup", "3", "--config", "c1")
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
