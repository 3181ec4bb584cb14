"""bench.py's reference arm (`--impl reference`) runs the unmodified reference CPU path
(oracle/_ref, or the oracle port) — no GPU needed — so its JSON-line contract is checked here:
the driver computes the headline ratio from this line and our arm's."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=600, env=e, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    return [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]


def test_reference_arm_json_line():
    lines = run_bench("--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "1")
    assert len(lines) == 1
    d = lines[0]
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 1 and d["higher_is_better"] is True
    assert d["unit"] == "TOPS" and d["value"] > 0 and d["config"]["M"] == 1024
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_exit_quietly():
    """Under torchrun only rank 0 prints the reference line; the others exit 0 without work."""
    lines = run_bench("--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "1",
                      env={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert lines == []


@pytest.mark.gpu
def test_our_arm_json_line():
    """Our arm on a short config-1 run: the keys the driver and the judge read."""
    lines = run_bench("--config", "c1", "--steps", "3", "--warmup", "3")
    assert len(lines) == 1
    d = lines[0]
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0 and d["gpu_launches"] >= 3
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and 0 < r["frac"] and r["peak"] > 0 and r["unit"] in ("GB/s", "TOPS")
    assert d["e2e"]["h2d_bytes_per_step"] == 2 * 1024 * 1024 and d["e2e"]["d2h_bytes_per_step"] == 4 * 1024 * 1024
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["kind"] in ("reference", "port")
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


def test_reference_arm_config_and_data_match_ours():
    """The driver compares the two arms' `config` (same_config) and `data`: both come from the
    same functions (bench.config_dict / bench.data_desc), the reference arm's line must equal what
    our arm prints for the same arguments, and both arms draw the same seeded inputs."""
    import argparse
    import numpy as np
    sys.path.insert(0, ROOT)
    import bench
    lines = run_bench("--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "1")
    d = lines[0]
    args = argparse.Namespace(shape=None, config="c1", mode="exact", adist="uniform", bdist="auto")
    assert d["config"] == bench.config_dict(args, 1)
    assert d["data"] == bench.data_desc(args, 1024)
    a1, a2 = bench.gen_a(64, 100, "uniform"), bench.gen_a(64, 100, "uniform")
    assert np.array_equal(a1, a2) and a1.dtype == np.uint8
    b = bench.gen_b(50, 100, "normal")
    assert b.dtype == np.int8 and abs(float(b.astype(np.float64).std()) - 32.0) < 3.0
