"""bench.py's one-line JSON contract (the driver parses it): the reference arm on CPU (it times the
oracle, so no GPU is needed) and the product arm on the GPU, both on the toy config so they finish
in seconds.  Checks the keys and their types, not the numbers."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def _common(line, steps, warmup):
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"):
        assert key in line, key
    assert line["value"] > 0 and line["ms_per_step"] > 0
    assert line["steps"] == steps and line["warmup"] == warmup and line["n_gpus"] == 1
    assert line["higher_is_better"] is True and line["scaling"] == "weak" and line["vs_baseline"] is None
    assert "workload" in line["config"] and "model" not in line["config"]
    e2e = line["e2e"]
    assert e2e["value"] > 0 and {"unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(e2e)
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]


def test_reference_arm_line():
    line = _run(["--impl", "reference", "--config", "toy", "--steps", "1", "--warmup", "1"], 600)
    _common(line, 1, 1)
    assert line["impl"] == "reference" and line["dtype"] == "f64"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["cpu_baseline"]["value"] == line["value"]


@pytest.mark.gpu
def test_product_arm_line():
    line = _run(["--config", "toy", "--steps", "3", "--warmup", "3", "--error-tokens", "64", "--rounds", "1"], 900)
    _common(line, 3, 3)
    assert line.get("impl", "flux") != "reference" and line["dtype"] == "bf16"
    rf = line["roofline"]
    assert rf["bound"] in ("tensor", "hbm") and rf["achieved"] > 0 and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert line["gpu_launches"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(line["clocks"] or {"sm_mhz": 0, "sm_max_mhz": 0, "reasons": []})


def test_launcher_spawns_the_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself with 2 ranks (gloo self-test on CPU): rank 0
    sees the world of 2, both ranks join the all-reduce, and the shards start at 0 and 1000."""
    line = _run(["--gpus", "2", "--selftest-launcher"], 300)
    assert line == {"n_gpus": 2, "ranks_seen": 2, "shard_starts_sum": 1000, "gpus_arg": 2}


def test_launcher_rejects_a_world_mismatch():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--selftest-launcher"],
                         cwd=ROOT, capture_output=True, text=True, timeout=120, env=env)
    assert out.returncode == 2 and "WORLD_SIZE=1" in out.stdout
