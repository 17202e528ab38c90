"""bench.py's JSON-line contract: the reference arm on CPU (C1, one step) and
the GPU arm on a small configuration (C1) with every key the driver and the
judge read."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "0"])
    assert d["impl"] == "reference" and d["unit"] == "DOF*stages/s" and d["value"] > 0
    for key in ("metric", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling", "dtype",
                "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["config"]["N_dof"] == 7840 and d["cpu_baseline"]["kind"] == "port"
    assert d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["parity"]["manufactured_max_rel"] < 1e-9


@pytest.mark.gpu
def test_gpu_arm_line():
    d = _run(["--config", "C1", "--steps", "4", "--warmup", "3"])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "kernels",
                "solve", "parity", "clocks", "cpu_baseline"):
        assert key in d, key
    assert d["steps"] == 4 and d["warmup"] == 3 and d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and 0 < r["frac"] < 1 and r["peak"] > 0
    assert any(k["kernel"].startswith("k_leaf_fd_mma") for k in d["kernels"])
    assert d["parity"]["ok"] and d["parity"]["sample_rel_l2"] < 1e-10
    assert d["cpu_baseline"]["value"] > 0
