"""The B200 arm of bench.py at a reduced size (`--scale`, tuning-only switch): the JSON line the
driver parses carries every key of the contract, the parity sample is green, the e2e leg's host
results equal the device-resident sweep's, and the torchrun launch path (one rank, NCCL
initialised) prints the same line."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks", "parity")


def _line(cmd, timeout=900):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [x for x in res.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    return json.loads(lines[0])


def test_default_arm_json_line_small_scale():
    d = _line([sys.executable, "bench.py", "--scale", "0.02", "--steps", "3", "--warmup", "3", "--e2e-steps", "1",
               "--no-sustained"])
    for k in KEYS:
        assert k in d, k
    assert d["config"]["workload"].startswith("config5") and d["n_gpus"] == 1 and d["dtype"] == "f64"
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["higher_is_better"] is True
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "frac_8tbs", "traffic"):
        assert k in r, k
    assert r["bound"] == "hbm" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    assert d["parity"]["ok"] and d["parity"]["max_rel_err"] <= 1e-12
    e = d["e2e"]
    assert e["matches_device_run"] and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert 0 < e["value"] < d["value"]  # host buffers, copies inside the timed region
    c = d["cpu_baseline"]
    assert c["kind"] == "port" and c["cores"] >= 1 and c["value"] > 0
    assert d["nonfinite_flag"] is False


def test_torchrun_single_rank_small_scale():
    d = _line([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr",
               "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "1", "--scale", "0.02", "--steps", "2",
               "--warmup", "3", "--no-e2e", "--no-cpu", "--no-sustained"])
    assert d["n_gpus"] == 1 and d["parity"]["ok"] and d["gpu_launches"] > 0
