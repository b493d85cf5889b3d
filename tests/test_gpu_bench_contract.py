"""The GPU arm of bench.py prints one JSON line with the keys the driver and
the judge read (round-2 contract: strong scaling, e2e over the same steps,
roofline with both models, top-level Gamma / Gibbs fields, clocks)."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpu_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--small", "--steps", "3",
                        "--warmup", "3", "--no-cpu-baseline"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "roofline",
              "e2e", "gpu_launches", "clocks", "breakdown", "gamma_cfg3", "gibbs_cfg5",
              "determinism"):
        assert k in d, k
    assert d["scaling"] == "strong" and d["n_gpus"] == 1 and d["steps"] == 3
    roof = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic", "models"):
        assert k in roof, k
    assert set(roof["models"]) == {"pipe", "issue_survey_8d"}
    assert abs(roof["frac"] - roof["achieved"] / roof["peak"]) < 1e-3
    e = d["e2e"]
    assert e["steps"] == 3 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] == 8 * 3 and d["determinism"]["identical_across_steps"]
    assert d["device_errors"] == 0
    assert "--small" in d["config"]["workload"] or "NOT a bench number" in d["config"]["workload"]
