"""The bench.py contract on the GPU: one JSON line with every key the driver and the judge read
(metric/value/unit/..., roofline, cpu_baseline, e2e, clocks, gpu_launches), with consistent
values.  A short run (few steps, small CPU budget)."""
import json
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_bench_json_contract():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "5", "--warmup", "3",
                        "--no-cmp", "--no-fs", "--cpu-seconds", "1", "--e2e-steps", "2"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "clocks", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] >= 3 and d["scaling"] == "weak"
    assert d["higher_is_better"] is True and d["dtype"] == "u8" and d["value"] > 0
    assert d["gpu_launches"] == 5                      # one search launch per timed step
    assert "workload" in d["config"]
    rf = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in rf, k
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9 and 0 < rf["frac"] < 1
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert e2e["value"] < d["value"]                   # host copies inside the timed region
    ck = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(ck)
    # value = blocks of all pairs / time per step
    cfg = d["config"]
    assert abs(d["value"] - cfg["pairs_per_gpu"] * cfg["blocks_per_pair"] / (d["ms_per_step"] * 1e-3)) < 1e-6 * d["value"]


def test_bench_graph_mode_small_config():
    """--graph: the timed steps replayed from one CUDA graph (small, launch-bound configs)."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c1", "--graph",
                        "--steps", "20", "--warmup", "3", "--no-cmp", "--no-fs", "--no-e2e", "--no-cpu"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")][0])
    assert d["config"]["cuda_graph"] is True and d["gpu_launches"] == 20 and d["value"] > 0
    assert "L2-resident" in d["config"]["l2"]
