"""GPU: bench.py keeps the driver's JSON-line contract (one line, the keys the
driver and the judge read), on the small C2 workload so it runs in seconds."""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.timeout(600)
def test_bench_json_line_contract(cuda):
    out = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--workload", "gat-pubmed", "--steps", "3",
         "--warmup", "3", "--no-cpu-baseline"],
        capture_output=True, text=True, cwd=ROOT, timeout=550)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "clocks", "e2e", "gpu_launches", "roofline"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["higher_is_better"] is False
    assert "workload" in d["config"]
    assert d["gpu_launches"] > 0
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in r, key
    assert r["bound"] in ("hbm", "tensor") and r["peak"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


@pytest.mark.timeout(900)
def test_bench_spawns_ranks_for_gpus_flag(cuda):
    """`bench.py --gpus 2` without torchrun launches two ranks itself and reports
    n_gpus 2 (validated with both ranks on this one GPU over gloo)."""
    import os

    env = dict(os.environ, HG_DIST_SHARED_GPU="1", HG_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--workload", "gat-pubmed",
         "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--reorder", "degree"],
        capture_output=True, text=True, cwd=ROOT, timeout=850, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2
    assert d["config"]["vertex_order"].startswith("degree-sorted")
    ex = d["exchange"]
    assert ex["recv_bytes_per_rank_per_step_max"] > 0
    assert ex["n_rows_max_over_mean"] <= 1.5
