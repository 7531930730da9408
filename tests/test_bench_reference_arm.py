"""CPU: bench.py --impl reference runs the reference's CPU path on the host
alone -- no GPU, no libhalfgnn.so -- and prints the contract's JSON line."""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.timeout(600)
def test_reference_arm_is_product_free():
    code = (
        "import sys, runpy, json\n"
        f"sys.argv = ['bench.py', '--impl', 'reference', '--workload', 'gat-pubmed', "
        "'--steps', '1', '--warmup', '1']\n"
        "runpy.run_path('bench.py', run_name='__main__')\n"
        "import paper_2411_01109_b200._native as nat\n"
        "assert nat._lib is None, 'reference arm loaded libhalfgnn.so'\n"
        "import torch\n"
        "assert not torch.cuda.is_initialized()\n")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         cwd=ROOT, timeout=550, env={"PATH": "/usr/bin:/bin",
                                                     "CUDA_VISIBLE_DEVICES": "",
                                                     "HOME": "/root"})
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1
    assert set(cb["core_counts"]) == {"os_cpu_count", "sched_affinity", "torch_threads"}
    assert d["e2e"]["h2d_bytes_per_step"] == 0
