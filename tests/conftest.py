"""Shared fixtures.  `-m gpu` tests need a B200 and the built libhalfgnn.so;
everything else runs on CPU (oracle vs golden vectors, host logic, gloo)."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = Path(__file__).resolve().parent / "golden"
for p in (str(ROOT),):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libhalfgnn.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def load_golden(name):
    with np.load(GOLDEN / name, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def golden_cases(name):
    d = load_golden(name)
    out = []
    for i in range(int(d["num_cases"])):
        pre = f"c{i}_"
        out.append({k[len(pre):]: v for k, v in d.items() if k.startswith(pre)})
    return out, d


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint16 if a.dtype == np.float16 else np.uint32)


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2411_01109_b200 import _native

    _native.lib()  # loud failure if the library is missing
    return torch.device("cuda:0")
