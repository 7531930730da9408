"""Pinned host -> device copy bandwidth on this box (the bound of bench.py's
e2e leg, which copies each epoch's features from pinned host memory)."""
import json

import torch

out = {}
for mb in (64, 283, 1024):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        d.copy_(h, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    out[f"{mb}MB"] = round(n * 10 / (e0.elapsed_time(e1) / 1e3) / 1e9, 2)
print(json.dumps({"h2d_GBps": out}))
