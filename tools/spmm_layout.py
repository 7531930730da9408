"""SpMM feature-row layout experiment on the Reddit-shaped graph: F columns
stored densely (row = 2F bytes) vs in rows padded to a 128-byte multiple (the
kernel reads F columns through the row stride).  L2 flushed between reps."""
from __future__ import annotations

import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2411_01109_b200 import device as D  # noqa: E402
from paper_2411_01109_b200 import graphgen  # noqa: E402


def timed(fn, reps=5):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    dg = graphgen.reddit_like(0)
    view = dg.view(False)
    fin, fout = dg.norm_tables("both", False, torch.float16)
    for f in map(int, (sys.argv[1] if len(sys.argv) > 1 else "16,24,32,40,48,56,64,96").split(",")):
        ld = (f + 63) // 64 * 64
        dense = torch.randn(dg.n, f, device="cuda", dtype=torch.float16)
        wide = torch.zeros(dg.n, ld, device="cuda", dtype=torch.float16)
        wide[:, :f] = dense
        yd = D.spmm_csr(view, dense, scaling="discretized", fout=fout)
        yw = D.spmm_csr(view, wide[:, :f], scaling="discretized", fout=fout)
        assert torch.equal(yd, yw)
        rec = {"F": f, "ld": ld,
               "dense_ms": round(timed(lambda: D.spmm_csr(view, dense, scaling="discretized", fout=fout)), 4),
               "padded_ms": round(timed(lambda: D.spmm_csr(view, wide[:, :f], scaling="discretized", fout=fout)), 4)}
        if ld != f:
            rec["full_ld_ms"] = round(timed(lambda: D.spmm_csr(view, wide, scaling="discretized", fout=fout)), 4)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
