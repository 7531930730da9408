"""Dev tool: time the fp32-guarded SpMM (and the reference-order kernel) on the
Reddit-shaped graph over F = 16..512, CUDA events, L2 flushed between reps."""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2411_01109_b200 import device as D  # noqa: E402
from paper_2411_01109_b200 import graphgen  # noqa: E402


def peak_hbm():
    p = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"
    try:
        return json.loads(p.read_text())["hbm_gbs"] * 1e9
    except Exception:
        return 6.65e12


def timeit(fn, reps, flush):
    ts = []
    for _ in range(reps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) / 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--feats", default="16,32,64,128,256,512")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--ref", action="store_true")
    ap.add_argument("--cap", type=int, default=512)
    ap.add_argument("--scale", type=float, default=1.0)
    args = ap.parse_args()
    t0 = time.time()
    n = int(graphgen.REDDIT_N * args.scale)
    e = int(graphgen.REDDIT_E * args.scale)
    dg = graphgen.reddit_like(0, n=n, e=e)
    torch.cuda.synchronize()
    print(f"graph N={dg.n} E={dg.num_edges} built in {time.time() - t0:.1f}s", flush=True)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    peak = peak_hbm()
    N, E = dg.n, dg.num_edges
    for f in map(int, args.feats.split(",")):
        x = torch.randn(N, f, device="cuda", dtype=torch.float16)
        fn = lambda: D.spmm(dg, x, None, "discretized", "both")  # noqa: E731
        fn()
        t = timeit(fn, args.reps, flush)
        byts = 4 * E + 8 * (N + 1) + 2 * f * E + 2 * f * N
        row = {"F": f, "ms": t * 1e3, "GBps": byts / t / 1e9, "frac": byts / t / peak}
        if args.ref:
            fr = lambda: D.spmm_edge_ref(dg, x, None, "discretized", "both")  # noqa: E731
            fr()
            tr = timeit(fr, max(2, args.reps // 2), flush)
            row.update(ref_ms=tr * 1e3, ref_GBps=byts / tr / 1e9)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
