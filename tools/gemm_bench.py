"""Dense per-layer GEMMs of the benched configs on the tcgen05 kernels vs
cuBLAS: forward (hg_gemm_tc, bias fused) and weight gradient (hg_gemm_wgrad,
bias gradient fused) at the C3/C4/C5 shapes.  `--ncu`: run each kernel a few
times untimed (a target for `ncu -k regex:k_gemm`)."""
from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2411_01109_b200 import device as D  # noqa: E402

SHAPES = [(232_965, 608, 64), (232_965, 64, 48), (2_449_029, 112, 64), (2_449_029, 64, 64),
          (2_449_029, 64, 48), (16_777_216, 128, 128)]


def timed(fn, reps=10):
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
    return statistics.median(ts) * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ncu", action="store_true")
    ap.add_argument("--shapes", default="")
    args = ap.parse_args()
    torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = False
    shapes = SHAPES if not args.shapes else [SHAPES[int(i)] for i in args.shapes.split(",")]
    for m, k, n in shapes:
        a = torch.randn(m, k, device="cuda", dtype=torch.float16)
        w = (torch.randn(k, n, device="cuda", dtype=torch.float16) * 0.1)
        b = torch.randn(n, device="cuda", dtype=torch.float16)
        g = torch.randn(m, n, device="cuda", dtype=torch.float16)
        wt = w.t().contiguous()
        if args.ncu:
            for _ in range(2):
                D.gemm_tc(a, wt, b)
                D.gemm_wgrad(a, g, bias=True)
            torch.cuda.synchronize()
            continue
        t_fwd = timed(lambda: D.gemm_tc(a, wt, b))
        t_fwd_cublas = timed(lambda: a @ w + b)
        t_wg = timed(lambda: D.gemm_wgrad(a, g, bias=True))
        t_wg_cublas = timed(lambda: (a.t() @ g, g.sum(0)))
        t_wg_nob = timed(lambda: D.gemm_wgrad(a, g))
        fwd_bytes = (m * k + m * n + k * n) * 2
        wg_bytes = (m * k + m * n) * 2
        print(json.dumps({"m": m, "k": k, "n": n,
                          "fwd_tcgen05_us": round(t_fwd, 1), "fwd_cublas_us": round(t_fwd_cublas, 1),
                          "fwd_tcgen05_GBps": round(fwd_bytes / t_fwd / 1e3, 1),
                          "wgrad_tcgen05_us": round(t_wg, 1), "wgrad_cublas_us": round(t_wg_cublas, 1),
                          "wgrad_nobias_us": round(t_wg_nob, 1),
                          "wgrad_tcgen05_GBps": round(wg_bytes / t_wg / 1e3, 1)}), flush=True)
        del a, g


if __name__ == "__main__":
    main()
