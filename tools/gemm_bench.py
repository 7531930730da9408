"""GCN layer GEMM + epilogue: cuBLAS (torch.matmul) followed by the fused
bias/scale pass vs the tcgen05 kernel with the epilogue fused (hg_gemm_tc)."""
from __future__ import annotations

import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2411_01109_b200 import device as D  # noqa: E402


def timed(fn, reps=20):
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
    torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = False
    for m, k, n in [(232_965, 608, 64), (232_965, 64, 48), (2_449_029, 104, 64),
                    (16_777_216, 128, 128)]:
        a = torch.randn(m, k, device="cuda", dtype=torch.float16)
        w = (torch.randn(k, n, device="cuda", dtype=torch.float16) * 0.1)
        b = torch.randn(n, device="cuda", dtype=torch.float16)
        s = torch.rand(m, device="cuda", dtype=torch.float16)
        wt = w.t().contiguous()
        t_cublas = timed(lambda: D.bias_scale_rows(a @ w, b, s))
        t_gemm_only = timed(lambda: a @ w)
        t_tc = timed(lambda: D.gemm_tc(a, wt, b, s))
        ref = D.bias_scale_rows(a @ w, b, s).float()
        got = D.gemm_tc(a, wt, b, s).float()
        bytes_ = (m * k + m * n + k * n) * 2
        print(json.dumps({"m": m, "k": k, "n": n, "cublas_plus_epilogue_us": round(t_cublas, 1),
                          "cublas_gemm_only_us": round(t_gemm_only, 1),
                          "tcgen05_fused_us": round(t_tc, 1),
                          "tcgen05_GBps": round(bytes_ / t_tc / 1e3, 1),
                          "tcgen05_TFLOPs": round(2 * m * k * n / t_tc / 1e6, 1),
                          "max_abs_diff_vs_cublas": float((ref - got).abs().max())}), flush=True)
        del a


if __name__ == "__main__":
    main()
