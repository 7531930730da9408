"""Where the RMAT SpMM loses against its gather floor: hg_spmm vs hg_gather_probe
on the C5 graph (F = 128, 64; plain and weighted, CSR and CSC), and on the same
column stream with rows merged in groups of `--merge` (fewer, longer rows:
the same gathers without the short-row latency chain).  Timing only."""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import bench  # noqa: E402
from paper_2411_01109_b200 import device as D  # noqa: E402


def t_ms(fn, reps=3):
    fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="gat-rmat")
    ap.add_argument("--merge", type=int, default=8)
    ap.add_argument("--feats", default="128,64")
    args = ap.parse_args()
    dg, _, _ = bench.build_workload(args.workload, 0)
    off = dg.offsets
    n = dg.n
    idx = torch.arange(0, n + 1, args.merge, device=off.device)
    if idx[-1] != n:
        idx = torch.cat([idx, torch.tensor([n], device=off.device)])
    merged = D.CsrView(off[idx].contiguous(), dg.cols, idx.numel() - 1, n)
    deg = (off[1:] - off[:-1])
    hist = {f"<={b}": int((deg <= b).sum()) for b in (0, 1, 2, 4, 8, 16, 32, 64)}
    res = {"n": n, "edges": dg.num_edges, "deg_hist": hist}
    for f in [int(v) for v in args.feats.split(",")]:
        x = torch.randn(n, f, device="cuda", dtype=torch.float16)
        w = torch.randn(dg.num_edges, 4, device="cuda", dtype=torch.float16)
        fwd, bwd = dg.view(False), dg.view(True)
        r = {}
        r["probe_csr"] = t_ms(lambda: D.gather_probe(fwd.cols, fwd.num_edges, x, f * 2))
        r["probe_csc"] = t_ms(lambda: D.gather_probe(bwd.cols, bwd.num_edges, x, f * 2))
        r["spmm_csr"] = t_ms(lambda: D.spmm_csr(fwd, x))
        r["spmm_csr_merged"] = t_ms(lambda: D.spmm_csr(merged, x))
        r["spmm_csr_w"] = t_ms(lambda: D.spmm_csr(fwd, x, w, None, 4))
        r["spmm_csc_w_perm"] = t_ms(lambda: D.spmm_csr(bwd, x, w, bwd.perm, 4))
        r["spmm_csc"] = t_ms(lambda: D.spmm_csr(bwd, x))
        res[f] = {k: round(v, 3) for k, v in r.items()}
        print(json.dumps({f: res[f]}), flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
