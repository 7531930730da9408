"""Per-layer timeline of the column-blocked, transfer-overlapped aggregation
(partition.py) for one rank of the C5 workload (RMAT-24 GAT,
4 heads) at P ranks, measured on ONE B200: the rank's CSR / CSC rows are cut
out of the full graph exactly as DistTrainer does, every column block's
hg_spmm_acc is timed with CUDA events (the rank's real edge subsets, real
feature widths), and the unblocked hg_spmm over the all-gathered buffer beside
it.  The NVLink transfer of each slab is NOT measured (one GPU): it is modelled
as slab bytes / B for the stated B values, broadcasts back to back in rank
order.  Prints one JSON document."""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2411_01109_b200 import device as D, graphgen  # noqa: E402
from paper_2411_01109_b200.partition import (block_bounds, block_groups, column_blocks,  # noqa: E402
                                             make_local_part)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def schedule(block_ms, bounds, splits, rank, bw_gbs, f):
    """Blocked pipeline: rank q's rows land after the broadcasts 0..q (own
    rows: no transfer); block g starts when its ranks' rows have landed and
    block g-1 is done."""
    land, t = [], 0.0
    for q in range(len(splits) - 1):
        if q != rank:
            t += (splits[q + 1] - splits[q]) * f * 2 / (bw_gbs * 1e6)   # ms
        land.append(0.0 if q == rank else t)
    t_end, rows = 0.0, []
    for g, ms in enumerate(block_ms):
        q0, q1 = list(splits).index(bounds[g]), list(splits).index(bounds[g + 1])
        arrive = max(land[q0:q1])
        start = max(t_end, arrive)
        t_end = start + ms
        rows.append({"block": g, "ranks": [q0, q1 - 1], "arrive_ms": round(arrive, 3),
                     "start_ms": round(start, 3), "end_ms": round(t_end, 3)})
    return t_end, t, rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--parts", type=int, default=8)
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--heads", type=int, default=4)
    ap.add_argument("--bw", default="450,700,900", help="modelled NVLink GB/s per rank")
    ap.add_argument("--no-reorder", action="store_true", help="keep the generated vertex ids")
    args = ap.parse_args()
    dg = graphgen.rmat(scale=args.scale, seed=0)
    if not args.no_reorder:   # as bench.py: degree-sorted, rank-interleaved relabelling
        dg = dg.relabel(D.locality_order(dg.offsets, dg.bwd.offsets, parts=args.parts))
    part = make_local_part(dg.offsets, dg.cols, dg.bwd.offsets, dg.bwd.cols, dg.bwd.perm,
                           args.rank, args.parts)
    n, h = dg.n, args.heads
    out = {"graph": f"RMAT scale {args.scale}, {dg.num_edges} edges", "parts": args.parts,
           "vertex_order": "as generated" if args.no_reorder else "degree-sorted, rank-interleaved",
           "rank": args.rank, "rank_rows": part.n_local, "rank_edges": part.fwd.num_edges,
           "transfer_model": "slab bytes / B, P broadcasts in rank order (not measured: 1 GPU)",
           "layers": []}
    # C5 GAT (hidden 32 x 4 heads, 16 classes): layer 1 aggregates F = 128,
    # layer 2 F = 4 x 16 = 64; backward aggregates the same widths over the CSC
    for name, f, transpose in (("layer1 fwd (z, F=128)", 128, False),
                               ("layer2 fwd (z, F=64)", 64, False),
                               ("layer2 bwd (dY, F=64)", 64, True),
                               ("layer1 bwd (dY, F=128)", 128, True)):
        view = part.bwd if transpose else part.fwd
        x = torch.randn(n, f, device="cuda", dtype=torch.float16)
        alpha = torch.rand(view.num_edges, h, device="cuda", dtype=torch.float16)
        full_ms = timed(lambda: D.spmm_csr(view, x, alpha, None, h, "post"))
        acc = torch.empty(part.n_local, f, device="cuda", dtype=torch.float32)
        layer = {"aggregation": name, "unblocked_spmm_ms": round(full_ms, 3),
                 "groups_chosen": block_groups(view, args.parts), "by_groups": {}}
        for groups in sorted({1, 2, 4, args.parts}):
            bounds = block_bounds(part.splits, groups)
            blocks = column_blocks(view, bounds)
            block_ms = []
            for q, b in enumerate(blocks):
                lo, hi = int(bounds[q]), int(bounds[q + 1])
                last = q == len(blocks) - 1
                block_ms.append(timed(lambda: D.spmm_csr_acc(
                    b, x[lo:hi], acc_in=None if q == 0 else acc, acc_out=None if last else acc,
                    w=alpha, w_index=b.perm, heads=h)))
            rec = {"block_ms": [round(v, 3) for v in block_ms],
                   "blocked_spmm_ms_sum": round(sum(block_ms), 3), "by_bw": {}}
            for bw in (float(v) for v in args.bw.split(",")):
                t_end, t_comm, rows = schedule(block_ms, bounds, part.splits, args.rank, bw, f)
                rec["by_bw"][str(int(bw))] = {
                    "allgather_ms": round(t_comm, 3), "serial_ms": round(t_comm + full_ms, 3),
                    "overlapped_ms": round(t_end, 3),
                    "saved_ms": round(t_comm + full_ms - t_end, 3), "timeline": rows}
            layer["by_groups"][str(groups)] = rec
        out["layers"].append(layer)
        del x, alpha, acc
    print(json.dumps(out))


if __name__ == "__main__":
    main()
