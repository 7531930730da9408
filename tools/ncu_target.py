"""Short ncu target: `--epochs` training epochs of a bench workload (default the
Reddit-shaped GCN), then standalone SpMM launches at `--feats` (discretized/
both) on that graph.  Never time under ncu."""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import bench  # noqa: E402
from paper_2411_01109_b200 import device as D  # noqa: E402
from paper_2411_01109_b200.models import GraphBundle, Trainer, TrainConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="gcn-reddit", choices=sorted(bench.WORKLOADS))
    ap.add_argument("--epochs", type=int, default=1)
    ap.add_argument("--feats", default="")
    ap.add_argument("--no-reorder", action="store_true")
    args = ap.parse_args()
    dg, x, labels = bench.build_workload(args.workload, 0)
    order = None
    if bench.WORKLOADS[args.workload].get("reorder") == "degree" and not args.no_reorder:
        order = D.locality_order(dg.offsets, dg.bwd.offsets)   # as bench.py
        dg = dg.relabel(order)
    cfg = TrainConfig(mode="half", seed=0, scaling="discretized", norm="both", numerics="fast",
                      grad_scale="auto", **bench.WORKLOADS[args.workload]["cfg"])
    tr = Trainer(GraphBundle.build(dg), x, labels, cfg, node_order=order)
    for _ in range(args.epochs):
        tr.step()
    for f in [int(v) for v in args.feats.split(",") if v]:
        xf = torch.randn(dg.n, f, device="cuda", dtype=torch.float16)
        D.spmm(dg, xf, None, "discretized", "both")
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
