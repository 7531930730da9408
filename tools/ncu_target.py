"""Short ncu target: one GCN epoch on the Reddit-shaped graph, then standalone
SpMM launches at F = 64 and 512 (discretized/both).  Never time under ncu."""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2411_01109_b200 import device as D  # noqa: E402
from paper_2411_01109_b200 import graphgen  # noqa: E402
from paper_2411_01109_b200.models import GraphBundle, Trainer, TrainConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--epochs", type=int, default=1)
    ap.add_argument("--feats", default="64,512")
    ap.add_argument("--gat", action="store_true")
    args = ap.parse_args()
    dg = graphgen.reddit_like(0)
    x, labels = graphgen.planted_features(dg.n, 602, 41, 0, "cuda")
    tr = Trainer(GraphBundle.build(dg), x, labels, TrainConfig(kind="gcn", hidden=64))
    for _ in range(args.epochs):
        tr.step()
    for f in map(int, args.feats.split(",")):
        xf = torch.randn(dg.n, f, device="cuda", dtype=torch.float16)
        D.spmm(dg, xf, None, "discretized", "both")
    if args.gat:
        rows, cols, feats, lab = graphgen.pubmed_like(0)
        from paper_2411_01109_b200.device import DeviceGraph

        g2 = DeviceGraph.from_edges(19717, rows, cols)
        tr2 = Trainer(GraphBundle.build(g2), feats, lab,
                      TrainConfig(kind="gat", hidden=16, heads=4, layers=3))
        tr2.step()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
