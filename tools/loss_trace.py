"""Loss traces of the bench workload: eager steps vs CUDA-graph replay from the
same state (diagnostic; prints JSON lines)."""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import bench  # noqa: E402
from paper_2411_01109_b200.models import GraphBundle, Trainer, TrainConfig  # noqa: E402


def torch32_gcn(dg, x, labels, cfg, epochs):
    """The same 2-layer GCN in plain torch fp32 (torch.sparse CSR, exact
    D_r^-1/2 A D_c^-1/2 values, torch.optim.Adam) from the same initial weights."""
    tr = Trainer(GraphBundle.build(dg, numerics="fast"), x, labels, cfg)
    off = dg.offsets
    deg_r = (off[1:] - off[:-1]).double()
    deg_c = torch.bincount(dg.cols.long(), minlength=dg.n).double()
    rows = torch.repeat_interleave(torch.arange(dg.n, device=off.device), off[1:] - off[:-1])
    inv = lambda d: torch.where(d > 0, 1.0 / d.sqrt(), torch.zeros_like(d))
    vals = (inv(deg_r)[rows] * inv(deg_c)[dg.cols.long()]).float()
    a = torch.sparse_csr_tensor(off, dg.cols.long(), vals, (dg.n, dg.n))
    ps = [p.master.detach().clone().requires_grad_(True) for p in tr.model.params()]
    opt = torch.optim.Adam(ps, lr=cfg.lr, betas=(0.9, 0.999), eps=1e-8)
    xf = tr.x.float()
    lab = tr.labels
    losses = []
    for _ in range(epochs):
        w1, b1, w2, b2 = ps
        h = torch.relu(torch.sparse.mm(a, xf @ w1 + b1))
        logits = torch.sparse.mm(a, h @ w2 + b2)[:, : tr.n_cls]
        loss = torch.nn.functional.cross_entropy(logits.double(), lab)
        opt.zero_grad()
        loss.backward()
        opt.step()
        losses.append(round(float(loss), 5))
    return losses


def gs(v):
    return v if v == "auto" else float(v)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="gcn-reddit")
    ap.add_argument("--epochs", type=int, default=45)
    ap.add_argument("--eager-first", type=int, default=4)
    ap.add_argument("--lr", type=float, default=1e-2)
    ap.add_argument("--grad-scale", default="1")
    args = ap.parse_args()
    dg, x, labels = bench.build_workload(args.workload, 0)
    cfg = TrainConfig(mode="half", seed=0, scaling="discretized", norm="both", numerics="fast",
                      lr=args.lr, grad_scale=gs(args.grad_scale), **bench.WORKLOADS[args.workload]["cfg"])
    out = {}
    for tag in ("eager", "graph"):
        tr = Trainer(GraphBundle.build(dg, numerics="fast"), x, labels, cfg)
        losses = []
        for i in range(args.epochs):
            if tag == "graph" and i == args.eager_first:
                tr.capture()
            losses.append(round(float(tr.step()[0]), 5))
        out[tag] = losses
        print(json.dumps({"workload": args.workload, "mode": tag, "losses": losses}), flush=True)
    if cfg.kind == "gcn":
        out["torch32"] = torch32_gcn(dg, x, labels, cfg, args.epochs)
        print(json.dumps({"workload": args.workload, "mode": "torch32",
                          "losses": out["torch32"]}), flush=True)
    same = out["eager"] == out["graph"]
    print(json.dumps({"identical": same}), flush=True)


if __name__ == "__main__":
    main()
