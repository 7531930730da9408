"""Experiment: vertex relabelling by descending degree (hot rows packed
together) vs the generated ids, for the C4 / C5 aggregations.  Times hg_spmm
(fast, discretized/both) on both labellings of the same graph."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2411_01109_b200 import device as D, graphgen  # noqa: E402
from paper_2411_01109_b200.device import DeviceGraph  # noqa: E402


def relabel(dg):
    deg = (dg.offsets[1:] - dg.offsets[:-1]) + (dg.bwd.offsets[1:] - dg.bwd.offsets[:-1])
    order = torch.argsort(deg, descending=True, stable=True)     # new -> old
    new_of_old = torch.empty_like(order)
    new_of_old[order] = torch.arange(order.numel(), device=order.device)
    rows = torch.repeat_interleave(torch.arange(dg.n, device="cuda"), dg.offsets[1:] - dg.offsets[:-1])
    r2, c2 = new_of_old[rows], new_of_old[dg.cols.long()]
    return DeviceGraph.from_edges(dg.n, r2, c2, device="cuda")


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


res = {}
for name, gen, fs in (("products", lambda: graphgen.products_like(seed=0), (112, 64)),
                      ("rmat24", lambda: graphgen.rmat(scale=24, seed=0), (128, 64))):
    dg = gen()
    dr = relabel(dg)
    for f in fs:
        x = torch.randn(dg.n, f, device="cuda", dtype=torch.float16)
        t0 = timeit(lambda: D.spmm(dg, x, None, "discretized", "both"))
        t1 = timeit(lambda: D.spmm(dr, x, None, "discretized", "both"))
        t0t = timeit(lambda: D.spmm(dg, x, None, "discretized", "both", transpose=True))
        t1t = timeit(lambda: D.spmm(dr, x, None, "discretized", "both", transpose=True))
        res[f"{name}_F{f}"] = {"generated_ms": round(t0, 3), "degree_sorted_ms": round(t1, 3),
                               "generated_T_ms": round(t0t, 3), "degree_sorted_T_ms": round(t1t, 3)}
        print(json.dumps(res), flush=True)
    del dg, dr
print(json.dumps(res))
