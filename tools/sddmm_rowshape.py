"""hg_sddmm_fast on the C5 RMAT graph, F = 128 / 64 over 4 heads: per-row
units only vs with short-row packs (device.sddmm), against the gather probe of
the same column stream.  Timing only."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2411_01109_b200 import device as D  # noqa: E402
from tools.spmm_rowshape import t_ms  # noqa: E402

dg, _, _ = bench.build_workload("gat-rmat", 0)
view = dg.view(False)
sched = view.schedule()
res = {}
for f in (128, 64):
    x = torch.randn(dg.n, f, device="cuda", dtype=torch.float16)
    y = torch.randn(dg.n, f, device="cuda", dtype=torch.float16)
    out = torch.empty((view.num_edges, 4), dtype=torch.float16, device="cuda")

    def units():
        D.nat.call("hg_sddmm_fast", D._p(view.offsets), D._p(view.cols), view.n_rows,
                   view.num_edges, D._p(sched.units), sched.num_units, None, 0, None, D._p(x), D._p(y),
                   D._p(out), f, 4, D._dtype_code(x), D._stream())

    res[f] = {"units": round(t_ms(units), 3),
              "packed": round(t_ms(lambda: D.sddmm(dg, x, y, heads=4, fast=True)), 3),
              "probe": round(t_ms(lambda: D.gather_probe(view.cols, view.num_edges, y, f * 2)), 3)}
    print(json.dumps({f: res[f]}), flush=True)
print(json.dumps(res))
