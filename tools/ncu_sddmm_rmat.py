"""ncu target: one fp32-guarded SDDMM (F=128, 4 heads, per-row units) on the C5
RMAT graph.  Never time under ncu."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2411_01109_b200 import device as D  # noqa: E402

f = int(sys.argv[1]) if len(sys.argv) > 1 else 128
dg, _, _ = bench.build_workload("gat-rmat", 0)
view = dg.view(False)
sched = view.schedule()
x = torch.randn(dg.n, f, device="cuda", dtype=torch.float16)
y = torch.randn(dg.n, f, device="cuda", dtype=torch.float16)
out = torch.empty((view.num_edges, 4), dtype=torch.float16, device="cuda")
D.nat.call("hg_sddmm_fast", D._p(view.offsets), D._p(view.cols), view.n_rows, view.num_edges,
           D._p(sched.units), sched.num_units, None, 0, None, D._p(x), D._p(y), D._p(out), f, 4,
           D._dtype_code(x), D._stream())
torch.cuda.synchronize()
