"""ncu target: one hg_spmm (F from argv, default 64, unweighted, CSR) on the C5
RMAT graph.  Never time under ncu."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2411_01109_b200 import device as D  # noqa: E402

f = int(sys.argv[1]) if len(sys.argv) > 1 else 64
dg, _, _ = bench.build_workload("gat-rmat", 0)
x = torch.randn(dg.n, f, device="cuda", dtype=torch.float16)
D.spmm_csr(dg.view(False), x)
torch.cuda.synchronize()
