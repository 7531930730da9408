"""ncu target: one standalone fp32-guarded SpMM per F on the Reddit-shaped
graph (discretized/both).  Never time under ncu."""
from __future__ import annotations

import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2411_01109_b200 import device as D  # noqa: E402
from paper_2411_01109_b200 import graphgen  # noqa: E402

if __name__ == "__main__":
    dg = graphgen.reddit_like(0)
    view = dg.view(False)
    fin, fout = dg.norm_tables("both", False, torch.float16)
    for f in map(int, sys.argv[1].split(",")):
        x = torch.randn(dg.n, f, device="cuda", dtype=torch.float16)
        D.spmm_csr(view, x, scaling="discretized", fout=fout)
    torch.cuda.synchronize()
