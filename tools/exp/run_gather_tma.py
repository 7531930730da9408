"""Random-row gather through TMA (tile::gather4, per-row cp.async.bulk) vs the
LSU probe (hg_gather_probe, LDG.256 teams) on the C3 column stream.
Experiment only; prints one JSON line of ms per pass."""
import ctypes
import json
import subprocess
import sys
from pathlib import Path

import torch

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
from paper_2411_01109_b200 import device as D, graphgen  # noqa: E402

so = HERE / "gather_tma.so"
if not so.exists() or so.stat().st_mtime < (HERE / "gather_tma.cu").stat().st_mtime:
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                    "-Xcompiler", "-fPIC", str(HERE / "gather_tma.cu"), "-o", str(so), "-lcuda"],
                   check=True)
lib = ctypes.CDLL(str(so))
dg = graphgen.reddit_like(0)
sink = torch.zeros(4, dtype=torch.int32, device="cuda")
res = {"edges": dg.num_edges}


def timeit(go, reps=5):
    go()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        go()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps, 4)


for f in (48, 64, 128):
    x = torch.randn(dg.n, f, device="cuda", dtype=torch.float16)
    rb = f * 2
    res[f"F{f}_ldg_probe"] = timeit(lambda: D.gather_probe(dg.cols, dg.num_edges, x, rb))
    for mode in (1, 2):
        for cps in (1, 2, 3):
            for nst in (2, 3, 4):
                smem = 1024 + 4 * nst * 128 * rb
                if smem * cps > 227 * 1024:
                    continue

                def go():
                    rc = lib.tma_probe(ctypes.c_void_p(dg.cols.data_ptr()),
                                       ctypes.c_int64(dg.num_edges), ctypes.c_void_p(x.data_ptr()),
                                       ctypes.c_int64(dg.n), ctypes.c_int64(rb), rb, mode, cps, nst,
                                       ctypes.c_void_p(sink.data_ptr()),
                                       ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
                    assert rc == 0, rc
                res[f"F{f}_mode{mode}_cps{cps}_nst{nst}"] = timeit(go)
    del x
print(json.dumps(res))
