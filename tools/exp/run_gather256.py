"""Random-row gather: 16-byte vs 32-byte lane loads (and 32-byte with
L1::no_allocate, lane code 33) on the C3 column stream.  Experiment only."""
import ctypes
import json
import subprocess
import sys
from pathlib import Path

import torch

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
import bench  # noqa: E402

so = HERE / "gather256.so"
if not so.exists() or so.stat().st_mtime < (HERE / "gather256.cu").stat().st_mtime:
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                    "-Xcompiler", "-fPIC", str(HERE / "gather256.cu"), "-o", str(so)], check=True)
lib = ctypes.CDLL(str(so))
dg, _, _ = bench.build_workload("gcn-reddit", 0)
sink = torch.zeros(4, dtype=torch.int32, device="cuda")
res = {}
for f in (32, 64, 128):
    x = torch.randn(dg.n, f, device="cuda", dtype=torch.float16)
    for lb in (16, 32, 33):   # 33: 32-byte lanes with L1::no_allocate
        for blocks in (148 * 8,):
            def go():
                rc = lib.probe(ctypes.c_void_p(dg.cols.data_ptr()), ctypes.c_int64(dg.num_edges),
                               ctypes.c_void_p(x.data_ptr()), ctypes.c_int64(f * 2), f * 2, lb,
                               ctypes.c_void_p(sink.data_ptr()), blocks,
                               ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
                assert rc == 0, rc
            go()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                go()
            e1.record()
            torch.cuda.synchronize()
            res[f"F{f}_lane{lb}_b{blocks}"] = round(e0.elapsed_time(e1) / 5, 4)
print(json.dumps(res))
