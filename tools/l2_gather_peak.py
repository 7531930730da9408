"""L2 random-gather peak: the best rate at which this GPU serves uniformly
random row gathers from an L2-resident table, measured with hg_gather_probe
(the SpMM's own load path: column ids streamed once from HBM, one team load
per row, nothing computed or stored).  Bytes are counted with the same gather
model as the SpMM roofline (4 B id + row bytes per gathered row), so
`bench.py` can report the SpMM against this roof (roofline.l2) as well as
against HBM copy bandwidth.

    python tools/l2_gather_peak.py            # prints one JSON line
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

ROW_BYTES = (16, 32, 64, 96, 128, 256, 512)


def measure(table_bytes=32 << 20, edges=1 << 25, reps=5, row_bytes=ROW_BYTES):
    """{row_bytes: GB/s} for uniform random ids over a table_bytes table."""
    import torch

    from paper_2411_01109_b200 import device as D

    g = torch.Generator(device="cuda")
    g.manual_seed(12345)
    out = {}
    for rb in row_bytes:
        rows = table_bytes // rb
        cols = torch.randint(0, rows, (edges,), generator=g, device="cuda", dtype=torch.int32)
        x = torch.zeros((rows, rb // 2), dtype=torch.float16, device="cuda")
        D.gather_probe(cols, edges, x, rb)
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        best = None
        for _ in range(reps):
            ev0.record()
            D.gather_probe(cols, edges, x, rb)
            ev1.record()
            torch.cuda.synchronize()
            t = ev0.elapsed_time(ev1) / 1e3
            best = t if best is None else min(best, t)
        out[rb] = (4 + rb) * edges / best / 1e9
        del cols, x
    return out


if __name__ == "__main__":
    res = measure()
    print(json.dumps({"what": "L2 random-gather peak (hg_gather_probe, uniform ids, 32 MB "
                              "table, 2^25 gathers, best of 5)",
                      "GBps_by_row_bytes": {str(k): round(v, 1) for k, v in res.items()}}))
