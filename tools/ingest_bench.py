"""Edge-list ingest throughput: a synthetic text of --edges lines
("%07d %07d\\n", built with numpy byte arithmetic) parsed on the GPU
(hg_count_lines + hg_parse_edges) and canonicalised (hg_build_csr), against the
oracle restatement of the reference loader on a --cpu-lines sample."""
from __future__ import annotations

import argparse
import json
import sys
import tempfile
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import oracle as O  # noqa: E402
from paper_2411_01109_b200 import device as D  # noqa: E402


def make_text(m, n, seed=0):
    rng = np.random.default_rng(seed)
    ab = rng.integers(0, n, (m, 2))
    buf = np.empty((m, 16), np.uint8)
    for k in range(7):
        p = 10 ** (6 - k)
        buf[:, k] = 48 + (ab[:, 0] // p) % 10
        buf[:, 8 + k] = 48 + (ab[:, 1] // p) % 10
    buf[:, 7] = 32
    buf[:, 15] = 10
    return buf.tobytes()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--edges", type=int, default=50_000_000)
    ap.add_argument("--vertices", type=int, default=4_000_000)
    ap.add_argument("--cpu-lines", type=int, default=300_000)
    args = ap.parse_args()
    text = make_text(args.edges, args.vertices)
    with tempfile.TemporaryDirectory() as tmp:
        p = Path(tmp) / "g.txt"
        p.write_bytes(text)
        dev = D.read_bytes_device(p)
        D.parse_edge_text(dev)  # warm-up (workspaces, module load)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            rows, cols, top = D.parse_edge_text(dev)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        parse_ms = min(ts)
        t0 = time.perf_counter()
        dg = D.DeviceGraph.from_edge_list(p, build_transpose=False)
        torch.cuda.synchronize()
        full_s = time.perf_counter() - t0
        sample = text[: 16 * args.cpu_lines]
        t0 = time.perf_counter()
        O.load_edge_list_text(sample, num_vertices=args.vertices)
        cpu_s = (time.perf_counter() - t0) * args.edges / args.cpu_lines
    print(json.dumps({
        "edges": args.edges, "bytes": len(text), "gpu_parse_ms": round(parse_ms, 3),
        "gpu_parse_GBps": round(len(text) / parse_ms / 1e6, 1),
        "file_to_csr_s": round(full_s, 3), "canonical_edges": dg.num_edges,
        "cpu_reference_loader_s_extrapolated": round(cpu_s, 1),
        "cpu_sample_lines": args.cpu_lines}))


if __name__ == "__main__":
    main()
