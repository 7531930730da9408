"""Benchmark: GCN training epoch on the Reddit-shaped graph (BASELINE config C3).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

A step is one full-batch training epoch -- forward, loss, backward, Adam -- of
the paper's 2-layer GCN (hidden 64, fp16, discretized/both norm) on a
synthetic Reddit-shaped graph (N=232,965, E=114,848,857, 602 features, 41
classes).  value = ms/epoch with inputs resident in HBM (device-timed, max over
ranks); e2e = the same through the public training loop with the features
copied from pinned host memory every epoch and the loss read back.

The dominant kernel is the fp32-guarded SpMM (k_spmm_fast); its roofline uses
the gather-model algorithmic bytes of every hg_spmm launch in the timed region
 over their CUDA-event durations, against MEASURED_PEAKS.json.
The CPU baseline times the numpy restatement of the reference (oracle/) on a
row-panel sample of the same workload and extrapolates the sparse part by E.
Under torchrun (N > 1) the graph is row-partitioned and features are
all-gathered over NCCL before every aggregation (partition.py).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "GCN/GAT ms/epoch at 1/2/4/8 B200; half2 SpMM GB/s vs HBM peak"
N_FEAT, N_CLASSES, HIDDEN = 602, 41, 64


def peaks():
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return d["hbm_gbs"] * 1e9, "measured"
    except Exception:
        return 6.65e12, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms during timing."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index=0):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def wait_first_sample(self, timeout=3.0):
        """Block until nvidia-smi has written its first sample (its start-up
        latency would otherwise leave a short timed region unsampled)."""
        t0 = time.time()
        while self.proc is not None and time.time() - t0 < timeout:
            try:
                if Path(self.path).read_text().strip():
                    return
            except OSError:
                pass
            time.sleep(0.02)

    def summary(self):
        rows = []
        try:
            for line in Path(self.path).read_text().splitlines():
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


def dist_env():
    """(world size, rank, local device).  HG_DIST_SHARED_GPU=1 puts every rank
    on cuda:0 (with HG_DIST_BACKEND=gloo: validating the N>1 path on one GPU;
    never a measurement)."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("HG_DIST_SHARED_GPU") == "1":
        local = 0
    return ws, rank, local


def max_over_ranks(dist, v, op="max"):
    """Max (or sum) of a host float over ranks (device tensor for NCCL, host
    for gloo)."""
    import torch

    dev = "cpu" if dist.get_backend() == "gloo" else "cuda"
    tt = torch.tensor([v], device=dev, dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(tt.item())


def load_traffic_profile(workload, ws):
    """ncu DRAM bytes per hg_spmm call of this workload's epoch from the newest
    committed `ncu --set full` summary (profiles/r*/ncu_spmm_summary.json), with
    its source; (None, None) when that workload was not captured at this world
    size (per-rank captures exist only for one GPU)."""
    if ws != 1:
        return None, None
    for rnd in ("r02", "r01"):
        p = ROOT / "profiles" / rnd / "ncu_spmm_summary.json"
        try:
            d = json.loads(p.read_text()).get(workload)
        except Exception:
            continue
        if d:
            return d["bytes_per_launch"], f"profiles/{rnd}/ncu_spmm_summary.json"
    return None, None


# ── CPU legs: the reference on the host cores (tools/refarm.py) ──


def cpu_leg_impl(cfg):
    """('reference', halfsparse) when the unmodified reference is installed
    under baseline/_ref and its Model covers the workload (2-layer, 1 head);
    else ('port', None): the numpy restatement in oracle/."""
    from tools import refarm as R

    H = R.load_reference()
    if H is not None and cfg.get("heads", 1) == 1 and cfg.get("layers", 2) == 2:
        return "reference", H
    return "port", None


def cpu_baseline(name, seed, budget_edges, torch_comparator=True):
    """cpu_baseline object of the B200 arm: one reference epoch on a random
    row-panel sample (after a small calibration epoch), extrapolated to the
    full graph; plus the torch-CPU fp32 comparator for GCN."""
    from tools import refarm as R

    w = WORKLOADS[name]
    hw = R.HostWorkload(name, seed, w["feat"], w["classes"])
    impl, H = cpu_leg_impl(w["cfg"])
    leg = R.CpuLeg(hw, impl, w["cfg"], H)
    ms = leg.step(budget_edges, sample_seed=seed + 17)
    cc = R.core_counts()
    out = {"value": round(ms, 1), "unit": "ms/epoch", "cores": cc["sched_affinity"],
           "kind": impl, "extrapolated": budget_edges < hw.num_edges,
           "sample": leg.describe(budget_edges), "core_counts": cc,
           "threads_note": "sparse operators single-threaded numpy; dense BLAS on all cores"}
    if torch_comparator and w["cfg"]["kind"] == "gcn":
        tl = R.CpuLeg(hw, "torch", w["cfg"])
        tms = tl.step(min(4 * budget_edges, hw.num_edges), sample_seed=seed + 18)
        out["torch_cpu_fp32"] = {"value": round(tms, 1), "unit": "ms/epoch",
                                 "cores": cc["torch_threads"], "sample": tl.describe(
                                     min(4 * budget_edges, hw.num_edges))}
    return out


def reference_arm(args, ws, rank):
    """--impl reference: the reference's own CPU path on this host's cores,
    rank 0 only (other ranks exit without work).  No GPU, no libhalfgnn.so:
    the graph rows are regenerated on the host (synth.py)."""
    if rank != 0:
        return
    from tools import refarm as R

    w = WORKLOADS[args.workload]
    hw = R.HostWorkload(args.workload, args.seed, w["feat"], w["classes"])
    impl, H = cpu_leg_impl(w["cfg"])
    leg = R.CpuLeg(hw, impl, w["cfg"], H)
    # per-step sample: >= 1M edges sampled over the timed steps in total, and
    # the whole run bounded to a few minutes (the dense part is full size)
    budget = args.ref_budget_edges or max(100_000, 2_000_000 // max(args.steps, 1))
    for i in range(args.warmup):
        leg.step(min(budget, 20_000), sample_seed=10_000 + i, warm=True)
    vals = [leg.step(budget, sample_seed=args.seed * 1000 + i) for i in range(args.steps)]
    v = round(statistics.median(vals), 1)
    cc = R.core_counts()
    line = {"metric": METRIC, "value": v, "unit": "ms/epoch", "impl": "reference",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": v,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "f16", "data": "synthetic (the B200 arm's graph rows, regenerated on the "
                                    "host by synth.py)",
            "config": workload_config(hw.n, hw.num_edges, name=args.workload),
            "extrapolated": budget < hw.num_edges,
            "scale_factor": round(hw.num_edges * leg.steps / max(leg.sampled_edges, 1), 1),
            "per_step_ms": [round(x, 1) for x in vals],
            "cpu_baseline": {"value": v, "unit": "ms/epoch", "cores": cc["sched_affinity"],
                             "kind": impl, "sample": leg.describe(budget),
                             "extrapolated": budget < hw.num_edges, "core_counts": cc},
            "e2e": {"value": v, "unit": "ms/epoch", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# BASELINE.json configs as bench workloads (C3 is the headline default).
WORKLOADS = {
    "gcn-reddit": dict(desc="GCN 2-layer train epoch, synthetic Reddit-shaped graph (C3)",
                       graph="reddit_like", feat=602, classes=41,
                       cfg=dict(kind="gcn", hidden=64), reorder="degree",
                       l2="inputs larger than L2 (column stream 459 MB, features 280 MB)"),
    "gin-products": dict(desc="GIN 2-layer train epoch, synthetic ogbn-products-shaped "
                              "power-law graph (C4)",
                         graph="products_like", feat=100, classes=47,
                         cfg=dict(kind="gin", hidden=64), reorder="degree",
                         l2="inputs larger than L2 (column stream 495 MB, features 490 MB)"),
    "gat-rmat": dict(desc="GAT 2-layer 4-head train epoch, synthetic RMAT scale-24 graph (C5)",
                     graph="rmat", feat=128, classes=16,
                     cfg=dict(kind="gat", hidden=32, heads=4), reorder="degree",
                     l2="inputs larger than L2 (column stream ~1 GB, features 4.3 GB)"),
    "gat-pubmed": dict(desc="GAT 3-layer 4-head train epoch, synthetic Pubmed-shaped graph (C2)",
                       graph="pubmed_like", feat=500, classes=3,
                       cfg=dict(kind="gat", hidden=16, heads=4, layers=3),
                       l2="inputs fit in L2; flushed between timed epochs is not applied"),
}


def workload_config(n, e, parallelism="dp1", name="gcn-reddit"):
    w = WORKLOADS[name]
    c = w["cfg"]
    return {"workload": w["desc"], "nodes": n, "edges": e, "feat": w["feat"],
            "hidden": c["hidden"], "heads": c.get("heads", 1), "layers": c.get("layers", 2),
            "classes": w["classes"], "reduction": "discretized/both",
            "numerics": "fp32-guarded SpMM", "l2": w["l2"], "parallelism": parallelism}


def build_workload(name, seed, device="cuda"):
    """(DeviceGraph, features [N, F] fp16 on device, labels) of a workload."""
    import torch

    from paper_2411_01109_b200 import graphgen
    from paper_2411_01109_b200.device import DeviceGraph

    w = WORKLOADS[name]
    if w["graph"] == "pubmed_like":
        rows, cols, feats, labels = graphgen.pubmed_like(seed)
        dg = DeviceGraph.from_edges(feats.shape[0], rows, cols, device=device)
        return dg, torch.from_numpy(feats).to(device).half(), torch.from_numpy(labels).to(device)
    dg = getattr(graphgen, w["graph"])(seed=seed, device=device)
    x, labels = graphgen.planted_features(dg.n, w["feat"], w["classes"], seed, device)
    return dg, x, labels


# ── B200 arm ─────────────────────────────────────────────────────────────


def spmm_sweep(dg, peak, feats=(16, 32, 64, 128, 256, 512), reps=3):
    import torch

    from paper_2411_01109_b200 import device as D

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = {}
    for f in feats:
        x = torch.randn(dg.n, f, device="cuda", dtype=torch.float16)
        D.spmm(dg, x, None, "discretized", "both")
        ts = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            D.spmm(dg, x, None, "discretized", "both")
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / 1e3)
        t = statistics.median(ts)
        byts = D.spmm_bytes(dg.n, dg.n, dg.num_edges, f)
        out[str(f)] = {"ms": round(t * 1e3, 4), "GBps": round(byts / t / 1e9, 1),
                       "frac": round(byts / t / peak, 4)}
        del x
    del flush
    return out


def parity_block(dg, f=64, n_random=2000, n_hubs=20, seed=0):
    """Parity of the benched aggregation on the benched graph: the fp32-guarded
    SpMM (discretized / both norm, F = 64, as the first GCN aggregation) on
    the top-degree hub rows (the split rows with fp32 carries) plus random rows,
    against a float64 segment sum computed here with torch (the Appendix-A
    rule |y - y64| <= 1e-2 max(1, |y64|))."""
    import torch

    from paper_2411_01109_b200 import device as D

    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(dg.n, f, device="cuda", dtype=torch.float16, generator=g)
    y = D.spmm(dg, x, None, "discretized", "both")
    fin, fout = dg.norm_tables("both", False, torch.float16)
    deg = dg.offsets[1:] - dg.offsets[:-1]
    hubs = torch.topk(deg, min(n_hubs, dg.n)).indices
    rnd = torch.randint(0, dg.n, (n_random,), device="cuda", generator=g)
    rows = torch.unique(torch.cat([hubs, rnd]))
    lo, cnt = dg.offsets[rows], deg[rows]
    seg = torch.repeat_interleave(torch.arange(rows.numel(), device="cuda"), cnt)
    starts = torch.cumsum(cnt, 0) - cnt
    eidx = lo[seg] + (torch.arange(seg.numel(), device="cuda") - starts[seg])
    c = dg.cols[eidx].long()
    contrib = x[c].double() * fin[c].double()[:, None]
    s64 = torch.zeros(rows.numel(), f, dtype=torch.float64, device="cuda").index_add_(0, seg, contrib)
    y64 = s64 * fout[rows].double()[:, None]
    err = ((y[rows].double() - y64).abs() / y64.abs().clamp(min=1.0)).max().item()
    return {"kernel": "hg_spmm (fast, discretized/both, F=64)", "rows_checked": int(rows.numel()),
            "hub_rows": int(hubs.numel()), "edges_checked": int(seg.numel()),
            "max_mixed_err": float(err), "bound": 1e-2, "ok": bool(err <= 1e-2),
            "reference": "float64 segment sum (torch, in this run)"}


def small_configs(args, peak):
    """C1 (Cora-shaped 2-layer GCN) and C2 (Pubmed-shaped 3-layer 4-head GAT):
    device-timed ms/epoch, plus the oracle port's epoch on the same graph."""
    import numpy as np
    import torch

    from paper_2411_01109_b200 import graphgen
    from paper_2411_01109_b200.device import DeviceGraph
    from paper_2411_01109_b200.models import GraphBundle, Trainer, TrainConfig

    out = {}
    specs = [("C1_gcn_cora", graphgen.cora_like, dict(kind="gcn", hidden=16)),
             ("C2_gat_pubmed_3x4", graphgen.pubmed_like,
              dict(kind="gat", hidden=16, heads=4, layers=3))]
    for name, gen, kw in specs:
        rows, cols, feats, labels = gen(0)
        n = feats.shape[0]
        dg = DeviceGraph.from_edges(n, rows, cols)
        tr = Trainer(GraphBundle.build(dg), feats, labels, TrainConfig(**kw))
        def timed(steps=20):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(steps):
                tr.step()
            b.record()
            torch.cuda.synchronize()
            return round(a.elapsed_time(b) / steps, 4)

        for _ in range(3):
            tr.step()
        eager = timed()
        tr.capture()
        rec = {"ms_per_epoch": timed(), "ms_per_epoch_eager": eager, "cuda_graph": True,
               "nodes": n, "edges": int(rows.size)}
        if not args.no_cpu_baseline:
            from tools import refarm as R

            impl, H = cpu_leg_impl(kw)
            r64, c64 = rows.astype(np.int64), cols.astype(np.int64)
            x16 = feats.astype(np.float16)
            if impl == "reference":
                s_, o_ = R.reference_epoch(H, n, r64, c64, x16, labels, kw["kind"], kw["hidden"])
            else:
                s_, o_ = R.port_epoch(n, r64, c64, x16, labels, kw["kind"], kw["hidden"],
                                      kw.get("heads", 1), kw.get("layers", 2))
            rec["cpu_ms_per_epoch"] = round((s_ + o_) * 1e3, 1)
            rec["cpu_kind"] = impl
        out[name] = rec
    return out


def b200_arm(args, ws, rank, local):
    import numpy as np
    import torch

    from paper_2411_01109_b200 import device as D
    from paper_2411_01109_b200 import graphgen
    from paper_2411_01109_b200.models import GraphBundle, Trainer, TrainConfig

    torch.cuda.set_device(local)
    dist = None
    # HG_FORCE_DIST=1: the partitioned trainer even at N=1 (a one-rank NCCL group:
    # validates the N>1 code path, graph capture of its collectives included)
    use_dist = ws > 1 or os.environ.get("HG_FORCE_DIST") == "1"
    if use_dist:
        import torch.distributed as dist

        for k, v in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29531"), ("RANK", "0"),
                     ("WORLD_SIZE", "1")):
            os.environ.setdefault(k, v)

        backend = os.environ.get("HG_DIST_BACKEND", "nccl")
        if backend == "nccl":
            # NCCL prints its version banner on stdout (NCCL_DEBUG=VERSION);
            # stdout must carry only the JSON line, so the communicator is
            # created (eagerly, device_id + a barrier) with fd 1 on stderr
            sys.stdout.flush()
            saved = os.dup(1)
            os.dup2(2, 1)
            try:
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
                dist.barrier()
                torch.cuda.synchronize()
            finally:
                sys.stdout.flush()
                os.dup2(saved, 1)
                os.close(saved)
        else:
            dist.init_process_group(backend)
    peak, peak_kind = peaks()
    t_setup = time.time()
    dg, x, labels = build_workload(args.workload, args.seed)
    cfg = TrainConfig(mode="half", seed=args.seed, scaling="discretized", norm="both",
                      numerics="fast", grad_scale="auto", **WORKLOADS[args.workload]["cfg"])
    # locality relabelling (device.locality_order): the same graph, features,
    # labels and split per original vertex; hot rows packed together
    reorder = args.reorder if args.reorder != "auto" else WORKLOADS[args.workload].get(
        "reorder", "none")
    order = None
    if reorder == "degree":
        order = D.locality_order(dg.offsets, dg.bwd.offsets, parts=ws)
        dg = dg.relabel(order)
    if use_dist:
        from paper_2411_01109_b200.partition import DistTrainer

        tr = DistTrainer(dg, x, labels, cfg, dist, node_order=order)
        parallelism = f"row-partition x{ws} ({dist.get_backend()} all-gather)"
    else:
        tr = Trainer(GraphBundle.build(dg, numerics="fast"), x, labels, cfg, node_order=order)
        parallelism = "dp1"
    if order is not None:
        x = x[order]   # the trainer's vertex order (the e2e feed copies these rows)
    for _ in range(args.warmup):
        tr.step()
    torch.cuda.synchronize()
    setup_s = time.time() - t_setup

    def barrier():
        if dist is not None:
            dist.barrier()

    def timed_steps(k):
        barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(k):
            loss, _ = tr.step()
        ev1.record()
        torch.cuda.synchronize()
        barrier()
        ms = ev0.elapsed_time(ev1) / k
        if dist is not None:
            ms = max_over_ranks(dist, ms)
        return ms, loss

    # clocks are sampled from before the first timed step to after the last
    clocks = ClockSampler(local).__enter__()
    clocks.wait_first_sample()

    # ---- eager pass: SpMM roofline (CUDA events around every hg_spmm) ----
    D.Probe.reset(timing=True)
    rb0 = tr.bundle.ex.recv_bytes if use_dist else 0
    eager_ms, _ = timed_steps(args.steps)
    recv_per_step = (tr.bundle.ex.recv_bytes - rb0) / args.steps if use_dist else 0.0
    if dist is not None:
        recv_max = max_over_ranks(dist, recv_per_step)
        recv_sum = max_over_ranks(dist, recv_per_step, op="sum")
    launches = D.Probe.launches
    spmm_b, spmm_s, spmm_n = D.Probe.summary()
    compulsory = D.Probe.compulsory_per_launch()
    # one more eager step holding its SpMM operands: the same gathers with the
    # arithmetic removed (hg_gather_probe) give the floor those launches could reach
    ceiling_s = None
    D.Probe.reset(timing=True, keep=True)
    timed_steps(1)
    _, probe_s, _ = D.Probe.summary()
    ceil = D.Probe.gather_ceiling()
    if ceil:
        ceiling_s = (ceil, probe_s)
    # the L2 random-gather roof (live), and the eager pass's calls priced at it
    from tools import l2_gather_peak

    l2_peak = l2_gather_peak.measure() if rank == 0 else None
    D.Probe.reset(timing=True)
    timed_steps(1)
    _, _, _ = D.Probe.summary()
    l2_ideal = D.Probe.l2_ideal_seconds(l2_peak) if l2_peak else None
    if l2_ideal is not None:   # scale to the eager pass's per-step SpMM time
        l2_ideal *= args.steps
    D.Probe.reset(timing=False)

    # ---- device-resident timing (value): the step replayed as a CUDA graph ----
    graphed = not args.no_graph and (not use_dist or dist.get_backend() == "nccl")
    if graphed:
        try:
            tr.capture()
            tr.step()
            torch.cuda.synchronize()
        except Exception as exc:  # a capture failure must not lose the measurement
            print(f"[bench] CUDA graph capture failed, timing eager steps: {exc}",
                  file=sys.stderr, flush=True)
            tr._graph = None
            graphed = False
    t_ms, loss = timed_steps(args.steps)
    clocks.__exit__(None, None, None)
    final_loss = float(loss)

    # ---- end to end through the public loop: host features in, loss out ----
    inner = tr.inner if use_dist else tr
    lo, hi = (tr.part.lo, tr.part.hi) if use_dist else (0, dg.n)
    host_x = inner.host_features(x[lo:hi].cpu())
    h2d = host_x.numel() * host_x.element_size()
    if dist is not None:  # whole-job bytes: every rank copies its own rows
        h2d = int(max_over_ranks(dist, float(h2d), op="sum"))
    def dist_feed(k):
        """k partitioned steps fed from pinned host memory: the next step's
        host->device copy runs on a side stream into a staging buffer while the
        current step computes (as Trainer.run_epochs does on one GPU); a
        device-to-device copy moves it into the captured graph's input."""
        cur_s, side = torch.cuda.current_stream(), torch.cuda.Stream()
        stage = [torch.empty_like(inner.x), torch.empty_like(inner.x)]
        copied = [torch.cuda.Event(), torch.cuda.Event()]
        used = [torch.cuda.Event(), torch.cuda.Event()]
        side.wait_stream(cur_s)
        with torch.cuda.stream(side):
            stage[0].copy_(host_x, non_blocking=True)
            copied[0].record()
        for i in range(k):
            cur, nxt = i % 2, 1 - i % 2
            if i + 1 < k:
                with torch.cuda.stream(side):
                    if i >= 1:
                        side.wait_event(used[nxt])
                    stage[nxt].copy_(host_x, non_blocking=True)
                    copied[nxt].record()
            cur_s.wait_event(copied[cur])
            inner.x.copy_(stage[cur])
            used[cur].record()
            loss, _ = tr.step()
            float(loss)

    # untimed warm-up of the same path (first copies out of the fresh pinned
    # buffer, the feed's side stream and events)
    if use_dist:
        dist_feed(min(2, args.warmup))
    else:
        tr.run_epochs(host_x, min(2, args.warmup))
    barrier()
    torch.cuda.synchronize()
    # wall-clock e2e: at least ~0.25 s of steps so sub-millisecond epochs are
    # not one host hiccup away from a different number (same on every rank)
    e2e_steps = max(args.steps, min(500, int(math.ceil(250.0 / max(t_ms, 1e-3)))))
    e0 = time.perf_counter()
    if use_dist:
        dist_feed(e2e_steps)
    else:
        tr.run_epochs(host_x, e2e_steps)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = (time.perf_counter() - e0) * 1e3 / e2e_steps
    if dist is not None:
        e2e_ms = max_over_ranks(dist, e2e_ms)

    result = None
    if rank == 0:
        achieved = spmm_b / spmm_s if spmm_s > 0 else 0.0
        traffic, traffic_src = load_traffic_profile(args.workload, ws)
        dram_gbs = traffic * spmm_n / spmm_s / 1e9 if traffic and spmm_s > 0 else None
        l2 = None
        if l2_peak:
            ideal = l2_ideal
            l2 = {"peak_GBps_by_row_bytes": {str(k): round(v, 1) for k, v in l2_peak.items()},
                  "frac": round(ideal / spmm_s, 4) if ideal and spmm_s > 0 else None,
                  "what": "tools/l2_gather_peak.py, run live: hg_gather_probe on uniform random "
                          "ids over a 32 MB L2-resident table (same gather-model bytes); frac = "
                          "time the step's hg_spmm calls would take at that rate for their row "
                          "widths / their measured time"}
        result = {
            "metric": METRIC, "value": round(t_ms, 4), "unit": "ms/epoch", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_ms, 4),
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "f16", "data": f"synthetic (seeded {WORKLOADS[args.workload]['graph']} graph, "
                                    "planted labels)",
            "config": dict(workload_config(dg.n, dg.num_edges, parallelism, args.workload),
                           vertex_order=("degree-sorted relabelling (device.locality_order, "
                                         "rank-interleaved; same graph, features, labels and "
                                         "split per original vertex)" if order is not None
                                         else "as generated")),
            "clocks": clocks.summary(),
            "e2e": {"value": round(e2e_ms, 4), "unit": "ms/epoch", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": 4 * ws, "steps": e2e_steps},
            "gpu_launches": int(launches),
            "ms_per_step_eager": round(eager_ms, 4), "cuda_graph": graphed,
            "roofline": {"bound": "hbm", "achieved": round(achieved / 1e9, 1),
                         "peak": round(peak / 1e9, 1), "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "kernel": "k_spmm_fast (hg_spmm)", "launches": spmm_n,
                         "peak_source": peak_kind,
                         "bytes_model": "4E+8(N+1)+2FE+2FN per SpMM launch, F = stored width",
                         "frac_note": ("achieved counts every gathered row (SURVEY 8(d) gather "
                                       "model); above 1 the rows are served from L2, not HBM -- "
                                       "read hbm_dram_frac for DRAM and l2.frac for the L2 "
                                       "gather roof" if achieved > peak else None),
                         "hbm_dram_frac": (round(dram_gbs * 1e9 / peak, 4)
                                           if dram_gbs else None),
                         "traffic_source": traffic_src,
                         "compulsory_bytes": round(compulsory),
                         "traffic_over_compulsory": (round(traffic / compulsory, 3)
                                                     if traffic and compulsory else None),
                         "compulsory_model": "4E+8(N+1)+2F(N_cols+N_rows): ids, X once, Y once",
                         "l2": l2,
                         "gather_ceiling": (None if ceiling_s is None else {
                             "spmm_ms_per_step": round(ceiling_s[1] * 1e3, 4),
                             "probe_ms_per_step": round(ceiling_s[0] * 1e3, 4),
                             "frac": round(ceiling_s[0] / ceiling_s[1], 4),
                             "what": "hg_gather_probe: the same column ids, feature buffers and "
                                     "widths as the step's hg_spmm calls, loads only (X warm in "
                                     "L2); frac = probe time / hg_spmm time"})},
            "exchange": (None if not use_dist else {
                "recv_bytes_per_rank_per_step_max": int(recv_max),
                "recv_bytes_per_step_total": int(recv_sum),
                "n_rows_max_over_mean": round(tr.part.n_max * ws / dg.n, 4),
                "what": "bytes each rank receives per epoch over the fabric: exact-count "
                        "feature / gradient all-gathers ((N - n_local) rows each) and the GAT "
                        "edge-value all-to-all; the static GIN input gathered once at load"}),
            "final_loss": round(final_loss, 5),
            "grad_scale": (tr.inner if use_dist else tr).grad_scale,
            "setup_s": round(setup_s, 1),
        }
    if rank == 0 and ws == 1 and args.workload in ("gcn-reddit", "gin-products", "gat-rmat"):
        result["parity"] = parity_block(dg)
    if not args.no_sweep and ws == 1 and args.workload == "gcn-reddit":
        result["spmm_sweep_reddit"] = spmm_sweep(dg, peak)
    if rank == 0 and ws == 1 and not args.no_small and args.workload == "gcn-reddit":
        result["small_configs"] = small_configs(args, peak)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(args.workload, args.seed, args.cpu_budget_edges)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def spawn_ranks(n):
    """`bench.py --gpus N` without torchrun: relaunch this command under
    torch.distributed.run with N ranks on this node (rank 0 prints the line)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="gcn-reddit")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-small", action="store_true", help="skip the C1/C2 epoch timings")
    ap.add_argument("--no-graph", action="store_true", help="time eager steps, no CUDA graph")
    ap.add_argument("--reorder", choices=("auto", "none", "degree"), default="auto",
                    help="vertex relabelling for gather locality (auto: the workload's default)")
    ap.add_argument("--cpu-budget-edges", type=int, default=500_000,
                    help="edges in the B200 arm's cpu_baseline sample")
    ap.add_argument("--ref-budget-edges", type=int, default=0,
                    help="edges per --impl reference step (0: max(100K, 2M / steps))")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    ws, rank, local = dist_env()
    if ws != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; launch with "
                         f"torchrun --nproc-per-node {args.gpus} or without torchrun")
    if args.impl == "reference":
        reference_arm(args, ws, rank)
        return
    b200_arm(args, ws, rank, local)


if __name__ == "__main__":
    main()
