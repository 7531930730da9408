"""The CPU legs of bench.py: the reference's own training epoch (halfsparse,
installed unmodified under baseline/_ref, or the numpy restatement in oracle/
when it is absent) and a torch-CPU fp32 CSR comparator, timed on a random
row-panel sample of the benched graph.

Nothing here touches the GPU or libhalfgnn.so: the graph rows are regenerated
on the host by synth.py (bit-identical to the rows the B200 arm trains on),
features and labels by the same planted-class recipe in numpy.  Per step, the
sparse operators' time (spmm_v / spmm_ve / sddmm, timed by wrapping the
reference module's functions; the oracle's own timer for the port) is scaled
by E / E_sample; the dense part (X.W over all N vertices, loss, Adam) is
measured at full size.  The result is labelled extrapolated.
"""
from __future__ import annotations

import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF_DIR = ROOT / "baseline" / "_ref"


def core_counts():
    try:
        aff = len(os.sched_getaffinity(0))
    except AttributeError:
        aff = os.cpu_count() or 1
    try:
        import torch

        tt = torch.get_num_threads()
    except Exception:
        tt = None
    return {"os_cpu_count": os.cpu_count(), "sched_affinity": aff, "torch_threads": tt}


def load_reference():
    """The unmodified reference package (baseline/_ref), or None."""
    if not (REF_DIR / "halfsparse" / "__init__.py").exists():
        return None
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    try:
        import halfsparse  # noqa: F401
        from halfsparse import kernels, models, sparse  # noqa: F401

        return sys.modules["halfsparse"]
    except Exception:
        return None


# ───────────────────────────── host workloads ────────────────────────────────


class HostWorkload:
    """A benched graph on the host: full-graph row offsets (for sampling), a
    function producing any ascending row subset's CSR, features, labels."""

    def __init__(self, name, seed, feat, classes):
        from paper_2411_01109_b200 import synth as S

        self.name, self.seed, self.feat, self.classes = name, seed, feat, classes
        if name == "gat-pubmed":
            from paper_2411_01109_b200.graphgen import pubmed_like

            r, c, x, labels = pubmed_like(seed)
            self.n = x.shape[0]
            off = np.zeros(self.n + 1, np.int64)
            np.cumsum(np.bincount(r, minlength=self.n), out=off[1:])
            self.offsets, self.num_edges, self.labels = off, int(r.size), labels
            self.x16 = x.astype(np.float16)

            def rows_of(rows, off=off, cols=c):
                d = off[rows + 1] - off[rows]
                o = np.concatenate([[0], np.cumsum(d)])
                idx = np.repeat(off[rows] - o[:-1], d) + np.arange(int(o[-1]))
                return o, cols[idx]
            self._rows = rows_of
            return
        if name == "gcn-reddit":
            deg = S.reddit_degrees(seed)
            self.n = deg.size
            self.offsets = np.concatenate([[0], np.cumsum(deg)])
            self._rows = lambda rows: S.reddit_rows(rows, deg, seed, self.n)
        else:  # no row-independent recipe: build the full graph on the host
            if name == "gin-products":
                off, cols = S.products_graph(seed)
            elif name == "gat-rmat":
                off, cols = S.rmat_graph(24, 16, seed)
            else:
                raise ValueError(f"no host recipe for {name}")
            self.n = off.size - 1
            self.offsets = off

            def rows_of(rows, off=off, cols=cols):
                d = off[rows + 1] - off[rows]
                o = np.concatenate([[0], np.cumsum(d)])
                idx = np.repeat(off[rows] - o[:-1], d) + np.arange(int(o[-1]))
                return o, cols[idx]
            self._rows = rows_of
        self.num_edges = int(self.offsets[-1])
        self.labels = (np.arange(self.n, dtype=np.int64) * classes) // self.n
        rng = np.random.default_rng(seed + 1)
        means = rng.normal(0.0, 1.0, (classes, feat))
        means = means / np.maximum(np.linalg.norm(means, axis=1, keepdims=True), 1e-12) * 4.0
        x = rng.standard_normal((self.n, feat), dtype=np.float32)
        x += means[self.labels].astype(np.float32)
        self.x16 = x.astype(np.float16)

    def sample(self, budget_edges, sample_seed):
        """(rows, cols) COO of a random row-panel sample (all n vertices)."""
        from paper_2411_01109_b200 import synth as S

        rows = S.sample_row_panels(self.offsets, budget_edges, panels=64, seed=sample_seed)
        off, cols = self._rows(rows)
        r = np.repeat(rows, np.diff(off))
        return r.astype(np.int64), cols.astype(np.int64)


# ─────────────────────────── the reference epoch ─────────────────────────────


class _SparseTimer:
    """Wraps halfsparse.kernels' sparse operators to accumulate their time."""

    NAMES = ("spmm_v", "spmm_ve", "sddmm", "spmm_vertex_grouped")

    def __init__(self, kernels):
        self.k = kernels
        self.t = 0.0
        self.saved = {}

    def __enter__(self):
        for nm in self.NAMES:
            f = getattr(self.k, nm)
            self.saved[nm] = f

            def wrap(*a, _f=f, **kw):
                t0 = time.perf_counter()
                try:
                    return _f(*a, **kw)
                finally:
                    self.t += time.perf_counter() - t0
            setattr(self.k, nm, wrap)
        return self

    def __exit__(self, *exc):
        for nm, f in self.saved.items():
            setattr(self.k, nm, f)


def reference_epoch(H, n, rows, cols, x16, labels, kind, hidden, seed=0, lam=0.1):
    """One training epoch through the reference's public API (models.py:633-684
    loop body: forward, convert, cross_entropy, backward, Adam.step) on the
    sampled graph.  Returns (sparse seconds, other seconds)."""
    M, K, SP = H.models, H.kernels, H.sparse
    g = SP.CooGraph(n, rows, cols)
    bundle = M.GraphBundle.build(g)
    n_cls = int(labels.max()) + 1
    n_cls += n_cls % 2                     # classes padded to even
    rng = np.random.default_rng(seed)
    model = M.Model(kind, rng, (x16.shape[1], hidden, n_cls),
                    K.Reduction("discretized", "both"), lam)
    opt = M.Adam(model.params(), lr=1e-2)
    x_data = x16
    t0 = time.perf_counter()
    with _SparseTimer(K) as st:
        xt = M.Tensor(x_data.astype(np.float16))
        logits = model.forward(bundle, xt, "half", "half2", None)
        logits = M.convert(logits, "float32")
        loss = M.cross_entropy(logits, labels)
        loss.backward(np.float32(1.0))
        opt.step()
    wall = time.perf_counter() - t0
    if not np.isfinite(float(loss.data)):
        raise RuntimeError("reference epoch produced a non-finite loss")
    return st.t, wall - st.t


def port_epoch(n, rows, cols, x16, labels, kind, hidden, heads=1, layers=2):
    """The same epoch through the numpy restatement (oracle/): (sparse s, other s)."""
    import oracle as O

    g = O.OracleGraph(n, rows, cols)
    timer = O.Timer()
    t0 = time.perf_counter()
    O.train_epochs(g, x16.astype(np.float32), labels, kind=kind, mode="half", epochs=1,
                   hidden=hidden, heads=heads, layers=layers, timer=timer)
    wall = time.perf_counter() - t0
    return timer.sparse, wall - timer.sparse


def torch_cpu_epoch(n, rows, cols, x16, labels, hidden, threads=None):
    """A plain torch-CPU fp32 GCN epoch (CSR sparse.mm, both-side degree norm,
    autograd through a custom Function whose backward is the transposed CSR
    product; Adam) on all host threads: SURVEY 8(d) item 3's stronger CPU
    comparator.  Returns (sparse s, other s)."""
    import torch

    if threads:
        torch.set_num_threads(threads)
    dout = np.bincount(rows, minlength=n).astype(np.float32)
    din = np.bincount(cols, minlength=n).astype(np.float32)
    fo = np.where(dout > 0, 1.0 / np.sqrt(np.maximum(dout, 1)), 0).astype(np.float32)
    fi = np.where(din > 0, 1.0 / np.sqrt(np.maximum(din, 1)), 0).astype(np.float32)
    vals = torch.from_numpy(fo[rows] * fi[cols])
    off = torch.from_numpy(np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=n))]))
    a = torch.sparse_csr_tensor(off, torch.from_numpy(cols), vals, (n, n))
    at = a.t().to_sparse_csr()
    spent = [0.0]

    class Agg(torch.autograd.Function):
        @staticmethod
        def forward(ctx, x):
            t0 = time.perf_counter()
            y = torch.sparse.mm(a, x)
            spent[0] += time.perf_counter() - t0
            return y

        @staticmethod
        def backward(ctx, g):
            t0 = time.perf_counter()
            y = torch.sparse.mm(at, g)
            spent[0] += time.perf_counter() - t0
            return y

    n_cls = int(labels.max()) + 1
    gen = torch.Generator().manual_seed(0)
    w1 = (torch.randn(x16.shape[1], hidden, generator=gen) * 0.05).requires_grad_()
    w2 = (torch.randn(hidden, n_cls, generator=gen) * 0.1).requires_grad_()
    opt = torch.optim.Adam([w1, w2], lr=1e-2)
    x = torch.from_numpy(x16.astype(np.float32))
    y = torch.from_numpy(labels)
    t0 = time.perf_counter()
    h = torch.relu(Agg.apply(x @ w1))
    out = Agg.apply(h @ w2)
    loss = torch.nn.functional.cross_entropy(out, y)
    opt.zero_grad()
    loss.backward()
    opt.step()
    wall = time.perf_counter() - t0
    return spent[0], wall - spent[0]


def extrapolate(sparse_s, other_s, e_sample, e_total, sparse_fixed=0.0, e_fixed=0):
    """ms/epoch at e_total edges: the non-sparse part as measured (full size),
    the sparse part linear in E through the calibration point (e_fixed,
    sparse_fixed) -- the sparse operators' per-call O(N) cost (output
    allocation, factor tables) does not scale with the sample."""
    slope = max(sparse_s - sparse_fixed, 0.0) / max(e_sample - e_fixed, 1)
    return (other_s + sparse_fixed + slope * (e_total - e_fixed)) * 1e3


class CpuLeg:
    """One CPU implementation (reference / port / torch) timed per step on a
    fresh random row-panel sample, with a one-off calibration epoch on a tiny
    sample that fixes the sparse operators' E-independent cost."""

    def __init__(self, w: HostWorkload, impl, cfg, H=None, calib_edges=2_000):
        self.w, self.impl, self.cfg, self.H = w, impl, cfg, H
        self.calib_edges = calib_edges
        self.fixed = None
        self.sampled_edges = 0
        self.steps = 0

    def _epoch(self, rows, cols):
        w, c = self.w, self.cfg
        if self.impl == "reference":
            return reference_epoch(self.H, w.n, rows, cols, w.x16, w.labels, c["kind"],
                                   c["hidden"])
        if self.impl == "torch":
            return torch_cpu_epoch(w.n, rows, cols, w.x16, w.labels, c["hidden"])
        return port_epoch(w.n, rows, cols, w.x16, w.labels, c["kind"], c["hidden"],
                          c.get("heads", 1), c.get("layers", 2))

    def calibrate(self):
        r, c = self.w.sample(self.calib_edges, 999_983)
        if self.impl == "torch":
            self._epoch(r, c)                      # first-call warm-up
        s, _ = self._epoch(r, c)
        self.fixed = (s, int(r.size))

    def step(self, budget_edges, sample_seed, warm=False):
        """One epoch on a fresh sample; returns extrapolated ms/epoch."""
        if self.fixed is None:
            self.calibrate()
        if budget_edges >= self.w.num_edges:
            r = np.repeat(np.arange(self.w.n), np.diff(self.w.offsets))
            _, c = self.w._rows(np.arange(self.w.n))
        else:
            r, c = self.w.sample(budget_edges, sample_seed)
        s, o = self._epoch(r, c)
        if not warm:
            self.sampled_edges += int(r.size)
            self.steps += 1
        if r.size >= self.w.num_edges:
            return (s + o) * 1e3
        return extrapolate(s, o, r.size, self.w.num_edges, *self.fixed)

    def describe(self, budget_edges):
        what = {"reference": "halfsparse (unmodified, baseline/_ref) public API: Model.forward, "
                             "convert, cross_entropy, backward, Adam.step",
                "port": "numpy restatement of the reference (oracle/)",
                "torch": "torch-CPU fp32 CSR GCN (torch.sparse.mm, autograd, Adam)"}[self.impl]
        if budget_edges >= self.w.num_edges:
            return f"{what}; full graph ({self.w.num_edges:,} edges) every step"
        return (f"{what}; every step a fresh random sample of 64 row panels holding "
                f"~{budget_edges:,} of {self.w.num_edges:,} edges (all {self.w.n:,} vertices, "
                f"all features); {self.sampled_edges:,} edges sampled over {self.steps} timed "
                f"steps; sparse-operator time extrapolated linearly in E through a "
                f"{self.fixed[1]:,}-edge calibration epoch (sparse {self.fixed[0]:.2f} s), "
                f"dense work (all vertices) measured at full size")
