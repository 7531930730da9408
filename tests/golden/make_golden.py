"""Generate golden vectors from the REAL reference package (halfsparse).

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

It imports halfsparse from /root/reference/pkg/src (read-only; nothing is
copied) and writes small .npz fixtures next to this script.  The fixtures are
committed; neither the GPU box nor the product code ever reads /root/reference.
Every fixture records the reference entry point that produced it.
"""
from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

from halfsparse import kernels as K  # noqa: E402
from halfsparse import models as M  # noqa: E402
from halfsparse import simt  # noqa: E402
from halfsparse import sparse as sp  # noqa: E402
from halfsparse.kernels import Reduction  # noqa: E402

REDUCTIONS = [("post", "none"), ("post", "left"), ("post", "right"), ("post", "both"),
              ("pre", "left"), ("pre", "right"), ("pre", "both"),
              ("discretized", "left"), ("discretized", "right"), ("discretized", "both")]


def random_graph(rng, n, density):
    mask = rng.random((n, n)) < density
    np.fill_diagonal(mask, False)
    r, c = np.nonzero(mask)
    return sp.CooGraph.from_edges(n, r, c)


def hub_graph(rng, n, hubs, hub_deg, density):
    """Random graph plus a few heavy rows (rows spanning several warps/CTAs)."""
    mask = rng.random((n, n)) < density
    np.fill_diagonal(mask, False)
    r, c = np.nonzero(mask)
    extra_r, extra_c = [], []
    for h in hubs:
        cols = rng.choice(n, size=min(hub_deg, n), replace=False)
        extra_r.append(np.full(cols.size, h))
        extra_c.append(cols)
    r = np.concatenate([r, *extra_r])
    c = np.concatenate([c, *extra_c])
    return sp.CooGraph.from_edges(n, r, c)


def save(name, **arrays):
    np.savez_compressed(OUT / name, **arrays)
    print(f"wrote {name}: {len(arrays)} arrays", file=sys.stderr)


def gen_graph_build():
    rng = np.random.default_rng(100)
    d = {}
    for i, (n, m) in enumerate([(1, 0), (5, 12), (40, 300), (300, 5000), (1000, 20000)]):
        rows = rng.integers(0, n, m)
        cols = rng.integers(0, n, m)
        g = sp.CooGraph.from_edges(n, rows, cols)
        csr = sp.coo_to_csr(g)
        gt, perm = sp.transpose(g, return_perm=True)
        sym = sp.symmetrize(g)
        loops = sp.add_self_loops(g)
        d.update({f"c{i}_n": np.int64(n), f"c{i}_rows_in": rows, f"c{i}_cols_in": cols,
                  f"c{i}_rows": g.rows, f"c{i}_cols": g.cols, f"c{i}_offsets": csr.offsets,
                  f"c{i}_t_rows": gt.rows, f"c{i}_t_cols": gt.cols, f"c{i}_perm": perm,
                  f"c{i}_coldeg": sp.col_degrees(g),
                  f"c{i}_sym_rows": sym.rows, f"c{i}_sym_cols": sym.cols,
                  f"c{i}_loop_rows": loops.rows, f"c{i}_loop_cols": loops.cols})
    d["num_cases"] = np.int64(5)
    save("graph_build.npz", **d)


def gen_factors():
    """kernels._ref_factors over degree lists 0..3000 plus large degrees."""
    rng = np.random.default_rng(101)
    deg = np.concatenate([np.arange(0, 3001), rng.integers(3001, 400_000, 40)]).astype(np.int64)
    n = deg.size
    rows = np.repeat(np.arange(n, dtype=np.int64), deg)
    d = {"deg": deg}
    for dtype, tag in ((np.float16, "h"), (np.float32, "f")):
        _, fr = K._ref_factors(n, rows, rows, Reduction("post", "right"), dtype)
        _, fb = K._ref_factors(n, rows, rows, Reduction("post", "both"), dtype)
        d[f"inv_{tag}"] = fr.astype(dtype)
        d[f"isqrt_{tag}"] = fb.astype(dtype)
    save("factors.npz", **d)


def gen_spmm():
    rng = np.random.default_rng(102)
    d = {}
    i = 0
    feats = [2, 4, 6, 16, 32, 64, 128]
    for trial in range(48):
        red = REDUCTIONS[trial % len(REDUCTIONS)]
        f = feats[trial % len(feats)]
        dtype = np.float16 if trial % 6 else np.float32
        if trial % 5 == 4:
            g = hub_graph(rng, int(rng.integers(200, 400)), [3, 7, 8], 350, 0.02)
        else:
            n = int(rng.integers(4, 90))
            g = random_graph(rng, n, float(rng.uniform(0.05, 0.5)))
        chunk = int(rng.choice([64, 128, 266]))
        wpc = int(rng.choice([1, 2, 4, 8]))
        x = sp.DenseTensor(rng.normal(0, 2, (g.n, f)).astype(dtype))
        weighted = trial % 3 == 1
        w = rng.normal(size=g.num_edges).astype(dtype) if weighted else None
        sched = simt.plan_edge_parallel(g, chunk, wpc)
        r = Reduction(*red)
        if weighted:
            y, _, st = K.spmm_ve(g, w, x, sched, r, return_staging=True)
        else:
            y, _, st = K.spmm_v(g, x, sched, r, return_staging=True)
        d.update({f"c{i}_n": np.int64(g.n), f"c{i}_rows": g.rows, f"c{i}_cols": g.cols,
                  f"c{i}_x": x.data, f"c{i}_y": y.data, f"c{i}_chunk": np.int64(chunk),
                  f"c{i}_wpc": np.int64(wpc), f"c{i}_scaling": np.array(red[0]),
                  f"c{i}_norm": np.array(red[1]), f"c{i}_st_rows": st.rows,
                  f"c{i}_st_vals": st.partials})
        if weighted:
            d[f"c{i}_w"] = w
        i += 1
    # known answers (test_acceptance.py:97-122, test_kernels.py:177-204)
    for deg, scaling in ((1024, "post"), (1024, "discretized"), (4, "post"), (4, "pre"),
                         (4, "discretized")):
        g = sp.CooGraph(deg + 1, np.zeros(deg, np.int64), np.arange(1, deg + 1, dtype=np.int64))
        x = sp.DenseTensor(np.full((deg + 1, 32), 30000.0, dtype=np.float16))
        sched = simt.plan_edge_parallel(g)
        y, _, st = K.spmm_v(g, x, sched, Reduction(scaling, "right"), return_staging=True)
        d.update({f"c{i}_n": np.int64(g.n), f"c{i}_rows": g.rows, f"c{i}_cols": g.cols,
                  f"c{i}_x": x.data, f"c{i}_y": y.data, f"c{i}_chunk": np.int64(128),
                  f"c{i}_wpc": np.int64(4), f"c{i}_scaling": np.array(scaling),
                  f"c{i}_norm": np.array("right"), f"c{i}_st_rows": st.rows,
                  f"c{i}_st_vals": st.partials})
        i += 1
    d["num_cases"] = np.int64(i)
    save("spmm_edge.npz", **d)


def gen_vertex():
    rng = np.random.default_rng(103)
    d = {}
    i = 0
    for trial in range(24):
        red = REDUCTIONS[trial % len(REDUCTIONS)]
        f = [2, 8, 16, 64][trial % 4]
        dtype = np.float16 if trial % 5 else np.float32
        if trial % 4 == 3:
            g = hub_graph(rng, 150, [0, 5], 140, 0.05)
        else:
            g = random_graph(rng, int(rng.integers(4, 100)), float(rng.uniform(0.05, 0.6)))
        csr = sp.coo_to_csr(g)
        x = sp.DenseTensor(rng.normal(0, 2, (g.n, f)).astype(dtype))
        y, _, st = K.spmm_vertex_grouped(csr, x, reduction=Reduction(*red), return_staging=True)
        d.update({f"c{i}_n": np.int64(g.n), f"c{i}_offsets": csr.offsets, f"c{i}_cols": csr.cols,
                  f"c{i}_x": x.data, f"c{i}_y": y.data, f"c{i}_scaling": np.array(red[0]),
                  f"c{i}_norm": np.array(red[1]), f"c{i}_st_rows": st.rows,
                  f"c{i}_st_vals": st.partials})
        i += 1
    d["num_cases"] = np.int64(i)
    save("spmm_vertex.npz", **d)


def gen_sddmm():
    rng = np.random.default_rng(104)
    d = {}
    feats = [2, 6, 8, 16, 32, 48, 64, 128, 256]
    for i, f in enumerate(feats):
        dtype = np.float16 if i % 4 else np.float32
        g = random_graph(rng, int(rng.integers(10, 70)), 0.3)
        x = sp.DenseTensor(rng.normal(0, 2, (g.n, f)).astype(dtype))
        y = sp.DenseTensor(rng.normal(0, 2, (g.n, f)).astype(dtype))
        out, _ = K.sddmm(g, x, y)
        d.update({f"c{i}_n": np.int64(g.n), f"c{i}_rows": g.rows, f"c{i}_cols": g.cols,
                  f"c{i}_x": x.data, f"c{i}_y": y.data, f"c{i}_out": out})
    d["num_cases"] = np.int64(len(feats))
    save("sddmm.npz", **d)


def gen_attention():
    """attention_scores -> leaky_relu -> edge_softmax forward and backward."""
    rng = np.random.default_rng(105)
    d = {}
    cases = []
    for n, dens in ((30, 0.3), (80, 0.2), (60, 0.9)):
        cases.append(random_graph(rng, n, dens))
    cases.append(hub_graph(rng, 400, [1, 2], 390, 0.01))   # rows of length ~390 (deep trees)
    cases.append(sp.CooGraph(4, np.zeros(4, np.int64), np.arange(4, dtype=np.int64)))
    for i, g in enumerate(cases):
        dtype = np.float16 if i != 2 else np.float32
        bundle = M.GraphBundle.build(g)
        s_l = M.Tensor(rng.normal(0, 2, (g.n, 1)).astype(dtype), requires_grad=True)
        s_r = M.Tensor(rng.normal(0, 2, (g.n, 1)).astype(dtype), requires_grad=True)
        if i == 4:
            s_l = M.Tensor(np.zeros((g.n, 1), dtype), requires_grad=True)
            s_r = M.Tensor(np.zeros((g.n, 1), dtype), requires_grad=True)
        e = M.attention_scores(bundle, s_l, s_r)
        e2 = M.leaky_relu(e, 0.2)
        alpha = M.edge_softmax(bundle, e2)
        seed = rng.normal(size=g.num_edges).astype(dtype)
        alpha.backward(seed)
        d.update({f"c{i}_n": np.int64(g.n), f"c{i}_rows": g.rows, f"c{i}_cols": g.cols,
                  f"c{i}_sl": s_l.data[:, 0], f"c{i}_sr": s_r.data[:, 0], f"c{i}_e": e.data,
                  f"c{i}_e2": e2.data, f"c{i}_alpha": alpha.data, f"c{i}_seed": seed,
                  f"c{i}_g_e2": e2.grad, f"c{i}_g_e": e.grad,
                  f"c{i}_g_sl": s_l.grad[:, 0], f"c{i}_g_sr": s_r.grad[:, 0]})
    d["num_cases"] = np.int64(len(cases))
    # exhaustive shadow_exp over every non-positive half (test_acceptance.py:247-253)
    allv = np.arange(65536, dtype=np.uint16).view(np.float16)
    nonpos = allv[allv <= 0]
    d["exp_in"] = nonpos
    d["exp_out"] = M.shadow_exp(nonpos)
    save("attention.npz", **d)


def harness_train(g, x, labels, cfg, n_cls, heads=1, layers=2):
    """models.train (models.py:633-684) with the SURVEY 8(c) harness changes:
    classes padded to n_cls, and multi-head / deeper GAT composed of GATLayers
    (concat in hidden layers, mean at the output)."""
    rng = np.random.default_rng(cfg.seed)
    n, fan_in = x.shape
    bundle = M.GraphBundle.build(g)
    red = Reduction(cfg.scaling, cfg.norm)
    if cfg.kind == "gat" and (heads > 1 or layers > 2):
        widths = [fan_in] + [cfg.hidden * heads] * (layers - 1)
        outs = [cfg.hidden] * (layers - 1) + [n_cls]
        stack = [[M.GATLayer(rng, widths[li], outs[li]) for _ in range(heads)]
                 for li in range(layers)]
        params = [p for lay in stack for hl in lay for p in hl.params()]

        def forward(x_t, mode, ov):
            h = x_t
            for li, lay in enumerate(stack):
                outs_h = [hl(bundle, h, mode, cfg.width, ov, f"gat{li}.{k}")
                          for k, hl in enumerate(lay)]
                if li + 1 < len(stack):
                    h = M.relu(_concat(outs_h))
                else:
                    h = _mean(outs_h)
            return h
    else:
        model = M.Model(cfg.kind, rng, (fan_in, cfg.hidden, n_cls), red, cfg.lam)
        params = model.params()

        def forward(x_t, mode, ov):
            return model.forward(bundle, x_t, mode, cfg.width, ov)

    opt = M.Adam(params, lr=cfg.lr)
    perm = rng.permutation(n)
    n_val = int(n * cfg.val_fraction)
    val_mask = np.zeros(n, dtype=bool)
    val_mask[perm[:n_val]] = True
    train_mask = ~val_mask
    dtype = np.float16 if cfg.mode == "half" else np.float32
    x_data = x.astype(np.float32)
    if cfg.mode == "half":
        x_data = M.to_half(x_data)
    losses, accs = [], []
    t0 = time.perf_counter()
    for epoch in range(cfg.epochs):
        xt = M.Tensor(x_data.astype(dtype))
        logits = forward(xt, cfg.mode, None)
        if cfg.mode == "half":
            logits = M.convert(logits, "float32")
        loss = M.cross_entropy(logits, labels)
        loss.backward(np.float32(1.0))
        opt.step()
        losses.append(float(loss.data))
        accs.append((M.accuracy(logits.data, labels, train_mask),
                     M.accuracy(logits.data, labels, val_mask)))
    return np.array(losses), np.array(accs), (time.perf_counter() - t0) / max(cfg.epochs, 1)


def _concat(ts):
    data = np.concatenate([t.data for t in ts], axis=1)
    out = M.Tensor(data, parents=tuple(ts))
    widths = [t.shape[1] for t in ts]

    def bwd(g):
        o = 0
        for t, wdt in zip(ts, widths):
            if t.requires_grad:
                t._accumulate(np.ascontiguousarray(g[:, o:o + wdt]))
            o += wdt
    out._backward = bwd
    return out


def _mean(ts):
    k = len(ts)
    dtype = ts[0].data.dtype
    data = (sum(t.data.astype(np.float64) for t in ts) / k).astype(dtype)
    out = M.Tensor(data, parents=tuple(ts))

    def bwd(g):
        gg = (g.astype(np.float64) / k).astype(dtype)
        for t in ts:
            if t.requires_grad:
                t._accumulate(gg)
    out._backward = bwd
    return out


def gen_training():
    d = {}
    # small SBM, all three kinds, both modes (the test_models.py shapes)
    g, x, labels = sp.synth_sbm(60, 2, 0.5, 0.1, 8, seed=1)
    d["sbm_rows"], d["sbm_cols"], d["sbm_x"], d["sbm_labels"] = g.rows, g.cols, x.data, labels
    for kind in ("gcn", "gin", "gat"):
        for mode in ("half", "float32"):
            cfg = M.TrainConfig(kind=kind, mode=mode, epochs=5, seed=3)
            losses, accs, _ = harness_train(g, x.data, labels, cfg, 2)
            d[f"sbm_{kind}_{mode}_loss"] = losses
            d[f"sbm_{kind}_{mode}_acc"] = accs
    # multi-head 3-layer GAT composition on the same small graph
    cfg = M.TrainConfig(kind="gat", mode="half", epochs=4, seed=5, hidden=4)
    losses, accs, _ = harness_train(g, x.data, labels, cfg, 2, heads=4, layers=3)
    d["sbm_gat4x3_half_loss"], d["sbm_gat4x3_half_acc"] = losses, accs
    # C1: Cora-shaped 2-layer GCN, 200 epochs, classes 7 -> 8
    g1, x1, l1 = sp.synth_sbm(2708, 7, 0.0085, 0.00026, 1433, 0)
    d["c1_num_edges"] = np.int64(g1.num_edges)
    for mode in ("half", "float32"):
        cfg = M.TrainConfig(kind="gcn", mode=mode, epochs=200, seed=0)
        losses, accs, sec = harness_train(g1, x1.data, l1, cfg, 8)
        d[f"c1_gcn_{mode}_loss"], d[f"c1_gcn_{mode}_acc"] = losses, accs
        d[f"c1_gcn_{mode}_sec_per_epoch"] = np.float64(sec)
    save("training.npz", **d)


def gen_c2(mode="half"):
    """C2 (Pubmed-shaped synth_sbm, 3-layer x 4-head x 16 GAT, classes 3 -> 4):
    200 epochs of the reference harness (models.py:633-684 composed from
    GATLayer, models.py:492-509).  About 40 min per mode on the build host;
    run as `make_golden.py c2 half` / `c2 float32` (one file per mode)."""
    g, x, labels = sp.synth_sbm(19717, 3, 0.00057, 5.71e-5, 500, 0)
    cfg = M.TrainConfig(kind="gat", mode=mode, epochs=200, seed=0, hidden=16)
    losses, accs, sec = harness_train(g, x.data, labels, cfg, 4, heads=4, layers=3)
    save(f"c2_{mode}.npz", num_edges=np.int64(g.num_edges), loss=losses, acc=accs,
         sec_per_epoch=np.float64(sec), config=np.str_(
             "synth_sbm(19717,3,0.00057,5.71e-5,500,0); GAT 3 layers x 4 heads x 16, "
             "concat + relu between layers, mean at the output; TrainConfig(seed=0, "
             f"mode={mode}, epochs=200); classes padded 3 -> 4"))


INGEST_CASES = [
    # (text, num_vertices, symmetrize)
    (b"# a comment\n0 1\n% another\n1 2\n\n2 0\n", None, False),    # test_sparse.py:127-131
    (b"0 1\nnot an edge\n", None, False),                               # :133-137
    (b"0\n", None, False),                                              # :139-143
    (b"0 1\n", 10, False),                                              # :145-148
    (b"0 1\n", None, True),                                             # :150-154
    (b"0 1\r\n1 2\r\n2 x\r\n", None, False),
    (b"0 1\r1 2\r3 -4\n", None, False),
    (b"  0\t 1  extra\n\t2 3 4 5\n\n   \n", None, False),
    (b"1_0 +2\n-0 003\n", None, False),
    (b"1__0 2\n", None, False),
    (b"_1 2\n", None, False),
    (b"1_ 2\n", None, False),
    (b"0 5\n", 3, False),
    (b"", None, False),
    (b"# only\n% comments\n", None, False),
    (b"# only\n", 4, False),
    (b"1 1\n0 1\n0 1\n", None, False),
    (b"0 1\n1 2", None, False),
    (b"0\x0b1\n2\x0c3\n4\x1f5\n", None, False),
    (b"0 1 # trailing\n#c\n  # indented\n2 1", None, True),
    (b"3 4\n1 2\n5 -1 x\n", None, False),
    (b"3 4\nx\n5 -1\n", None, False),
    (b"7 8\n+ 1\n", None, False),
    (b"7 8\n- 1\n", None, False),
    (b"0 99999999999999999999\n1 2\n", None, False),
    (b"0 99999999999999999999\nbad line\n", None, False),
    (b"-99999999999999999999 1\n", None, False),
    (b"\r\n\r\n0 1\r\n\r", None, False),
    (b"0 1\n2 3\n", 3, False),
]


def gen_ingest():
    """sparse.load_edge_list on small texts (the loader tests plus whitespace,
    newline, int() syntax, error-order and overflow cases) and one large
    randomized file; errors recorded as '<Type>: <message>' with the path
    replaced by '<path>'."""
    import tempfile

    rng = np.random.default_rng(11)
    parts = []
    for i in range(3000):
        k = rng.integers(0, 20)
        if k == 0:
            parts.append(b"# comment line\n")
        elif k == 1:
            parts.append(b"\n")
        else:
            ws = [b" ", b"\t", b"  ", b" \t "][rng.integers(0, 4)]
            parts.append(b"%d%s%d%s" % (rng.integers(0, 500), ws, rng.integers(0, 500),
                                         [b"\n", b"\r\n", b" \n"][rng.integers(0, 3)]))
    cases = INGEST_CASES + [(b"".join(parts), None, False), (b"".join(parts), 600, True)]
    d = {"num_cases": np.int64(len(cases))}
    with tempfile.TemporaryDirectory() as tmp:
        for i, (text, nv, sym) in enumerate(cases):
            p = Path(tmp) / f"c{i}.txt"
            p.write_bytes(text)
            d[f"c{i}_text"] = np.frombuffer(text, dtype=np.uint8).copy()
            d[f"c{i}_nv"] = np.int64(-1 if nv is None else nv)
            d[f"c{i}_sym"] = np.bool_(sym)
            try:
                g = sp.load_edge_list(p, num_vertices=nv, symmetrize_edges=sym)
                d[f"c{i}_n"] = np.int64(g.n)
                d[f"c{i}_rows"], d[f"c{i}_cols"] = g.rows, g.cols
                d[f"c{i}_err"] = np.str_("")
            except Exception as exc:  # record the reference's failure
                d[f"c{i}_n"] = np.int64(-1)
                d[f"c{i}_err"] = np.str_(f"{type(exc).__name__}: {str(exc).replace(str(p), '<path>')}")
    save("ingest.npz", **d)


if __name__ == "__main__":
    which = sys.argv[1:] or ["graph", "factors", "spmm", "vertex", "sddmm", "attention", "training",
                             "ingest"]
    if which[0] == "c2":
        gen_c2(*which[1:])
        sys.exit(0)
    for w in which:
        globals()[f"gen_{w}" if w != "graph" else "gen_graph_build"]()
