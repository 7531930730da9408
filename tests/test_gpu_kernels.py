"""GPU parity: every CUDA operator against the reference's golden vectors and
the CPU oracle.  Bit-exact for graph construction, schedules, factor tables,
reference-order SpMM, SDDMM and edge softmax; the fp32-guarded SpMM within the
SURVEY Appendix A tolerance (|y - y_f64| <= 1e-2 * max(1, |y_f64|))."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle as O
from conftest import bits, golden_cases, load_golden

pytestmark = pytest.mark.gpu

TOL = 1e-2  # SURVEY Appendix A, rule (1)


def _dg(n, rows, cols, dev):
    from paper_2411_01109_b200.device import DeviceGraph

    return DeviceGraph.from_edges(n, np.asarray(rows), np.asarray(cols), device=dev)


def _t(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


# ── graph construction ───────────────────────────────────────────────────


def test_build_csr_and_transpose_golden(cuda):
    from paper_2411_01109_b200 import device as D

    cases, _ = golden_cases("graph_build.npz")
    for c in cases:
        n = int(c["n"])
        off, cols, rows = D.build_csr(n, _t(c["rows_in"], cuda), _t(c["cols_in"], cuda), True)
        np.testing.assert_array_equal(off.cpu().numpy(), c["offsets"])
        np.testing.assert_array_equal(cols.cpu().numpy(), c["cols"])
        np.testing.assert_array_equal(rows.cpu().numpy(), c["rows"])
        t_off, t_cols, perm = D.transpose_csr(off, cols, n)
        np.testing.assert_array_equal(perm.cpu().numpy(), c["perm"])
        np.testing.assert_array_equal(t_cols.cpu().numpy(), c["t_cols"])
        np.testing.assert_array_equal(np.diff(t_off.cpu().numpy()), c["coldeg"])
        # symmetrize / self loops = canonicalisation of the concatenation
        r, cc = c["rows"], c["cols"]
        off2, cols2, rows2 = D.build_csr(n, _t(np.r_[r, cc], cuda), _t(np.r_[cc, r], cuda), True)
        np.testing.assert_array_equal(rows2.cpu().numpy(), c["sym_rows"])
        np.testing.assert_array_equal(cols2.cpu().numpy(), c["sym_cols"])
        v = np.arange(n)
        off3, cols3, rows3 = D.build_csr(n, _t(np.r_[r, v], cuda), _t(np.r_[cc, v], cuda), True)
        np.testing.assert_array_equal(rows3.cpu().numpy(), c["loop_rows"])
        np.testing.assert_array_equal(cols3.cpu().numpy(), c["loop_cols"])


def test_build_csr_errors(cuda):
    from paper_2411_01109_b200 import device as D

    with pytest.raises(ValueError, match="negative vertex id"):
        D.build_csr(4, _t(np.array([0, -1]), cuda), _t(np.array([1, 2]), cuda))
    with pytest.raises(ValueError, match="out of range"):
        D.build_csr(4, _t(np.array([0, 4]), cuda), _t(np.array([1, 2]), cuda))


def test_build_csr_large_random_vs_oracle(cuda):
    from paper_2411_01109_b200 import device as D

    rng = np.random.default_rng(7)
    n, m = 200_000, 3_000_000
    rows = rng.integers(0, n, m)
    cols = (rows + rng.integers(-50, 50, m)) % n
    off, c32, r64 = D.build_csr(n, _t(rows, cuda), _t(cols, cuda), True)
    wr, wc = O.canonical_edges(n, rows, cols)
    np.testing.assert_array_equal(r64.cpu().numpy(), wr)
    np.testing.assert_array_equal(c32.cpu().numpy(), wc)
    np.testing.assert_array_equal(off.cpu().numpy(), O.csr_offsets(n, wr))
    _, _, perm = D.transpose_csr(off, c32, n)
    np.testing.assert_array_equal(perm.cpu().numpy(), O.transpose_perm(n, wr, wc)[2])


def test_factors_golden(cuda):
    from paper_2411_01109_b200 import device as D

    g = load_golden("factors.npz")
    deg = g["deg"]
    off = _t(np.r_[0, np.cumsum(deg)].astype(np.int64), cuda)
    for dt, tag in ((torch.float16, "h"), (torch.float32, "f")):
        inv = D.degree_factors(off, "inv", dt).cpu().numpy()
        isq = D.degree_factors(off, "inv_sqrt", dt).cpu().numpy()
        np.testing.assert_array_equal(bits(inv), bits(g[f"inv_{tag}"]))
        np.testing.assert_array_equal(bits(isq), bits(g[f"isqrt_{tag}"]))


@pytest.mark.parametrize("cap", [4, 32, 512])
def test_schedule_matches_restatement(cuda, cap):
    from paper_2411_01109_b200 import device as D

    rng = np.random.default_rng(cap)
    deg = np.concatenate([np.zeros(50, np.int64), rng.integers(0, 3 * cap, 3000),
                          np.array([20 * cap + 3, 7 * cap])])
    rng.shuffle(deg)
    off = np.r_[0, np.cumsum(deg)].astype(np.int64)
    s = D.build_schedule(_t(off, cuda), cap)
    units, split_rows, slots = O.schedule_units(off, cap)
    np.testing.assert_array_equal(s.units.cpu().numpy(), units)
    np.testing.assert_array_equal(s.split_rows.cpu().numpy(), split_rows)
    assert s.num_slots == slots


def _short_row_graph(seed, n):
    """Mostly short and empty rows (packs) with a few long and split rows."""
    rng = np.random.default_rng(seed)
    deg = rng.choice([0, 0, 0, 1, 2, 3, 5, 9, 17, 32], size=n)
    deg[n // 3: n // 3 + min(n // 3, 1000)] = 0   # a run of empty rows (empty-only packs)
    deg[rng.integers(0, n, 6)] = [33, 100, 600, 2000, 40, 5000]
    rows = np.repeat(np.arange(n), deg)
    return O.canonical_edges(n, rows, rng.integers(0, n, rows.size))


@pytest.mark.parametrize("n", [16, 1001, 40000])
def test_schedule_packs_match_restatement(cuda, n):
    from paper_2411_01109_b200 import device as D

    r, c = _short_row_graph(n, n)
    off = O.csr_offsets(n, r)
    s = D.build_schedule(_t(off, cuda), 512, 16, 64)
    units, split_rows, slots, packs = O.schedule_units(off, 512, 16, 64)
    np.testing.assert_array_equal(s.units.cpu().numpy(), units)
    np.testing.assert_array_equal(s.split_rows.cpu().numpy(), split_rows)
    np.testing.assert_array_equal(s.packs.cpu().numpy(), packs)
    assert s.num_slots == slots
    # every row is covered exactly once by units or packs
    cover = np.zeros(n, np.int64)
    np.add.at(cover, units[:, 0][units[:, 3] < 0], 1)
    np.add.at(cover, split_rows[:, 0], 1)
    for r0, _, _, cnt in packs:
        cover[r0:r0 + cnt] += 1
    assert (cover == 1).all()


@pytest.mark.parametrize("pack_edges", [0, 64, 512])
@pytest.mark.parametrize("f", [8, 48, 64, 128, 512])
@pytest.mark.parametrize("mode", ["plain", "weighted", "perm", "sumw"])
def test_spmm_packed_rows_bitwise_equal_units(cuda, f, mode, pack_edges):
    """Packed short rows (one team walking a run of rows as one edge stream)
    give bit-identical output to the same rows as separate units, for every
    team width, weights direct / through perm, output factors, ReLU and the
    summed second weight block."""
    from paper_2411_01109_b200 import device as D

    n = 30000
    r, c = _short_row_graph(f, n)
    dg = _dg(n, r, c, cuda)
    heads = 4 if f % 32 == 0 else 1
    if mode == "sumw" and f > 256:
        pytest.skip("summed weights need F/8 <= 32")
    x = torch.randn(n, f, device=cuda, dtype=torch.float16)
    fout = torch.rand(n, device=cuda, dtype=torch.float16)
    view = dg.view(mode in ("perm", "sumw"))
    e = r.size
    w = widx = w2 = out2 = None
    kw = {}
    if mode == "weighted":
        w = torch.randn(e, heads, device=cuda, dtype=torch.float16)
    elif mode in ("perm", "sumw"):
        ae = torch.randn(e, 2 * heads, device=cuda, dtype=torch.float16)
        w, widx = ae[:, :heads], view.perm
        if mode == "sumw":
            kw = dict(w2_off=heads)
    outs = []
    saved = (D.PACK_EDGES_WIDE, D.PACK_EDGES_NARROW, D.PACK_MIN_ROWS)
    D.PACK_EDGES_WIDE = D.PACK_EDGES_NARROW = pack_edges
    D.PACK_MIN_ROWS = 0
    for packing in (False, True):
        D.PACKING = packing
        try:
            extra = {}
            if mode == "sumw":
                extra["out2"] = torch.empty(n, heads, device=cuda, dtype=torch.float16)
            y = D.spmm_csr(view, x, w, widx, heads if w is not None else 1, "discretized",
                           fout=fout, relu=(mode == "plain"), **kw, **extra)
            outs.append((y, extra.get("out2")))
        finally:
            D.PACKING = True
    D.PACK_EDGES_WIDE, D.PACK_EDGES_NARROW, D.PACK_MIN_ROWS = saved
    if mode in ("plain", "weighted"):  # (the empty run is in CSR rows)
        assert view.schedule(pack_edges=pack_edges).num_packs > 0
    np.testing.assert_array_equal(bits(outs[0][0].cpu().numpy()), bits(outs[1][0].cpu().numpy()))
    if mode == "sumw":
        np.testing.assert_array_equal(bits(outs[0][1].cpu().numpy()),
                                      bits(outs[1][1].cpu().numpy()))


# ── reference-order SpMM (bit-exact) ─────────────────────────────────────


def test_spmm_edge_ref_golden(cuda):
    from paper_2411_01109_b200 import device as D

    cases, _ = golden_cases("spmm_edge.npz")
    for i, c in enumerate(cases):
        n = int(c["n"])
        dg = _dg(n, c["rows"], c["cols"], cuda)
        x = _t(c["x"], cuda)
        w = _t(c["w"], cuda) if "w" in c else None
        y, st_rows, st_vals = D.spmm_edge_ref(dg, x, w, str(c["scaling"]), str(c["norm"]),
                                              warp_chunk=int(c["chunk"]),
                                              warps_per_cta=int(c["wpc"]), staging=True)
        np.testing.assert_array_equal(bits(y.cpu().numpy()), bits(c["y"]), err_msg=f"case {i}")
        np.testing.assert_array_equal(st_rows.cpu().numpy(), c["st_rows"], err_msg=f"case {i}")
        np.testing.assert_array_equal(bits(st_vals.cpu().numpy()), bits(c["st_vals"]),
                                      err_msg=f"case {i}")


def test_spmm_vertex_ref_golden(cuda):
    from paper_2411_01109_b200 import device as D
    from paper_2411_01109_b200.device import DeviceGraph

    cases, _ = golden_cases("spmm_vertex.npz")
    for i, c in enumerate(cases):
        n = int(c["n"])
        rows = O.rows_from_offsets(c["offsets"])
        dg = DeviceGraph.from_edges(n, rows, c["cols"], device=cuda)
        y, st_rows, st_vals = D.spmm_vertex_ref(dg, _t(c["x"], cuda), str(c["scaling"]),
                                                str(c["norm"]), staging=True)
        np.testing.assert_array_equal(bits(y.cpu().numpy()), bits(c["y"]), err_msg=f"case {i}")
        np.testing.assert_array_equal(st_rows.cpu().numpy(), c["st_rows"])
        np.testing.assert_array_equal(bits(st_vals.cpu().numpy()), bits(c["st_vals"]))


@pytest.mark.parametrize("scaling,norm", [("post", "both"), ("discretized", "both"),
                                          ("pre", "right"), ("post", "none")])
@pytest.mark.parametrize("f", [16, 64, 256])
def test_spmm_edge_ref_vs_oracle_powerlaw(cuda, scaling, norm, f):
    from paper_2411_01109_b200 import device as D

    rng = np.random.default_rng(f)
    n = 3000
    deg = np.minimum(rng.zipf(1.8, n), 2500)
    rows = np.repeat(np.arange(n), deg)
    cols = rng.integers(0, n, rows.size)
    r, c = O.canonical_edges(n, rows, cols)
    x = rng.normal(0, 1, (n, f)).astype(np.float16)
    want, wrows, wvals = O.spmm_edge_parallel(n, r, c, x, None, 128, 4, scaling, norm)
    dg = _dg(n, r, c, cuda)
    y, srow, sval = D.spmm_edge_ref(dg, _t(x, cuda), None, scaling, norm, staging=True)
    np.testing.assert_array_equal(bits(y.cpu().numpy()), bits(want))
    np.testing.assert_array_equal(srow.cpu().numpy(), wrows)
    np.testing.assert_array_equal(bits(sval.cpu().numpy()), bits(wvals))


def test_hub_known_answers(cuda):
    """test_acceptance.py:97-122: post -> INF in exactly the hub row, discretized 29904."""
    from paper_2411_01109_b200 import device as D

    n = 1025
    dg = _dg(n, np.zeros(n - 1, np.int64), np.arange(1, n), cuda)
    x = torch.full((n, 32), 30000.0, dtype=torch.float16, device=cuda)
    y_post = D.spmm_edge_ref(dg, x, None, "post", "right").cpu().numpy()
    assert np.isinf(y_post[0]).all() and np.isinf(y_post).sum() == 32
    y_disc = D.spmm_edge_ref(dg, x, None, "discretized", "right").cpu().numpy()
    assert np.isfinite(y_disc).all() and float(y_disc[0, 0]) == 29904.0
    # the fp32-guarded kernel keeps the post-mode overflow of raw sums and is exact otherwise
    yf = D.spmm(dg, x, None, "post", "right").cpu().numpy()
    assert np.isinf(yf[0]).all() and np.isinf(yf).sum() == 32
    yd = D.spmm(dg, x, None, "discretized", "right").cpu().numpy()
    assert float(yd[0, 0]) == 30000.0


# ── fp32-guarded SpMM (tolerance) ────────────────────────────────────────


def _powerlaw(rng, n, alpha=1.7, cap=5000):
    deg = np.minimum(rng.zipf(alpha, n), cap)
    deg[rng.random(n) < 0.1] = 0
    rows = np.repeat(np.arange(n), deg)
    cols = rng.integers(0, n, rows.size)
    return O.canonical_edges(n, rows, cols)


def _check_tol(got, want, label):
    err = np.abs(got.astype(np.float64) - want)
    lim = TOL * np.maximum(1.0, np.abs(want))
    bad = ~(err <= lim)
    assert not bad.any(), f"{label}: {bad.sum()} entries outside tolerance, max err {err.max()}"


@pytest.mark.parametrize("f", [2, 6, 8, 16, 24, 40, 42, 48, 56, 64, 96, 128, 192, 256, 512, 1024])
@pytest.mark.parametrize("scaling,norm", [("post", "none"), ("discretized", "both"),
                                          ("pre", "left"), ("post", "right")])
def test_spmm_fast_vs_f64(cuda, f, scaling, norm):
    from paper_2411_01109_b200 import device as D

    rng = np.random.default_rng(f * 7 + len(norm))
    n = 4000
    r, c = _powerlaw(rng, n)
    x = rng.normal(0, 1, (n, f)).astype(np.float16)
    dg = _dg(n, r, c, cuda)
    fin, fout = O.norm_factors(n, r, c, norm, np.float16)
    want = O.spmm_f64(n, r, c, x, None, fin, fout)
    got = D.spmm(dg, _t(x, cuda), None, scaling, norm).cpu().numpy()
    _check_tol(got, want, f"F={f} {scaling}/{norm}")
    # rule (2): agreement with the reference order up to the reference's own error
    ref = O.spmm_edge_parallel(n, r, c, x, None, 128, 4, scaling, norm)[0].astype(np.float64)
    slack = TOL * np.maximum(1.0, np.abs(ref)) + np.abs(ref - want)
    assert np.all(np.abs(got - ref) <= slack + 1e-12)


@pytest.mark.parametrize("heads,fh", [(1, 16), (1, 64), (4, 16), (4, 64), (8, 8), (2, 6)])
def test_spmm_fast_weighted_heads(cuda, heads, fh):
    from paper_2411_01109_b200 import device as D

    rng = np.random.default_rng(heads * 100 + fh)
    n = 2000
    r, c = _powerlaw(rng, n, cap=1500)
    f = heads * fh
    x = rng.normal(0, 1, (n, f)).astype(np.float16)
    w = rng.uniform(0.5, 1.5, (r.size, heads)).astype(np.float16)
    dg = _dg(n, r, c, cuda)
    got = D.spmm(dg, _t(x, cuda), _t(w, cuda), heads=heads).cpu().numpy()
    want = np.concatenate([O.spmm_f64(n, r, c, x[:, h * fh:(h + 1) * fh], w[:, h])
                           for h in range(heads)], axis=1)
    _check_tol(got, want, f"heads={heads} fh={fh}")
    # transposed traversal with weights read through perm (spmm_weighted backward)
    got_t = D.spmm(dg, _t(x, cuda), _t(w, cuda), heads=heads, transpose=True,
                   weight_via_perm=True).cpu().numpy()
    tr, tc, perm = O.transpose_perm(n, r, c)
    want_t = np.concatenate([O.spmm_f64(n, tr, tc, x[:, h * fh:(h + 1) * fh], w[perm, h])
                             for h in range(heads)], axis=1)
    _check_tol(got_t, want_t, f"transposed heads={heads} fh={fh}")


def test_spmm_fast_deterministic(cuda):
    from paper_2411_01109_b200 import device as D

    rng = np.random.default_rng(3)
    n = 5000
    r, c = _powerlaw(rng, n, alpha=1.5, cap=20000)
    dg = _dg(n, r, c, cuda)
    x = torch.randn(n, 64, device=cuda, dtype=torch.float16)
    a = D.spmm(dg, x, None, "discretized", "both")
    for _ in range(3):
        assert torch.equal(a, D.spmm(dg, x, None, "discretized", "both"))


def test_spmm_empty_and_isolated(cuda):
    from paper_2411_01109_b200 import device as D
    from paper_2411_01109_b200.device import DeviceGraph

    dg = DeviceGraph.from_edges(4, np.zeros(0, np.int64), np.zeros(0, np.int64), device=cuda)
    x = torch.ones(4, 8, dtype=torch.float16, device=cuda)
    assert not D.spmm(dg, x).any()
    assert not D.spmm_edge_ref(dg, x).any()
    dg = DeviceGraph.from_edges(5, np.array([0]), np.array([1]), device=cuda)
    x = torch.ones(5, 4, dtype=torch.float16, device=cuda)
    y = D.spmm(dg, x, None, "post", "both").cpu().numpy()
    assert y[0, 0] == 1.0 and not y[1:].any()


# ── SDDMM / attention / softmax (bit-exact) ──────────────────────────────


def test_sddmm_golden(cuda):
    from paper_2411_01109_b200 import device as D

    cases, _ = golden_cases("sddmm.npz")
    for i, c in enumerate(cases):
        dg = _dg(int(c["n"]), c["rows"], c["cols"], cuda)
        out = D.sddmm(dg, _t(c["x"], cuda), _t(c["y"], cuda)).cpu().numpy()
        np.testing.assert_array_equal(bits(out), bits(c["out"]), err_msg=f"case {i}")


@pytest.mark.parametrize("heads,fh", [(1, 256), (1, 512), (4, 64), (2, 48), (8, 16), (4, 128)])
def test_sddmm_heads_vs_oracle(cuda, heads, fh):
    from paper_2411_01109_b200 import device as D

    rng = np.random.default_rng(fh + heads)
    n = 700
    r, c = _powerlaw(rng, n, cap=600)
    f = heads * fh
    x = rng.normal(0, 1, (n, f)).astype(np.float16)
    y = rng.normal(0, 1, (n, f)).astype(np.float16)
    dg = _dg(n, r, c, cuda)
    got = D.sddmm(dg, _t(x, cuda), _t(y, cuda), heads=heads).cpu().numpy()
    want = O.sddmm(r, c, x, y, heads=heads)
    np.testing.assert_array_equal(bits(got), bits(want))


def test_attention_softmax_golden(cuda):
    from paper_2411_01109_b200 import device as D

    cases, d = golden_cases("attention.npz")
    for i, c in enumerate(cases):
        dg = _dg(int(c["n"]), c["rows"], c["cols"], cuda)
        sl = _t(c["sl"][:, None], cuda)
        sr = _t(c["sr"][:, None], cuda)
        e2 = D.attention_logits(dg, sl, sr)[:, 0]
        np.testing.assert_array_equal(bits(e2.cpu().numpy()), bits(c["e2"]), err_msg=f"case {i}")
        alpha = D.edge_softmax_fwd(dg, e2)
        np.testing.assert_array_equal(bits(alpha.cpu().numpy()), bits(c["alpha"]))
        de = D.edge_softmax_bwd(dg, alpha, _t(c["seed"], cuda))
        np.testing.assert_array_equal(bits(de.cpu().numpy()), bits(c["g_e2"]))


def test_shadow_exp_exhaustive(cuda):
    """Every non-positive half through the softmax exp path: row i holds
    scores [v_i, 0] so ex = rnd(exp(v_i)) (test_acceptance.py:247-253)."""
    from paper_2411_01109_b200 import device as D

    vals = load_golden("attention.npz")["exp_in"]
    n = vals.size
    rows = np.repeat(np.arange(n), 2)
    cols = np.stack([np.arange(n), (np.arange(n) + 1) % n], 1).reshape(-1)
    r, c = O.canonical_edges(n, rows, cols)
    dg = _dg(n, r, c, cuda)
    e = np.zeros(r.size, np.float16)
    diag = c == r
    e[diag] = vals[r[diag]]
    alpha = D.edge_softmax_fwd(dg, _t(e, cuda)).cpu().numpy()
    want = O.edge_softmax_fwd(O.csr_offsets(n, r), e)
    np.testing.assert_array_equal(bits(alpha), bits(want))


def test_softmax_heads_long_rows_vs_oracle(cuda):
    from paper_2411_01109_b200 import device as D

    rng = np.random.default_rng(11)
    n = 600
    r, c = _powerlaw(rng, n, alpha=1.4, cap=590)
    dg = _dg(n, r, c, cuda)
    e = rng.uniform(-6, 6, (r.size, 4)).astype(np.float16)
    g = rng.normal(size=(r.size, 4)).astype(np.float16)
    off = O.csr_offsets(n, r)
    alpha = D.edge_softmax_fwd(dg, _t(e, cuda))
    np.testing.assert_array_equal(bits(alpha.cpu().numpy()), bits(O.edge_softmax_fwd(off, e)))
    de = D.edge_softmax_bwd(dg, alpha, _t(g, cuda)).cpu().numpy()
    np.testing.assert_array_equal(bits(de), bits(O.edge_softmax_bwd(off, alpha.cpu().numpy(), g)))


def test_scale_f64_matches_numpy(cuda):
    from paper_2411_01109_b200 import device as D

    allv = np.arange(65536, dtype=np.uint16).view(np.float16)
    allv = allv[np.isfinite(allv)]
    got = D.scale_f64(_t(allv, cuda), 0.2).cpu().numpy()
    want = (allv.astype(np.float64) * 0.2).astype(np.float16)
    np.testing.assert_array_equal(bits(got), bits(want))


def test_softmax_and_rowsum_long_rows(cuda):
    """Rows above device.LONG_ROW take the one-CTA-per-row kernels; the tree
    order (and so every bit) must not change."""
    from paper_2411_01109_b200 import device as D

    rng = np.random.default_rng(99)
    n = 80_000
    deg = rng.integers(0, 6, n)
    deg[[3, 17, 500]] = [5000, 20_000, 70_001]
    rows = np.repeat(np.arange(n), deg)
    cols = rng.integers(0, n, rows.size)
    r, c = O.canonical_edges(n, rows, cols)
    dg = _dg(n, r, c, cuda)
    assert dg.fwd.long_rows().numel() == 3
    e = rng.uniform(-8, 8, (r.size, 2)).astype(np.float16)
    g = rng.normal(size=(r.size, 2)).astype(np.float16)
    off = O.csr_offsets(n, r)
    alpha = D.edge_softmax_fwd(dg, _t(e, cuda))
    np.testing.assert_array_equal(bits(alpha.cpu().numpy()), bits(O.edge_softmax_fwd(off, e)))
    de = D.edge_softmax_bwd(dg, alpha, _t(g, cuda)).cpu().numpy()
    np.testing.assert_array_equal(bits(de), bits(O.edge_softmax_bwd(off, alpha.cpu().numpy(), g)))
    rs = D.edge_rowsum(dg, _t(g, cuda)).cpu().numpy().astype(np.float64)
    want = np.zeros((n, 2))
    np.add.at(want, r, g.astype(np.float64))
    np.testing.assert_allclose(rs, want, rtol=2e-3, atol=2e-2)


@pytest.mark.parametrize("heads,fh", [(1, 64), (4, 16), (4, 32), (3, 6), (2, 160)])
def test_head_dots_fwd_bwd(cuda, heads, fh):
    from paper_2411_01109_b200 import device as D

    rng = np.random.default_rng(heads * fh)
    n = 5000
    z = rng.normal(size=(n, heads * fh)).astype(np.float16)
    a_l = rng.normal(size=(heads, fh)).astype(np.float16)
    a_r = rng.normal(size=(heads, fh)).astype(np.float16)
    zt, alt, art = _t(z, cuda), _t(a_l, cuda), _t(a_r, cuda)
    s_l, s_r = D.head_dots(zt, alt, art, heads)
    zh = z.reshape(n, heads, fh).astype(np.float64)
    want_l = (zh * a_l.astype(np.float64)[None]).sum(-1)
    np.testing.assert_allclose(s_l.cpu().numpy().astype(np.float64), want_l, rtol=2e-3, atol=2e-2)
    g_l = rng.normal(size=(n, heads)).astype(np.float16)
    g_r = rng.normal(size=(n, heads)).astype(np.float16)
    gz, ga_l, ga_r = D.head_dots_bwd(zt, alt, art, _t(g_l, cuda), _t(g_r, cuda), heads)
    want_gz = ((g_l.astype(np.float64)[:, :, None] * a_l[None]).astype(np.float16).astype(np.float64)
               + (g_r.astype(np.float64)[:, :, None] * a_r[None]).astype(np.float16)).astype(np.float16)
    np.testing.assert_array_equal(bits(gz.cpu().numpy()), bits(want_gz.reshape(n, -1)))
    want_ga = (zh * g_l.astype(np.float64)[:, :, None]).sum(0)
    np.testing.assert_allclose(ga_l.cpu().numpy().astype(np.float64), want_ga, rtol=3e-3, atol=0.1)
    a1 = D.head_dots_bwd(zt, alt, art, _t(g_l, cuda), _t(g_r, cuda), heads)
    assert torch.equal(a1[1], ga_l) and torch.equal(a1[2], ga_r)  # deterministic


# ── dense-side helpers (GCN epilogue, loss) ──────────────────────────────


@pytest.mark.parametrize("dtype", [np.float16, np.float32])
@pytest.mark.parametrize("f", [6, 8, 48, 64, 602])
def test_bias_scale_rows_bits(cuda, dtype, f):
    """rnd(rnd(x + b) * s): add_bias (models.py:161-166) then the left-norm
    input scaling (kernels.py:358-361), each an fp64 op rounded once."""
    from paper_2411_01109_b200 import device as D

    rng = np.random.default_rng(f)
    n = 1537
    x = rng.normal(0, 30, (n, f)).astype(dtype)
    b = rng.normal(0, 3, f).astype(dtype)
    s = rng.uniform(0, 1, n).astype(dtype)
    s[::7] = 0
    step1 = (x.astype(np.float64) + b.astype(np.float64)).astype(dtype)
    want = (step1.astype(np.float64) * s.astype(np.float64)[:, None]).astype(dtype)
    got = D.bias_scale_rows(_t(x, cuda), _t(b, cuda), _t(s, cuda)).cpu().numpy()
    np.testing.assert_array_equal(bits(got), bits(want))
    only_b = D.bias_scale_rows(_t(x, cuda), _t(b, cuda), None).cpu().numpy()
    np.testing.assert_array_equal(bits(only_b), bits(step1))


@pytest.mark.parametrize("dtype", [np.float16, np.float32])
@pytest.mark.parametrize("n,f", [(0, 8), (1, 8), (1000, 6), (233_000, 64), (50_000, 48),
                                 (3000, 4096)])
def test_col_sums(cuda, dtype, n, f):
    """add_bias backward: fp32 column sums rounded once (models.py:168-170);
    checked against float64 with the fp32 accumulation bound; deterministic."""
    from paper_2411_01109_b200 import device as D

    rng = np.random.default_rng(n + f)
    x = rng.normal(0, 1, (n, f)).astype(dtype)
    xt = _t(x, cuda)
    got = D.col_sums(xt).cpu().numpy().astype(np.float64)
    want = x.astype(np.float64).sum(0)
    bound = 1e-6 * np.abs(x).astype(np.float64).sum(0) + np.abs(want) * (
        2.0 ** -11 if dtype == np.float16 else 2.0 ** -23) + 1e-30
    assert np.all(np.abs(got - want) <= bound)
    assert torch.equal(D.col_sums(xt), D.col_sums(xt))


@pytest.mark.parametrize("c,ld", [(7, 8), (42, 48), (47, 48), (3, 4), (100, 104), (300, 304)])
@pytest.mark.parametrize("scale", [1.0, 2048.0])
def test_softmax_xent_fp16_logits(cuda, c, ld, scale):
    """convert -> cross_entropy -> backward -> convert-backward in one kernel
    (models.py:203-217, 552-572): nll in fp64, grad = fp16(fp32((p-y)/n) * S)."""
    from paper_2411_01109_b200 import device as D

    rng = np.random.default_rng(c)
    n = 3001
    z = rng.normal(0, 4, (n, ld)).astype(np.float16)
    lab = rng.integers(0, c, n)
    nll, g = D.softmax_xent(_t(z, cuda), _t(lab, cuda), c, n, scale=scale)
    zz = z[:, :c].astype(np.float64)
    zz = zz - zz.max(1, keepdims=True)
    se = np.exp(zz).sum(1)
    p = np.exp(zz) / se[:, None]
    p[np.arange(n), lab] -= 1.0
    want = np.zeros((n, ld), np.float16)
    want[:, :c] = ((p / n).astype(np.float32) * np.float32(scale)).astype(np.float16)
    got = g.cpu().numpy()
    assert got.dtype == np.float16
    diff = np.abs(bits(got).astype(np.int32) - bits(want).astype(np.int32))
    assert diff.max() <= 1 and (diff > 0).mean() < 1e-3
    want_nll = np.log(se) - zz[np.arange(n), lab]
    np.testing.assert_allclose(nll.cpu().numpy(), want_nll, rtol=1e-12, atol=1e-12)
    # fp32 logits / fp32 grad path
    nll32, g32 = D.softmax_xent(_t(z.astype(np.float32), cuda), _t(lab, cuda), c, n)
    assert g32.dtype == torch.float32
    np.testing.assert_allclose(g32.cpu().numpy()[:, :c], (p / n).astype(np.float32),
                               rtol=1e-6, atol=1e-12)


@pytest.mark.parametrize("f,ld", [(48, 64), (24, 32), (6, 8), (40, 64), (64, 72)])
def test_spmm_fast_row_strides(cuda, f, ld):
    """x / y as column slices of wider rows (hg_spmm ldx / ldy): identical
    values to the dense layout; padding columns of y untouched."""
    from paper_2411_01109_b200 import device as D

    rng = np.random.default_rng(f * ld)
    n = 3000
    deg = np.minimum(rng.zipf(1.6, n), 2500)
    rows = np.repeat(np.arange(n), deg)
    r, c = O.canonical_edges(n, rows, rng.integers(0, n, rows.size))
    dg = _dg(n, r, c, cuda)
    view = dg.view(False)
    fin, fout = dg.norm_tables("both", False, torch.float16)
    x = torch.randn(n, f, device=cuda, dtype=torch.float16)
    wide = torch.randn(n, ld, device=cuda, dtype=torch.float16)
    wide[:, :f] = x
    want = D.spmm_csr(view, x, scaling="discretized", fout=fout)
    ybuf = torch.full((n, ld), 7.0, device=cuda, dtype=torch.float16)
    got = D.spmm_csr(view, wide[:, :f], scaling="discretized", fout=fout, out=ybuf[:, :f])
    assert torch.equal(got, want)
    assert torch.equal(ybuf[:, :f], want)
    assert bool((ybuf[:, f:] == 7.0).all())


# ── fp32-guarded GAT attention (numerics="fast") ─────────────────────────


def _hub_graph(seed, n=6000):
    """Degrees covering all three row classes: <= 32, (32, 4096], > 4096."""
    rng = np.random.default_rng(seed)
    deg = np.minimum(rng.zipf(1.8, n), 3000)
    deg[:3] = [5000, 4097, 4096]
    deg[3:6] = [33, 32, 0]
    rows = np.repeat(np.arange(n), deg)
    return O.canonical_edges(n, rows, rng.integers(0, n, rows.size))


@pytest.mark.parametrize("heads", [1, 4, 8])
def test_gat_attention_fast_vs_f64(cuda, heads):
    from paper_2411_01109_b200 import device as D

    n = 6000
    r, c = _hub_graph(heads, n)
    dg = _dg(n, r, c, cuda)
    rng = np.random.default_rng(heads)
    sl = rng.normal(0, 3, (n, heads)).astype(np.float16)
    sr = rng.normal(0, 3, (n, heads)).astype(np.float16)
    alpha = D.gat_attention_fwd(dg.view(False), _t(sl, cuda), _t(sr, cuda), 0.2).cpu().numpy()
    # float64 reference
    lg = sl.astype(np.float64)[r] + sr.astype(np.float64)[c]
    lg = np.where(lg > 0, lg, 0.2 * lg)
    off = O.csr_offsets(n, r)
    want = np.zeros_like(lg)
    for v in range(n):
        s, e = off[v], off[v + 1]
        if e > s:
            z = np.exp(lg[s:e] - lg[s:e].max(0))
            want[s:e] = z / z.sum(0)
    a = alpha.astype(np.float64)
    assert np.all(np.abs(a - want) <= 2.0 ** -10 * want + 1e-7)
    # rows sum to 1 within fp16 rounding
    rs = np.add.reduceat(a, off[:-1][np.diff(off) > 0], axis=0)
    assert np.all(np.abs(rs - 1.0) <= 2e-3)

    # backward: de = alpha (g - sum alpha g) leaky'(l); ds_l / ds_r row / col sums
    g = rng.normal(0, 1, (r.size, heads)).astype(np.float16)
    de, dsl = D.gat_attention_bwd(dg.view(False), _t(sl, cuda), _t(sr, cuda), _t(alpha, cuda),
                                  _t(g, cuda), 0.2)
    gg = g.astype(np.float64)
    dd = np.zeros_like(gg)
    for v in range(n):
        s, e = off[v], off[v + 1]
        if e > s:
            dd[s:e] = a[s:e] * (gg[s:e] - (a[s:e] * gg[s:e]).sum(0))
    raw = sl.astype(np.float64)[r] + sr.astype(np.float64)[c]
    dd = np.where(raw > 0, dd, 0.2 * dd)
    de = de.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(de - dd) <= 2.0 ** -10 * np.abs(dd) + 2e-4)
    want_l = np.zeros((n, heads))
    np.add.at(want_l, r, dd)
    got_l = dsl.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(got_l - want_l) <= 2e-3 * np.maximum(1, np.abs(want_l)))
    bwd = dg.view(True)
    got_r = D.edge_sums_fast(bwd, _t(de.astype(np.float16), cuda), bwd.perm).cpu().numpy()
    want_r = np.zeros((n, heads))
    np.add.at(want_r, c, de)
    assert np.all(np.abs(got_r.astype(np.float64) - want_r) <= 2e-3 * np.maximum(1, np.abs(want_r)))


@pytest.mark.parametrize("f", [8, 48, 64, 256])
@pytest.mark.parametrize("mode", ["plain", "sumw"])
def test_spmm_fused_followup_bitwise(cuda, f, mode):
    """hg_spmm with split_counters / slot_split (the last unit of each split
    row folds the carries) == the separate follow-up launch, bit for bit, and
    the counters are left zero (graph replays reuse them)."""
    from paper_2411_01109_b200 import device as D

    n = 6000
    r, c = _hub_graph(f, n)
    if mode == "sumw":   # hubs on the CSC side (the transposed view this mode reads)
        r, c = O.canonical_edges(n, c, r)
    dg = _dg(n, r, c, cuda)
    view = dg.view(mode == "sumw")
    heads = 4 if f % 64 == 0 else 1
    x = torch.randn(n, f, device=cuda, dtype=torch.float16)
    fout = torch.rand(n, device=cuda, dtype=torch.float16)
    kw, extra = {}, {}
    w = widx = None
    if mode == "sumw":
        if f > 256:
            pytest.skip("summed weights need F/8 <= 32")
        ae = torch.randn(r.size, 2 * heads, device=cuda, dtype=torch.float16)
        w, widx = ae[:, :heads], view.perm
        kw = dict(w2_off=heads)
    outs = []
    saved = D.FUSED_FOLLOWUP
    try:
        for fused in (False, True):
            D.FUSED_FOLLOWUP = fused
            if mode == "sumw":
                extra = {"out2": torch.empty(n, heads, device=cuda, dtype=torch.float16)}
            for _ in range(2):   # second call reuses the (re-armed) counters
                y = D.spmm_csr(view, x, w, widx, heads if w is not None else 1, "discretized",
                               fout=fout, **kw, **extra)
            outs.append((y, extra.get("out2")))
    finally:
        D.FUSED_FOLLOWUP = saved
    sched = view.schedule(D.DEFAULT_SPLIT_CAP, -1)
    assert sched.split_rows.shape[0] > 0
    cnt, _ = sched.finish_state()
    assert int(cnt.abs().sum()) == 0
    assert torch.equal(outs[0][0].view(torch.int16), outs[1][0].view(torch.int16))
    if mode == "sumw":
        assert torch.equal(outs[0][1].view(torch.int16), outs[1][1].view(torch.int16))


@pytest.mark.parametrize("heads,fh", [(1, 16), (4, 16), (4, 32), (2, 64), (3, 16), (1, 256)])
@pytest.mark.parametrize("packs", [False, True])
def test_spmm_head_dot_store_bitwise(cuda, heads, fh, packs):
    """hg_spmm with the head-dot store (hd_gl..) == hg_spmm then hg_head_dots_bwd
    accumulating into its output, bit for bit: every row class (split hub rows,
    fused and separate follow-up, packs), multi-head weights through a perm;
    and head_dots_bwd(dz=False) gives the same da."""
    from paper_2411_01109_b200 import device as D

    n, f = 6000, heads * fh
    r, c = _hub_graph(heads + fh, n)
    r, c = O.canonical_edges(n, c, r)   # hubs on the CSC side (the view aggregated)
    dg = _dg(n, r, c, cuda)
    view = dg.view(True)
    rng = np.random.default_rng(heads * fh)
    x = _t(rng.normal(0, 1, (n, f)).astype(np.float16), cuda)
    z = _t(rng.normal(0, 1, (n, f)).astype(np.float16), cuda)
    w = _t(rng.uniform(0, 1, (r.size, heads)).astype(np.float16), cuda)
    gl = _t(rng.normal(0, 2, (n, heads)).astype(np.float16), cuda)
    gr = _t(rng.normal(0, 2, (n, heads)).astype(np.float16), cuda)
    al = _t(rng.normal(0, 0.5, f).astype(np.float16), cuda)
    ar = _t(rng.normal(0, 0.5, f).astype(np.float16), cuda)
    saved = D.PACK_MIN_ROWS, D.FUSED_FOLLOWUP
    D.PACK_MIN_ROWS = 0 if packs else 1 << 40
    try:
        for fused in (False, True):
            D.FUSED_FOLLOWUP = fused
            want = D.spmm_csr(view, x, w, view.perm, heads, "post")
            want, wl, wr = D.head_dots_bwd(z, al, ar, gl, gr, heads, gz_acc=want)
            got = D.spmm_csr(view, x, w, view.perm, heads, "post", head_dots=(gl, gr, al, ar))
            assert torch.equal(got.view(torch.int16), want.view(torch.int16))
            none, gotl, gotr = D.head_dots_bwd(z, al, ar, gl, gr, heads, dz=False)
            assert none is None
            assert torch.equal(gotl.view(torch.int16), wl.view(torch.int16))
            assert torch.equal(gotr.view(torch.int16), wr.view(torch.int16))
    finally:
        D.PACK_MIN_ROWS, D.FUSED_FOLLOWUP = saved
    assert view.schedule(D.DEFAULT_SPLIT_CAP, -1).split_rows.shape[0] > 0
    with pytest.raises(ValueError, match="head-dot store"):
        D.spmm_csr(view, x, w, view.perm, heads, "post", relu=True, head_dots=(gl, gr, al, ar))


@pytest.mark.parametrize("f", [16, 48, 64, 128])
@pytest.mark.parametrize("parts,packs", [(2, False), (3, True), (8, False), (8, True)])
def test_spmm_acc_column_blocks_chain(cuda, f, parts, packs):
    """hg_spmm_acc chained over the column blocks of a CSR (partition.column_blocks)
    == hg_spmm on the whole CSR: bitwise on every row that is one work unit in
    each block (short rows, packed or not), within the Appendix-A bound of
    float64 on split hub rows; block concatenation restores every row."""
    from paper_2411_01109_b200 import device as D
    from paper_2411_01109_b200.partition import column_blocks

    n = 6000
    r, c = _hub_graph(parts + f, n)
    dg = _dg(n, r, c, cuda)
    view = dg.view(False)
    splits = np.linspace(0, n, parts + 1).astype(np.int64)
    blocks = column_blocks(view, splits)
    # structure: rows of the blocks concatenated in q order = the original rows
    off = view.offsets.cpu().numpy()
    cols = view.cols.cpu().numpy()
    bo = [b.offsets.cpu().numpy() for b in blocks]
    bc = [b.cols.cpu().numpy() for b in blocks]
    for row in (0, 1, 2, 3, 7, 100, 5999):
        cat = np.concatenate([bc[q][bo[q][row]:bo[q][row + 1]] + splits[q] for q in range(parts)])
        np.testing.assert_array_equal(cat, cols[off[row]:off[row + 1]])
    x = torch.randn(n, f, device=cuda, dtype=torch.float16)
    fout = torch.rand(n, device=cuda, dtype=torch.float16)
    saved = D.PACK_MIN_ROWS
    D.PACK_MIN_ROWS = 0 if packs else 1 << 40
    try:
        want = D.spmm_csr(view, x, None, None, 1, "discretized", fout=fout)
        acc = torch.empty(n, f, device=cuda, dtype=torch.float32)
        got = None
        for q, b in enumerate(blocks):
            got = D.spmm_csr_acc(b, x[int(splits[q]):int(splits[q + 1])],
                                 acc_in=None if q == 0 else acc,
                                 acc_out=None if q == parts - 1 else acc, scaling="discretized",
                                 fout=fout if q == parts - 1 else None)
    finally:
        D.PACK_MIN_ROWS = saved
    deg = np.diff(off)
    single = deg <= D.DEFAULT_SPLIT_CAP
    g, w = got.cpu().numpy(), want.cpu().numpy()
    np.testing.assert_array_equal(bits(g[single]), bits(w[single]))
    fo = fout.cpu().numpy().astype(np.float64)
    f64 = O.spmm_f64(n, r, c, x.cpu().numpy(), None, None, fo)
    gg, ww = g.astype(np.float64), w.astype(np.float64)
    assert np.all(np.abs(gg - f64) <= 1e-2 * np.maximum(1.0, np.abs(f64)) + np.abs(ww - f64))


@pytest.mark.parametrize("heads,fh", [(1, 64), (4, 32), (4, 16), (8, 8), (2, 6), (4, 128)])
@pytest.mark.parametrize("packs", [False, True])
def test_gat_fused_forward_bitwise_equals_composed(cuda, heads, fh, packs):
    """hg_gat_attention_stats + hg_gat_aggregate (alpha formed in the gather
    loop) == hg_gat_attention_fwd + hg_spmm(w = alpha), bit for bit: alpha,
    the aggregation (all three row classes, split hub rows with carries, packed
    short rows) and the fused ReLU."""
    from paper_2411_01109_b200 import device as D

    n = 6000
    r, c = _hub_graph(heads + fh, n)
    dg = _dg(n, r, c, cuda)
    rng = np.random.default_rng(fh)
    sl = _t(rng.normal(0, 3, (n, heads)).astype(np.float16), cuda)
    sr = _t(rng.normal(0, 3, (n, heads)).astype(np.float16), cuda)
    z = _t(rng.normal(0, 1, (n, heads * fh)).astype(np.float16), cuda)
    saved = D.PACK_MIN_ROWS
    D.PACK_MIN_ROWS = 0 if packs else 1 << 40
    try:
        view = dg.view(False)
        for relu in (False, True):
            alpha = D.gat_attention_fwd(view, sl, sr, 0.2)
            want = D.spmm_csr(view, z, alpha, None, heads, "post", relu=relu)
            stats = D.gat_attention_stats(view, sl, sr, 0.2)
            got, galpha = D.gat_aggregate(view, z, sl, sr, stats, heads, 0.2, relu=relu)
            assert torch.equal(galpha.view(torch.int16), alpha.view(torch.int16))
            assert torch.equal(got.view(torch.int16), want.view(torch.int16))
        if packs and fh * heads * 2 < 256:
            assert view.schedule(pack_edges=D.PACK_EDGES_NARROW).num_packs > 0
    finally:
        D.PACK_MIN_ROWS = saved


@pytest.mark.parametrize("heads,f", [(4, 16), (2, 3), (8, 8), (4, 24), (3, 40)])
def test_head_mean_bits(cuda, heads, f):
    from paper_2411_01109_b200 import device as D

    rng = np.random.default_rng(f)
    y = rng.normal(0, 100, (777, heads * f)).astype(np.float16)
    got = D.head_mean(_t(y, cuda), heads).cpu().numpy()
    want = (y.reshape(777, heads, f).astype(np.float64).sum(1) / heads).astype(np.float16)
    np.testing.assert_array_equal(bits(got), bits(want))
    g = rng.normal(0, 1, (777, f)).astype(np.float16)
    gin = D.head_mean_bwd(_t(g, cuda), heads).cpu().numpy()
    np.testing.assert_array_equal(bits(gin), bits(np.tile((g.astype(np.float64) / heads).astype(np.float16), (1, heads))))


# ── GPU ingest of edge-list text (sparse.load_edge_list) ─────────────────


def test_edge_list_ingest_golden(cuda, tmp_path):
    """load_edge_list (GPU parse + canonicalise) == the reference's loader on
    every recorded text: edges, vertex count, error type and message."""
    from paper_2411_01109_b200 import sparse as sp
    from paper_2411_01109_b200.device import DeviceGraph

    cases, _ = golden_cases("ingest.npz")
    for i, c in enumerate(cases):
        p = tmp_path / f"c{i}.txt"
        p.write_bytes(c["text"].tobytes())
        nv = None if int(c["nv"]) < 0 else int(c["nv"])
        want_err = str(c["err"])
        if want_err:
            kind = want_err.split(":")[0]
            with pytest.raises((ValueError, OverflowError)) as err:
                sp.load_edge_list(p, num_vertices=nv, symmetrize_edges=bool(c["sym"]))
            assert type(err.value).__name__ == kind, (i, err.value)
            if kind == "ValueError":
                assert f"ValueError: {err.value}".replace(str(p), "<path>") == want_err, i
            continue
        g = sp.load_edge_list(p, num_vertices=nv, symmetrize_edges=bool(c["sym"]))
        assert g.n == int(c["n"]), i
        np.testing.assert_array_equal(g.rows, c["rows"])
        np.testing.assert_array_equal(g.cols, c["cols"])
        dg = DeviceGraph.from_edge_list(p, nv, bool(c["sym"]))
        np.testing.assert_array_equal(dg.cols.cpu().numpy(), c["cols"])


def test_edge_list_ingest_large(cuda, tmp_path):
    """2M-edge randomized text (mixed whitespace, CRLF, comments): GPU parse ==
    the oracle restatement of the reference loader."""
    from paper_2411_01109_b200.device import DeviceGraph, parse_edge_text, read_bytes_device

    rng = np.random.default_rng(5)
    m = 2_000_000
    a = rng.integers(0, 300_000, m)
    b = rng.integers(0, 300_000, m)
    seps = np.array([" ", "\t", "  "])[rng.integers(0, 3, m)]
    ends = np.array(["\n", "\r\n", " \n"])[rng.integers(0, 3, m)]
    lines = np.char.add(np.char.add(np.char.add(a.astype(str), seps), b.astype(str)), ends)
    lines[::1000] = "# comment\n"
    text = "".join(lines.tolist()).encode()
    p = tmp_path / "big.txt"
    p.write_bytes(text)
    rows, cols, top = parse_edge_text(read_bytes_device(p), str(p))
    keep = np.ones(m, bool)
    keep[::1000] = False
    np.testing.assert_array_equal(rows.cpu().numpy(), a[keep])
    np.testing.assert_array_equal(cols.cpu().numpy(), b[keep])
    assert top == max(a[keep].max(), b[keep].max())
    n, r, c = O.load_edge_list_text(text)
    dg = DeviceGraph.from_edge_list(p)
    assert dg.n == n
    np.testing.assert_array_equal(dg.offsets.cpu().numpy(), O.csr_offsets(n, r))
    np.testing.assert_array_equal(dg.cols.cpu().numpy(), c)


def test_load_tensor_device_roundtrip(cuda, tmp_path):
    """HSDT files (sparse.save_tensor) load straight into HBM bit for bit."""
    from paper_2411_01109_b200 import sparse as sp
    from paper_2411_01109_b200.device import load_tensor_device

    rng = np.random.default_rng(0)
    for dt in (np.float16, np.float32):
        t = sp.DenseTensor(rng.normal(0, 5, (123, 37)).astype(dt))
        p = tmp_path / f"t{np.dtype(dt).itemsize}.hsdt"
        sp.save_tensor(t, p)
        got = load_tensor_device(p).cpu().numpy()
        np.testing.assert_array_equal(bits(got), bits(t.data))
    p.write_bytes(p.read_bytes()[:-4])
    with pytest.raises(ValueError, match="payload"):
        load_tensor_device(p)


@pytest.mark.parametrize("heads,fh", [(1, 8), (1, 16), (1, 64), (1, 256), (4, 32), (4, 8),
                                      (2, 128), (8, 16), (2, 6), (1, 512)])
def test_sddmm_fast_vs_f64(cuda, heads, fh):
    """hg_sddmm_fast (fp32 accumulation + butterfly head reduction) within one
    fp16 rounding of the float64 dot, on a power-law graph; layouts outside
    the butterfly kernel fall back to the exact kernel."""
    from paper_2411_01109_b200 import device as D

    n = 3000
    rng = np.random.default_rng(fh * heads)
    deg = np.minimum(rng.zipf(1.7, n), 2000)
    rows = np.repeat(np.arange(n), deg)
    r, c = O.canonical_edges(n, rows, rng.integers(0, n, rows.size))
    dg = _dg(n, r, c, cuda)
    f = heads * fh
    x = rng.normal(0, 1, (n, f)).astype(np.float16)
    y = rng.normal(0, 1, (n, f)).astype(np.float16)
    got = D.sddmm(dg, _t(x, cuda), _t(y, cuda), heads=heads, fast=True).cpu().numpy()
    got = got.reshape(r.size, heads).astype(np.float64)
    prod = x.astype(np.float64)[r] * y.astype(np.float64)[c]
    want = prod.reshape(r.size, heads, fh).sum(-1)
    bound = 2.0 ** -11 * np.abs(want) + 1e-6 * np.abs(prod).reshape(r.size, heads, fh).sum(-1) + 1e-7
    if fh % 2 or fh == 6 or f > 256:  # exact (fp16 tree) fallback layouts: SURVEY App. A rule
        # fp16 pair/tree sums: error grows with the sum of |products|
        bound = np.maximum(bound, 2.0 ** -8 * np.abs(prod).reshape(r.size, heads, fh).sum(-1))
    assert np.all(np.abs(got - want) <= bound)


@pytest.mark.parametrize("heads,fh", [(1, 8), (4, 32), (4, 16), (2, 64), (8, 8), (1, 2), (4, 6),
                                     (1, 256), (3, 4)])
@pytest.mark.parametrize("dtype", [torch.float16, torch.float32])
def test_sddmm_packed_bitwise_equal_units(cuda, heads, fh, dtype):
    """hg_sddmm_fast with short-row packs (one team per 16-row block, X row per
    edge) is bitwise the per-row unit kernel, on empty / short / long / split
    rows; layouts outside the butterfly kernel run unpacked."""
    from paper_2411_01109_b200 import device as D

    n = 20000
    r, c = _short_row_graph(fh * heads + 1, n)
    dg = _dg(n, r, c, cuda)
    f = heads * fh
    x = torch.randn(n, f, device=cuda).to(dtype)
    y = torch.randn(n, f, device=cuda).to(dtype)
    saved = (D.PACK_MIN_ROWS, D.LANE32)
    try:
        D.LANE32 = False   # packs run with the 16-byte-lane kernels only
        D.PACK_MIN_ROWS = 1 << 40
        want = D.sddmm(dg, x, y, heads=heads, fast=True)
        D.PACK_MIN_ROWS = 0
        got = D.sddmm(dg, x, y, heads=heads, fast=True)
    finally:
        D.PACK_MIN_ROWS, D.LANE32 = saved
    it = torch.int16 if dtype == torch.float16 else torch.int32
    assert torch.equal(got.contiguous().view(it), want.contiguous().view(it))
    if D._butterfly_layout(x, y, f, heads):
        assert dg.view(False).schedule(D.DEFAULT_SPLIT_CAP, D.PACK_EDGES_WIDE).num_packs > 0


# ── tcgen05 GEMM with the GCN epilogue (hg_gemm_tc) ──────────────────────


@pytest.mark.parametrize("m,k,n", [(1000, 608, 64), (300, 64, 48), (4097, 1440, 16), (129, 16, 256),
                                   (5000, 104, 128), (77, 200, 32)])
@pytest.mark.parametrize("epi", ["none", "bias", "both", "relu"])
def test_gemm_tc_vs_f64(cuda, m, k, n, epi):
    """tcgen05 GEMM + fused epilogue against float64: the accumulation differs
    from the reference only in fp32 summation order, so each output is within
    one fp16 rounding step of rnd(rnd(rnd(A B) + b) * s) computed in float64."""
    from paper_2411_01109_b200 import device as D

    rng = np.random.default_rng(m + k + n)
    a = rng.normal(0, 1, (m, k)).astype(np.float16)
    w = rng.normal(0, 0.2, (k, n)).astype(np.float16)
    b = rng.normal(0, 1, n).astype(np.float16) if epi != "none" else None
    s = rng.uniform(0, 1, m).astype(np.float16) if epi == "both" else None
    got = D.gemm_tc(_t(a, cuda), _t(np.ascontiguousarray(w.T), cuda),
                    None if b is None else _t(b, cuda), None if s is None else _t(s, cuda),
                    relu=epi == "relu")
    got = got.cpu().numpy().astype(np.float64)
    acc = a.astype(np.float64) @ w.astype(np.float64)
    h = acc.astype(np.float16).astype(np.float64)
    # a different fp32 summation order may move rnd(acc) by one ulp; that ulp
    # survives the bias add (even through cancellation) and scales with s
    slack = 2.0 ** -10 * np.abs(h) + 1e-6 * (np.abs(a.astype(np.float64)) @ np.abs(w.astype(np.float64)))
    if b is not None:
        h = (h + b.astype(np.float64)).astype(np.float16).astype(np.float64)
        slack = slack + 2.0 ** -10 * np.abs(h)
    if s is not None:
        sc = s.astype(np.float64)[:, None]
        h = (h * sc).astype(np.float16).astype(np.float64)
        slack = slack * sc + 2.0 ** -10 * np.abs(h)
    if epi == "relu":
        h = np.maximum(h, 0.0)
    assert np.all(np.abs(got - h) <= slack + 2.0 ** -24)


@pytest.mark.parametrize("f", [256, 520])
def test_spmm_column_slabs_vs_f64(cuda, f):
    """X larger than half the L2 makes hg_spmm aggregate in column slabs (each
    pass's gathers stay L2-resident): same tolerance as the one-pass kernel,
    checked on sampled rows (incl. split heavy rows)."""
    from paper_2411_01109_b200 import device as D, graphgen

    dg = graphgen.reddit_like(9, n=200_000, e=3_000_000)
    assert 2 * f * dg.n > 63 * 2**20  # above the slab threshold on B200
    x = torch.randn(dg.n, f, device=cuda, dtype=torch.float16)
    y = D.spmm(dg, x, None, "discretized", "both")
    assert torch.equal(y, D.spmm(dg, x, None, "discretized", "both"))
    off = dg.offsets.cpu().numpy()
    cols = dg.cols.cpu().numpy()
    deg = np.diff(off)
    rng = np.random.default_rng(f)
    rows = np.concatenate([np.argsort(deg)[-5:], rng.integers(0, dg.n, 300)])
    fin, fout = dg.norm_tables("both", False, torch.float16)
    fin, fout = fin.cpu().numpy().astype(np.float64), fout.cpu().numpy().astype(np.float64)
    xs = (x.cpu().numpy().astype(np.float64) * fin[:, None]).astype(np.float16).astype(np.float64)
    yh = y.cpu().numpy().astype(np.float64)
    for r in rows:
        c = cols[off[r]:off[r + 1]]
        want = xs[c].sum(0) * fout[r]
        assert np.all(np.abs(yh[r] - want) <= TOL * np.maximum(1.0, np.abs(want))), r


@pytest.mark.parametrize("count", [8, 1000, 999, 2_449_029 * 104 // 64])
def test_scale_combine_bits(cuda, count):
    """GIN combine (models.py:220-240) forward bit-exact; backward gx / ga
    bit-exact, the (1+eps) gradient an fp64 sum within one fp16 rounding."""
    from paper_2411_01109_b200 import device as D

    rng = np.random.default_rng(count)
    x = rng.normal(0, 3, count).astype(np.float16)
    a = rng.normal(0, 30, count).astype(np.float16)
    g = rng.normal(0, 1, count).astype(np.float16)
    ope = np.array(1.0009765625, dtype=np.float16)
    lam = 0.1
    got = D.scale_combine(_t(x, cuda), _t(a, cuda), _t(ope, cuda), lam).cpu().numpy()
    u = (x.astype(np.float64) * float(ope)).astype(np.float16).astype(np.float64)
    v = (a.astype(np.float64) * lam).astype(np.float16).astype(np.float64)
    np.testing.assert_array_equal(bits(got), bits((u + v).astype(np.float16)))
    gx, ga, gope = D.scale_combine_bwd(_t(x, cuda), _t(g, cuda), _t(ope, cuda), lam)
    np.testing.assert_array_equal(bits(gx.cpu().numpy()),
                                  bits((g.astype(np.float64) * float(ope)).astype(np.float16)))
    np.testing.assert_array_equal(bits(ga.cpu().numpy()),
                                  bits((g.astype(np.float64) * lam).astype(np.float16)))
    want = np.float64((x.astype(np.float64) * g.astype(np.float64)).sum())
    assert abs(float(gope.cpu()) - want) <= 2.0 ** -10 * abs(want) + 1e-3
    _, _, only = D.scale_combine_bwd(_t(x, cuda), _t(g, cuda), _t(ope, cuda), lam, False, False)
    assert torch.equal(only, gope)


def test_relu_grad(cuda):
    from paper_2411_01109_b200 import device as D

    rng = np.random.default_rng(1)
    pre = rng.normal(0, 1, 4099).astype(np.float16)
    y = np.maximum(pre, 0).astype(np.float16)
    g = rng.normal(0, 1, 4099).astype(np.float16)
    got = D.relu_grad(_t(y, cuda), _t(g, cuda)).cpu().numpy()
    np.testing.assert_array_equal(bits(got), bits(np.where(pre > 0, g, np.float16(0))))


@pytest.mark.parametrize("m,k,heads,fh", [(1, 8, 1, 16), (300, 128, 4, 32), (5000, 64, 8, 16),
                                          (1031, 608, 2, 64), (2000, 128, 2, 128),
                                          (700, 64, 3, 16), (129, 72, 1, 16)])
def test_gemm_tc_dots_vs_f64(cuda, m, k, heads, fh):
    """hg_gemm_tc_dots: z equals hg_gemm_tc bit for bit, and the epilogue's head
    dots are rnd(sum_f z_h[f] a[h, f]) over the ROUNDED z -- exact products, fp32
    sums -- within one fp16 step of the float64 value (and of hg_head_dots)."""
    from paper_2411_01109_b200 import device as D

    rng = np.random.default_rng(m + k + heads)
    n = heads * fh
    a = _t(rng.normal(0, 1, (m, k)).astype(np.float16), cuda)
    bt = _t(rng.normal(0, 0.2, (n, k)).astype(np.float16), cuda)
    al = _t(rng.normal(0, 0.3, (heads, fh)).astype(np.float16), cuda)
    ar = _t(rng.normal(0, 0.3, (heads, fh)).astype(np.float16), cuda)
    z, sl, sr = D.gemm_tc_dots(a, bt, al, ar, heads)
    assert torch.equal(z.view(torch.int16), D.gemm_tc(a, bt).view(torch.int16))
    zh = z.double().reshape(m, heads, fh)
    hl, hr = D.head_dots(z, al, ar, heads)
    for got, vec, other in ((sl, al, hl), (sr, ar, hr)):
        want = (zh * vec.double()[None]).sum(-1)
        mag = (zh.abs() * vec.double().abs()[None]).sum(-1)
        h = want.half().double()
        slack = 2.0 ** -10 * h.abs() + 1e-6 * mag + 2.0 ** -24
        assert bool(((got.double() - h).abs() <= slack).all())
        assert bool(((got.double() - other.double()).abs() <= 2 * slack).all())
    with pytest.raises(ValueError, match="multiples of 16"):
        D.gemm_tc_dots(a, bt.new_zeros(24, k), al.new_zeros(24), ar.new_zeros(24), 2)
    with pytest.raises(ValueError, match="odd head counts"):
        D.gemm_tc_dots(a, bt.new_zeros(96, k), al.new_zeros(96), ar.new_zeros(96), 3)


@pytest.mark.parametrize("m,k,n", [(1, 16, 16), (300, 64, 128), (5000, 128, 64), (1031, 48, 256)])
def test_gemm_tc_masked_bitwise(cuda, m, k, n):
    """hg_gemm_tc_masked == relu_grad(mask, hg_gemm_tc(...)) bit for bit: the
    ReLU backward folded into the dX epilogue (+0 where mask <= 0 or NaN)."""
    from paper_2411_01109_b200 import device as D

    rng = np.random.default_rng(m + n)
    a = _t(rng.normal(0, 1, (m, k)).astype(np.float16), cuda)
    bt = _t(rng.normal(0, 0.2, (n, k)).astype(np.float16), cuda)
    y = rng.normal(0, 1, (m, n)).astype(np.float16)
    y[rng.random((m, n)) < 0.05] = 0.0
    y[rng.random((m, n)) < 0.01] = np.nan
    y = _t(y, cuda)
    want = D.relu_grad(y, D.gemm_tc(a, bt))
    got = D.gemm_tc_masked(a, bt, y)
    assert torch.equal(got.view(torch.int16), want.view(torch.int16))


def test_gemm_tc_from_autograd_worker_thread(cuda):
    """hg_gemm_tc encodes its TMA descriptors through the driver API; it must
    work from autograd's backward worker thread (no context bound there)."""
    from paper_2411_01109_b200 import models as M

    x = torch.randn(3000, 64, device=cuda, dtype=torch.float16, requires_grad=True)
    w = (torch.randn(64, 48, device=cuda, dtype=torch.float16) * 0.1).requires_grad_(True)
    b = torch.zeros(48, device=cuda, dtype=torch.float16, requires_grad=True)
    y = M._LinearTCFn.apply(x, w, b, True)
    y.float().sum().backward()
    ref = torch.relu(x.detach().float() @ w.detach().float() + b.detach().float())
    assert torch.allclose(y.float(), ref, atol=2e-2, rtol=1e-2)
    g = (ref > 0).float()
    assert torch.allclose(x.grad.float(), g @ w.detach().float().t(), atol=2e-2, rtol=1e-2)


def _wgrad_check(got, a, b):
    """got = rnd(a^T b) up to the fp32 summation order: within one fp16 step
    of the float64 value rounded once, plus an fp32-accumulation slack."""
    acc = a.astype(np.float64).T @ b.astype(np.float64)
    h = acc.astype(np.float16).astype(np.float64)
    slack = 2.0 ** -10 * np.abs(h) + 1e-6 * (np.abs(a.astype(np.float64)).T
                                              @ np.abs(b.astype(np.float64))) + 2.0 ** -24
    bad = np.abs(got.astype(np.float64) - h) > slack
    assert not bad.any(), f"{bad.sum()} of {bad.size} outside; max |d| {np.abs(got - h).max()}"


@pytest.mark.parametrize("k,m,n", [(233, 608, 64), (5000, 64, 48), (100_000, 608, 64),
                                   (7, 24, 8), (3000, 128, 128), (4097, 1032, 256),
                                   (70_001, 112, 48), (19_717, 512, 64), (40, 8, 200)])
def test_gemm_wgrad_vs_f64(cuda, k, m, n):
    """hg_gemm_wgrad (dW = x^T g, split over the vertices, MN-major tcgen05
    operands) and its fused bias gradient (column sums of g) vs float64:
    ragged K, M and N, several M-tile groups, N from 8 to 256."""
    from paper_2411_01109_b200 import device as D

    rng = np.random.default_rng(k + m + n)
    a = rng.normal(0, 1, (k, m)).astype(np.float16)
    b = rng.normal(0, 1, (k, n)).astype(np.float16)
    dw, db = D.gemm_wgrad(_t(a, cuda), _t(b, cuda), bias=True)
    _wgrad_check(dw.cpu().numpy(), a, b)
    _wgrad_check(db.cpu().numpy()[None, :], np.ones((k, 1), np.float16), b)
    # deterministic: same bits on a second call
    dw2 = D.gemm_wgrad(_t(a, cuda), _t(b, cuda))
    assert torch.equal(dw, dw2)


def test_gemm_wgrad_accumulate_and_empty(cuda):
    """accumulate: out = rnd(out + rnd(a^T b)) (Tensor._accumulate); K = 0 gives
    zeros, or leaves an accumulated output unchanged; strided (sliced) operands."""
    from paper_2411_01109_b200 import device as D

    rng = np.random.default_rng(5)
    a = rng.normal(0, 1, (3000, 64)).astype(np.float16)
    b = rng.normal(0, 1, (3000, 32)).astype(np.float16)
    prev = rng.normal(0, 4, (64, 32)).astype(np.float16)
    prevb = rng.normal(0, 4, 32).astype(np.float16)
    out, outb = _t(prev, cuda), _t(prevb, cuda)
    fresh, freshb = D.gemm_wgrad(_t(a, cuda), _t(b, cuda), bias=True)
    D.gemm_wgrad(_t(a, cuda), _t(b, cuda), out=out, bias_out=outb, accumulate=True)
    assert torch.equal(out, (prev_t := _t(prev, cuda)) + fresh)
    assert torch.equal(outb, _t(prevb, cuda) + freshb)
    z = D.gemm_wgrad(torch.empty(0, 16, device=cuda, dtype=torch.float16),
                     torch.empty(0, 8, device=cuda, dtype=torch.float16))
    assert z.shape == (16, 8) and not z.any()
    keep = prev_t.clone()
    D.gemm_wgrad(torch.empty(0, 64, device=cuda, dtype=torch.float16),
                 torch.empty(0, 32, device=cuda, dtype=torch.float16), out=keep, accumulate=True)
    assert torch.equal(keep, prev_t)
    wide = _t(rng.normal(0, 1, (3000, 96)).astype(np.float16), cuda)
    got = D.gemm_wgrad(wide[:, 16:80], _t(b, cuda))   # pitch 96, 16-byte aligned start
    _wgrad_check(got.cpu().numpy(), wide[:, 16:80].cpu().numpy(), b)
    with pytest.raises(ValueError, match="multiple of 8"):
        D.gemm_wgrad(torch.zeros(8, 16, device=cuda, dtype=torch.float16),
                     torch.zeros(8, 12, device=cuda, dtype=torch.float16))


@pytest.mark.parametrize("n", [8, 24, 40, 56, 200])
def test_gemm_tc_widths_8_mod_16(cuda, n):
    """hg_gemm_tc with N = 8 (mod 16): runs as the next multiple of 16 and
    stores only N columns (bias read only for those)."""
    from paper_2411_01109_b200 import device as D

    rng = np.random.default_rng(n)
    a = rng.normal(0, 1, (1000, 72)).astype(np.float16)
    wt = rng.normal(0, 0.2, (n, 72)).astype(np.float16)
    bias = rng.normal(0, 1, n).astype(np.float16)
    got = D.gemm_tc(_t(a, cuda), _t(wt, cuda), _t(bias, cuda)).cpu().numpy().astype(np.float64)
    acc = a.astype(np.float64) @ wt.astype(np.float64).T
    h = (acc.astype(np.float16).astype(np.float64) + bias).astype(np.float16).astype(np.float64)
    assert got.shape == (1000, n)
    assert np.all(np.abs(got - h) <= 2.0 ** -9 * np.abs(h) + 1e-3)


def test_linear_tc_backward_on_tensor_cores(cuda):
    """_LinearTCFn / _MatmulTCFn backward: dx, dW, db all from the tcgen05
    kernels; with ParamGroup-style leaves (persistent .grad) the weight and
    bias gradients accumulate in place and match a fresh computation."""
    from paper_2411_01109_b200 import models as M

    rng = np.random.default_rng(9)
    x = _t(rng.normal(0, 1, (4000, 64)).astype(np.float16), cuda).requires_grad_(True)
    w = _t((rng.normal(0, 0.1, (64, 40))).astype(np.float16), cuda).requires_grad_(True)
    b = _t(rng.normal(0, 1, 40).astype(np.float16), cuda).requires_grad_(True)
    g = _t(rng.normal(0, 1, (4000, 40)).astype(np.float16), cuda)
    y = M._LinearTCFn.apply(x, w, b, False)
    y.backward(g)
    gw, gb, gx = w.grad.clone(), b.grad.clone(), x.grad.clone()
    xf, wf, gf = x.detach().double(), w.detach().double(), g.double()
    assert torch.allclose(gx.double(), gf @ wf.t(), atol=2e-2, rtol=1e-2)
    assert torch.allclose(gw.double(), xf.t() @ gf, atol=0.5, rtol=2e-3)
    assert torch.allclose(gb.double(), gf.sum(0), atol=0.5, rtol=2e-3)
    # in place: pre-existing grads accumulate, autograd's own add not needed
    y = M._LinearTCFn.apply(x, w, b, False)
    y.backward(g)
    assert torch.equal(w.grad, gw + gw) and torch.equal(b.grad, gb + gb)
    # plain matmul (GAT projection, no bias) takes the same kernels
    z = M.matmul(x, w)
    assert z.grad_fn is not None and "MatmulTC" in type(z.grad_fn).__name__


@pytest.mark.parametrize("shape", [(1000,), (1000, 4), (999, 3), (500, 8)])
def test_gather_rows(cuda, shape):
    from paper_2411_01109_b200 import device as D

    rng = np.random.default_rng(len(shape))
    src = rng.normal(0, 1, shape).astype(np.float16)
    idx = rng.permutation(shape[0]).astype(np.int32)
    got = D.gather_rows(_t(src, cuda), _t(idx, cuda)).cpu().numpy()
    np.testing.assert_array_equal(bits(got), bits(src[idx]))


@pytest.mark.parametrize("f", [8, 48, 64, 128, 256])
def test_gather_probe_runs_and_times_below_spmm(cuda, f):
    """hg_gather_probe (bench's gather floor) runs for every team width, leaves
    its sink alone, and the Probe ceiling path returns a time."""
    from paper_2411_01109_b200 import device as D

    n = 20000
    r, c = _hub_graph(f, n)
    dg = _dg(n, r, c, cuda)
    x = torch.randn(n, f, device=cuda, dtype=torch.float16)
    view = dg.view(False)
    D.gather_probe(view.cols, view.num_edges, x, f * 2)
    D.gather_probe(view.cols, 0, x, f * 2)
    with pytest.raises(Exception):
        D.gather_probe(view.cols, view.num_edges, x, 1024)
    D.Probe.reset(timing=True, keep=True)
    D.spmm_csr(view, x, None, None, 1, "post")
    ceil = D.Probe.gather_ceiling()
    D.Probe.reset()
    torch.cuda.synchronize()
    assert ceil is not None and ceil > 0


@pytest.mark.parametrize("heads,fh", [(4, 32), (4, 16), (2, 64), (1, 128), (8, 8)])
def test_spmm_interleaved_weights_and_second_sums(cuda, heads, fh):
    """hg_spmm over interleaved [E, 2H] (w | w2) rows read through perm: the
    aggregation equals the one with dense weights, and out2 equals the column
    sums of w2 (hg_edge_sums_fast) -- incl. split heavy rows."""
    from paper_2411_01109_b200 import device as D

    n = 5000
    r, c = _hub_graph(heads + fh, n)
    dg = _dg(n, r, c, cuda)
    bwd = dg.view(True)
    e = r.size
    ae = torch.randn(e, 2 * heads, device=cuda, dtype=torch.float16)
    g = torch.randn(n, heads * fh, device=cuda, dtype=torch.float16)
    s2 = torch.empty(n, heads, device=cuda, dtype=torch.float16)
    got = D.spmm_csr(bwd, g, ae[:, :heads], bwd.perm, heads, "post", w2_off=heads, out2=s2)
    want = D.spmm_csr(bwd, g, ae[:, :heads].contiguous(), bwd.perm, heads, "post")
    assert torch.equal(got, want)
    want2 = D.edge_sums_fast(bwd, ae[:, heads:].contiguous(), bwd.perm)
    assert torch.allclose(s2.float(), want2.float(), atol=2e-2, rtol=2e-3)


def test_allgather_features_c_abi_one_rank(cuda):
    """hg_allgather_features through the C ABI with a communicator made by
    hg_nccl_comm_init (libnccl bound at run time): one rank (this box has one
    GPU) -- the group of exact-count broadcasts copies the rank's rows into
    place; bad splits are rejected."""
    from paper_2411_01109_b200 import device as D

    assert D.NcclComm.available()
    comm = D.NcclComm(1, 0, D.NcclComm.unique_id())
    try:
        x = torch.randn(1000, 48, device=cuda, dtype=torch.float16)
        full = D.allgather_features(comm, x, [0, 1000])
        torch.cuda.synchronize()
        assert torch.equal(full, x)
        with pytest.raises(ValueError, match="splits"):
            D.allgather_features(comm, x, [5, 1000])
    finally:
        comm.close()
