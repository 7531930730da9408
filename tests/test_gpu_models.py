"""GPU: the reference-facing API (kernels.*, sparse.*, models.*) on the B200.
Mirrors the reference's own tests (pkg/tests/test_kernels.py, test_models.py,
test_acceptance.py) -- same inputs, same expected values -- and compares
training traces with the golden traces recorded from the reference."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle as O
from conftest import bits, load_golden

pytestmark = pytest.mark.gpu

REDUCTIONS = [("post", "none"), ("post", "left"), ("post", "right"), ("post", "both"),
              ("pre", "left"), ("pre", "right"), ("pre", "both"),
              ("discretized", "left"), ("discretized", "right"), ("discretized", "both")]


def _random_graph(rng, n, density=0.2):
    from paper_2411_01109_b200 import sparse as sp

    mask = rng.random((n, n)) < density
    np.fill_diagonal(mask, False)
    return sp.CooGraph.from_edges(n, *np.nonzero(mask))


def _feats(rng, n, f, dtype=np.float16):
    from paper_2411_01109_b200 import sparse as sp

    return sp.DenseTensor(rng.normal(0, 2, size=(n, f)).astype(dtype))


# ── kernels API (test_kernels.py) ────────────────────────────────────────


@pytest.mark.parametrize("red", REDUCTIONS, ids=lambda r: "-".join(r))
@pytest.mark.parametrize("f", [4, 32])
def test_spmm_v_matches_oracle_bits(cuda, red, f):
    from paper_2411_01109_b200 import kernels as K, simt

    rng = np.random.default_rng(f * 13 + 1)
    g = _random_graph(rng, 48)
    x = _feats(rng, 48, f)
    sched = simt.plan_edge_parallel(g, warp_chunk=64, warps_per_cta=2)
    got, _ = K.spmm_v(g, x, schedule=sched, reduction=K.Reduction(*red))
    want = O.spmm_edge_parallel(g.n, g.rows, g.cols, x.data, None, 64, 2, *red)[0]
    np.testing.assert_array_equal(bits(got.data), bits(want))


def test_float32_mode_bit_exact(cuda):
    from paper_2411_01109_b200 import kernels as K

    rng = np.random.default_rng(17)
    g = _random_graph(rng, 30)
    x = _feats(rng, 30, 8, np.float32)
    got, _ = K.spmm_v(g, x, reduction=K.Reduction("discretized", "both"))
    want = O.spmm_edge_parallel(g.n, g.rows, g.cols, x.data, None, 128, 4, "discretized", "both")[0]
    np.testing.assert_array_equal(bits(got.data), bits(want))


def test_edge_metrics_hand_counted(cuda):
    """test_kernels.py:210-243: 130 single-edge rows, chunk 128, F=32."""
    from paper_2411_01109_b200 import kernels as K, simt, sparse as sp

    rows = np.arange(130, dtype=np.int64)
    g = sp.CooGraph(131, rows, rows + 1)
    x = sp.DenseTensor(np.ones((131, 32), dtype=np.float16))
    sched = simt.plan_edge_parallel(g, warp_chunk=128, warps_per_cta=4)
    _, m = K.spmm_v(g, x, schedule=sched)
    assert (m.load_transactions, m.load_bytes) == (70, 5 * 256 + 65 * 128)
    assert (m.barrier_waits, m.intra_cta_rounds, m.staging_writes) == (2, 0, 1)
    _, m = K.spmm_ve(g, np.ones(130, dtype=np.float16), x, schedule=sched)
    assert (m.load_transactions, m.load_bytes) == (73, 9600 + 3 * 128)


def test_intra_cta_chain_of_eight(cuda):
    """test_kernels.py:256-273: one 512-edge row, chunk 64, 8 warps/CTA."""
    from paper_2411_01109_b200 import kernels as K, simt, sparse as sp

    g = sp.CooGraph(513, np.zeros(512, dtype=np.int64), np.arange(1, 513, dtype=np.int64))
    x = sp.DenseTensor(np.ones((513, 4), dtype=np.float16))
    sched = simt.plan_edge_parallel(g, warp_chunk=64, warps_per_cta=8)
    y, m, st = K.spmm_v(g, x, schedule=sched, return_staging=True)
    assert m.intra_cta_rounds == 3 and m.staging_writes == 1
    assert st.capacity == 1 and st.rows.tolist() == [0]
    assert float(st.partials[0, 0]) == 512.0 and float(y.data[0, 0]) == 512.0


def test_vertex_conflict_writes(cuda):
    """test_kernels.py:287-311: 70-edge row -> groups 32+32+6."""
    from paper_2411_01109_b200 import kernels as K, sparse as sp

    g = sp.CooGraph(80, np.zeros(70, dtype=np.int64), np.arange(1, 71, dtype=np.int64))
    csr = sp.coo_to_csr(g)
    x = sp.DenseTensor(np.ones((80, 4), dtype=np.float16))
    y, m, st = K.spmm_vertex_grouped(csr, x, write_mode="staging", return_staging=True)
    assert (m.staging_writes, m.atomic_writes, st.capacity) == (3, 0, 3)
    assert st.rows.tolist() == [0, 0, 0] and float(y.data[0, 0]) == 70.0
    _, m = K.spmm_vertex_grouped(csr, x, write_mode="atomic_model")
    assert (m.atomic_writes, m.staging_writes) == (2, 0)


def test_equivalences_and_padding(cuda):
    from paper_2411_01109_b200 import kernels as K, sparse as sp

    rng = np.random.default_rng(12)
    g = _random_graph(rng, 50)
    x = _feats(rng, 50, 16)
    ones = np.ones(g.num_edges, dtype=np.float16)
    for red in (K.Reduction("post", "both"), K.Reduction("discretized", "right")):
        yv, _ = K.spmm_v(g, x, reduction=red)
        yw, _ = K.spmm_ve(g, ones, x, reduction=red)
        np.testing.assert_array_equal(bits(yv.data), bits(yw.data))
    x6 = _feats(rng, 50, 6)
    y, _ = K.spmm_v(g, x6, reduction=K.Reduction("post", "both"))
    yp, _ = K.spmm_v(g, sp.pad_features(x6, 4), reduction=K.Reduction("post", "both"))
    np.testing.assert_array_equal(bits(y.data), bits(yp.data)[:, :6])
    a, b = _feats(rng, 50, 32), _feats(rng, 50, 32)
    w2, m2 = K.sddmm(g, a, b, width="half2")
    w8, m8 = K.sddmm(g, a, b, width="half8")
    np.testing.assert_array_equal(bits(w2), bits(w8))
    assert m2.shuffle_rounds == 4 * g.num_edges and m8.shuffle_rounds == 2 * g.num_edges


def test_scaling_worked_example(cuda):
    from paper_2411_01109_b200 import kernels as K, sparse as sp

    g = sp.CooGraph(5, np.zeros(4, dtype=np.int64), np.arange(1, 5, dtype=np.int64))
    x = sp.DenseTensor(np.full((5, 32), 30000.0, dtype=np.float16))
    assert np.isinf(K.spmm_v(g, x, reduction=K.Reduction("post", "right"))[0].data[0]).all()
    for scaling in ("pre", "discretized"):
        for numerics in ("reference", "fast"):
            y, _ = K.spmm_v(g, x, reduction=K.Reduction(scaling, "right"), numerics=numerics)
            assert np.all(y.data[0] == 30000.0) and not y.data[1:].any()


def test_validation_errors(cuda):
    from paper_2411_01109_b200 import kernels as K, simt, sparse as sp

    g = sp.CooGraph(3, np.array([0]), np.array([1]))
    with pytest.raises(ValueError):
        K.spmm_v(g, sp.DenseTensor(np.ones((3, 5), np.float16)))
    with pytest.raises(ValueError):
        K.spmm_v(g, sp.DenseTensor(np.ones((3, 4), np.float16)), width="half8")
    with pytest.raises(ValueError, match="rows"):
        K.spmm_v(g, sp.DenseTensor(np.ones((4, 4), np.float16)))
    with pytest.raises(ValueError, match="CSR"):
        K.spmm_vertex_grouped(g, sp.DenseTensor(np.ones((3, 4), np.float16)))
    with pytest.raises(ValueError, match="modes"):
        K.sddmm(g, sp.DenseTensor(np.ones((3, 4), np.float16)),
                sp.DenseTensor(np.ones((3, 4), np.float32)))
    csr = sp.coo_to_csr(g)
    with pytest.raises(ValueError):
        K.spmm_v(g, sp.DenseTensor(np.ones((3, 4), np.float16)),
                 schedule=simt.plan_vertex_grouped(csr))
    with pytest.raises(ValueError, match="negative"):
        sp.CooGraph.from_edges(3, [0, -1], [1, 2])


def test_sparse_api_matches_oracle(cuda):
    from paper_2411_01109_b200 import sparse as sp

    rng = np.random.default_rng(5)
    n = 300
    rows, cols = rng.integers(0, n, 4000), rng.integers(0, n, 4000)
    g = sp.CooGraph.from_edges(n, rows, cols)
    wr, wc = O.canonical_edges(n, rows, cols)
    np.testing.assert_array_equal(g.rows, wr)
    np.testing.assert_array_equal(g.cols, wc)
    np.testing.assert_array_equal(sp.coo_to_csr(g).offsets, O.csr_offsets(n, wr))
    gt, perm = sp.transpose(g, return_perm=True)
    tr, tc, tp = O.transpose_perm(n, wr, wc)
    np.testing.assert_array_equal(gt.rows, tr)
    np.testing.assert_array_equal(gt.cols, tc)
    np.testing.assert_array_equal(perm, tp)
    np.testing.assert_array_equal(sp.col_degrees(g), np.bincount(wc, minlength=n))
    s = sp.symmetrize(g)
    np.testing.assert_array_equal(s.rows, O.symmetrize(n, wr, wc)[0])
    lp = sp.add_self_loops(g)
    np.testing.assert_array_equal(lp.cols, O.add_self_loops(n, wr, wc)[1])


# ── autograd ops (test_models.py) ────────────────────────────────────────


def _bundle(seed=0, n=24, density=0.25, numerics="reference"):
    from paper_2411_01109_b200 import sparse as sp
    from paper_2411_01109_b200.models import GraphBundle

    rng = np.random.default_rng(seed)
    mask = rng.random((n, n)) < density
    np.fill_diagonal(mask, False)
    g = sp.CooGraph.from_edges(n, *np.nonzero(mask))
    return GraphBundle.build(g, numerics=numerics), g


@pytest.mark.parametrize("numerics", ["reference", "fast"])
def test_spmm_agg_backward_is_transposed(cuda, numerics):
    from paper_2411_01109_b200 import models as M
    from paper_2411_01109_b200.kernels import Reduction

    bundle, g = _bundle(2, numerics=numerics)
    rng = np.random.default_rng(3)
    x = torch.tensor(rng.normal(size=(g.n, 4)).astype(np.float32), device=cuda,
                     requires_grad=True)
    y = M.spmm_agg(bundle, x, Reduction("post", "both"))
    seed = rng.normal(size=(g.n, 4)).astype(np.float32)
    y.backward(torch.tensor(seed, device=cuda))
    deg_r = np.bincount(g.rows, minlength=g.n).astype(np.float64)
    deg_c = np.bincount(g.cols, minlength=g.n).astype(np.float64)
    fin = np.where(deg_r > 0, 1 / np.sqrt(np.maximum(deg_r, 1)), 0)
    fout = np.where(deg_c > 0, 1 / np.sqrt(np.maximum(deg_c, 1)), 0)
    tr, tc, _ = O.transpose_perm(g.n, g.rows, g.cols)
    want = O.spmm_f64(g.n, tr, tc, seed, None, fin, fout)
    np.testing.assert_allclose(x.grad.cpu().numpy(), want, rtol=1e-3, atol=1e-4)


@pytest.mark.parametrize("numerics", ["reference", "fast"])
def test_spmm_weighted_grads(cuda, numerics):
    from paper_2411_01109_b200 import models as M

    bundle, g = _bundle(5, numerics=numerics)
    rng = np.random.default_rng(6)
    w = torch.tensor(rng.normal(size=g.num_edges).astype(np.float32), device=cuda,
                     requires_grad=True)
    x = torch.tensor(rng.normal(size=(g.n, 4)).astype(np.float32), device=cuda,
                     requires_grad=True)
    y = M.spmm_weighted(bundle, w, x)
    seed = rng.normal(size=(g.n, 4)).astype(np.float32)
    y.backward(torch.tensor(seed, device=cuda))
    want_w = np.einsum("ef,ef->e", seed.astype(np.float64)[g.rows],
                       x.detach().cpu().numpy().astype(np.float64)[g.cols])
    np.testing.assert_allclose(w.grad.cpu().numpy(), want_w, rtol=1e-3, atol=1e-4)
    a = np.zeros((g.n, g.n))
    a[g.rows, g.cols] = w.detach().cpu().numpy()
    np.testing.assert_allclose(x.grad.cpu().numpy(), a.T @ seed, rtol=1e-3, atol=1e-4)


def test_attention_backward_degree_sums(cuda):
    from paper_2411_01109_b200 import models as M

    for numerics in ("reference", "fast"):
        bundle, g = _bundle(9, numerics=numerics)
        s_l = torch.zeros((g.n, 1), dtype=torch.float16, device=cuda, requires_grad=True)
        s_r = torch.zeros((g.n, 1), dtype=torch.float16, device=cuda, requires_grad=True)
        e = M.attention_scores(bundle, s_l, s_r)
        e.backward(torch.ones(g.num_edges, dtype=torch.float16, device=cuda))
        np.testing.assert_array_equal(s_l.grad[:, 0].cpu().numpy(),
                                      np.bincount(g.rows, minlength=g.n))
        np.testing.assert_array_equal(s_r.grad[:, 0].cpu().numpy(),
                                      np.bincount(g.cols, minlength=g.n))


def test_attention_golden_through_models(cuda):
    """attention_scores -> leaky_relu -> edge_softmax fwd+bwd against the
    reference's own tape values, bit for bit (reference numerics)."""
    from paper_2411_01109_b200 import models as M
    from paper_2411_01109_b200 import sparse as sp
    from conftest import golden_cases

    cases, _ = golden_cases("attention.npz")
    for i, c in enumerate(cases):
        g = sp.CooGraph(int(c["n"]), c["rows"], c["cols"])
        bundle = M.GraphBundle.build(g, numerics="reference")
        dt = torch.float16 if c["sl"].dtype == np.float16 else torch.float32
        s_l = torch.tensor(c["sl"][:, None], device=cuda, requires_grad=True)
        s_r = torch.tensor(c["sr"][:, None], device=cuda, requires_grad=True)
        e = M.attention_scores(bundle, s_l, s_r)
        e2 = M.leaky_relu(e, 0.2)
        alpha = M.edge_softmax(bundle, e2)
        np.testing.assert_array_equal(bits(alpha.detach().cpu().numpy()), bits(c["alpha"]))
        alpha.backward(torch.tensor(c["seed"], device=cuda, dtype=dt))
        np.testing.assert_array_equal(bits(s_l.grad[:, 0].cpu().numpy()), bits(c["g_sl"]),
                                      err_msg=f"case {i}")
        np.testing.assert_array_equal(bits(s_r.grad[:, 0].cpu().numpy()), bits(c["g_sr"]),
                                      err_msg=f"case {i}")


def test_edge_softmax_uniform(cuda):
    from paper_2411_01109_b200 import models as M, sparse as sp

    g = sp.CooGraph(4, np.zeros(4, dtype=np.int64), np.arange(4, dtype=np.int64))
    bundle = M.GraphBundle.build(g)
    e = torch.zeros(4, dtype=torch.float16, device=cuda, requires_grad=True)
    alpha = M.edge_softmax(bundle, e)
    assert alpha.detach().cpu().tolist() == [0.25] * 4
    alpha.backward(torch.ones(4, dtype=torch.float16, device=cuda))
    assert not e.grad.any()


# ── training (test_models.py TestTrain, test_acceptance.py C4) ───────────


def _sbm_golden():
    d = load_golden("training.npz")
    from paper_2411_01109_b200 import sparse as sp

    g = sp.CooGraph(60, d["sbm_rows"], d["sbm_cols"])
    return g, d["sbm_x"], d["sbm_labels"], d


@pytest.mark.parametrize("kind", ["gcn", "gin", "gat"])
@pytest.mark.parametrize("mode", ["half", "float32"])
def test_training_trace_matches_reference(cuda, kind, mode):
    """5 epochs, reference numerics: losses within 2e-3 of the reference's."""
    from paper_2411_01109_b200 import models as M

    g, x, labels, d = _sbm_golden()
    cfg = M.TrainConfig(kind=kind, mode=mode, epochs=5, seed=3, numerics="reference")
    res = M.train(g, x, labels, cfg)
    want = d[f"sbm_{kind}_{mode}_loss"]
    np.testing.assert_allclose(res.losses, want, atol=2e-3)
    cfg_fast = M.TrainConfig(kind=kind, mode=mode, epochs=5, seed=3, numerics="fast")
    np.testing.assert_allclose(M.train(g, x, labels, cfg_fast).losses, want, atol=5e-3)


def test_multihead_gat_trace(cuda):
    from paper_2411_01109_b200 import models as M

    g, x, labels, d = _sbm_golden()
    cfg = M.TrainConfig(kind="gat", mode="half", epochs=4, seed=5, hidden=4, heads=4, layers=3,
                        numerics="reference")
    res = M.train(g, x, labels, cfg)
    np.testing.assert_allclose(res.losses, d["sbm_gat4x3_half_loss"], atol=3e-3)


def test_c1_gcn_accuracy_parity(cuda):
    """C1 (Cora-shaped, 7 -> 8 classes) 200 epochs: final train/val accuracy
    within 0.5 pt of the reference trainer's (north_star tolerance)."""
    from paper_2411_01109_b200 import graphgen, models as M, sparse as sp

    d = load_golden("training.npz")
    rows, cols, feats, labels = graphgen.cora_like(0)
    assert rows.size == int(d["c1_num_edges"])
    g = sp.CooGraph(2708, rows, cols)
    for numerics in ("fast", "reference"):
        res = M.train(g, feats, labels, M.TrainConfig(kind="gcn", epochs=200, seed=0,
                                                      numerics=numerics))
        want_train, want_val = d["c1_gcn_half_acc"][-1]
        assert abs(res.train_acc - want_train) <= 0.005, (numerics, res.train_acc, want_train)
        assert abs(res.val_acc - want_val) <= 0.005, (numerics, res.val_acc, want_val)
        assert all(row[5] == 0 for row in res.trace)


@pytest.mark.timeout(900)
def test_c2_gat_accuracy_parity(cuda):
    """C2 (Pubmed-shaped synth_sbm, 3-layer x 4-head x 16 GAT, classes 3 -> 4)
    200 epochs: final train / val accuracy within 0.5 pt of the reference
    harness's 200-epoch run (tests/golden/c2_half.npz, make_golden.py c2 half:
    reference GATLayers composed with concat / mean, models.py:492-509,
    633-684), in both numerics; the loss trace follows the reference's."""
    from paper_2411_01109_b200 import graphgen, models as M, sparse as sp

    d = load_golden("c2_half.npz")
    rows, cols, feats, labels = graphgen.pubmed_like(0)
    assert rows.size == int(d["num_edges"])
    g = sp.CooGraph(19717, rows, cols)
    want_train, want_val = d["acc"][-1]
    for numerics, atol in (("reference", 5e-3), ("fast", 1e-2)):
        res = M.train(g, feats, labels, M.TrainConfig(kind="gat", hidden=16, heads=4, layers=3,
                                                      epochs=200, seed=0, numerics=numerics))
        assert abs(res.train_acc - want_train) <= 0.005, (numerics, res.train_acc, want_train)
        assert abs(res.val_acc - want_val) <= 0.005, (numerics, res.val_acc, want_val)
        np.testing.assert_allclose(res.losses, d["loss"], atol=atol, rtol=0)
        assert all(row[5] == 0 for row in res.trace)


def test_conversions_and_nan_abort(cuda):
    from paper_2411_01109_b200 import graphgen, models as M, sparse as sp

    g, x, labels, _ = _sbm_golden()
    r = M.train(g, x, labels, M.TrainConfig(kind="gat", epochs=3))
    assert (r.conversions.forward, r.conversions.backward) == (3, 3)
    r = M.train(g, x, labels, M.TrainConfig(mode="float32", epochs=3))
    assert r.conversions.total == 0
    # test_models.py:337-350: GIN lam=1, x1000, post scaling overflows -> NaN at epoch 0
    rows, cols, f8, lab = graphgen.synth_sbm(60, 2, 0.5, 0.1, 8, 3)
    g2 = sp.CooGraph(60, rows, cols)
    big = f8 * 1000.0
    with pytest.raises(M.NanLossError) as err:
        M.train(g2, big, lab, M.TrainConfig(kind="gin", epochs=5, lam=1.0, scaling="post",
                                            norm="right"))
    assert err.value.epoch == 0 and sum(err.value.counters.inf.values()) > 0
    ok = M.train(g2, big, lab, M.TrainConfig(kind="gin", epochs=5, lam=1.0,
                                             scaling="discretized", norm="right"))
    assert all(row[4] == 0 and row[5] == 0 for row in ok.trace)


def test_smoke_entry(cuda):
    import __graft_entry__

    __graft_entry__.smoke()


def test_cuda_graph_step_matches_eager(cuda):
    """A captured training step replays to the same losses as eager steps."""
    from paper_2411_01109_b200 import graphgen, models as M
    from paper_2411_01109_b200.device import DeviceGraph

    rows, cols, feats, labels = graphgen.synth_sbm(300, 3, 0.05, 0.005, 12, 4)
    dg = DeviceGraph.from_edges(300, rows, cols)
    for kind, kw in (("gcn", {}), ("gat", {"heads": 2, "layers": 3}), ("gin", {})):
        cfg = M.TrainConfig(kind=kind, hidden=8, **kw)
        a = M.Trainer(M.GraphBundle.build(dg), feats, labels, cfg)
        b = M.Trainer(M.GraphBundle.build(dg), feats, labels, cfg)
        la = [float(a.step()[0]) for _ in range(6)]
        lb = [float(b.step()[0])]
        b.capture()
        lb += [float(b.step()[0]) for _ in range(5)]
        np.testing.assert_allclose(la, lb, rtol=0, atol=1e-6, err_msg=kind)


@pytest.mark.parametrize("kind,kw", [("gcn", {}), ("gin", {}), ("gat", {"heads": 4, "layers": 3})])
def test_training_step_dense_math_on_own_kernels(cuda, kind, kw):
    """A fast-numerics half training step (the benched path) launches no
    cuBLAS / library GEMM: forward, dx and dW GEMMs all run on hg_gemm_tc /
    hg_gemm_wgrad (tcgen05).  The kernel list goes to HG_KERNEL_LIST if set."""
    import os

    from torch.profiler import ProfilerActivity, profile

    from paper_2411_01109_b200 import graphgen, models as M
    from paper_2411_01109_b200.device import DeviceGraph

    rows, cols, feats, labels = graphgen.synth_sbm(3000, 3, 0.01, 0.001, 100, 1)
    dg = DeviceGraph.from_edges(3000, rows, cols)
    cfg = M.TrainConfig(kind=kind, hidden=16, numerics="fast", grad_scale="auto", **kw)
    tr = M.Trainer(M.GraphBundle.build(dg, numerics="fast"), feats, labels, cfg)
    for _ in range(2):
        tr.step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        tr.step()
        torch.cuda.synchronize()
    names = sorted({e.name for e in prof.events() if e.device_type.name == "CUDA"})
    if os.environ.get("HG_KERNEL_LIST"):
        with open(os.environ["HG_KERNEL_LIST"], "a") as f:
            f.write(f"== {kind}\n" + "\n".join(names) + "\n")
    lib = [n for n in names if any(t in n.lower() for t in ("nvjet", "cublas", "cutlass", "sgemm",
                                                            "hgemm", "gemv", "gemmk"))]
    assert not lib, lib
    assert any("k_gemm_wgrad" in n for n in names) and any("k_gemm_tc" in n for n in names)


def test_locality_relabel_same_graph_and_training(cuda):
    """DeviceGraph.relabel(locality_order): the relabelled graph is the same
    graph (edge set maps exactly), its aggregation equals the original's row
    for row within the fast-path bound of float64, and training with
    node_order (features / labels / split per original vertex) reaches the
    same accuracy and a close loss trace."""
    import oracle as O
    from paper_2411_01109_b200 import device as D, graphgen, models as M
    from paper_2411_01109_b200.device import DeviceGraph

    rows, cols, feats, labels = graphgen.synth_sbm(2000, 4, 0.02, 0.002, 32, 3)
    dg = DeviceGraph.from_edges(2000, rows, cols)
    order = D.locality_order(dg.offsets, dg.bwd.offsets)
    dr = dg.relabel(order)
    o = order.cpu().numpy()
    new_of_old = np.empty_like(o)
    new_of_old[o] = np.arange(o.size)
    r0 = np.repeat(np.arange(2000), np.diff(dg.offsets.cpu().numpy()))
    e0 = set(zip(new_of_old[r0].tolist(), new_of_old[dg.cols.cpu().numpy()].tolist()))
    r1 = np.repeat(np.arange(2000), np.diff(dr.offsets.cpu().numpy()))
    assert e0 == set(zip(r1.tolist(), dr.cols.cpu().numpy().tolist()))
    x = torch.randn(2000, 64, device=cuda, dtype=torch.float16)
    y0 = D.spmm(dg, x, None, "discretized", "both").double().cpu().numpy()
    y1 = D.spmm(dr, x[order], None, "discretized", "both").double().cpu().numpy()[new_of_old]
    assert np.all(np.abs(y1 - y0) <= 1e-2 * np.maximum(1.0, np.abs(y0)))
    cfg = M.TrainConfig(kind="gcn", hidden=16, epochs=30, numerics="fast")
    a = M.Trainer(M.GraphBundle.build(dg), feats, labels, cfg)
    b = M.Trainer(M.GraphBundle.build(dr), feats, labels, cfg, node_order=order)
    assert bool((b.labels.cpu() == torch.as_tensor(labels)[order.cpu()]).all())
    la = [float(a.step()[0]) for _ in range(30)]
    lb = [float(b.step()[0]) for _ in range(30)]
    np.testing.assert_allclose(la, lb, rtol=0, atol=5e-3)


def test_gin_combine_epilogue_bitwise(cuda):
    """GIN's scale_combine folded into the aggregation's row store (forward)
    and the residual gradient add into the transposed aggregation's store
    (backward) train bit for bit like the separate passes (packs and split
    rows included)."""
    from paper_2411_01109_b200 import device as D, graphgen, models as M
    from paper_2411_01109_b200.device import DeviceGraph

    rows, cols, feats, labels = graphgen.synth_sbm(3000, 3, 0.05, 0.003, 40, 6)
    hub = np.repeat(np.arange(3), 900)
    rows = np.concatenate([rows, hub]).astype(np.int64)
    cols = np.concatenate([cols, np.random.default_rng(0).integers(0, 3000, hub.size)])
    dg = DeviceGraph.from_edges(3000, rows, cols)
    cfg = M.TrainConfig(kind="gin", hidden=16, numerics="fast")
    saved = (M.FUSED_GIN_COMBINE, D.PACK_MIN_ROWS)
    out = []
    try:
        D.PACK_MIN_ROWS = 0
        for fused in (False, True):
            M.FUSED_GIN_COMBINE = fused
            tr = M.Trainer(M.GraphBundle.build(dg), feats, labels, cfg)
            losses = [float(tr.step()[0]) for _ in range(4)]
            out.append((losses, tr.group.master.clone()))
    finally:
        M.FUSED_GIN_COMBINE, D.PACK_MIN_ROWS = saved
    assert out[0][0] == out[1][0]
    assert torch.equal(out[0][1], out[1][1])


def test_run_epochs_host_feed_matches_steps(cuda):
    """Double-buffered host feeding (e2e path) trains exactly like step()."""
    from paper_2411_01109_b200 import graphgen, models as M
    from paper_2411_01109_b200.device import DeviceGraph

    rows, cols, feats, labels = graphgen.synth_sbm(200, 2, 0.05, 0.005, 10, 2)
    dg = DeviceGraph.from_edges(200, rows, cols)
    cfg = M.TrainConfig(kind="gcn", hidden=8)
    a = M.Trainer(M.GraphBundle.build(dg), feats, labels, cfg)
    b = M.Trainer(M.GraphBundle.build(dg), feats, labels, cfg)
    la = [float(a.step()[0]) for _ in range(5)]
    lb = b.run_epochs(b.host_features(feats), 5)
    assert la == lb


def test_synthetic_generators_shapes(cuda):
    """C3/C4/C5 generators (small instances): exact edge counts, canonical CSR,
    symmetry for the products-shaped graph, determinism for a seed."""
    from paper_2411_01109_b200 import graphgen

    g = graphgen.reddit_like(0, n=5000, e=200_000)
    assert g.n == 5000 and g.num_edges == 200_000
    off = g.offsets.cpu().numpy()
    cols = g.cols.cpu().numpy()
    rows = np.repeat(np.arange(g.n), np.diff(off))
    assert np.all(np.diff(rows * g.n + cols) > 0)  # sorted, unique
    p = graphgen.products_like(1, n=20000, undirected=100_000)
    pr = np.repeat(np.arange(p.n), np.diff(p.offsets.cpu().numpy()))
    pc = p.cols.cpu().numpy()
    fwd = set(zip(pr.tolist(), pc.tolist()))
    assert all((c, r) in fwd for r, c in list(fwd)[:5000])
    r1 = graphgen.rmat(scale=12, edge_factor=8, seed=3)
    r2 = graphgen.rmat(scale=12, edge_factor=8, seed=3)
    assert r1.n == 4096 and 0 < r1.num_edges <= 8 * 4096
    assert torch.equal(r1.cols, r2.cols) and torch.equal(r1.offsets, r2.offsets)
    deg = np.diff(r1.offsets.cpu().numpy())
    assert deg.max() > 20 * max(1, int(np.median(deg)))  # power-law skew


def test_run_epochs_with_graphs_matches_eager(cuda):
    from paper_2411_01109_b200 import graphgen, models as M
    from paper_2411_01109_b200.device import DeviceGraph

    rows, cols, feats, labels = graphgen.synth_sbm(200, 2, 0.05, 0.005, 10, 5)
    dg = DeviceGraph.from_edges(200, rows, cols)
    cfg = M.TrainConfig(kind="gat", hidden=8, heads=2)
    a = M.Trainer(M.GraphBundle.build(dg), feats, labels, cfg)
    b = M.Trainer(M.GraphBundle.build(dg), feats, labels, cfg)
    la = [float(a.step()[0]) for _ in range(7)]
    lb = [float(b.step()[0])]
    b.capture()
    lb += b.run_epochs(b.host_features(feats), 6)
    np.testing.assert_allclose(la, lb, rtol=0, atol=1e-6)


def _torch_fp32_gcn_losses(tr, dg, epochs, lr):
    """Plain torch fp32 GCN (torch.sparse CSR with exact D_r^-1/2 A D_c^-1/2
    values, torch.optim.Adam) from the trainer's initial fp32 masters."""
    off = dg.offsets
    deg_r = (off[1:] - off[:-1]).double()
    deg_c = torch.bincount(dg.cols.long(), minlength=dg.n).double()
    rows = torch.repeat_interleave(torch.arange(dg.n, device=off.device), off[1:] - off[:-1])

    def inv(d):
        return torch.where(d > 0, 1.0 / d.sqrt(), torch.zeros_like(d))

    vals = (inv(deg_r)[rows] * inv(deg_c)[dg.cols.long()]).float()
    a = torch.sparse_csr_tensor(off, dg.cols.long(), vals, (dg.n, dg.n))
    ps = [p.master.detach().clone().requires_grad_(True) for p in tr.model.params()]
    opt = torch.optim.Adam(ps, lr=lr, betas=(0.9, 0.999), eps=1e-8)
    xf = tr.x.float()
    out = []
    for _ in range(epochs):
        w1, b1, w2, b2 = ps
        h = torch.relu(torch.sparse.mm(a, xf @ w1 + b1))
        logits = torch.sparse.mm(a, h @ w2 + b2)[:, : tr.n_cls]
        loss = torch.nn.functional.cross_entropy(logits.double(), tr.labels)
        opt.zero_grad()
        loss.backward()
        opt.step()
        out.append(float(loss.detach()))
    return out


def test_gcn_large_graph_tracks_torch_fp32_with_grad_scale(cuda):
    """Reddit-shaped degrees at 1/4 scale (58K nodes, 7M edges, rows split
    across work units): with the static loss scale the fp16 fast path trains
    like a plain torch fp32 GCN from the same weights; without it the
    reference's (p - y)/N gradient sits in fp16 subnormals and the first
    update already deviates."""
    from paper_2411_01109_b200 import graphgen, models as M

    dg = graphgen.reddit_like(3, n=58_000, e=7_000_000)
    x, labels = graphgen.planted_features(dg.n, 96, 12, 3, "cuda")
    kw = dict(kind="gcn", hidden=32, numerics="fast")
    tr = M.Trainer(M.GraphBundle.build(dg), x, labels, M.TrainConfig(grad_scale="auto", **kw))
    assert tr.grad_scale == 512.0
    want = _torch_fp32_gcn_losses(tr, dg, 12, 1e-2)
    got = [float(tr.step()[0]) for _ in range(12)]
    np.testing.assert_allclose(got, want, rtol=0, atol=2e-3)
    # same start, no scale: identical first loss, worse-tracking second step
    t1 = M.Trainer(M.GraphBundle.build(dg), x, labels, M.TrainConfig(**kw))
    l1 = [float(t1.step()[0]) for _ in range(2)]
    assert l1[0] == got[0]
    assert abs(l1[1] - want[1]) > abs(got[1] - want[1])


@pytest.mark.parametrize("fh", [8, 16, 32])
def test_gat_head_dot_folds_bitwise(cuda, fh):
    """The GAT layer with the projection's head dots in the GEMM epilogue and
    their dz term in the transposed aggregation's store (HG_FUSED_GAT_DZ) ==
    the separate hg_head_dots_bwd accumulate: bitwise the same outputs and
    gradients of every parameter."""
    from paper_2411_01109_b200 import graphgen, models as M
    from paper_2411_01109_b200.device import DeviceGraph

    rows, cols, feats, labels = graphgen.synth_sbm(3000, 3, 0.01, 0.001, 32, 5)
    dg = DeviceGraph.from_edges(3000, rows, cols)
    b = M.GraphBundle.build(dg)
    rng = np.random.default_rng(1)
    layer = M.GATLayer(rng, 32, fh, heads=4, store_in=32, store_out=fh)
    x = torch.from_numpy(feats).cuda().half()
    res = []
    saved = M.FUSED_GAT_DZ
    try:
        for dz in (False, True):
            M.FUSED_GAT_DZ = dz
            for p in layer.params():
                p.published = None
            y = layer(b, x, "half", "half2", None, "gat", relu_out=True)
            (y.float() * torch.linspace(-1, 1, y.numel(), device=cuda).view_as(y)).sum().backward()
            res.append([y.detach()] + [p.published.grad.clone() for p in layer.params()])
    finally:
        M.FUSED_GAT_DZ = saved
    for a, c in zip(*res):
        assert torch.equal(a.view(torch.int16), c.view(torch.int16))


@pytest.mark.parametrize("kind,hidden,layers", [("gat", 16, 2), ("gat", 16, 3), ("gat", 8, 3),
                                                ("gin", 32, 2), ("gin", 16, 3),
                                                ("gcn", 16, 2), ("gcn", 64, 3)])
def test_relu_backward_fold_bitwise(cuda, kind, hidden, layers):
    """A ReLU's backward folded into its only consumer's dX GEMM
    (hg_gemm_tc_masked, relu_grad skipped by the producer: between GAT layers,
    between GCN layers, and between GIN's two MLP linears) trains bit for bit
    like the separate relu_grad pass: losses and every parameter."""
    from paper_2411_01109_b200 import graphgen, models as M
    from paper_2411_01109_b200.device import DeviceGraph

    rows, cols, feats, labels = graphgen.synth_sbm(3000, 4, 0.01, 0.001, 32, 9)
    dg = DeviceGraph.from_edges(3000, rows, cols)
    runs = []
    saved = M.FUSED_RELU_BWD
    try:
        for fold in (False, True):
            M.FUSED_RELU_BWD = fold
            tr = M.Trainer(M.GraphBundle.build(dg), feats, labels,
                           M.TrainConfig(kind=kind, hidden=hidden, layers=layers, epochs=3,
                                         seed=3, **({"heads": 4} if kind == "gat" else {})))
            losses = [float(tr.step()[0]) for _ in range(3)]
            runs.append((losses, [p.master.clone() for p in tr.model.params()]))
    finally:
        M.FUSED_RELU_BWD = saved
    assert runs[0][0] == runs[1][0]
    for p0, p1 in zip(runs[0][1], runs[1][1]):
        assert torch.equal(p0, p1)


@pytest.mark.parametrize("fh", [8, 16])
def test_gat_core_fused_matches_composed(cuda, fh):
    """The single-node GAT core (_GATCoreFn, ReLU fused) against the composed
    ops (taken when overflow counters watch): same outputs and gradients up to
    fp16 rounding order.  fh=16: the projection also forms the head dots in its
    GEMM epilogue (_GATProjFn, hg_gemm_tc_dots)."""
    from paper_2411_01109_b200 import graphgen, models as M
    from paper_2411_01109_b200.device import DeviceGraph

    rows, cols, feats, labels = graphgen.synth_sbm(400, 3, 0.05, 0.005, 24, 7)
    dg = DeviceGraph.from_edges(400, rows, cols)
    b = M.GraphBundle.build(dg)
    rng = np.random.default_rng(0)
    layer = M.GATLayer(rng, 24, fh, heads=4, store_in=24, store_out=fh)
    x = torch.from_numpy(feats).cuda().half()
    assert M._dots_shapes(x, layer.w.publish("half"), 4) == (fh == 16)
    outs, grads = [], []
    for ov in (None, M.OverflowCounters()):
        for p in layer.params():
            p.published = None
        y = layer(b, x, "half", "half2", ov, "gat", relu_out=True)
        (y.float() * torch.linspace(-1, 1, y.numel(), device=cuda).view_as(y)).sum().backward()
        outs.append(y.detach().float())
        grads.append([p.published.grad.float().clone() for p in layer.params()])
    assert torch.allclose(outs[0], outs[1], atol=2e-3, rtol=2e-3)
    for g0, g1 in zip(*grads):
        assert torch.allclose(g0, g1, atol=2e-2, rtol=2e-2)
