"""GPU: the reference's acceptance criteria (pkg/tests/test_acceptance.py)
re-run through the B200 build with the same inputs and tolerances:

  C1  200 random graphs, every kernel kind, bit-exact (test_acceptance.py:47-91)
      -- here against the oracle restatement (pinned to the reference's goldens)
  C4  training parity half vs float32, 3 models x 3 seeds, 200 epochs, and the
      128x-input NaN variant (173-223)
  C5  attention softmax ranges over 10^4 neighbourhoods (229-268)
  C6  analytic gradients vs central differences on 6 vertices (274-343)
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle as O
from conftest import bits

pytestmark = pytest.mark.gpu

DIFFERENTIAL_TRIALS = 200
PARITY_EPOCHS = 200
PARITY_SEEDS = (0, 1, 2)
PARITY_ACC_TOL = 0.010
ROWSUM_TOL = 2.0 ** -8
GRAD_EPS = 3e-3
GRAD_REL_TOL = 0.02
GRAD_FLOOR = 1e-3
SCALINGS = ("post", "pre", "discretized")
NORMS = ("none", "left", "right", "both")


def _random_reduction(rng):
    scaling = str(rng.choice(SCALINGS))
    norms = [n for n in NORMS if not (scaling == "discretized" and n == "none")]
    return scaling, str(rng.choice(norms))


@pytest.mark.timeout(600)
def test_criterion_1_bit_exact_random_graphs(cuda):
    from paper_2411_01109_b200 import kernels as K, simt, sparse as sp
    from paper_2411_01109_b200.kernels import Reduction

    kinds = ("spmm_v", "spmm_ve", "sddmm", "vertex_staging", "vertex_atomic")
    for i in range(DIFFERENTIAL_TRIALS):
        rng = np.random.default_rng(1000 + i)
        n = int(rng.integers(4, 65))
        mask = rng.random((n, n)) < rng.uniform(0.05, 0.5)
        np.fill_diagonal(mask, False)
        r, c = np.nonzero(mask)
        g = sp.CooGraph.from_edges(n, r, c)
        f = int(rng.choice([2, 4, 16, 32, 64]))
        dtype = np.float16 if i % 4 else np.float32
        xa = rng.normal(0, 2, (n, f)).astype(dtype)
        x = sp.DenseTensor(xa)
        scaling, norm = _random_reduction(rng)
        red = Reduction(scaling, norm)
        kind = kinds[i % len(kinds)]
        label = f"trial {i}: {kind} n={n} f={f} {scaling}/{norm} {x.mode}"
        if kind in ("spmm_v", "spmm_ve"):
            chunk, warps = int(rng.choice([64, 128, 266])), int(rng.choice([1, 2, 4, 8]))
            sched = simt.plan_edge_parallel(g, chunk, warps)
            w = None
            if kind == "spmm_ve":
                w = rng.normal(size=g.num_edges).astype(dtype)
                got, _ = K.spmm_ve(g, w, x, sched, red)
            else:
                got, _ = K.spmm_v(g, x, sched, red)
            want = O.spmm_edge_parallel(n, g.rows, g.cols, xa, w, chunk, warps, scaling, norm)[0]
            assert np.array_equal(bits(got.data), bits(want)), label
        elif kind == "sddmm":
            ya = rng.normal(0, 2, (n, f)).astype(dtype)
            got, _ = K.sddmm(g, x, sp.DenseTensor(ya))
            assert np.array_equal(bits(got), bits(O.sddmm(g.rows, g.cols, xa, ya))), label
        else:
            csr = sp.coo_to_csr(g)
            mode = "staging" if kind == "vertex_staging" else "atomic_model"
            got, _ = K.spmm_vertex_grouped(csr, x, reduction=red, write_mode=mode)
            want = O.spmm_vertex_grouped(n, O.csr_offsets(n, g.rows), g.cols, xa, scaling,
                                         norm)[0]
            assert np.array_equal(bits(got.data), bits(want)), label


@pytest.mark.timeout(900)
@pytest.mark.parametrize("numerics", ["fast", "reference"])
def test_criterion_4_training_parity(cuda, numerics):
    from paper_2411_01109_b200 import models as M, sparse as sp

    worst = 0.0
    for kind in ("gcn", "gin", "gat"):
        for seed in PARITY_SEEDS:
            g, x, labels = sp.synth_sbm(1000, 2, 0.05, 0.005, 32, seed=seed)
            half = M.train(g, x.data, labels, M.TrainConfig(
                kind=kind, mode="half", epochs=PARITY_EPOCHS, seed=seed, numerics=numerics))
            full = M.train(g, x.data, labels, M.TrainConfig(
                kind=kind, mode="float32", epochs=PARITY_EPOCHS, seed=seed, numerics=numerics))
            delta = abs(half.train_acc - full.train_acc)
            worst = max(worst, delta)
            assert delta <= PARITY_ACC_TOL, (kind, seed, delta)
            assert all(row[5] == 0 for row in half.trace), (kind, seed, "NaN seen")
            assert np.isfinite(half.losses).all()
    # 128x inputs: post scaling overflows at once, discretized finishes clean
    g, x, labels = sp.synth_sbm(1000, 2, 0.9, 0.05, 32, seed=5)
    big = x.data * 128.0
    with pytest.raises(M.NanLossError) as err:
        M.train(g, big, labels, M.TrainConfig(kind="gcn", mode="half", epochs=30, scaling="post",
                                              norm="right", seed=0, numerics=numerics))
    assert err.value.epoch == 0
    assert sum(err.value.counters.inf.values()) > 0
    survived = M.train(g, big, labels, M.TrainConfig(
        kind="gcn", mode="half", epochs=30, scaling="discretized", norm="right", seed=0,
        numerics=numerics))
    assert all(row[5] == 0 for row in survived.trace)
    assert survived.train_acc >= 0.9


def test_criterion_5_softmax_ranges(cuda):
    """10^4 neighbourhoods, degrees 1..32, scores in [-4, 4]: alpha in (0, 1] and
    row sums within 2^-8 -- for the reference-order softmax and for the fast
    fused attention; one conversion pair per GAT epoch."""
    from paper_2411_01109_b200 import device as D, models as M, sparse as sp

    rng = np.random.default_rng(50)
    n = 10_000
    deg = rng.integers(1, 33, size=n)
    rows = np.repeat(np.arange(n, dtype=np.int64), deg)
    cols = rng.integers(0, n, size=rows.size)
    g = sp.CooGraph.from_edges(n, rows, cols)
    assert np.unique(g.rows).size == n
    bundle = M.GraphBundle.build(g, numerics="reference")
    e = torch.from_numpy(rng.uniform(-4, 4, g.num_edges).astype(np.float16)).cuda()
    for alpha in (M.edge_softmax(bundle, e).cpu().numpy().astype(np.float64),
                  D.gat_attention_fwd(g.device().view(False),
                                      torch.zeros(n, 1, dtype=torch.float16, device="cuda"),
                                      torch.from_numpy(rng.uniform(-4, 4, (n, 1)).astype(np.float16)).cuda(),
                                      0.2).cpu().numpy()[:, 0].astype(np.float64)):
        assert (alpha > 0).all() and (alpha <= 1.0).all()
        sums = np.zeros(n)
        np.add.at(sums, g.rows, alpha)
        assert float(np.abs(sums - 1.0).max()) <= ROWSUM_TOL
    gg, xx, ll = sp.synth_sbm(60, 2, 0.5, 0.1, 8, seed=1)
    r = M.train(gg, xx.data, ll, M.TrainConfig(kind="gat", mode="half", epochs=4))
    assert (r.conversions.forward, r.conversions.backward) == (4, 4)


def _grad_setup(kind, numerics):
    from paper_2411_01109_b200 import models as M, sparse as sp

    rows = np.array([0, 0, 1, 2, 2, 3, 4, 4, 5])
    cols = np.array([1, 2, 0, 3, 4, 5, 0, 2, 1])
    g = sp.CooGraph(6, rows, cols)
    labels = torch.tensor([0, 1, 0, 1, 0, 1], device="cuda")
    x32 = torch.from_numpy(np.random.default_rng(7).normal(size=(6, 4)).astype(np.float32)).cuda()
    bundle = M.GraphBundle.build(g, numerics=numerics)
    model = M.Model(kind, np.random.default_rng(11), (4, 4, 2), in_store=8)
    xs = torch.zeros(6, 8, device="cuda")
    xs[:, :4] = x32

    def loss_value():
        with torch.no_grad():
            logits = model.forward(bundle, xs, "float32")
            return float(M.cross_entropy(logits, labels, 2))

    return bundle, model, xs, labels, loss_value


@pytest.mark.parametrize("numerics", ["fast", "reference"])
@pytest.mark.parametrize("kind", ["gcn", "gin", "gat"])
def test_criterion_6_gradcheck(cuda, kind, numerics):
    """float32 mode on 6 vertices: every parameter's analytic gradient within 2%
    of the central difference (elements with |numeric| > 1e-3)."""
    from paper_2411_01109_b200 import models as M

    bundle, model, xs, labels, loss_value = _grad_setup(kind, numerics)
    logits = model.forward(bundle, xs, "float32")
    M.cross_entropy(logits, labels, 2).backward()
    analytic = [p.grad32().clone() for p in model.params()]
    worst = 0.0
    for p, ana in zip(model.params(), analytic):
        flat = p.master.view(-1)
        for i in range(flat.numel()):
            orig = float(flat[i])
            flat[i] = orig + GRAD_EPS
            fp = loss_value()
            flat[i] = orig - GRAD_EPS
            fm = loss_value()
            flat[i] = orig
            num = (fp - fm) / (2 * GRAD_EPS)
            if abs(num) > GRAD_FLOOR:
                worst = max(worst, abs(float(ana.view(-1)[i]) - num) / abs(num))
    assert worst <= GRAD_REL_TOL, (kind, numerics, worst)
