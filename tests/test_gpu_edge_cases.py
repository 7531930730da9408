"""GPU edge cases for the fast-path kernels: empty graphs, isolated rows, single
edges, minimal feature widths, degenerate GEMM shapes -- the boundary cases the
reference's own tests exercise for its operators (test_kernels.py:372-386,
test_sparse.py), applied to the kernels added for numerics="fast"."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import bits

pytestmark = pytest.mark.gpu


def _dg(n, rows, cols, dev):
    from paper_2411_01109_b200.device import DeviceGraph

    return DeviceGraph.from_edges(n, np.asarray(rows, np.int64), np.asarray(cols, np.int64),
                                  device=dev)


@pytest.mark.parametrize("n,edges", [(1, []), (5, []), (5, [(2, 3)]), (6, [(0, 0), (5, 5)])])
def test_fast_kernels_on_tiny_graphs(cuda, n, edges):
    from paper_2411_01109_b200 import device as D

    r = [e[0] for e in edges]
    c = [e[1] for e in edges]
    dg = _dg(n, r, c, cuda)
    x = torch.randn(n, 16, device=cuda, dtype=torch.float16)
    y = D.spmm(dg, x, None, "discretized", "both")
    want = torch.zeros(n, 16, dtype=torch.float64)
    deg_r = np.bincount(np.asarray(r, np.int64), minlength=n)
    deg_c = np.bincount(np.asarray(c, np.int64), minlength=n)
    for a, b in edges:
        want[a] += x[b].double().cpu() / np.sqrt(deg_c[b]) / np.sqrt(deg_r[a])
    assert torch.allclose(y.double().cpu(), want, atol=2e-2, rtol=1e-2)
    isolated = torch.from_numpy(deg_r == 0)
    assert bool((y.cpu()[isolated] == 0).all())
    # fast GAT attention: rows with edges sum to 1, isolated rows produce nothing
    sl = torch.randn(n, 4, device=cuda, dtype=torch.float16)
    sr = torch.randn(n, 4, device=cuda, dtype=torch.float16)
    alpha = D.gat_attention_fwd(dg.view(False), sl, sr)
    assert alpha.shape == (len(edges), 4)
    if edges:
        assert bool(((alpha.float() - 1).abs() < 1e-3).all())  # each row here has one edge
    g = torch.randn(len(edges), 4, device=cuda, dtype=torch.float16)
    de, dsl = D.gat_attention_bwd(dg.view(False), sl, sr, alpha, g)
    assert bool((de.float().abs() < 1e-3).all())  # single-edge softmax has zero gradient
    assert bool((dsl.float().abs() < 1e-3).all())
    bwd = dg.view(True)
    dsr = D.edge_sums_fast(bwd, de, bwd.perm)
    assert dsr.shape == (n, 4) and bool((dsr.float().abs() < 1e-3).all())
    s = D.sddmm(dg, x, x, heads=2, fast=True)
    assert s.shape == (len(edges), 2)


def test_gemm_tc_degenerate_shapes(cuda):
    from paper_2411_01109_b200 import device as D

    for m, k, n in [(0, 64, 16), (1, 8, 16), (3, 16, 32), (127, 72, 64), (129, 8, 256)]:
        a = torch.randn(m, k, device=cuda, dtype=torch.float16)
        bt = torch.randn(n, k, device=cuda, dtype=torch.float16)
        got = D.gemm_tc(a, bt)
        assert got.shape == (m, n)
        if m:
            want = (a.float() @ bt.float().t())
            assert torch.allclose(got.float(), want, atol=5e-2, rtol=1e-2)
    with pytest.raises(ValueError, match="multiple of 8"):
        D.gemm_tc(torch.randn(4, 8, device=cuda, dtype=torch.float16),
                  torch.randn(12, 8, device=cuda, dtype=torch.float16))


def test_softmax_xent_single_class_and_padding(cuda):
    from paper_2411_01109_b200 import device as D

    z = torch.randn(10, 8, device=cuda, dtype=torch.float16)
    lab = torch.zeros(10, dtype=torch.int64, device=cuda)
    nll, g = D.softmax_xent(z, lab, 1, 10)
    assert bool((nll.abs() < 1e-12).all())            # one active class: p = 1
    assert bool((g == 0).all())                          # no gradient, padding zeroed


def test_elementwise_helpers_empty(cuda):
    from paper_2411_01109_b200 import device as D

    e = torch.empty(0, device=cuda, dtype=torch.float16)
    one = torch.ones((), device=cuda, dtype=torch.float16)
    assert D.scale_combine(e, e, one, 0.1).numel() == 0
    gx, ga, gope = D.scale_combine_bwd(e, e, one, 0.1)
    assert gx.numel() == 0 and float(gope) == 0.0
    assert D.relu_grad(e, e).numel() == 0
    assert D.col_sums(torch.empty(0, 8, device=cuda, dtype=torch.float16)).tolist() == [0.0] * 8


def test_parse_edge_text_degenerate(cuda):
    from paper_2411_01109_b200.device import parse_edge_text

    for text, want in [(b"", []), (b"\n\n\r\n", []), (b"# x\n% y", []), (b"7 8", [(7, 8)]),
                       (b"  3\t4  \r", [(3, 4)]), (b"0 1\n" * 3, [(0, 1)] * 3)]:
        t = torch.frombuffer(bytearray(text), dtype=torch.uint8).to(cuda) if text else \
            torch.empty(0, dtype=torch.uint8, device=cuda)
        r, c, top = parse_edge_text(t)
        assert list(zip(r.tolist(), c.tolist())) == want
        assert top == (max(max(p) for p in want) if want else -1)
