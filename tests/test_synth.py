"""CPU: the counter-based workload generators.  graphgen.py's device recipe
(torch int64 ops) run on CPU tensors, with the GPU CSR builder replaced by its
numpy definition, reproduces synth.py's host graphs bit for bit; row subsets
reproduce the full graph's rows; RMAT scrambling is a bijection that balances
nnz-partitioned row counts."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2411_01109_b200 import graphgen as G
from paper_2411_01109_b200 import synth as S


class _HostGraph:
    def __init__(self, n, offsets, cols):
        self.n, self.offsets, self.cols = n, offsets, cols


def _build_csr_cpu(n, rows, cols, want_rows=False):
    off, c = S.csr_from_pairs(n, rows.numpy(), cols.numpy())
    r = np.repeat(np.arange(n), np.diff(off))
    return (torch.from_numpy(off), torch.from_numpy(c.astype(np.int32)),
            torch.from_numpy(r) if want_rows else None)


@pytest.fixture
def cpu_graphgen(monkeypatch):
    monkeypatch.setattr(G, "build_csr", _build_csr_cpu)
    monkeypatch.setattr(G, "DeviceGraph", _HostGraph)
    return G


def test_hash_device_recipe_matches_host():
    idx = torch.arange(0, 1 << 20, dtype=torch.int64) * 104729 + (1 << 40)
    got = G._h(7, 3, idx).numpy().view(np.uint64)
    want = S.h(7, 3, idx.numpy().astype(np.uint64))
    assert np.array_equal(got, want)
    assert np.array_equal(G._mulhi32(G._h(7, 3, idx), 232965).numpy(),
                          S.mulhi32(want, 232965))
    assert np.array_equal(G._unit53(G._h(7, 3, idx)).numpy(), S.unit53(want))


def test_reddit_device_recipe_equals_host(cpu_graphgen):
    n, e = 3000, 150_000
    g = cpu_graphgen.reddit_like(seed=2, device="cpu", n=n, e=e)
    off, cols = S.reddit_graph(seed=2, n=n, e=e)
    assert np.array_equal(g.offsets.numpy(), off)
    assert np.array_equal(g.cols.numpy().astype(np.int64), cols)
    assert off[-1] == e
    assert np.array_equal(np.diff(off), S.reddit_degrees(2, n, e))
    # any subset of rows reproduces those rows exactly
    rows = S.sample_row_panels(off, 20_000, panels=8, seed=5)
    so, sc = S.reddit_rows(rows, S.reddit_degrees(2, n, e), seed=2, n=n)
    want = np.concatenate([cols[off[r]:off[r + 1]] for r in rows])
    assert np.array_equal(sc, want)
    assert np.array_equal(np.diff(so), np.diff(off)[rows])


def test_products_device_recipe_equals_host(cpu_graphgen):
    n, u = 20_000, 90_000
    g = cpu_graphgen.products_like(seed=1, device="cpu", n=n, undirected=u, max_degree=2000)
    off, cols = S.products_graph(seed=1, n=n, undirected=u, max_degree=2000)
    assert off[-1] == 2 * u
    assert np.array_equal(g.offsets.numpy(), off)
    assert np.array_equal(g.cols.numpy().astype(np.int64), cols)
    # symmetric, no self loops
    r = np.repeat(np.arange(n), np.diff(off))
    assert not np.any(r == cols)
    assert np.array_equal(np.sort(r * n + cols), np.sort(cols * n + r))


def test_rmat_device_recipe_equals_host(cpu_graphgen):
    g = cpu_graphgen.rmat(scale=12, edge_factor=8, seed=3, device="cpu")
    off, cols = S.rmat_graph(scale=12, edge_factor=8, seed=3)
    assert np.array_equal(g.offsets.numpy(), off)
    assert np.array_equal(g.cols.numpy().astype(np.int64), cols)


def test_scramble_is_a_bijection():
    for scale in (1, 5, 12, 20):
        v = np.arange(1 << scale, dtype=np.int64)
        s = S.scramble(v, 11, scale)
        assert np.array_equal(np.sort(s), v)
        assert np.array_equal(G._scramble(torch.from_numpy(v), 11, scale).numpy(), s)


def test_rmat_scrambled_partitions_balance_rows():
    """Graph500 scrambling spreads the hubs: on a scale-18 RMAT the nnz-balanced
    split at P=8 (SURVEY 8(e) rule) gives near-equal row counts, so an
    exact-count feature all-gather is not inflated."""
    import oracle as O

    off, _ = S.rmat_graph(scale=18, edge_factor=16, seed=0)
    n = off.size - 1
    for p in (2, 4, 8):
        s = O.partition_splits(off, p)
        sizes = np.diff(s)
        assert p * sizes.max() / n <= 1.1, (p, sizes)
    off_u, _ = S.rmat_graph(scale=18, edge_factor=16, seed=0, scrambled=False)
    s = O.partition_splits(off_u, 8)
    assert 8 * np.diff(s).max() / n > 2.0   # what the unscrambled ids did
