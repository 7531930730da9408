"""CPU, world_size 2 over gloo: the row-partitioned execution path
(partition.py) -- split points, padded column remapping, feature / gradient /
edge-value all-to-alls, global loss and weight-gradient all-reduce -- gives the
same training step as one process.  The CUDA kernels are swapped for a host
implementation of the same row-owned semantics (HostOps below, test-only), so
this checks the exchange logic, not the kernels (those are the -m gpu tests)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O


class HostOps:
    """Row-owned host compute over one CsrView (fp64 accumulation, one rounding)."""

    @staticmethod
    def _rows(view):
        deg = view.offsets[1:] - view.offsets[:-1]
        return torch.repeat_interleave(torch.arange(view.n_rows), deg)

    @staticmethod
    def spmm(view, x, w, w_index, heads, scaling, fin, fout):
        xs = x.double()
        if fin is not None:
            xs = (x * fin[:, None]).to(x.dtype).double()
        rows = HostOps._rows(view)
        contrib = xs[view.cols.long()]
        if w is not None:
            idx = torch.arange(view.num_edges) if w_index is None else w_index.long()
            wt = w.reshape(w.shape[0], -1)[idx].double()
            f = x.shape[1]
            contrib = contrib * wt.repeat_interleave(f // heads, dim=1)
        s = torch.zeros((view.n_rows, x.shape[1]), dtype=torch.float64)
        s.index_add_(0, rows, contrib)
        if fout is None:
            return s.to(x.dtype)
        if scaling == "post":
            h = s.to(x.dtype)
            return torch.where(fout[:, None] > 0, h * fout[:, None], h)
        return (s * fout.double()[:, None]).to(x.dtype)


def _host_xent(logits, labels, n_active, denom, scale=1.0, grad_dtype=None):
    z = logits[:, :n_active].double()
    z = z - z.max(dim=1, keepdim=True).values
    ez = torch.exp(z)
    se = ez.sum(dim=1)
    nll = torch.log(se) - z.gather(1, labels[:, None])[:, 0]
    g = ez / se[:, None]
    g[torch.arange(z.shape[0]), labels] -= 1.0
    grad = torch.zeros(logits.shape, dtype=grad_dtype or logits.dtype)
    grad[:, :n_active] = ((g / denom).float() * scale).to(grad.dtype)
    return nll, grad


def _rows_of(view):
    deg = (view.offsets[1:] - view.offsets[:-1]).numpy()
    return np.repeat(np.arange(view.n_rows), deg)


def _host_sddmm(view, x_rows, y_cols, heads):
    out = O.sddmm(_rows_of(view), view.cols.numpy().astype(np.int64), x_rows.numpy(),
                  y_cols.numpy(), heads=heads)
    return torch.from_numpy(np.ascontiguousarray(out.reshape(view.num_edges, heads)))


def _host_attn(view, s_l, s_r, slope):
    rows, cols = _rows_of(view), view.cols.numpy().astype(np.int64)
    sl, sr = s_l.numpy(), s_r.numpy()
    e = np.stack([O.attention_scores(rows, cols, sl[:, h], sr[:, h]) for h in range(sl.shape[1])], 1)
    return torch.from_numpy(np.ascontiguousarray(O.leaky_relu(e, slope)))


def _host_softmax_fwd(view, e):
    return torch.from_numpy(O.edge_softmax_fwd(view.offsets.numpy(), e.numpy()))


def _host_softmax_bwd(view, alpha, g):
    return torch.from_numpy(O.edge_softmax_bwd(view.offsets.numpy(), alpha.numpy(), g.numpy()))


def _host_edge_sums(view, v, perm):
    v2 = v.reshape(v.shape[0], -1).double()
    if perm is not None:
        v2 = v2[perm.long()]
    out = torch.zeros((view.n_rows, v2.shape[1]), dtype=torch.float64)
    out.index_add_(0, torch.from_numpy(_rows_of(view)), v2[: view.num_edges])
    return out.to(v.dtype)


def _host_head_dots(z, a_l, a_r, heads):
    zh = z.view(z.shape[0], heads, -1).double()
    return ((zh * a_l.double()[None]).sum(-1).to(z.dtype),
            (zh * a_r.double()[None]).sum(-1).to(z.dtype))


def _host_head_dots_bwd(z, a_l, a_r, g_l, g_r, heads):
    n = z.shape[0]
    zh = z.view(n, heads, -1).double()
    gz = ((g_l.double()[:, :, None] * a_l.double()[None]).to(z.dtype)
          + (g_r.double()[:, :, None] * a_r.double()[None]).to(z.dtype)).reshape(n, -1)
    ga_l = (zh * g_l.double()[:, :, None]).sum(0).to(z.dtype)
    ga_r = (zh * g_r.double()[:, :, None]).sum(0).to(z.dtype)
    return gz, ga_l, ga_r


HostOps.head_dots_bwd = staticmethod(_host_head_dots_bwd)
HostOps.xent = staticmethod(_host_xent)
HostOps.sddmm = staticmethod(_host_sddmm)
HostOps.attn = staticmethod(_host_attn)
HostOps.softmax_fwd = staticmethod(_host_softmax_fwd)
HostOps.softmax_bwd = staticmethod(_host_softmax_bwd)
HostOps.edge_sums = staticmethod(_host_edge_sums)
HostOps.head_dots = staticmethod(_host_head_dots)
HostOps.scale = staticmethod(lambda x, s: (x.double() * s).to(x.dtype))
HostOps.row_scale = staticmethod(lambda x, s: (x.double() * s.double()[:, None]).to(x.dtype))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _graph():
    rng = np.random.default_rng(21)
    n = 120
    deg = np.minimum(rng.zipf(1.6, n), 90)
    rows = np.repeat(np.arange(n), deg)
    cols = rng.integers(0, n, rows.size)
    r, c = O.canonical_edges(n, rows, cols)
    x = rng.normal(size=(n, 10)).astype(np.float32)
    labels = (np.arange(n) * 3) // n
    return n, r, c, x, labels


class HostGraph:
    """The slice of DeviceGraph that DistTrainer uses, built on the host."""

    def __init__(self, n, r, c):
        self.n = n
        self.offsets = torch.from_numpy(O.csr_offsets(n, r))
        self.cols = torch.from_numpy(c.astype(np.int32))
        tr, tc, perm = O.transpose_perm(n, r, c)

        class _B:
            pass

        self.bwd = _B()
        self.bwd.offsets = torch.from_numpy(O.csr_offsets(n, tr))
        self.bwd.cols = torch.from_numpy(tc.astype(np.int32))
        self.bwd.perm = torch.from_numpy(perm.astype(np.int32))
        self._deg = {"row": np.diff(O.csr_offsets(n, r)), "col": np.bincount(c, minlength=n)}

    def factor(self, kind, side, dtype):
        np_dt = np.float16 if dtype == torch.float16 else np.float32
        f = O.degree_factor(self._deg[side], kind, np_dt).astype(np_dt)
        return torch.from_numpy(f)


def _run(rank, world, port, out_q, kind="gcn"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_01109_b200.models import TrainConfig
        from paper_2411_01109_b200.partition import DistTrainer

        n, r, c, x, labels = _graph()
        g = HostGraph(n, r, c)
        extra = {"heads": 2} if kind == "gat" else {}
        cfg = TrainConfig(kind=kind, mode="float32", hidden=8, device="cpu", seed=1, **extra)
        tr = DistTrainer(g, torch.from_numpy(x), labels, cfg, dist, ops=HostOps)
        losses = []
        first = None
        if kind == "gin":   # the static raw input was gathered once at load time
            g0 = tr.bundle.ex.gathers
            assert tr.bundle._gathered(tr.inner.x) is tr.bundle._static[1]
            assert tr.bundle.ex.gathers == g0
        ex = tr.bundle.ex
        b0 = ex.recv_bytes
        for _ in range(3):
            loss, logits = tr.step()
            losses.append(float(loss))
            first = logits.numpy() if first is None else first
        parts = [None] * world
        dist.all_gather_object(parts, (tr.part.lo, tr.part.hi, first, logits.numpy(),
                                       ex.recv_bytes - b0))
        if rank == 0:
            out_q.put((losses, parts, [p.master.numpy() for p in tr.inner.opt.params]))
    finally:
        dist.destroy_process_group()


def _run_world(world, kind="gcn"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run, args=(r, world, port, q, kind)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.timeout(400)
@pytest.mark.parametrize("kind,world", [("gcn", 2), ("gat", 2), ("gcn", 3)])
def test_multi_rank_step_matches_single_rank(kind, world):
    l1, parts1, w1 = _run_world(1, kind)
    l2, parts2, w2 = _run_world(world, kind)
    assert parts1[0][4] == 0            # one rank receives nothing
    assert all(p[4] > 0 for p in parts2)
    n = _graph()[0]
    # nnz-balanced split points (bit-exact rule)
    offsets = O.csr_offsets(n, _graph()[1])
    s = O.partition_splits(offsets, world)
    assert [(p[0], p[1]) for p in parts2] == [(int(s[q]), int(s[q + 1])) for q in range(world)]
    # step 1 (same weights): row-owned aggregation + global tables give
    # identical logits, rank by rank
    np.testing.assert_array_equal(parts1[0][2], np.concatenate([p[2] for p in parts2], axis=0))
    # later steps differ only through the all-reduce summation order of the grads
    np.testing.assert_allclose(parts1[0][3], np.concatenate([p[3] for p in parts2], axis=0),
                               rtol=1e-5, atol=1e-6)
    # loss / weight gradients are all-reduced sums: equal up to summation order
    np.testing.assert_allclose(l1, l2, rtol=1e-6, atol=1e-7)
    for a, b in zip(w1, w2):
        np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-6)


def test_static_input_gathered_once():
    """GIN's raw features are static: DistBundle reads the copy gathered at load
    time instead of gathering again every epoch."""
    from paper_2411_01109_b200.partition import DistBundle

    class _Ex:
        gathers = 0

        def gather_rows(self, x):
            self.gathers += 1
            return torch.cat([x, x])

    class _Part:
        rank, parts = 0, 1

    ex = _Ex()
    b = DistBundle(_Part(), ex, None)
    x = torch.ones(3, 4)
    full = ex.gather_rows(x)
    b.set_static(x, full)
    assert b._gathered(x) is full and ex.gathers == 1
    y = torch.ones(3, 4)
    assert b._gathered(y).shape == (6, 4) and ex.gathers == 2
    assert b._gathered(x[:2]) is not full           # a different view is not the input


def test_column_blocks_restore_rows():
    """partition.column_blocks (CPU tensors): block q holds each row's edges
    whose column rank q owns, rebased to s_q; concatenating the blocks' rows in
    q order restores every CSR row."""
    import numpy as np
    import torch

    from paper_2411_01109_b200.device import CsrView
    from paper_2411_01109_b200.partition import column_blocks, split_points

    rng = np.random.default_rng(3)
    n = 500
    deg = rng.integers(0, 40, n)
    rows = np.repeat(np.arange(n), deg)
    cols = rng.integers(0, n, rows.size)
    key = np.unique(rows * n + cols)
    rows, cols = key // n, key % n
    off = np.zeros(n + 1, np.int64)
    np.add.at(off, rows + 1, 1)
    off = np.cumsum(off)
    view = CsrView(torch.from_numpy(off), torch.from_numpy(cols.astype(np.int32)), n, n)
    for parts in (1, 2, 5):
        splits = split_points(torch.from_numpy(off), parts)
        blocks = column_blocks(view, splits)
        assert len(blocks) == parts
        assert sum(b.num_edges for b in blocks) == cols.size
        for q, b in enumerate(blocks):
            assert b.n_rows == n and b.n_cols == splits[q + 1] - splits[q]
            bc = b.cols.numpy()
            assert bc.size == 0 or (bc.min() >= 0 and bc.max() < b.n_cols)
        for r in range(n):
            cat = np.concatenate([blocks[q].cols.numpy()[int(blocks[q].offsets[r]):
                                                        int(blocks[q].offsets[r + 1])]
                                  + splits[q] for q in range(parts)])
            np.testing.assert_array_equal(cat, cols[off[r]:off[r + 1]])


def test_locality_order_permutation_and_rank_interleave():
    """device.locality_order (CPU tensors): a permutation, vertices by
    descending total degree (stable); with parts > 1 each part's contiguous
    id range holds every parts-th vertex of that order (hubs shared out)."""
    import torch

    from paper_2411_01109_b200.device import locality_order

    g = torch.Generator().manual_seed(0)
    n = 1003
    deg = torch.randint(0, 50, (n,), generator=g)
    off = torch.zeros(n + 1, dtype=torch.int64)
    off[1:] = torch.cumsum(deg, 0)
    tdeg = torch.randint(0, 50, (n,), generator=g)
    toff = torch.zeros(n + 1, dtype=torch.int64)
    toff[1:] = torch.cumsum(tdeg, 0)
    o1 = locality_order(off, toff)
    assert sorted(o1.tolist()) == list(range(n))
    tot = (deg + tdeg)[o1]
    assert bool((tot[:-1] >= tot[1:]).all())
    for parts in (2, 3, 8):
        op = locality_order(off, toff, parts=parts)
        assert sorted(op.tolist()) == list(range(n))
        pos = 0
        for p in range(parts):
            share = o1[p::parts]
            assert op[pos:pos + share.numel()].tolist() == share.tolist()
            pos += share.numel()
