"""Row-partitioned multi-GPU execution.

One process per GPU.  Rank p owns the contiguous vertex range [s_p, s_{p+1})
with s_p = searchsorted(offsets, (p*E)//P, 'left') (nnz-balanced, bit-exact
with oracle.partition_splits): its CSR rows (global column ids), the CSC rows
of the same vertices (for the backward pass), its feature rows and labels.

Exchange: before each aggregation the ranks' feature rows are all-gathered
with exact per-rank counts (NCCL over NVLink: one group of P broadcasts, the
all-gather-v idiom) into an [N, F] buffer in global row order, so the local
CSR keeps its global column ids and the SpMM reads the gathered buffer in
place; each rank receives exactly (N - n_local) * F * 2 bytes per gather, no
padding to the largest partition.  Backward all-gathers the output gradient
the same way and aggregates over the local CSC rows.  A static input (GIN's
first aggregation reads the raw features) is gathered once when it is loaded
(`DistTrainer.refresh_inputs`), not every epoch.  GAT additionally sends per-edge values (alpha, d_e) to the
owner of each edge's column with one all-to-all (each edge travels once,
E/P per rank instead of the E an all-gather would deliver).
Weight gradients and the loss are all-reduced (the data-parallel sum).

Comm/compute overlap (`overlap=True`, the default on CUDA): each
rank's CSR (and CSC) rows are also split into G column blocks, runs of
consecutive ranks' columns (`column_blocks`, G from the rows' degree:
`block_groups`).  An aggregation then receives the feature rows as P ordered
async NCCL broadcasts and runs block g as soon as its ranks' rows have landed,
carrying the rows' fp32 sums from block to block (hg_spmm_acc) and rounding
once after the last: the SpMM of the first blocks overlaps the transfer of
the later ones.  The blocks run in ascending
column order, so every row that is a single work unit in each block sums in
exactly the unblocked order (bitwise equal); split hub rows regroup their
fp32 carries (within the fast-path tolerance).
Degree-factor tables are global (computed once from the full graph), which
makes the concatenated rank outputs bit-identical to the 1-GPU result.

The compute callbacks default to the CUDA kernels; `ops=` lets the CPU/gloo
tests drive the same exchange logic with a host implementation.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

from . import device as D
from .device import CsrView


def split_points(offsets, parts: int) -> np.ndarray:
    """s_0 = 0, s_P = N, s_p = searchsorted(offsets, (p*E)//P, 'left')."""
    off = offsets if isinstance(offsets, torch.Tensor) else torch.as_tensor(offsets)
    n = off.numel() - 1
    e = int(off[-1])
    targets = torch.tensor([(p * e) // parts for p in range(1, parts)], dtype=off.dtype,
                           device=off.device)
    mid = torch.searchsorted(off, targets, right=False).cpu().numpy()
    return np.concatenate([[0], mid, [n]]).astype(np.int64)


def remap_to_padded(ids: torch.Tensor, splits: np.ndarray, stride: int) -> torch.Tensor:
    """(The round-1 padded all-gather layout; kept for the exchange-layout
    tests.)"""
    return _remap_to_padded(ids, splits, stride)


def _remap_to_padded(ids: torch.Tensor, splits: np.ndarray, stride: int) -> torch.Tensor:
    """Global id -> q*stride + (id - splits[q]) where q owns id."""
    bounds = torch.as_tensor(splits[1:-1], dtype=torch.int64, device=ids.device)
    ids64 = ids.to(torch.int64)
    q = torch.searchsorted(bounds, ids64, right=True)
    base = torch.as_tensor(splits[:-1], dtype=torch.int64, device=ids.device)[q]
    return (q * stride + (ids64 - base)).to(torch.int32)


@dataclass
class LocalPart:
    rank: int
    parts: int
    splits: np.ndarray        # vertex split points [P+1]
    edge_splits: np.ndarray   # CSR edge offsets of the split points [P+1]
    n_max: int                # rows of the largest partition (balance diagnostic)
    e_max: int                # largest per-rank edge count
    fwd: CsrView              # local CSR rows, global column ids
    bwd: CsrView              # local CSC rows, global column ids, perm -> received edge buffer
    send_index: torch.Tensor  # local CSR edges grouped by the rank owning their column
    send_counts: list         # edges sent to each rank
    recv_counts: list         # edges received from each rank (this rank's CSC edges)

    @property
    def lo(self):
        return int(self.splits[self.rank])

    @property
    def hi(self):
        return int(self.splits[self.rank + 1])

    @property
    def n_local(self):
        return self.hi - self.lo


def make_local_part(offsets, cols, t_offsets, t_cols, perm, rank, parts) -> LocalPart:
    """Slice rank `rank`'s CSR/CSC rows out of the global arrays (column ids
    stay global: the gathered buffers are in global row order)."""
    splits = split_points(offsets, parts)
    eoff = offsets[torch.as_tensor(splits, device=offsets.device)].cpu().numpy()
    n_max = int(np.diff(splits).max())
    e_max = int(np.diff(eoff).max()) if parts > 0 else 0
    lo, hi = int(splits[rank]), int(splits[rank + 1])
    f_off = (offsets[lo:hi + 1] - offsets[lo]).contiguous()
    n = int(splits[-1])
    # fresh allocations (not views at an edge offset): the kernels vector-load
    # column ids from 16-byte-aligned bases
    f_cols = cols[int(offsets[lo]):int(offsets[hi])].clone()
    t_lo, t_hi = int(t_offsets[lo]), int(t_offsets[hi])
    b_off = (t_offsets[lo:hi + 1] - t_offsets[lo]).contiguous()
    b_cols = t_cols[t_lo:t_hi].clone()
    # Edge values for the column owner travel by all-to-all (SURVEY 8(e)
    # option A): rank q sends rank p the values of its edges whose column p
    # owns, in ascending global edge id; concatenated over q that is p's CSC
    # edges sorted by global edge id, and recv_pos maps each CSC slot into it.
    dev = offsets.device
    g_ids = perm[t_lo:t_hi].to(torch.int64)
    order = torch.argsort(g_ids, stable=True)
    sorted_g = g_ids[order]
    eoff_t = torch.as_tensor(eoff, dtype=torch.int64, device=dev)
    bounds = torch.searchsorted(sorted_g, eoff_t, right=False)
    recv_counts = (bounds[1:] - bounds[:-1]).cpu().tolist()
    recv_pos = torch.empty_like(order)
    recv_pos[order] = torch.arange(order.numel(), device=dev)
    my_cols = cols[int(offsets[lo]):int(offsets[hi])].to(torch.int64)
    owner = torch.searchsorted(torch.as_tensor(splits[1:-1], dtype=torch.int64, device=dev),
                               my_cols, right=True)
    send_index = torch.argsort(owner, stable=True)
    send_counts = torch.bincount(owner, minlength=parts).cpu().tolist()
    fwd = CsrView(f_off, f_cols, hi - lo, n)
    bwd = CsrView(b_off, b_cols, hi - lo, n, perm=recv_pos.to(torch.int32))
    return LocalPart(rank, parts, splits, eoff, n_max, e_max, fwd, bwd, send_index,
                     send_counts, recv_counts)


def block_bounds(splits: np.ndarray, groups: int) -> np.ndarray:
    """Column-block boundaries: `groups` runs of consecutive ranks (as equal in
    rank count as possible), given as vertex ids (a subset of the splits)."""
    parts = len(splits) - 1
    g = max(1, min(groups, parts))
    idx = np.round(np.linspace(0, parts, g + 1)).astype(np.int64)
    return np.asarray(splits)[idx]


def block_groups(view: CsrView, parts: int) -> int:
    """Column blocks worth running for a rank's rows: each block re-reads and
    re-writes the rows' fp32 sums and walks every row once (C5 rank 0 at P = 8,
    F = 128: 1.57 ms unblocked, +0.77 ms per extra block), so blocks pay only
    while they keep ~4 edges per row.  Measured per-block SpMM times with the
    transfer modelled at 900 GB/s (tools/overlap_timeline.py, profiles/r02):
    C5 (15.6 edges per row) 5.61 ms serial -> 5.17 ms at 4 blocks, 7.20 ms at 8."""
    deg = view.num_edges / max(1, view.n_rows)
    return max(1, min(parts, int(deg // 4)))


def column_blocks(view: CsrView, splits: np.ndarray) -> list:
    """Split a CSR whose rows hold sorted global column ids into CSRs by column
    range: block q keeps, row by row and in order, the edges with a column in
    [splits[q], splits[q+1]) (a rank's range, or a run of ranks'), column ids
    rebased to splits[q] (they index that range of the gathered rows).
    Concatenating the blocks' rows in q order gives back each original row."""
    off, cols = view.offsets, view.cols
    dev = cols.device
    n, e = view.n_rows, cols.numel()
    parts = len(splits) - 1
    c64 = cols.to(torch.int64)
    owner = torch.searchsorted(torch.as_tensor(splits[1:-1], dtype=torch.int64, device=dev), c64,
                               right=True)
    rows = torch.repeat_interleave(torch.arange(n, device=dev), (off[1:] - off[:-1]).to(torch.int64),
                                   output_size=e)
    counts = torch.bincount(owner * n + rows, minlength=parts * n).view(parts, n)
    order = torch.argsort(owner, stable=True)          # grouped by owner, CSR order inside
    per_block = counts.sum(1).cpu().tolist()
    out, start = [], 0
    for q in range(parts):
        seg = order[start:start + per_block[q]]
        start += per_block[q]
        o_q = torch.zeros(n + 1, dtype=off.dtype, device=dev)
        o_q[1:] = torch.cumsum(counts[q], 0)
        c_q = (c64[seg] - int(splits[q])).to(torch.int32).clone()
        # perm: block slot -> edge of the unblocked view (edge weights follow it)
        out.append(CsrView(o_q, c_q, n, int(splits[q + 1] - splits[q]),
                           perm=seg.to(torch.int32).clone()))
    return out


class Exchange:
    """Exact-count all-gathers over a torch.distributed process group.  NCCL
    moves device tensors over NVLink (all_gather into per-rank views of
    different sizes = one NCCL group of broadcasts); a gloo group (CPU tests,
    or several ranks sharing one GPU for validation) stages through the host,
    padding to the largest partition there only.  `recv_bytes` counts the
    bytes this rank received (feature rows and edge values)."""

    def __init__(self, dist, part: LocalPart):
        self.dist = dist
        self.part = part
        self.staged = dist.get_backend() == "gloo"
        self.recv_bytes = 0
        self.gathers = 0

    def _views(self, out):
        s = self.part.splits
        return [out[int(s[q]):int(s[q + 1])] for q in range(self.part.parts)]

    def gather_rows(self, x_local: torch.Tensor) -> torch.Tensor:
        """[n_local, ...] -> [N, ...] in global row order."""
        p = self.part
        x_local = x_local.contiguous()
        tail = tuple(x_local.shape[1:])
        n = int(p.splits[-1])
        out = x_local.new_empty((n,) + tail)
        row = x_local[0].numel() * x_local.element_size() if x_local.shape[0] else 0
        self.recv_bytes += (n - p.n_local) * row
        self.gathers += 1
        if self.staged:
            send = x_local.new_zeros((p.n_max,) + tail, device="cpu")
            send[: p.n_local] = x_local.cpu()
            host = send.new_empty((p.parts * p.n_max,) + tail)
            self.dist.all_gather_into_tensor(host, send)
            for q, v in enumerate(self._views(out)):
                v.copy_(host[q * p.n_max: q * p.n_max + v.shape[0]])
        else:
            self.dist.all_gather(self._views(out), x_local)
        return out

    def gather_async(self, x_local: torch.Tensor):
        """(full, waits): the all-gathered [N, ...] rows in global order, filled
        by P async NCCL broadcasts issued in rank order on the process group's
        stream (this rank's rows copied in place); waits[q]() makes the current
        stream wait until ranks 0..q have landed, so an aggregation over the
        rows already there overlaps the transfer of the rest.  gloo: one staged
        all-gather, no waits."""
        p = self.part
        x_local = x_local.contiguous()
        if self.staged:
            return self.gather_rows(x_local), [None] * p.parts
        tail = tuple(x_local.shape[1:])
        row = x_local[0].numel() * x_local.element_size() if x_local.shape[0] else 0
        n = int(p.splits[-1])
        self.recv_bytes += (n - p.n_local) * row
        self.gathers += 1
        full = x_local.new_empty((n,) + tail)
        views = self._views(full)
        views[p.rank].copy_(x_local)
        waits = []
        for q in range(p.parts):
            work = self.dist.broadcast(views[q], src=q, async_op=True)
            waits.append(None if q == p.rank else work.wait)
        return full, waits

    def gather_edges(self, v_local: torch.Tensor) -> torch.Tensor:
        """Per-edge values ([E_local, ...], CSR order) -> the values of this
        rank's CSC edges in received order (index with part.bwd.perm): one
        all-to-all, each edge sent once to its column's owner."""
        p = self.part
        send = v_local.index_select(0, p.send_index).contiguous()
        out = v_local.new_empty((sum(p.recv_counts),) + tuple(v_local.shape[1:]))
        row = v_local[0].numel() * v_local.element_size() if v_local.shape[0] else 0
        self.recv_bytes += (sum(p.recv_counts) - p.recv_counts[p.rank]) * row
        if self.staged and out.is_cuda:
            host = out.cpu()
            self.dist.all_to_all_single(host, send.cpu(), p.recv_counts, p.send_counts)
            out.copy_(host)
        else:
            self.dist.all_to_all_single(out, send, p.recv_counts, p.send_counts)
        return out

    def all_reduce_(self, t: torch.Tensor, op=None) -> torch.Tensor:
        kw = {} if op is None else {"op": op}
        if self.staged and t.is_cuda:
            host = t.cpu()
            self.dist.all_reduce(host, **kw)
            t.copy_(host)
        else:
            self.dist.all_reduce(t, **kw)
        return t


class CudaOps:
    """Compute callbacks on one rank's views (the B200 kernels)."""

    @staticmethod
    def spmm(view, x, w, w_index, heads, scaling, fin, fout):
        return D.spmm_csr(view, x, w, w_index, heads, scaling, fin, fout)

    @staticmethod
    def sddmm(view, x_rows, y_cols, heads):
        sched = view.schedule()
        out = torch.empty((view.num_edges, heads), dtype=x_rows.dtype, device=x_rows.device)
        D.nat.call("hg_sddmm", D._p(view.offsets), D._p(view.cols), view.n_rows,
                   view.num_edges, D._p(sched.units), sched.num_units, D._p(x_rows),
                   D._p(y_cols), D._p(out), x_rows.shape[1], heads, D._dtype_code(x_rows),
                   D._stream())
        return out

    @staticmethod
    def attn(view, s_l, s_r, slope):
        heads = s_l.shape[1]
        out = torch.empty((view.num_edges, heads), dtype=s_l.dtype, device=s_l.device)
        D.nat.call("hg_attn_scores", D._p(view.offsets), D._p(view.cols), view.n_rows,
                   view.num_edges, D._p(s_l), D._p(s_r), heads, float(slope), D._p(out),
                   D._dtype_code(s_l), D._stream())
        return out

    @staticmethod
    def softmax_fwd(view, e):
        return D.softmax_fwd_view(view, e)

    @staticmethod
    def softmax_bwd(view, alpha, g):
        return D.softmax_bwd_view(view, alpha, g)

    @staticmethod
    def row_scale(x, s):
        return D.bias_scale_rows(x, None, s)

    @staticmethod
    def xent(logits, labels, n_active, denom, scale=1.0, grad_dtype=None):
        return D.softmax_xent(logits, labels, n_active, denom, scale, grad_dtype)

    @staticmethod
    def head_dots(z, a_l, a_r, heads):
        return D.head_dots(z, a_l, a_r, heads)

    @staticmethod
    def scale(x, s):
        return D.scale_f64(x, s)

    @staticmethod
    def edge_sums(view, v, perm):
        return D.rowsum_view(view, v, perm)

    @staticmethod
    def head_dots_bwd(z, a_l, a_r, g_l, g_r, heads):
        return D.head_dots_bwd(z, a_l, a_r, g_l, g_r, heads)


class DistBundle:
    """GraphBundle interface over one rank's partition: inputs and outputs are
    the rank's local rows (or local edges); exchanges happen inside."""

    numerics = "fast"

    def __init__(self, part: LocalPart, exchange: Exchange, tables, ops=CudaOps, overlap=None):
        self.part = part
        self.ex = exchange
        self.ops = ops
        self._tables = tables  # callable (kind, side, dtype) -> global table [N]
        self._cache = {}
        self._static = None    # (local input tensor, its gathered [N, F] copy)
        # column-blocked, transfer-overlapped unweighted aggregation (CUDA ops, P > 1)
        if overlap is None:
            env = os.environ.get("HG_DIST_OVERLAP", "1")
            # "force": the blocked path even for one part (a one-rank NCCL group
            # then exercises the async-broadcast exchange, e.g. under graph capture)
            overlap = "force" if env == "force" else env != "0"
        self.overlap = (bool(overlap) and ops is CudaOps
                        and (part.parts > 1 or overlap == "force"))
        self._blocks = {}

    def blocks(self, transpose):
        """(bounds, column blocks) of the local CSR (forward) or CSC (backward):
        block_groups() runs of consecutive ranks' columns."""
        b = self._blocks.get(transpose)
        if b is None:
            view = self.part.bwd if transpose else self.part.fwd
            bounds = block_bounds(self.part.splits, block_groups(view, self.part.parts))
            b = (bounds, column_blocks(view, bounds))
            self._blocks[transpose] = b
        return b

    def _block_windex(self, transpose, via_perm):
        """Per block: the row of the weight array each block edge reads -- the
        unblocked edge (block perm) or, for weights received in CSC order, that
        edge's slot in the receive buffer (view.perm after the block perm)."""
        key = ("widx", transpose, via_perm)
        w = self._blocks.get(key)
        if w is None:
            view = self.part.bwd if transpose else self.part.fwd
            w = [(view.perm.long()[b.perm.long()].to(torch.int32).clone() if via_perm
                  else b.perm) for b in self.blocks(transpose)[1]]
            self._blocks[key] = w
        return w

    def _blocked_agg(self, xs_local, scaling, fout, transpose, full=None, w=None,
                     via_perm=False, heads=1):
        """Aggregation of the gathered rows block by block: block q as soon as
        slab q has landed, rows' fp32 sums carried from block to block
        (hg_spmm_acc), rounded (scaling, out factor) after the last.  Edge
        weights (GAT's alpha) follow each block edge to its unblocked slot."""
        bounds, blocks = self.blocks(transpose)
        widx = self._block_windex(transpose, via_perm) if w is not None else None
        waits = [None] * self.part.parts
        if full is None:          # (a static input was gathered earlier)
            full, waits = self.ex.gather_async(xs_local)
        f = full.shape[1]
        n = self.part.n_local
        acc = torch.empty((n, f), dtype=torch.float32, device=full.device) if len(blocks) > 1 \
            else None
        splits = [int(v) for v in self.part.splits]
        out = None
        last = len(blocks) - 1
        for q, view in enumerate(blocks):
            lo, hi = int(bounds[q]), int(bounds[q + 1])
            for r in range(splits.index(lo), splits.index(hi)):   # the block's ranks landed
                if waits[r] is not None:
                    waits[r]()
            out = D.spmm_csr_acc(view, full[lo:hi], acc_in=None if q == 0 else acc,
                                 acc_out=None if q == last else acc, scaling=scaling,
                                 fout=fout if q == last else None, w=w,
                                 w_index=None if widx is None else widx[q], heads=heads)
        return out

    def set_static(self, x_local, x_full):
        """Register a gathered copy of a static input (GIN's raw features):
        aggregations of x_local read x_full instead of gathering again."""
        self._static = (x_local, x_full)

    def _gathered(self, x):
        st = self._static
        if st is not None and x.data_ptr() == st[0].data_ptr() and x.shape == st[0].shape:
            return st[1]
        return self.ex.gather_rows(x.contiguous())

    @property
    def n(self):
        return self.part.n_local

    @property
    def num_edges(self):
        return self.part.fwd.num_edges

    def norm_tables(self, norm, transpose, dtype):
        key = (norm, transpose, dtype)
        t = self._cache.get(key)
        if t is None:
            kind = "inv_sqrt" if norm == "both" else "inv"
            row_side, col_side = ("col", "row") if transpose else ("row", "col")
            fin = self._tables(kind, col_side, dtype) if norm in ("left", "both") else None
            fout = self._tables(kind, row_side, dtype)[self.part.lo:self.part.hi].contiguous() \
                if norm in ("right", "both") else None
            t = (fin, fout)
            self._cache[key] = t
        return t

    def local_in_scale(self, norm, transpose, dtype):
        """The left-norm input scale of this rank's own rows (global table)."""
        if norm not in ("left", "both"):
            return None
        key = ("fin_local", norm, transpose, dtype)
        t = self._cache.get(key)
        if t is None:
            kind = "inv_sqrt" if norm == "both" else "inv"
            side = "row" if transpose else "col"
            t = self._tables(kind, side, dtype)[self.part.lo:self.part.hi].contiguous()
            self._cache[key] = t
        return t

    @property
    def fused_bias_agg(self):
        """GCN layers run the tcgen05 GEMM + epilogue on local rows (CUDA ops only)."""
        return self.ops is CudaOps

    def _gather_scaled(self, xs, scaling, norm, transpose, heads=1, w=None, widx=None):
        view = self.part.bwd if transpose else self.part.fwd
        _, fout = self.norm_tables(norm, transpose, xs.dtype)
        if self.overlap and w is None and xs.shape[1] % 4 == 0:
            return self._blocked_agg(xs, scaling, fout, transpose)
        return self.ops.spmm(view, self.ex.gather_rows(xs.contiguous()), w, widx, heads,
                             scaling, None, fout)

    @property
    def fused_gat(self):
        """GAT layers use the fp32-guarded fused attention (CUDA ops only)."""
        return self.ops is CudaOps

    def gat_attention(self, s_l, s_r, slope):
        """Row-owned fused attention over the local rows; the column scores s_r
        are all-gathered (N x H, small)."""
        return D.gat_attention_fwd(self.part.fwd, s_l.contiguous(),
                                   self.ex.gather_rows(s_r.contiguous()), slope)

    def gat_attention_bwd(self, s_l, s_r, alpha, g, slope):
        """(ds_l, ds_r): row sums locally; the column owner sums d_e over its CSC
        rows after the all-to-all that sends each edge value to its column's
        owner."""
        de, ds_l = D.gat_attention_bwd(self.part.fwd, s_l.contiguous(),
                                       self.ex.gather_rows(s_r.contiguous()), alpha, g, slope)
        bwd = self.part.bwd
        ds_r = D.edge_sums_fast(bwd, self.ex.gather_edges(de), bwd.perm)
        return ds_l, ds_r

    def bias_spmm(self, h, b, scaling, norm):
        """spmm(add_bias(h, b)): bias and input scale applied to the local rows
        before the all-gather (hg_bias_scale_rows), then the gathered SpMM."""
        xs = D.bias_scale_rows(h, b, self.local_in_scale(norm, False, h.dtype))
        return self._gather_scaled(xs, scaling, norm, False)

    def gcn_agg_tc(self, x, w, b, reduction):
        """GCN layer forward: tcgen05 GEMM + bias + input scale on the local rows,
        all-gather of the scaled rows, SpMM over the local CSR rows."""
        fin = self.local_in_scale(reduction.norm, False, x.dtype)
        wt = getattr(w, "_hg_t", None)   # ParamGroup's transposed published copy
        xs = D.gemm_tc(x, wt if wt is not None else w.t().contiguous(), b, fin)
        return self._gather_scaled(xs, reduction.scaling, reduction.norm, False)

    def spmm(self, x, w=None, scaling="post", norm="none", transpose=False, heads=1,
             weight_via_perm=False):
        view = self.part.bwd if transpose else self.part.fwd
        fin_local = self.local_in_scale(norm, transpose, x.dtype)
        row_scale = getattr(self.ops, "row_scale", None)
        if fin_local is not None and row_scale is not None:
            # X' = rnd(X * in_scale) on the local rows before the gather (the
            # same elementwise rounding hg_spmm applies, done once per row
            # instead of on every rank's gathered copy)
            widx = None
            if w is not None and weight_via_perm:
                w = self.ex.gather_edges(w.contiguous())
                widx = view.perm
            return self._gather_scaled(row_scale(x.contiguous(), fin_local), scaling, norm,
                                       transpose, heads, w, widx)
        fin, fout = self.norm_tables(norm, transpose, x.dtype)
        if self.overlap and fin is None and x.shape[1] % 4 == 0:
            st = self._static
            static = (st[1] if st is not None and x.data_ptr() == st[0].data_ptr()
                      and x.shape == st[0].shape else None)
            if w is not None:
                w = self.ex.gather_edges(w.contiguous()) if weight_via_perm else w.contiguous()
            return self._blocked_agg(x, scaling, fout, transpose, full=static, w=w,
                                     via_perm=weight_via_perm, heads=heads)
        x_full = self._gathered(x)
        widx = None
        if w is not None and weight_via_perm:
            w = self.ex.gather_edges(w.contiguous())
            widx = view.perm
        return self.ops.spmm(view, x_full, w, widx, heads, scaling, fin, fout)

    def sddmm(self, x, y, heads=1):
        out = self.ops.sddmm(self.part.fwd, x.contiguous(), self.ex.gather_rows(y.contiguous()),
                             heads)
        return out[:, 0] if heads == 1 else out

    def attn_logits(self, s_l, s_r, slope):
        return self.ops.attn(self.part.fwd, s_l.contiguous(),
                             self.ex.gather_rows(s_r.contiguous()), slope)

    def head_dots(self, z, a_l, a_r, heads):
        return self.ops.head_dots(z, a_l, a_r, heads)

    def scale(self, x, s):
        return self.ops.scale(x, s)

    def head_dots_bwd(self, z, a_l, a_r, g_l, g_r, heads):
        return self.ops.head_dots_bwd(z, a_l, a_r, g_l, g_r, heads)

    def softmax_fwd(self, e):
        return self.ops.softmax_fwd(self.part.fwd, e.contiguous())

    def softmax_bwd(self, alpha, g):
        return self.ops.softmax_bwd(self.part.fwd, alpha, g)

    def edge_sums(self, v, transpose=False):
        v = v.contiguous()
        if not transpose:
            return self.ops.edge_sums(self.part.fwd, v, None)
        return self.ops.edge_sums(self.part.bwd, self.ex.gather_edges(v), self.part.bwd.perm)


class DistTrainer:
    """Trainer over a row partition: same model init, masks and optimiser as
    the 1-GPU Trainer (identical RNG stream); the loss is the global mean, the
    weight gradients are all-reduced before Adam."""

    def __init__(self, dg: D.DeviceGraph, features, labels, config, dist, ops=CudaOps,
                 node_order=None):
        from .models import Trainer

        self.dist = dist
        rank, parts = dist.get_rank(), dist.get_world_size()
        part = make_local_part(dg.offsets, dg.cols, dg.bwd.offsets, dg.bwd.cols, dg.bwd.perm,
                               rank, parts)
        self.part = part
        self.bundle = DistBundle(part, Exchange(dist, part),
                                 lambda k, side, dt: dg.factor(k, side, dt), ops)
        self.inner = Trainer(self.bundle, features, labels, config, row_slice=(part.lo, part.hi),
                             node_order=node_order)
        self.n_total = dg.n
        self._graph = None
        self._graph_out = None
        self.refresh_inputs()

    @property
    def x(self):
        return self.inner.x

    def refresh_inputs(self):
        """Gather the static input once (after features are loaded or replaced):
        GIN's first aggregation reads the raw features, which do not change
        between epochs; other models need nothing."""
        if self.inner.cfg.kind == "gin":
            self.bundle.set_static(self.inner.x, self.bundle.ex.gather_rows(self.inner.x))

    def load_features(self, feats, out=None):
        lo, hi = self.part.lo, self.part.hi
        out = self.inner.load_features(feats[lo:hi], out=self.inner.x)
        self.refresh_inputs()
        return out

    def step(self, overflow=None):
        if self._graph is not None and overflow is None:
            self._graph.replay()
            return self._graph_out
        return self._step_eager(overflow)

    def capture(self):
        """Record one step -- exchanges (NCCL all-gathers / all-reduces) included
        -- as a CUDA graph; later step() calls replay it.  Call after an eager
        step.  Needs an NCCL group (gloo's host staging cannot be captured)."""
        if self.dist.get_backend() != "nccl":
            raise RuntimeError("graph capture of the partitioned step needs the NCCL backend")
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            out = self._step_eager()
        self._graph, self._graph_out = graph, out
        return graph

    def _step_eager(self, overflow=None):
        tr = self.inner
        cfg = tr.cfg
        tr.group.publish_if_stale()
        logits = tr.model.forward(self.bundle, tr.x, cfg.mode, cfg.width, overflow)
        loss = tr.loss_backward(logits, self.bundle.ops.xent, self.n_total)
        if not tr.group.check_grads():
            raise RuntimeError("autograd did not accumulate into the flat gradient buffer")
        # data-parallel sum of the weight gradients: one fp32 all-reduce of the
        # group's flat gradient buffer
        flat = tr.group.grad.to(torch.float32)
        self.bundle.ex.all_reduce_(flat)
        tr.opt.step(flat_grad=flat)
        total = loss.detach().clone()
        self.bundle.ex.all_reduce_(total)
        return total, logits.detach()
