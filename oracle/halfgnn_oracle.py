"""Numpy restatement of the halfsparse hot path -- TEST INFRASTRUCTURE ONLY.

Every function names the reference code it restates (paths relative to
/root/reference/pkg/src/halfsparse/).  Values are carried in float64 and
rounded to the mode dtype (float16 / float32) once per arithmetic step, the
reference's numeric convention (kernels.py:90-101, halfnum.py:152-168).
Vectorisation is our own: loops run over the position inside a warp chunk /
neighbour group / tree level, vectorised across warps, groups and rows.

Pinned against tests/golden/*.npz (produced by the real reference) in
tests/test_oracle_golden.py.
"""
from __future__ import annotations

import time

import numpy as np

F16, F32 = np.float16, np.float32
SCALINGS = ("post", "pre", "discretized")
NORMS = ("none", "left", "right", "both")


def rnd(a, dtype):
    """One round-to-nearest-even to `dtype`, result widened to float64."""
    with np.errstate(over="ignore", invalid="ignore"):
        return np.asarray(a, dtype=np.float64).astype(dtype).astype(np.float64)


# ── graph construction (sparse.py:56-140) ────────────────────────────────


def canonical_edges(n, rows, cols):
    """CooGraph.from_edges (sparse.py:56-69): sort by (row, col), drop duplicates."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    if rows.size == 0:
        return rows, cols
    if rows.min() < 0 or cols.min() < 0:
        raise ValueError("negative vertex id")
    if max(rows.max(), cols.max()) >= n:
        raise ValueError("vertex id out of range")
    keys = np.unique(rows * np.int64(n) + cols)
    return keys // n, keys % n


def load_edge_list_text(text: bytes, num_vertices=None, symmetrize_edges=False, where="<path>"):
    """sparse.load_edge_list (sparse.py:143-177) over the file's bytes: Python
    universal-newline lines, str.strip / str.split fields, int() ids, the same
    errors and messages.  Returns (n, rows, cols) canonical."""
    import io

    src, dst = [], []
    for lineno, line in enumerate(io.TextIOWrapper(io.BytesIO(text), newline=None), start=1):
        t = line.strip()
        if not t or t[0] in "#%":
            continue
        parts = t.split()
        if len(parts) < 2:
            raise ValueError(f"{where}:{lineno}: expected 'src dst'")
        try:
            a, b = int(parts[0]), int(parts[1])
        except ValueError as exc:
            raise ValueError(f"{where}:{lineno}: non-integer vertex id") from exc
        if a < 0 or b < 0:
            raise ValueError(f"{where}:{lineno}: negative vertex id")
        src.append(a)
        dst.append(b)
    rows = np.asarray(src, dtype=np.int64)
    cols = np.asarray(dst, dtype=np.int64)
    n = int(num_vertices) if num_vertices is not None else int(
        max(rows.max(initial=-1), cols.max(initial=-1)) + 1)
    if n <= 0:
        raise ValueError(f"{where}: empty graph and no vertex count given")
    if rows.size and max(rows.max(), cols.max()) >= n:
        bad = np.argmax((rows >= n) | (cols >= n))
        raise ValueError(f"{where}: vertex id out of range at edge {bad}")
    r, c = canonical_edges(n, rows, cols)
    if symmetrize_edges:
        r, c = symmetrize(n, r, c)
    return n, r, c


def csr_offsets(n, rows):
    """coo_to_csr (sparse.py:97-101): offsets = [0, cumsum(bincount(rows))]."""
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(np.asarray(rows, np.int64), minlength=n), out=off[1:])
    return off


def rows_from_offsets(offsets):
    """csr_to_coo (sparse.py:104-106)."""
    return np.repeat(np.arange(offsets.size - 1, dtype=np.int64), np.diff(offsets))


def transpose_perm(n, rows, cols):
    """transpose(g, return_perm=True) (sparse.py:109-120): stable argsort of col*n+row."""
    perm = np.argsort(np.asarray(cols, np.int64) * np.int64(n) + rows, kind="stable")
    return cols[perm], rows[perm], perm


def symmetrize(n, rows, cols):
    """sparse.py:136-140."""
    return canonical_edges(n, np.concatenate([rows, cols]), np.concatenate([cols, rows]))


def add_self_loops(n, rows, cols):
    """sparse.py:128-133."""
    v = np.arange(n, dtype=np.int64)
    return canonical_edges(n, np.concatenate([rows, v]), np.concatenate([cols, v]))


def degree_factor(deg, kind, dtype):
    """_degree_factors (kernels.py:118-140): fp32 1/d or 1/sqrt(d), 0 for d == 0,
    rounded once to the mode.  kind: 'inv' | 'inv_sqrt'."""
    d = np.asarray(deg).astype(np.float32)
    with np.errstate(divide="ignore"):
        inv = np.float32(1.0) / d if kind == "inv" else np.float32(1.0) / np.sqrt(d)
    inv = np.where(d > 0, inv, np.float32(0.0)).astype(np.float32)
    return rnd(inv, dtype)


def norm_factors(n, rows, cols, norm, dtype):
    """(in_scale, out_factor) of a Reduction norm (kernels.py:118-140)."""
    deg_r = np.bincount(rows, minlength=n)
    deg_c = np.bincount(cols, minlength=n)
    fin = fout = None
    if norm in ("left", "both"):
        fin = degree_factor(deg_c, "inv" if norm == "left" else "inv_sqrt", dtype)
    if norm in ("right", "both"):
        fout = degree_factor(deg_r, "inv" if norm == "right" else "inv_sqrt", dtype)
    return fin, fout


def check_reduction(scaling, norm):
    """Reduction.__post_init__ (kernels.py:61-67)."""
    if scaling not in SCALINGS:
        raise ValueError(f"unknown scaling {scaling!r}")
    if norm not in NORMS:
        raise ValueError(f"unknown norm {norm!r}")
    if scaling == "discretized" and norm == "none":
        raise ValueError("discretized scaling requires a degree norm")


def discretize_batch(feat):
    """simt.subwarp_layout(F).subwarps (simt.py:86-98): edges per warp iteration."""
    return 1 if feat > 64 else 32 // (feat // 2)


# ── adjacent-pair trees (kernels.py:252-262, 445-454; models.py:343-357) ──


def _aligned_tree(values, member, count, dtype):
    """Adjacent-pair tree with pass-through, evaluated as the implicit tree over
    power-of-two aligned ranges: at stride s, member m (m % 2s == 0) absorbs
    member m+s when it exists.  values: (K, F) rows grouped contiguously;
    member: position of each row inside its group; count: group size per row.
    Returns the updated array; each group's root sits at its member-0 row."""
    v = values.copy()
    s = 1
    cmax = int(count.max(initial=1))
    while s < cmax:
        idx = np.flatnonzero((member % (2 * s) == 0) & (member + s < count))
        if idx.size:
            v[idx] = rnd(v[idx] + v[idx + s], dtype)
        s *= 2
    return v


def row_tree_sum(vals, offsets, dtype):
    """_row_tree_sum (models.py:343-357) over CSR-ordered edge values (E,) or (E, H)."""
    vals = np.asarray(vals, dtype=np.float64)
    n = offsets.size - 1
    deg = np.diff(offsets)
    rows = rows_from_offsets(offsets)
    pos = np.arange(rows.size) - offsets[rows]
    squeeze = vals.ndim == 1
    v2 = vals.reshape(rows.size, -1)
    tree = _aligned_tree(v2, pos, deg[rows], dtype)
    out = np.zeros((n, v2.shape[1]))
    nz = deg > 0
    out[nz] = tree[offsets[:-1][nz]]
    return out[:, 0] if squeeze else out


# ── SpMM, edge-parallel reference order (kernels.py:328-401, 603-688) ────


def spmm_edge_parallel(n, rows, cols, x, w=None, warp_chunk=128, warps_per_cta=4,
                       scaling="post", norm="none", fin=None, fout=None, factors=True):
    """halfsparse.kernels.spmm_v / spmm_ve, bit-exact.

    rows/cols: canonical COO.  x: (n, F) float16/float32.  w: per-edge weights
    (same dtype) or None.  If factors is True, (fin, fout) are derived from the
    graph's degrees for `norm`; otherwise the given tables are used.
    Returns (y, carry_rows, carry_vals) -- the StagingBuffer of kernels.py:70-87.
    """
    check_reduction(scaling, norm)
    dtype = x.dtype.type
    feat = x.shape[1]
    e_cnt = rows.size
    if factors:
        fin, fout = norm_factors(n, rows, cols, norm, dtype)
    y = np.zeros((n, feat))
    if e_cnt == 0:
        return y.astype(dtype), np.zeros(0, np.int64), np.zeros((0, feat), dtype)
    xw = x.astype(np.float64)
    if fin is not None:
        xw = rnd(xw * fin[:, None], dtype)
    mult = np.ones(e_cnt) if w is None else np.asarray(w).astype(np.float64)
    if scaling == "pre" and fout is not None:
        mult = fout[rows] if w is None else rnd(mult * fout[rows], dtype)

    chunk, wpc = warp_chunk, warps_per_cta
    eid = np.arange(e_cnt)
    warp = eid // chunk
    start = np.ones(e_cnt, dtype=bool)
    start[1:] = (rows[1:] != rows[:-1]) | (warp[1:] != warp[:-1])
    seg_of = np.cumsum(start) - 1
    seg_start = np.flatnonzero(start)
    seg_len = np.diff(np.append(seg_start, e_cnt))
    seg_row = rows[seg_start]
    seg_cta = warp[seg_start] // wpc
    pos = eid - seg_start[seg_of]

    acc = np.zeros((seg_start.size, feat))
    disc = scaling == "discretized"
    if disc:
        kb = discretize_batch(feat)
        raw = np.zeros_like(acc)
        fo_seg = None if fout is None else fout[seg_row]
    for p in range(min(chunk, e_cnt)):
        e = np.arange(p, e_cnt, chunk)           # one edge per warp
        s = seg_of[e]
        contrib = mult[e][:, None] * xw[cols[e]]
        if disc:
            raw[s] = rnd(contrib + raw[s], dtype)
            closing = ((pos[e] + 1) % kb == 0) | (pos[e] + 1 == seg_len[s])
            cs = s[closing]
            if fo_seg is None:
                acc[cs] = rnd(raw[cs] + acc[cs], dtype)
            else:
                acc[cs] = rnd(raw[cs] * fo_seg[cs][:, None] + acc[cs], dtype)
            raw[cs] = 0.0
        else:
            acc[s] = rnd(contrib + acc[s], dtype)

    # chains: consecutive segments of one row inside one CTA
    brk = np.ones(seg_start.size, dtype=bool)
    brk[1:] = (seg_cta[1:] != seg_cta[:-1]) | (seg_row[1:] != seg_row[:-1])
    chain_of = np.cumsum(brk) - 1
    chain_first = np.flatnonzero(brk)
    chain_cnt = np.diff(np.append(chain_first, seg_start.size))
    member = np.arange(seg_start.size) - chain_first[chain_of]
    merged = _aligned_tree(acc, member, chain_cnt[chain_of], dtype)
    chain_val = merged[chain_first]
    chain_row = seg_row[chain_first]
    chain_cta = seg_cta[chain_first]
    is_carry = np.ones(chain_first.size, dtype=bool)
    is_carry[:-1] = chain_cta[1:] != chain_cta[:-1]
    y[chain_row[~is_carry]] = chain_val[~is_carry]
    carry_rows = chain_row[is_carry]
    carry_vals = chain_val[is_carry]
    # follow-up: fold carries into their rows in ascending CTA order
    first = np.ones(carry_rows.size, dtype=bool)
    first[1:] = carry_rows[1:] != carry_rows[:-1]
    rank = np.arange(carry_rows.size) - np.flatnonzero(first)[np.cumsum(first) - 1]
    for r in range(int(rank.max(initial=-1)) + 1):
        sel = rank == r
        y[carry_rows[sel]] = rnd(y[carry_rows[sel]] + carry_vals[sel], dtype)
    if scaling == "post" and fout is not None:
        sc = np.flatnonzero(fout > 0)
        y[sc] = rnd(y[sc] * fout[sc, None], dtype)
    with np.errstate(over="ignore"):
        return y.astype(dtype), carry_rows.astype(np.int64), carry_vals.astype(dtype)


# ── SpMM, vertex-grouped reference order (kernels.py:463-559, 709-740) ───


def spmm_vertex_grouped(n, offsets, cols, x, scaling="post", norm="none", group=32):
    """halfsparse.kernels.spmm_vertex_grouped, bit-exact.
    Returns (y, staging_rows, staging_partials)."""
    check_reduction(scaling, norm)
    dtype = x.dtype.type
    feat = x.shape[1]
    rows = rows_from_offsets(offsets)
    fin, fout = norm_factors(n, rows, cols, norm, dtype)
    xw = x.astype(np.float64)
    if fin is not None:
        xw = rnd(xw * fin[:, None], dtype)
    deg = np.diff(offsets)
    ngrp = -(-deg // group)
    g_row = np.repeat(np.arange(n, dtype=np.int64), ngrp)
    g_idx = np.arange(g_row.size) - np.repeat(np.cumsum(ngrp) - ngrp, ngrp)
    g_beg = offsets[g_row] + g_idx * group
    g_len = np.minimum(group, offsets[g_row + 1] - g_beg)
    m = np.ones(rows.size) if not (scaling == "pre" and fout is not None) else fout[rows]
    acc = np.zeros((g_row.size, feat))
    for p in range(group):
        live = np.flatnonzero(g_len > p)
        e = g_beg[live] + p
        acc[live] = rnd(m[e][:, None] * xw[cols[e]] + acc[live], dtype)
    part = acc
    if scaling == "discretized" and fout is not None:
        part = rnd(acc * fout[g_row][:, None], dtype)
    y = np.zeros((n, feat))
    y[g_row[g_idx == 0]] = part[g_idx == 0]
    for j in range(1, int(g_idx.max(initial=0)) + 1):
        sel = g_idx == j
        y[g_row[sel]] = rnd(y[g_row[sel]] + part[sel], dtype)
    if scaling == "post" and fout is not None:
        sc = np.flatnonzero(fout > 0)
        y[sc] = rnd(y[sc] * fout[sc, None], dtype)
    multi = ngrp[g_row] > 1
    with np.errstate(over="ignore"):
        return y.astype(dtype), g_row[multi], part[multi].astype(dtype)


def spmm_f64(n, rows, cols, x, w=None, fin=None, fout=None):
    """Float64 segment-sum oracle: fout * (A_w @ (fin * x)), no rounding
    (tests/oracles.py:105-135 computed sparsely)."""
    xw = np.asarray(x, np.float64)
    if fin is not None:
        xw = xw * np.asarray(fin, np.float64)[:, None]
    wt = np.ones(rows.size) if w is None else np.asarray(w, np.float64)
    y = np.zeros((n, xw.shape[1]))
    if rows.size:
        order = np.argsort(rows, kind="stable")
        contrib = wt[order][:, None] * xw[cols[order]]
        r = rows[order]
        starts = np.flatnonzero(np.r_[True, r[1:] != r[:-1]])
        y[r[starts]] = np.add.reduceat(contrib, starts, axis=0)
    if fout is not None:
        y = y * np.asarray(fout, np.float64)[:, None]
    return y


# ── SDDMM and attention (kernels.py:407-455; models.py:188-200, 317-412) ─


def sddmm(rows, cols, x, y, heads=1):
    """kernels.sddmm per head: products rounded, adjacent pair sums, aligned tree."""
    dtype = x.dtype.type
    feat = x.shape[1]
    fh = feat // heads
    out = np.zeros((rows.size, heads))
    for h in range(heads):
        xs = x[:, h * fh:(h + 1) * fh].astype(np.float64)
        ys = y[:, h * fh:(h + 1) * fh].astype(np.float64)
        prods = rnd(xs[rows] * ys[cols], dtype)
        v = rnd(prods[:, 0::2] + prods[:, 1::2], dtype)
        m = v.shape[1]
        s = 1
        while s < m:
            for i in range(0, m - s, 2 * s):
                v[:, i] = rnd(v[:, i] + v[:, i + s], dtype)
            s *= 2
        out[:, h] = v[:, 0]
    out = out.astype(dtype)
    return out[:, 0] if heads == 1 else out


def leaky_relu(x, slope=0.2):
    """models.leaky_relu forward (models.py:188-192)."""
    dtype = x.dtype.type
    lo = rnd(x.astype(np.float64) * slope, dtype).astype(dtype)
    return np.where(x > 0, x, lo)


def leaky_relu_bwd(x, g, slope=0.2):
    """models.py:194-197 (mask from the forward input)."""
    dtype = g.dtype.type
    return np.where(x > 0, g, rnd(g.astype(np.float64) * slope, dtype).astype(dtype))


def attention_scores(rows, cols, s_l, s_r):
    """models.attention_scores forward (F=2 SDDMM of [s_l|1].[1|s_r]): rnd(s_l[r]+s_r[c])."""
    dtype = s_l.dtype.type
    return rnd(s_l.astype(np.float64)[rows] + s_r.astype(np.float64)[cols], dtype).astype(dtype)


def edge_softmax_fwd(offsets, e):
    """models.edge_softmax forward (models.py:389-401); e: (E,) or (E, H)."""
    dtype = e.dtype.type
    n = offsets.size - 1
    rows = rows_from_offsets(offsets)
    e64 = e.astype(np.float64).reshape(rows.size, -1)
    m = np.full((n, e64.shape[1]), -np.inf)
    np.maximum.at(m, rows, e64)
    shifted = rnd(e64 - m[rows], dtype)
    with np.errstate(invalid="ignore"):
        ex = rnd(np.exp(shifted), dtype)
    den = row_tree_sum(ex, offsets, dtype).reshape(n, -1)
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        alpha = rnd(ex / den[rows], dtype)
    return alpha.astype(dtype).reshape(e.shape)


def edge_softmax_bwd(offsets, alpha, g):
    """models.edge_softmax backward (models.py:403-410)."""
    dtype = alpha.dtype.type
    rows = rows_from_offsets(offsets)
    a = alpha.astype(np.float64).reshape(rows.size, -1)
    g64 = g.astype(np.float64).reshape(rows.size, -1)
    prod = rnd(a * g64, dtype)
    s = row_tree_sum(prod, offsets, dtype).reshape(offsets.size - 1, -1)
    inner = rnd(g64 - s[rows], dtype)
    return rnd(a * inner, dtype).astype(dtype).reshape(alpha.shape)


# ── scheduler and partitioner restatements (build-specified integer maps) ─


def schedule_units(offsets, cap, pack_rows=0, pack_edges=0):
    """Restatement of hg_schedule_build (include/halfgnn.h): the degree-bucketed
    work units that replace simt.plan_edge_parallel / plan_vertex_grouped
    (simt.py:158-201) for the fp32-guarded kernels.  Returns (units (U,4) int32,
    split_rows (S,4) int32, num_slots), plus packs (P,4) int32 {first_row,
    begin, end, rows} when pack_rows > 0 (aligned blocks of pack_rows rows with
    at most pack_edges edges in total; their rows get no units)."""
    offsets = np.asarray(offsets, np.int64)
    n = offsets.size - 1
    deg = np.diff(offsets)
    nparts = np.where(deg == 0, 1, -(-deg // cap))
    packs = np.zeros((0, 4), np.int32)
    if pack_rows:
        nb = -(-n // pack_rows)
        r0 = np.arange(nb) * pack_rows
        blk = offsets[np.minimum(r0 + pack_rows, n)] - offsets[r0] <= pack_edges
        nparts = np.where(np.repeat(blk, pack_rows)[:n], 0, nparts)
        r0 = np.flatnonzero(blk) * pack_rows
        cnt = np.minimum(pack_rows, n - r0)
        packs = np.stack([r0, offsets[r0], offsets[r0 + cnt], cnt], axis=1).astype(np.int32)
    ubase = np.cumsum(nparts) - nparts
    row = np.repeat(np.arange(n, dtype=np.int64), nparts)
    part = np.arange(row.size) - ubase[row]
    beg = offsets[row] + part * cap
    end = np.minimum(beg + cap, offsets[row + 1])
    split = nparts > 1
    sparts = np.where(split, nparts, 0)
    sbase = np.cumsum(sparts) - sparts
    slot = np.where(split[row], sbase[row] + part, -1)
    length = end - beg
    cls = np.zeros(row.size, dtype=np.int64)
    nzl = length > 0
    cls[nzl] = np.floor(np.log2(length[nzl])).astype(np.int64) + 1
    order = np.argsort(32 - cls, kind="stable")
    units = np.stack([row, beg, end, slot], axis=1)[order].astype(np.int32)
    srows = np.flatnonzero(split)
    split_rows = np.stack([srows, sbase[srows], nparts[srows], np.zeros_like(srows)],
                          axis=1).astype(np.int32)
    if pack_rows:
        return units, split_rows.reshape(-1, 4), int(sparts.sum()), packs.reshape(-1, 4)
    return units, split_rows.reshape(-1, 4), int(sparts.sum())


def partition_splits(offsets, parts):
    """Row split points of the nnz-balanced P-way partition:
    s_0 = 0, s_P = N, s_p = searchsorted(offsets, (p*E)//P, 'left')."""
    offsets = np.asarray(offsets, np.int64)
    n, e = offsets.size - 1, int(offsets[-1])
    s = [0]
    for p in range(1, parts):
        s.append(int(np.searchsorted(offsets, (p * e) // parts, side="left")))
    s.append(n)
    return np.asarray(s, dtype=np.int64)


# ── training loop restatement (models.py:130-684) ─────────────────────────


def glorot(rng, fan_in, fan_out, shape=None):
    """models._glorot (models.py:436-438)."""
    lim = np.sqrt(6.0 / (fan_in + fan_out))
    return rng.uniform(-lim, lim, size=shape or (fan_in, fan_out)).astype(np.float32)


def init_params(kind, rng, dims, heads=1, layers=2):
    """Model.__init__ parameter draws (models.py:518-532), in RNG order.
    Multi-head / deeper GAT: one GATLayer per head per layer, drawn in
    (layer, head) order; a builder extension (the reference is 2 layers, 1 head)."""
    fan_in, hidden, n_cls = dims
    widths = [fan_in] + [hidden * (heads if kind == "gat" else 1)] * (layers - 1)
    outs = [hidden] * (layers - 1) + [n_cls]
    params = []
    for li in range(layers):
        fi, fo = widths[li], outs[li]
        if kind == "gcn":
            params.append({"w": glorot(rng, fi, fo), "b": np.zeros(fo, np.float32)})
        elif kind == "gin":
            params.append({"ope": np.float32(1.0),
                           "w1": glorot(rng, fi, fo), "b1": np.zeros(fo, np.float32),
                           "w2": glorot(rng, fo, fo), "b2": np.zeros(fo, np.float32)})
        elif kind == "gat":
            hp = []
            for _ in range(heads):
                hp.append({"w": glorot(rng, fi, fo), "a_l": glorot(rng, fo, 1),
                           "a_r": glorot(rng, fo, 1)})
            params.append(hp)
        else:
            raise ValueError(f"unknown model kind {kind!r}")
    return params


class OracleGraph:
    """GraphBundle.build (models.py:256-264) as plain arrays."""

    def __init__(self, n, rows, cols, warp_chunk=128, warps_per_cta=4):
        self.n, self.rows, self.cols = n, np.asarray(rows, np.int64), np.asarray(cols, np.int64)
        self.offsets = csr_offsets(n, self.rows)
        self.t_rows, self.t_cols, self.perm = transpose_perm(n, self.rows, self.cols)
        self.t_offsets = csr_offsets(n, self.t_rows)
        self.chunk, self.wpc = warp_chunk, warps_per_cta

    def spmm(self, x, w=None, scaling="post", norm="none", transpose=False):
        if transpose:
            return spmm_edge_parallel(self.n, self.t_rows, self.t_cols, x, w, self.chunk,
                                      self.wpc, scaling, norm)[0]
        return spmm_edge_parallel(self.n, self.rows, self.cols, x, w, self.chunk, self.wpc,
                                  scaling, norm)[0]


_MIRROR = {"none": "none", "left": "right", "right": "left", "both": "both"}


def _mm(a, b, dtype):
    """models.matmul (models.py:141-158): fp32 accumulate, one rounding."""
    with np.errstate(over="ignore", invalid="ignore"):
        return (a.astype(np.float32) @ b.astype(np.float32)).astype(dtype)


def _bias(x, b, dtype):
    return rnd(x.astype(np.float64) + b.astype(np.float64), dtype).astype(dtype)


def _bias_grad(g, dtype):
    return np.asarray(g.astype(np.float32).sum(axis=0)).astype(dtype)


def _acc(a, b):
    """Tape grad accumulation (models.py:107-109): a + b in the mode dtype."""
    if a is None:
        return b
    with np.errstate(over="ignore", invalid="ignore"):
        return a + b


class Timer:
    def __init__(self):
        self.sparse = 0.0
        self.dense = 0.0

    def run(self, cat, fn, *a, **k):
        t0 = time.perf_counter()
        out = fn(*a, **k)
        setattr(self, cat, getattr(self, cat) + time.perf_counter() - t0)
        return out


def train_epochs(graph, x, labels, kind="gcn", mode="half", epochs=1, hidden=16, lr=1e-2,
                 seed=0, scaling="discretized", norm="both", lam=0.1, heads=1, layers=2,
                 n_cls=None, val_fraction=0.2, timer=None):
    """Restatement of models.train (models.py:633-684) with the SURVEY 8(c)
    harness extensions: classes padded to even (n_cls = C + C % 2), multi-head
    GAT by per-head GATLayers (concat in hidden layers, mean at the output).
    Returns dict(losses, train_acc, val_acc, logits)."""
    dtype = F16 if mode == "half" else F32
    timer = timer or Timer()
    rng = np.random.default_rng(seed)
    n, fan_in = x.shape
    c = int(labels.max()) + 1
    n_cls = n_cls or c + c % 2
    params = init_params(kind, rng, (fan_in, hidden, n_cls), heads, layers)
    perm = rng.permutation(n)
    val = np.zeros(n, dtype=bool)
    val[perm[: int(n * val_fraction)]] = True
    train = ~val
    adam = [_AdamState(p) for p in _flat(params)]
    x_in = x.astype(np.float32).astype(dtype)
    losses = []
    logits32 = None
    for t in range(1, epochs + 1):
        pub = [rnd(p, dtype).astype(dtype) if mode == "half" else np.asarray(p, np.float32)
               for p in _flat(params)]
        logits, cache = _forward(kind, graph, x_in, _unflat(params, pub), dtype, scaling, norm,
                                 lam, heads, timer)
        logits32 = logits.astype(np.float32)
        z = logits32.astype(np.float64)
        z = z - z.max(axis=1, keepdims=True)
        sumexp = np.exp(z).sum(axis=1)
        p = np.exp(z) / sumexp[:, None]
        nll = np.log(sumexp) - z[np.arange(n), labels]
        loss = np.float32(nll.mean())
        if not np.isfinite(loss):
            raise FloatingPointError(f"loss is NaN at epoch {t - 1}")
        grad = p.copy()
        grad[np.arange(n), labels] -= 1.0
        g_logits = (grad / n).astype(np.float32).astype(dtype)
        grads = _backward(kind, graph, cache, g_logits, dtype, scaling, norm, lam, heads, timer)
        for st, g in zip(adam, _flat(grads)):
            st.step(np.asarray(g).astype(np.float32), lr, t)
        params = _unflat(params, [st.master for st in adam])
        losses.append(float(loss))
    pred = logits32.argmax(axis=1)
    return {"losses": losses, "train_acc": float((pred[train] == labels[train]).mean()),
            "val_acc": float((pred[val] == labels[val]).mean()) if val.any() else 0.0,
            "logits": logits32}


class _AdamState:
    """models.Adam (models.py:575-592) for one parameter."""

    def __init__(self, p):
        self.master = np.array(p, dtype=np.float32)
        self.m = np.zeros_like(self.master)
        self.v = np.zeros_like(self.master)

    def step(self, g, lr, t, b1=0.9, b2=0.999, eps=1e-8):
        self.m += (1 - b1) * (g - self.m)
        self.v += (1 - b2) * (g * g - self.v)
        mhat = self.m / (1 - b1**t)
        vhat = self.v / (1 - b2**t)
        self.master -= (lr * mhat / (np.sqrt(vhat) + eps)).astype(np.float32)


def _flat(params):
    out = []
    for layer in params:
        items = layer if isinstance(layer, list) else [layer]
        for d in items:
            out.extend(d[k] for k in sorted(d))
    return out


def _unflat(params, flat):
    it = iter(flat)
    res = []
    for layer in params:
        if isinstance(layer, list):
            res.append([{k: next(it) for k in sorted(d)} for d in layer])
        else:
            res.append({k: next(it) for k in sorted(layer)})
    return res


def _forward(kind, graph, x, params, dtype, scaling, norm, lam, heads, timer):
    cache = []
    h = x
    for li, p in enumerate(params):
        last = li == len(params) - 1
        c = {"x": h}
        if kind == "gcn":
            lin = timer.run("dense", _mm, h, p["w"], dtype)
            lin = _bias(lin, p["b"], dtype)
            out = timer.run("sparse", graph.spmm, lin, None, scaling, norm)
        elif kind == "gin":
            agg = timer.run("sparse", graph.spmm, h, None, scaling, "right")
            u = rnd(h.astype(np.float64) * float(p["ope"]), dtype)
            v = rnd(agg.astype(np.float64) * lam, dtype)
            mixed = rnd(u + v, dtype).astype(dtype)
            h1 = _bias(timer.run("dense", _mm, mixed, p["w1"], dtype), p["b1"], dtype)
            r1 = np.where(h1 > 0, h1, np.zeros_like(h1))
            out = _bias(timer.run("dense", _mm, r1, p["w2"], dtype), p["b2"], dtype)
            c.update(mixed=mixed, h1=h1, r1=r1)
        else:
            outs, hc = [], []
            for hp in p:
                z = timer.run("dense", _mm, h, hp["w"], dtype)
                s_l = _mm(z, hp["a_l"], dtype)
                s_r = _mm(z, hp["a_r"], dtype)
                e = timer.run("sparse", attention_scores, graph.rows, graph.cols, s_l[:, 0], s_r[:, 0])
                e2 = leaky_relu(e)
                alpha = timer.run("sparse", edge_softmax_fwd, graph.offsets, e2)
                o = timer.run("sparse", graph.spmm, z, alpha, "post", "none")
                outs.append(o)
                hc.append(dict(z=z, e=e, alpha=alpha))
            c["heads"] = hc
            if last and len(p) > 1:
                out = rnd(sum(o.astype(np.float64) for o in outs) / len(p), dtype).astype(dtype)
            elif last:
                out = outs[0]
            else:
                out = np.concatenate(outs, axis=1)
        c["out"] = out
        if not last:
            c["pre_relu"] = out
            out = np.where(out > 0, out, np.zeros_like(out))
        cache.append(c)
        h = out
    _attach_params(cache, params)
    return h, cache


def _backward(kind, graph, cache, g, dtype, scaling, norm, lam, heads, timer):
    grads = [None] * len(cache)
    ones2 = np.ones((graph.n, 2), dtype=dtype)
    for li in range(len(cache) - 1, -1, -1):
        c = cache[li]
        need_x = li > 0
        if li < len(cache) - 1:  # relu between layers
            g = np.where(c["pre_relu"] > 0, g, np.zeros_like(g))
        x = c["x"]
        if kind == "gcn":
            gl = timer.run("sparse", graph.spmm, g, None, scaling, _MIRROR[norm], True)
            gb = _bias_grad(gl, dtype)
            w = c["w"]
            gw = timer.run("dense", _mm, x.T, gl, dtype)
            gx = timer.run("dense", _mm, gl, w.T, dtype) if need_x else None
            grads[li] = {"b": gb, "w": gw}
        elif kind == "gin":
            gb2 = _bias_grad(g, dtype)
            gw2 = _mm(c["r1"].T, g, dtype)
            gr1 = _mm(g, c["w2"].T, dtype)
            gh1 = np.where(c["h1"] > 0, gr1, np.zeros_like(gr1))
            gb1 = _bias_grad(gh1, dtype)
            gw1 = _mm(c["mixed"].T, gh1, dtype)
            gm = _mm(gh1, c["w1"].T, dtype)
            g64 = gm.astype(np.float64)
            gx = None
            if need_x:
                gx = rnd(g64 * float(c["ope"]), dtype).astype(dtype)
            gagg = rnd(g64 * lam, dtype).astype(dtype)
            gope = rnd(np.float64((x.astype(np.float64) * g64).sum()), dtype).astype(dtype)
            if need_x:
                gx2 = timer.run("sparse", graph.spmm, gagg, None, scaling, "left", True)
                gx = _acc(gx, gx2)
            grads[li] = {"b1": gb1, "b2": gb2, "ope": gope, "w1": gw1, "w2": gw2}
        else:
            hs = c["heads"]
            nh = len(hs)
            last = li == len(cache) - 1
            fo = hs[0]["z"].shape[1]
            hg = []
            gx = None
            for hi, hc in enumerate(hs):
                if last and nh > 1:
                    go = rnd(g.astype(np.float64) / nh, dtype).astype(dtype)
                elif last:
                    go = g
                else:
                    go = np.ascontiguousarray(g[:, hi * fo:(hi + 1) * fo])
                z, alpha, e = hc["z"], hc["alpha"], hc["e"]
                hp = c["hp"][hi]
                g_alpha = timer.run("sparse", sddmm, graph.rows, graph.cols, go, z)
                gz = timer.run("sparse", graph.spmm, go, alpha[graph.perm], "post", "none", True)
                g_e2 = timer.run("sparse", edge_softmax_bwd, graph.offsets, alpha, g_alpha)
                g_e = leaky_relu_bwd(e, g_e2)
                gsl = graph.spmm(ones2, g_e, "post", "none")[:, :1]
                gsr = graph.spmm(ones2, g_e[graph.perm], "post", "none", True)[:, :1]
                gz = _acc(gz, _mm(gsr, hp["a_r"].T, dtype))
                g_ar = _mm(z.T, gsr, dtype)
                gz = _acc(gz, _mm(gsl, hp["a_l"].T, dtype))
                g_al = _mm(z.T, gsl, dtype)
                gw = timer.run("dense", _mm, x.T, gz, dtype)
                if need_x:
                    gx = _acc(gx, _mm(gz, hp["w"].T, dtype))
                hg.append({"a_l": g_al, "a_r": g_ar, "w": gw})
            grads[li] = hg
        g = gx
    return grads


def _attach_params(cache, params):
    for c, p in zip(cache, params):
        if isinstance(p, list):
            c["hp"] = p
        else:
            c.update({k: v for k, v in p.items()})
