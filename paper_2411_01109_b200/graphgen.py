"""Deterministic synthetic graphs of the BASELINE.json shapes.

C1/C2 use the reference's own SBM recipe (sparse.synth_sbm, sparse.py:269-298)
restated with the identical numpy RNG stream, so the graphs, features and
labels are the ones the reference trains on.  C3-C5 are generated on the GPU
(torch RNG, seeded) and canonicalised by the GPU CSR builder:

  C3 reddit_like     N=232,965  E=114,848,857  heavy-tailed (lognormal) row degrees
  C4 products_like   N=2,449,029, Chung-Lu power law, 61,859,140 undirected edges,
                     symmetrised (~123.7M directed nnz)
  C5 rmat            Graph500 RMAT (a,b,c)=(0.57,0.19,0.19), scale 24, edge factor 16
Labels for C3-C5 are planted classes with class-mean features.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from .device import DeviceGraph, build_csr

REDDIT_N, REDDIT_E = 232_965, 114_848_857
PRODUCTS_N, PRODUCTS_UNDIRECTED_E = 2_449_029, 61_859_140


def synth_sbm(n, classes, p_in, p_out, feat_dim, seed, chunk=1 << 24):
    """sparse.synth_sbm (sparse.py:269-298) with the same RNG consumption,
    evaluated in chunks of vertex pairs (bounded memory, identical stream).
    Returns (rows, cols) canonical int64, features float32 [n, feat_dim], labels."""
    if classes < 1 or n < classes:
        raise ValueError("need at least one vertex per class")
    if not (0.0 <= p_out <= p_in <= 1.0):
        raise ValueError("need 0 <= p_out <= p_in <= 1")
    rng = np.random.default_rng(seed)
    labels = (np.arange(n, dtype=np.int64) * classes) // n
    src_parts, dst_parts = [], []
    # pairs (i, j), i < j, in np.triu_indices order: row-major over i
    i = 0
    while i < n - 1:
        # rows [i, i2) hold at most `chunk` pairs
        i2 = i
        cnt = 0
        while i2 < n - 1 and cnt + (n - 1 - i2) <= chunk:
            cnt += n - 1 - i2
            i2 += 1
        if i2 == i:
            i2 = i + 1
            cnt = n - 1 - i
        lens = (n - 1 - np.arange(i, i2)).astype(np.int64)
        ii = np.repeat(np.arange(i, i2, dtype=np.int64), lens)
        starts = np.cumsum(lens) - lens
        jj = np.arange(cnt, dtype=np.int64) - np.repeat(starts, lens) + np.repeat(
            np.arange(i, i2, dtype=np.int64) + 1, lens)
        p = np.where(labels[ii] == labels[jj], p_in, p_out)
        keep = rng.random(cnt) < p
        src_parts.append(ii[keep])
        dst_parts.append(jj[keep])
        i = i2
    src = np.concatenate(src_parts) if src_parts else np.zeros(0, np.int64)
    dst = np.concatenate(dst_parts) if dst_parts else np.zeros(0, np.int64)
    keys = np.unique(np.concatenate([src * n + dst, dst * n + src]))
    rows, cols = keys // n, keys % n
    means = rng.normal(0.0, 1.0, size=(classes, feat_dim))
    norms = np.linalg.norm(means, axis=1, keepdims=True)
    means = means / np.where(norms == 0, 1.0, norms) * 4.0
    feats = means[labels] + rng.normal(0.0, 1.0, size=(n, feat_dim))
    return rows, cols, feats.astype(np.float32), labels


def cora_like(seed=0):
    """C1: synth_sbm(2708, 7, 0.0085, 0.00026, 1433, seed)."""
    return synth_sbm(2708, 7, 0.0085, 0.00026, 1433, seed)


def pubmed_like(seed=0):
    """C2: synth_sbm(19717, 3, 0.00057, 5.71e-5, 500, seed)."""
    return synth_sbm(19717, 3, 0.00057, 5.71e-5, 500, seed)


def _gen(seed, device):
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def _exact_degree_graph(n, deg, gen, device, max_rounds=8):
    """Rows with exactly deg[r] distinct uniform columns: draw, canonicalise on
    the GPU, top up each row's shortfall, repeat."""
    deg = deg.to(device)
    rows = torch.repeat_interleave(torch.arange(n, device=device), deg)
    cols = torch.randint(0, n, (rows.numel(),), generator=gen, device=device)
    for _ in range(max_rounds):
        offsets, c32, r64 = build_csr(n, rows, cols, want_rows=True)
        have = offsets[1:] - offsets[:-1]
        short = deg - have
        if int(short.sum().item()) == 0:
            return offsets, c32
        extra_r = torch.repeat_interleave(torch.arange(n, device=device), short.clamp_min(0))
        extra_c = torch.randint(0, n, (extra_r.numel(),), generator=gen, device=device)
        rows = torch.cat([r64, extra_r])
        cols = torch.cat([c32.to(torch.int64), extra_c])
        del offsets, c32, r64
    offsets, c32, _ = build_csr(n, rows, cols)
    return offsets, c32


def reddit_like(seed=0, device="cuda", n=REDDIT_N, e=REDDIT_E):
    """C3: lognormal row degrees (mean 493, clipped [1, 2e4]) rescaled
    to sum to E exactly, uniform columns, exactly E unique edges."""
    gen = _gen(seed, device)
    mean = e / n
    sigma = 1.0
    mu = math.log(mean) - sigma * sigma / 2
    raw = torch.empty(n, device=device, dtype=torch.float64).log_normal_(mu, sigma, generator=gen)
    raw = raw.clamp(1.0, 2.0e4)
    deg = torch.floor(raw * (e / raw.sum())).clamp(1, min(20000, n)).to(torch.int64)
    rem = e - int(deg.sum().item())
    # hand out the remainder one edge at a time to the rows with headroom
    while rem != 0:
        step = 1 if rem > 0 else -1
        room = (deg < min(20000, n)) if step > 0 else (deg > 1)
        idx = torch.nonzero(room).flatten()[: abs(rem)]
        deg[idx] += step
        rem -= step * idx.numel()
    offsets, cols = _exact_degree_graph(n, deg, gen, device)
    return DeviceGraph(n, offsets, cols)


def products_like(seed=0, device="cuda", n=PRODUCTS_N, undirected=PRODUCTS_UNDIRECTED_E,
                  exponent=2.1, max_degree=17_000):
    """C4: Chung-Lu power-law graph with exactly `undirected` distinct undirected
    edges (no self loops), symmetrised.  Expected degrees follow
    rank^(-1/(exponent-1)) scaled to the target mean and clipped to
    [1, max_degree] (ogbn-products' maximum degree is ~17K); endpoints are
    drawn proportionally, duplicates are topped up until the count is exact."""
    gen = _gen(seed, device)
    ranks = torch.arange(1, n + 1, device=device, dtype=torch.float64)
    w = ranks.pow(-1.0 / (exponent - 1.0))
    mean = 2.0 * undirected / n
    for _ in range(20):  # rescale so the clipped weights keep the target mean
        w = (w * (mean * n / w.clamp(1.0, max_degree).sum())).clamp(min=1e-9)
    w = w.clamp(1.0, max_degree)
    prob = (w / w.sum()).float()
    perm = torch.randperm(n, generator=gen, device=device)
    keys = torch.empty(0, dtype=torch.int64, device=device)
    need = undirected
    for _ in range(16):
        m = int(need * 1.15) + 1024
        a = perm[torch.multinomial(prob, m, replacement=True, generator=gen)]
        b = perm[torch.multinomial(prob, m, replacement=True, generator=gen)]
        keep = a != b
        lo, hi = torch.minimum(a, b)[keep], torch.maximum(a, b)[keep]
        keys = torch.unique(torch.cat([keys, lo * n + hi]))
        need = undirected - keys.numel()
        if need <= 0:
            break
    if keys.numel() > undirected:  # drop a random surplus
        pick = torch.randperm(keys.numel(), generator=gen, device=device)[:undirected]
        keys = keys[pick]
    src, dst = keys // n, keys % n
    offsets, c32, _ = build_csr(n, torch.cat([src, dst]), torch.cat([dst, src]))
    return DeviceGraph(n, offsets, c32)


def rmat(scale=24, edge_factor=16, seed=0, device="cuda", abc=(0.57, 0.19, 0.19)):
    """C5: Graph500 RMAT, deduplicated (self loops kept as generated)."""
    gen = _gen(seed, device)
    n = 1 << scale
    m = edge_factor * n
    a, b, c = abc
    rows = torch.zeros(m, dtype=torch.int64, device=device)
    cols = torch.zeros(m, dtype=torch.int64, device=device)
    for bit in range(scale):
        u = torch.rand(m, generator=gen, device=device)
        right = ((u >= a) & (u < a + b)) | (u >= a + b + c)
        down = u >= a + b
        rows |= down.to(torch.int64) << bit
        cols |= right.to(torch.int64) << bit
    offsets, c32, _ = build_csr(n, rows, cols)
    return DeviceGraph(n, offsets, c32)


def planted_features(n, feat, classes, seed=0, device="cuda", dtype=torch.float16):
    """Labels = contiguous class blocks; features = class mean (norm 4) + N(0,1)."""
    gen = _gen(seed + 1, device)
    labels = (torch.arange(n, device=device) * classes) // n
    means = torch.randn(classes, feat, generator=gen, device=device)
    means = means / means.norm(dim=1, keepdim=True).clamp_min(1e-12) * 4.0
    x = means[labels] + torch.randn(n, feat, generator=gen, device=device)
    return x.to(dtype), labels
