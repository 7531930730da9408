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

from . import synth as S
from .device import DeviceGraph, build_csr

REDDIT_N, REDDIT_E = S.REDDIT_N, S.REDDIT_E
PRODUCTS_N, PRODUCTS_UNDIRECTED_E = S.PRODUCTS_N, S.PRODUCTS_UNDIRECTED_E


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


# ── counter-based draws on the device, bit-identical to synth.h (numpy) ──

def _s64(c):
    return c - (1 << 64) if c >= 1 << 63 else c


def _srl(z, k):
    """Logical right shift of int64 tensors holding uint64 bit patterns."""
    return (z >> k) & ((1 << (64 - k)) - 1)


def _h(seed, stream, idx):
    """synth.h(seed, stream, idx) on int64 tensors (wrapping arithmetic)."""
    z = idx + _s64(S.key_base(seed, stream))
    z = z ^ _srl(z, 30)
    z = z * _s64(S.MIX1)
    z = z ^ _srl(z, 27)
    z = z * _s64(S.MIX2)
    return z ^ _srl(z, 31)


def _mulhi32(hv, n):
    return (_srl(hv, 32) * n) >> 32


def _unit53(hv):
    return _srl(hv, 11).to(torch.float64) * (1.0 / (1 << 53))


def reddit_like(seed=0, device="cuda", n=REDDIT_N, e=REDDIT_E):
    """C3 (synth.reddit_rows): lognormal row degrees (host numpy,
    mean 493, clipped [1, 2e4], rescaled to sum to E), each row's columns the
    first deg distinct counter-based uniform draws; exactly E unique edges.
    Bit-identical to synth.reddit_graph."""
    deg = torch.from_numpy(S.reddit_degrees(seed, n, e)).to(device)
    ar = torch.arange(n, device=device)
    nxt = torch.zeros(n, dtype=torch.int64, device=device)
    need = deg
    rows = torch.zeros(0, dtype=torch.int64, device=device)
    cols = torch.zeros(0, dtype=torch.int64, device=device)
    while True:
        cnt = need.clamp_min(0)
        total = int(cnt.sum().item())
        if total == 0:
            break
        rid = torch.repeat_interleave(ar, cnt)
        start = torch.cumsum(cnt, 0) - cnt
        k = torch.arange(total, device=device) - start[rid] + nxt[rid]
        nxt = nxt + cnt
        c = _mulhi32(_h(seed, S.S_REDDIT, (rid << 32) | k), n)
        offsets, c32, r64 = build_csr(n, torch.cat([rows, rid]), torch.cat([cols, c]),
                                      want_rows=True)
        rows, cols = r64, c32.to(torch.int64)
        del rid, k, c
        need = deg - (offsets[1:] - offsets[:-1])
    return DeviceGraph(n, offsets, c32)


def products_like(seed=0, device="cuda", n=PRODUCTS_N, undirected=PRODUCTS_UNDIRECTED_E,
                  exponent=2.1, max_degree=17_000):
    """C4 (synth.products_graph): Chung-Lu power-law graph with exactly
    `undirected` distinct undirected edges (no self loops), symmetrised.
    Expected degrees follow rank^(-1/(exponent-1)) scaled to the target mean and
    clipped to [1, max_degree] (ogbn-products' maximum degree is ~17K);
    endpoints by inverse CDF of counter-based uniforms, vertex ids permuted;
    the first `undirected` distinct pairs in draw order are kept.
    Bit-identical to synth.products_graph."""
    cdf_h, total = S.products_cdf(n, undirected, exponent, max_degree)
    cdf = torch.from_numpy(cdf_h).to(device)
    perm = torch.from_numpy(S.products_perm(seed, n)).to(device)
    keys = torch.zeros(0, dtype=torch.int64, device=device)
    first = torch.zeros(0, dtype=torch.int64, device=device)
    t0 = 0
    while keys.numel() < undirected:
        m = S.products_batch(undirected - keys.numel())
        t = torch.arange(t0, t0 + m, device=device)
        ia = torch.searchsorted(cdf, _unit53(_h(seed, S.S_PROD_A, t)) * total, right=True)
        ib = torch.searchsorted(cdf, _unit53(_h(seed, S.S_PROD_B, t)) * total, right=True)
        a, b = perm[ia.clamp_max(n - 1)], perm[ib.clamp_max(n - 1)]
        del ia, ib
        ok = a != b
        k = torch.minimum(a, b)[ok] * n + torch.maximum(a, b)[ok]
        tt = t[ok]
        del a, b, ok, t
        allk, allt = torch.cat([keys, k]), torch.cat([first, tt])
        del k, tt
        sk, order = torch.sort(allk, stable=True)
        st = allt[order]
        del allk, allt, order
        head = torch.ones_like(sk, dtype=torch.bool)
        head[1:] = sk[1:] != sk[:-1]
        keys, first = sk[head], st[head]
        del sk, st, head
        t0 += m
    if keys.numel() > undirected:
        keep = torch.argsort(first)[:undirected].sort().values
        keys = keys[keep]
    src, dst = keys // n, keys % n
    del keys, first
    offsets, c32, _ = build_csr(n, torch.cat([src, dst]), torch.cat([dst, src]))
    return DeviceGraph(n, offsets, c32)


def rmat(scale=24, edge_factor=16, seed=0, device="cuda", abc=S.RMAT_ABC, scrambled=True):
    """C5: Graph500 RMAT, deduplicated (self loops kept as generated), vertex
    ids scrambled by a seeded bijection as Graph500 does (hubs spread over the
    id range, so row partitions balance).  Bit-identical to synth.rmat_graph."""
    n = 1 << scale
    m = edge_factor * n
    ta, tab, tabc = S.rmat_thresholds(abc)
    t = torch.arange(m, device=device)
    rows = torch.zeros(m, dtype=torch.int64, device=device)
    cols = torch.zeros(m, dtype=torch.int64, device=device)
    for bit in range(scale):
        u = _srl(_h(seed, S.S_RMAT + bit, t), 40)
        rows |= (u >= tab).to(torch.int64) << bit
        cols |= (((u >= ta) & (u < tab)) | (u >= tabc)).to(torch.int64) << bit
        del u
    del t
    if scrambled:
        rows, cols = _scramble(rows, seed, scale), _scramble(cols, seed, scale)
    offsets, c32, _ = build_csr(n, rows, cols)
    return DeviceGraph(n, offsets, c32)


def _scramble(v, seed, scale):
    """synth.scramble on the device."""
    mask = (1 << scale) - 1
    k1, k2, k3 = S.scramble_consts(seed, scale)
    s1, s2 = max(1, scale // 2), max(1, scale // 2 + 1)
    x = (v * k1) & mask
    x = x ^ (x >> s1)
    x = (x * k2) & mask
    x = x ^ (x >> s2)
    return x ^ k3


def planted_features(n, feat, classes, seed=0, device="cuda", dtype=torch.float16):
    """Labels = contiguous class blocks; features = class mean (norm 4) + N(0,1)."""
    gen = _gen(seed + 1, device)
    labels = (torch.arange(n, device=device) * classes) // n
    means = torch.randn(classes, feat, generator=gen, device=device)
    means = means / means.norm(dim=1, keepdim=True).clamp_min(1e-12) * 4.0
    x = means[labels] + torch.randn(n, feat, generator=gen, device=device)
    return x.to(dtype), labels
