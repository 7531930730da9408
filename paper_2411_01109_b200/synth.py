"""Counter-based synthetic workloads, defined so that the host
(numpy) and the device (torch int64 on CUDA, graphgen.py) produce the SAME
graph bit for bit.

Every random draw is `h(seed, stream, index)`, a splitmix64 finalizer of a
64-bit counter, so any subset of rows can be regenerated on its own: the
CPU reference arm of bench.py rebuilds exactly the sampled rows of the graph
the B200 arm trains on, without the GPU or libhalfgnn.so, and the GPU tests
compare the device-built CSR of the full benched graphs with a numpy build.

Pure numpy: importing this module loads no native code.

  reddit   C3: lognormal row degrees (numpy RNG on the host, both sides),
           row r's columns = the first deg[r] distinct values of
           col(r, k) = mulhi32(h(seed, REDDIT, r<<32 | k), n), k = 0, 1, ...
  products C4: Chung-Lu: endpoints by inverse CDF of host-computed float64
           weights, u = (h >> 11) * 2^-53; the first U distinct undirected
           pairs (a != b) in draw order; symmetrised
  rmat     C5: Graph500 RMAT, one 24-bit uniform per (edge, level), integer
           thresholds, vertex ids scrambled by a seeded bijection on `scale` bits
"""
from __future__ import annotations

import math

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
SEED_MUL = 0xD1B54A32D192ED03
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB

# stream ids (one per independent draw sequence)
S_REDDIT = 1
S_PROD_A, S_PROD_B = 2, 3
S_RMAT = 16          # + level (0 .. scale-1)
S_SCRAMBLE = 15

REDDIT_N, REDDIT_E = 232_965, 114_848_857
PRODUCTS_N, PRODUCTS_UNDIRECTED_E = 2_449_029, 61_859_140
RMAT_ABC = (0.57, 0.19, 0.19)


def key_base(seed: int, stream: int) -> int:
    """The counter offset of (seed, stream): h(seed, stream, i) = mix64(base + i)."""
    return (seed * SEED_MUL + stream * GOLDEN) & M64


def mix64(z: np.ndarray) -> np.ndarray:
    """splitmix64 finalizer over uint64 (wrapping arithmetic)."""
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= np.uint64(MIX1)
        z ^= z >> np.uint64(27)
        z *= np.uint64(MIX2)
        z ^= z >> np.uint64(31)
    return z


def h(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        return mix64(np.asarray(idx).astype(np.uint64) + np.uint64(key_base(seed, stream)))


def mulhi32(hv: np.ndarray, n: int) -> np.ndarray:
    """floor((hv >> 32) * n / 2^32): a value in [0, n)."""
    return (((hv >> np.uint64(32)) * np.uint64(n)) >> np.uint64(32)).astype(np.int64)


def unit53(hv: np.ndarray) -> np.ndarray:
    return (hv >> np.uint64(11)).astype(np.float64) * (1.0 / (1 << 53))


# ───────────────────────────── C3: Reddit-shaped ─────────────────────────────


def reddit_degrees(seed=0, n=REDDIT_N, e=REDDIT_E, dmax=20_000) -> np.ndarray:
    """Lognormal row degrees (mean e/n, sigma 1) clipped to [1, dmax] and
    rescaled to sum to e exactly; the remainder goes one edge at a time to the
    lowest-numbered rows with headroom."""
    rng = np.random.default_rng(seed)
    sigma = 1.0
    mu = math.log(e / n) - sigma * sigma / 2
    raw = np.clip(rng.lognormal(mu, sigma, n), 1.0, 2.0e4)
    cap = min(dmax, n)
    deg = np.clip(np.floor(raw * (e / raw.sum())), 1, cap).astype(np.int64)
    rem = e - int(deg.sum())
    while rem != 0:
        step = 1 if rem > 0 else -1
        room = np.nonzero(deg < cap if step > 0 else deg > 1)[0][: abs(rem)]
        deg[room] += step
        rem -= step * room.size
    return deg


def reddit_rows(rows: np.ndarray, deg: np.ndarray, seed=0, n=REDDIT_N):
    """CSR (offsets, cols) of the given rows (ascending) of the C3 graph: each
    row's first deg distinct draws, sorted.  Rows are independent, so any
    subset reproduces those rows of the full graph exactly."""
    rows = np.asarray(rows, dtype=np.int64)
    want = deg[rows]
    nxt = np.zeros(rows.size, dtype=np.int64)   # next draw index per row
    have_r = np.zeros(0, np.int64)
    have_c = np.zeros(0, np.int64)
    need = want.copy()
    while True:
        cnt = need
        if int(cnt.sum()) == 0:
            break
        rid = np.repeat(np.arange(rows.size, dtype=np.int64), cnt)
        k = np.arange(rid.size, dtype=np.int64) - np.repeat(np.cumsum(cnt) - cnt, cnt) + nxt[rid]
        nxt += cnt
        c = mulhi32(h(seed, S_REDDIT, (rows[rid].astype(np.uint64) << np.uint64(32))
                      | k.astype(np.uint64)), n)
        keys = sorted_unique(np.concatenate([have_r * n + have_c, rid * n + c]))
        have_r, have_c = keys // n, keys % n
        need = want - np.bincount(have_r, minlength=rows.size)
    offsets = np.zeros(rows.size + 1, dtype=np.int64)
    np.cumsum(np.bincount(have_r, minlength=rows.size), out=offsets[1:])
    return offsets, have_c


def reddit_graph(seed=0, n=REDDIT_N, e=REDDIT_E):
    """The whole C3 CSR on the host (about 30 s and 5 GB at full size)."""
    deg = reddit_degrees(seed, n, e)
    return reddit_rows(np.arange(n), deg, seed, n)


# ───────────────────────────── C4: products-shaped ───────────────────────────


def products_cdf(n=PRODUCTS_N, undirected=PRODUCTS_UNDIRECTED_E, exponent=2.1,
                 max_degree=17_000):
    """Chung-Lu expected degrees rank^(-1/(exponent-1)) rescaled to the target
    mean and clipped to [1, max_degree]: (cumulative weights float64, total)."""
    ranks = np.arange(1, n + 1, dtype=np.float64)
    w = ranks ** (-1.0 / (exponent - 1.0))
    mean = 2.0 * undirected / n
    for _ in range(20):
        w = np.maximum(w * (mean * n / np.clip(w, 1.0, max_degree).sum()), 1e-9)
    w = np.clip(w, 1.0, max_degree)
    cdf = np.cumsum(w)
    return cdf, float(cdf[-1])


def products_perm(seed=0, n=PRODUCTS_N):
    return np.random.default_rng(seed).permutation(n).astype(np.int64)


def products_draws(t0, m, cdf, total, perm, seed=0):
    """Endpoints (a, b) of draws t0 .. t0+m-1."""
    t = np.arange(t0, t0 + m, dtype=np.uint64)
    n = perm.size
    ia = np.minimum(np.searchsorted(cdf, unit53(h(seed, S_PROD_A, t)) * total, side="right"), n - 1)
    ib = np.minimum(np.searchsorted(cdf, unit53(h(seed, S_PROD_B, t)) * total, side="right"), n - 1)
    return perm[ia], perm[ib]


def products_batch(need):
    return int(need * 1.15) + 1024


def products_graph(seed=0, n=PRODUCTS_N, undirected=PRODUCTS_UNDIRECTED_E, **kw):
    """The C4 CSR on the host: the first `undirected` distinct pairs in draw
    order, symmetrised."""
    cdf, total = products_cdf(n, undirected, **kw)
    perm = products_perm(seed, n)
    keys = np.zeros(0, np.int64)
    first = np.zeros(0, np.int64)
    t0 = 0
    while keys.size < undirected:
        m = products_batch(undirected - keys.size)
        a, b = products_draws(t0, m, cdf, total, perm, seed)
        ok = a != b
        k = np.minimum(a, b)[ok] * n + np.maximum(a, b)[ok]
        t = np.arange(t0, t0 + m, dtype=np.int64)[ok]
        allk = np.concatenate([keys, k])
        allt = np.concatenate([first, t])
        order = np.argsort(allk, kind="stable")
        sk = allk[order]
        head = np.ones(sk.size, dtype=bool)
        head[1:] = sk[1:] != sk[:-1]
        keys, first = sk[head], allt[order][head]
        t0 += m
    if keys.size > undirected:
        keep = np.sort(np.argsort(first, kind="stable")[:undirected])
        keys = keys[keep]
    src, dst = keys // n, keys % n
    return csr_from_pairs(n, np.concatenate([src, dst]), np.concatenate([dst, src]))


# ───────────────────────────────── C5: RMAT ──────────────────────────────────


def rmat_thresholds(abc=RMAT_ABC):
    a, b, c = abc
    ta = int(round(a * (1 << 24)))
    tab = int(round((a + b) * (1 << 24)))
    tabc = int(round((a + b + c) * (1 << 24)))
    return ta, tab, tabc


def scramble_consts(seed, scale):
    mask = (1 << scale) - 1
    x = int(h(seed, S_SCRAMBLE, np.arange(3, dtype=np.uint64))[0])
    y = int(h(seed, S_SCRAMBLE, np.arange(3, dtype=np.uint64))[1])
    z = int(h(seed, S_SCRAMBLE, np.arange(3, dtype=np.uint64))[2])
    return (x | 1) & mask, (y | 1) & mask, z & mask


def scramble(v: np.ndarray, seed: int, scale: int) -> np.ndarray:
    """A seeded bijection on [0, 2^scale) (Graph500 vertex scrambling):
    odd multiplies mod 2^scale, xor-shifts and an xor, all invertible."""
    mask = np.uint64((1 << scale) - 1)
    k1, k2, k3 = (np.uint64(c) for c in scramble_consts(seed, scale))
    s1, s2 = np.uint64(max(1, scale // 2)), np.uint64(max(1, scale // 2 + 1))
    x = v.astype(np.uint64)
    with np.errstate(over="ignore"):
        x = (x * k1) & mask
        x ^= x >> s1
        x = (x * k2) & mask
        x ^= x >> s2
        x ^= k3
    return x.astype(np.int64)


def rmat_edges(t0, m, scale=24, seed=0, abc=RMAT_ABC, scrambled=True):
    """(rows, cols) of generated edges t0 .. t0+m-1 (before dedup)."""
    ta, tab, tabc = rmat_thresholds(abc)
    t = np.arange(t0, t0 + m, dtype=np.uint64)
    rows = np.zeros(m, np.int64)
    cols = np.zeros(m, np.int64)
    for bit in range(scale):
        u = (h(seed, S_RMAT + bit, t) >> np.uint64(40)).astype(np.int64)
        right = ((u >= ta) & (u < tab)) | (u >= tabc)
        down = u >= tab
        rows |= down.astype(np.int64) << bit
        cols |= right.astype(np.int64) << bit
    if scrambled:
        rows, cols = scramble(rows, seed, scale), scramble(cols, seed, scale)
    return rows, cols


def rmat_graph(scale=24, edge_factor=16, seed=0, abc=RMAT_ABC, scrambled=True):
    n = 1 << scale
    r, c = rmat_edges(0, edge_factor * n, scale, seed, abc, scrambled)
    return csr_from_pairs(n, r, c)


# ───────────────────────────────── helpers ───────────────────────────────────


def sorted_unique(keys):
    """np.unique of int64 keys by sort + run heads (numpy 2's hash-based
    np.unique is ~30x slower at 1e7+ keys)."""
    k = np.sort(keys)
    if k.size:
        k = k[np.concatenate([[True], k[1:] != k[:-1]])]
    return k


def csr_from_pairs(n, rows, cols):
    """Canonical CSR (sorted, unique) of an edge list: the CooGraph.from_edges
    rule (reference sparse.py:56-69) followed by coo_to_csr (sparse.py:97-106)."""
    keys = sorted_unique(rows.astype(np.int64) * n + cols.astype(np.int64))
    r, c = keys // n, keys % n
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=offsets[1:])
    return offsets, c


def sample_row_panels(offsets, budget_edges, panels=64, seed=1234):
    """Random contiguous row panels holding about budget_edges edges in total
    (rows ascending, disjoint): a bounded, unbiased sample of a row-partitioned
    workload (leading rows would over-weight hubs on power-law graphs)."""
    n = offsets.size - 1
    e = int(offsets[-1])
    rng = np.random.default_rng(seed)
    per = max(1, budget_edges // panels)
    picked = np.zeros(n, dtype=bool)
    got = 0
    tries = 0
    while got < budget_edges and tries < 100 * panels:
        tries += 1
        start = int(rng.integers(0, n))
        end = int(np.searchsorted(offsets, offsets[start] + per, side="left"))
        end = min(max(end, start + 1), n)
        seg = ~picked[start:end]
        if not seg.any():
            continue
        idx = np.arange(start, end)[seg]
        picked[idx] = True
        got += int((offsets[idx + 1] - offsets[idx]).sum())
        if got >= e:
            break
    return np.nonzero(picked)[0]
