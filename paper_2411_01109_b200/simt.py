"""Schedule objects and counting metrics of the reference API (simt.py of halfsparse).

On B200 the work decomposition that actually runs is the degree-bucketed
unit schedule built on the GPU (device.build_schedule / hg_schedule_build) for
the fp32-guarded kernels, and the reference's own warp-chunk geometry for the
bit-exact reference-order kernels.  This module keeps the reference's
Schedule / KernelMetrics types and planning functions so callers written
against halfsparse keep working (simt.py:101-201); the counters are the
reference's analytic cost model (GPU timing comes from CUDA events and ncu).
"""
from __future__ import annotations

import json
import math
from dataclasses import asdict, dataclass, field

import numpy as np

EDGE_PARALLEL_MIN_CHUNK = 64
DEFAULT_WARP_CHUNK = 128
DEFAULT_WARPS_PER_CTA = 4
WARP_SIZE = 32
VERTEX_GROUP_SIZE = 32
WIDTH_LANES = {"half": 1, "half2": 2, "half4": 4, "half8": 8}
_NZE_COO_BYTES, _NZE_CSR_BYTES = 8, 4


def warp_load_bytes(width: str) -> int:
    """Bytes one coalesced warp load moves at a given vector width (simt.py:39-43)."""
    lanes = WIDTH_LANES.get(width)
    if lanes is None:
        raise ValueError(f"unknown width {width!r}")
    return 2 * lanes * WARP_SIZE


def feature_transactions(n_values: int, width: str) -> int:
    per = WARP_SIZE * WIDTH_LANES[width]
    return 0 if n_values <= 0 else (n_values + per - 1) // per


def sddmm_reduction_rounds(feature_len: int, width: str) -> int:
    """Shuffle rounds per edge: log2 of the threads holding partials (simt.py:52-66)."""
    lanes = WIDTH_LANES.get(width)
    if lanes is None:
        raise ValueError(f"unknown width {width!r}")
    if feature_len <= 0 or feature_len % lanes:
        raise ValueError(f"feature length {feature_len} not divisible by {width} lanes ({lanes})")
    return max(0, int(feature_len // lanes - 1).bit_length())


def intra_cta_rounds(subwarp_count: int) -> int:
    if subwarp_count <= 0 or subwarp_count & (subwarp_count - 1):
        raise ValueError(f"sub-warp count must be a power of two, got {subwarp_count}")
    return int(math.log2(subwarp_count))


@dataclass(frozen=True)
class SubWarpLayout:
    feature_len: int
    threads_per_edge: int
    subwarps: int
    feature_chunk: int


def subwarp_layout(feature_len: int) -> SubWarpLayout:
    """simt.py:86-98: F/2 half2 threads per edge, 32/(F/2) edges per warp step."""
    if feature_len <= 0 or feature_len % 2:
        raise ValueError(f"feature length must be even and positive, got {feature_len}")
    if feature_len > 2 * WARP_SIZE:
        return SubWarpLayout(feature_len, WARP_SIZE, 1, 2 * WARP_SIZE)
    t = feature_len // 2
    return SubWarpLayout(feature_len, t, WARP_SIZE // t, feature_len)


@dataclass
class KernelMetrics:
    load_transactions: int = 0
    load_bytes: int = 0
    coalesced_bytes_per_warp_load: int = 0
    barrier_waits: int = 0
    shuffle_rounds: int = 0
    intra_cta_rounds: int = 0
    atomic_writes: int = 0
    staging_writes: int = 0

    def to_json(self) -> str:
        return json.dumps(asdict(self), sort_keys=True)

    def as_dict(self) -> dict:
        return asdict(self)


@dataclass
class Schedule:
    """Warp/CTA ownership plan (simt.py:124-155).  edge_parallel: warp w owns
    edges [starts[w], ends[w]); vertex_grouped: warp w owns CSR slots of row
    group_rows[w]."""

    kind: str
    warp_chunk: int
    warps_per_cta: int
    starts: np.ndarray
    ends: np.ndarray
    group_rows: np.ndarray | None = None
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def num_warps(self):
        return int(self.starts.size)

    @property
    def num_ctas(self):
        return (self.num_warps + self.warps_per_cta - 1) // self.warps_per_cta if self.num_warps else 0

    def cta_of(self, warp):
        return warp // self.warps_per_cta

    def warp_range(self, cta):
        lo = cta * self.warps_per_cta
        return lo, min(lo + self.warps_per_cta, self.num_warps)


def plan_edge_parallel(g, warp_chunk: int = DEFAULT_WARP_CHUNK,
                       warps_per_cta: int = DEFAULT_WARPS_PER_CTA) -> Schedule:
    if warp_chunk < EDGE_PARALLEL_MIN_CHUNK or warp_chunk % 2:
        raise ValueError(
            f"warp_chunk must be >= {EDGE_PARALLEL_MIN_CHUNK} and even, got {warp_chunk}")
    if warps_per_cta < 1:
        raise ValueError("warps_per_cta must be positive")
    e = g.num_edges
    starts = np.arange(0, e, warp_chunk, dtype=np.int64)
    return Schedule("edge_parallel", warp_chunk, warps_per_cta, starts,
                    np.minimum(starts + warp_chunk, e))


def plan_vertex_grouped(csr, warps_per_cta: int = DEFAULT_WARPS_PER_CTA) -> Schedule:
    if warps_per_cta < 1:
        raise ValueError("warps_per_cta must be positive")
    deg = np.diff(csr.offsets)
    ng = (deg + VERTEX_GROUP_SIZE - 1) // VERTEX_GROUP_SIZE
    rows = np.repeat(np.arange(csr.n, dtype=np.int64), ng)
    k = np.arange(rows.size, dtype=np.int64) - np.repeat(np.cumsum(ng) - ng, ng)
    starts = csr.offsets[rows] + k * VERTEX_GROUP_SIZE
    ends = np.minimum(starts + VERTEX_GROUP_SIZE, csr.offsets[rows + 1])
    return Schedule("vertex_grouped", VERTEX_GROUP_SIZE, warps_per_cta, starts, ends,
                    group_rows=rows)


def check_spmm_rules(g, sched: Schedule) -> None:
    """Edge-parallel ownership rules (simt.py:204-231)."""
    if sched.kind != "edge_parallel":
        raise ValueError("rule check applies to edge-parallel schedules")
    e = g.num_edges
    cover = np.zeros(e + 1, dtype=np.int64)
    np.add.at(cover, sched.starts, 1)
    np.add.at(cover, sched.ends, -1)
    owned = np.cumsum(cover)[:e]
    if e and not np.all(owned == 1):
        raise AssertionError("edge ownership is not a partition")
    for w in range(sched.num_warps):
        seg = g.rows[sched.starts[w]:sched.ends[w]]
        if seg.size and np.any(np.diff(seg) < 0):
            raise AssertionError(f"warp {w}: row ids decrease")
    cta = np.repeat(np.arange(sched.num_warps) // sched.warps_per_cta, sched.ends - sched.starts)
    lo = np.full(g.n, np.iinfo(np.int64).max)
    hi = np.full(g.n, -1)
    np.minimum.at(lo, g.rows, cta)
    np.maximum.at(hi, g.rows, cta)
    for row in np.unique(g.rows):
        span = np.unique(cta[g.rows == row])
        if span.size != hi[row] - lo[row] + 1:
            raise AssertionError(f"row {row} spans non-consecutive CTAs")


# ── counting model (cost-model outputs kept for API compatibility) ───────


def edge_metrics(g, sched: Schedule, feat: int, width: str, weighted: bool) -> KernelMetrics:
    """The reference's edge-parallel SpMM counters (kernels.py:300-322)."""
    m = KernelMetrics(coalesced_bytes_per_warp_load=warp_load_bytes(width))
    if g.num_edges == 0:
        return m
    owned = (sched.ends - sched.starts).astype(np.int64)
    nze = -(-owned // WARP_SIZE)
    m.load_transactions += int(nze.sum())
    m.load_bytes += int(nze.sum()) * WARP_SIZE * _NZE_COO_BYTES
    if weighted:
        wt = -(-owned // (WARP_SIZE * WIDTH_LANES[width]))
        m.load_transactions += int(wt.sum())
        m.load_bytes += int(wt.sum()) * warp_load_bytes(width)
    k = subwarp_layout(feat).subwarps
    iters = int((-(-owned // k)).sum())
    per = feature_transactions(k * feat, width)
    m.load_transactions += iters * per
    m.load_bytes += iters * per * warp_load_bytes(width)
    m.barrier_waits += sched.num_warps
    # chain lengths: segments of one row inside one CTA
    rows = g.rows
    warp = np.arange(rows.size) // sched.warp_chunk
    start = np.r_[True, (rows[1:] != rows[:-1]) | (warp[1:] != warp[:-1])]
    seg_row = rows[start]
    seg_cta = warp[start] // sched.warps_per_cta
    brk = np.r_[True, (seg_cta[1:] != seg_cta[:-1]) | (seg_row[1:] != seg_row[:-1])]
    chain_len = np.diff(np.r_[np.flatnonzero(brk), brk.size])
    m.intra_cta_rounds += int(sum(int(c - 1).bit_length() for c in chain_len[chain_len > 1]))
    m.staging_writes += sched.num_ctas
    return m


def sddmm_metrics(g, sched: Schedule, feat: int, width: str) -> KernelMetrics:
    """kernels.py:428-441."""
    m = KernelMetrics(coalesced_bytes_per_warp_load=warp_load_bytes(width),
                      shuffle_rounds=sddmm_reduction_rounds(feat, width) * g.num_edges)
    lanes_t = feature_transactions(feat, width)
    owned = (sched.ends - sched.starts).astype(np.int64)
    nze = int((-(-owned // WARP_SIZE)).sum())
    m.load_transactions = nze + 2 * g.num_edges * lanes_t
    m.load_bytes = nze * WARP_SIZE * _NZE_COO_BYTES + 2 * g.num_edges * lanes_t * warp_load_bytes(width)
    m.barrier_waits = sched.num_warps
    return m


def vertex_metrics(csr, sched: Schedule, feat: int, width: str, write_mode: str) -> KernelMetrics:
    """kernels.py:493-504, 546-556."""
    m = KernelMetrics(coalesced_bytes_per_warp_load=warp_load_bytes(width))
    ng = sched.num_warps
    glen = int((sched.ends - sched.starts).sum())
    per = feature_transactions(feat, width)
    m.load_transactions = ng + per * glen
    m.load_bytes = ng * WARP_SIZE * _NZE_CSR_BYTES + per * glen * warp_load_bytes(width)
    m.barrier_waits = ng
    if csr.num_edges:
        gpr = np.bincount(sched.group_rows, minlength=csr.n)
        if write_mode == "staging":
            m.staging_writes = int(gpr[gpr > 1].sum())
        else:
            m.atomic_writes = int(np.maximum(gpr - 1, 0).sum())
    return m
