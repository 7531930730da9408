"""Operator API of the reference (halfsparse/kernels.py) backed by sm_100a kernels.

spmm_v / spmm_ve / sddmm / spmm_vertex_grouped accept the reference's host
containers (CooGraph / CsrGraph / DenseTensor), validate eagerly with the
reference's messages, run on the GPU and return the reference's result types
(DenseTensor, KernelMetrics[, StagingBuffer]).

numerics="reference" (default here) runs the bit-exact reference-order
kernels: hg_spmm_edge_ref reproduces _spmm_edge_parallel's rounding sequence
for the given schedule, hg_spmm_vertex_ref spmm_vertex_grouped's, hg_sddmm
sddmm's.  numerics="fast" runs the fp32-guarded row-owned kernel (hg_spmm),
within the SURVEY Appendix A tolerance of the float64 result.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import simt
from .simt import KernelMetrics, Schedule
from .sparse import CooGraph, CsrGraph, DenseTensor, csr_to_coo

SCALINGS = ("post", "pre", "discretized")
NORMS = ("none", "left", "right", "both")
WRITE_MODES = ("staging", "atomic_model")
NUMERICS = ("reference", "fast")


@dataclass(frozen=True)
class Reduction:
    """Scaling placement x degree-norm side of one SpMM call (kernels.py:54-67)."""

    scaling: str = "post"
    norm: str = "none"

    def __post_init__(self):
        if self.scaling not in SCALINGS:
            raise ValueError(f"unknown scaling {self.scaling!r}")
        if self.norm not in NORMS:
            raise ValueError(f"unknown norm {self.norm!r}")
        if self.scaling == "discretized" and self.norm == "none":
            raise ValueError("discretized scaling requires a degree norm")


@dataclass
class StagingBuffer:
    """Carry-out slots (kernels.py:70-87): one per CTA (edge-parallel) or per
    neighbour group of a multi-group row (vertex-grouped)."""

    rows: np.ndarray
    partials: np.ndarray

    @property
    def capacity(self):
        return int(self.rows.size)

    def slot_for(self, owner: int) -> int:
        return owner


def _check_width(feat, width):
    lanes = simt.WIDTH_LANES.get(width)
    if lanes is None:
        raise ValueError(f"unknown width {width!r}")
    if feat % 2 or feat % lanes:
        raise ValueError(f"feature length {feat} must be even and divisible by {width} lanes")


def _torch_of(arr):
    import torch

    return torch.from_numpy(np.ascontiguousarray(arr)).cuda()


def _edge_parallel(g, w_e, x, schedule, reduction, width, return_staging, numerics):
    from . import device as D

    if numerics not in NUMERICS:
        raise ValueError(f"unknown numerics {numerics!r}")
    feat = x.cols
    _check_width(feat, width)
    if x.rows != g.n:
        raise ValueError(f"feature tensor has {x.rows} rows for {g.n} vertices")
    sched = schedule if schedule is not None else simt.plan_edge_parallel(g)
    if sched.kind != "edge_parallel":
        raise ValueError("expected an edge-parallel schedule")
    if w_e is not None:
        w_e = np.asarray(w_e)
        if w_e.shape != (g.num_edges,):
            raise ValueError("edge weights must be one value per edge")
        if w_e.dtype != x.data.dtype:
            raise ValueError(f"edge weights must be {x.mode}")
    metrics = simt.edge_metrics(g, sched, feat, width, w_e is not None)
    if g.num_edges == 0:
        out = DenseTensor(np.zeros((g.n, feat), dtype=x.data.dtype))
        empty = StagingBuffer(np.zeros(0, np.int64), np.zeros((0, feat), dtype=x.data.dtype))
        return (out, metrics, empty) if return_staging else (out, metrics)
    dg = g.device()
    xt = _torch_of(x.data)
    wt = None if w_e is None else _torch_of(w_e)
    if numerics == "reference":
        y, srows, svals = D.spmm_edge_ref(dg, xt, wt, reduction.scaling, reduction.norm,
                                          warp_chunk=sched.warp_chunk,
                                          warps_per_cta=sched.warps_per_cta, staging=True)
        staging = StagingBuffer(srows.cpu().numpy(), svals.cpu().numpy())
    else:
        y = D.spmm(dg, xt, wt, reduction.scaling, reduction.norm)
        staging = StagingBuffer(np.zeros(0, np.int64), np.zeros((0, feat), x.data.dtype))
    out = DenseTensor(y.cpu().numpy())
    return (out, metrics, staging) if return_staging else (out, metrics)


def spmm_v(g, x, schedule=None, reduction=Reduction(), width="half2", return_staging=False,
           numerics="reference"):
    """Y[r] = reduce over edges (r, c) of X[c] (kernels.py:394-396)."""
    return _edge_parallel(g, None, x, schedule, reduction, width, return_staging, numerics)


def spmm_ve(g, w_e, x, schedule=None, reduction=Reduction(), width="half2",
            return_staging=False, numerics="reference"):
    """Y[r] = reduce over edges (r, c) of w_e * X[c] (kernels.py:399-401)."""
    return _edge_parallel(g, w_e, x, schedule, reduction, width, return_staging, numerics)


def sddmm(g, x, y, schedule=None, width="half2"):
    """W[e] = X[row(e)] . Y[col(e)], the reference's tree order, bit-exact (kernels.py:407-455)."""
    from . import device as D

    if x.mode != y.mode:
        raise ValueError("operand modes differ")
    if x.cols != y.cols:
        raise ValueError("operand feature lengths differ")
    if x.rows != g.n or y.rows != g.n:
        raise ValueError("operand rows must match the vertex count")
    _check_width(x.cols, width)
    sched = schedule if schedule is not None else simt.plan_edge_parallel(g)
    if sched.kind != "edge_parallel":
        raise ValueError("expected an edge-parallel schedule")
    metrics = simt.sddmm_metrics(g, sched, x.cols, width)
    if g.num_edges == 0:
        return np.zeros(0, dtype=x.data.dtype), metrics
    out = D.sddmm(g.device(), _torch_of(x.data), _torch_of(y.data))
    return out.cpu().numpy(), metrics


def spmm_vertex_grouped(csr, x, schedule=None, reduction=Reduction(), write_mode="staging",
                        width="half2", return_staging=False):
    """Neighbour-group SpMM (kernels.py:463-559), bit-exact; both write modes
    give identical values, only the counters differ."""
    from . import device as D

    if not isinstance(csr, CsrGraph):
        raise ValueError("vertex-grouped kernel expects a CSR graph")
    if write_mode not in WRITE_MODES:
        raise ValueError(f"unknown write mode {write_mode!r}")
    feat = x.cols
    _check_width(feat, width)
    if x.rows != csr.n:
        raise ValueError(f"feature tensor has {x.rows} rows for {csr.n} vertices")
    sched = schedule if schedule is not None else simt.plan_vertex_grouped(csr)
    if sched.kind != "vertex_grouped":
        raise ValueError("expected a vertex-grouped schedule")
    metrics = simt.vertex_metrics(csr, sched, feat, width, write_mode)
    if csr.num_edges == 0:
        out = DenseTensor(np.zeros((csr.n, feat), dtype=x.data.dtype))
        empty = StagingBuffer(np.zeros(0, np.int64), np.zeros((0, feat), dtype=x.data.dtype))
        return (out, metrics, empty) if return_staging else (out, metrics)
    g = csr_to_coo(csr)
    y, srows, svals = D.spmm_vertex_ref(g.device(), _torch_of(x.data), reduction.scaling,
                                        reduction.norm, staging=True)
    out = DenseTensor(y.cpu().numpy())
    if write_mode == "staging":
        staging = StagingBuffer(srows.cpu().numpy(), svals.cpu().numpy())
    else:
        staging = StagingBuffer(np.zeros(0, np.int64), np.zeros((0, feat), dtype=x.data.dtype))
    return (out, metrics, staging) if return_staging else (out, metrics)


def scalar_reference(kind, g, x, schedule=None, w_e=None, y=None, reduction=Reduction(),
                     write_mode="staging"):
    """The reference's order-faithful results (kernels.py:565-580), produced by
    the bit-exact reference-order GPU kernels."""
    if kind in ("spmm_v", "spmm_ve"):
        out, _ = _edge_parallel(g, w_e if kind == "spmm_ve" else None, x, schedule, reduction,
                                "half2", False, "reference")
        return out
    if kind == "sddmm":
        return sddmm(g, x, y)[0]
    if kind == "spmm_vertex_grouped":
        return spmm_vertex_grouped(g, x, schedule, reduction, write_mode)[0]
    raise ValueError(f"unknown reference kind {kind!r}")
