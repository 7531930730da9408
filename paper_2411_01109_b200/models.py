"""Mixed-precision GNN training on the B200 kernels (halfsparse/models.py API).

torch autograd replaces the reference's tape (models.py:85-127); the sparse
operators are torch.autograd.Functions over libhalfgnn:

  spmm_agg        forward hg_spmm on the CSR, backward on the CSC with the
                  norm mirrored (the exact adjoint, models.py:274-290)
  spmm_weighted   forward weighted SpMM; backward SDDMM for dw and a
                  transposed weighted SpMM reading w through perm (293-314)
  attention       hg_attn_scores (+ leaky ReLU fused), backward row/column
                  sums (317-340)
  edge_softmax    hg_edge_softmax_fwd / _bwd, bit-exact (382-412)

Dense GEMMs use cuBLAS on the tensor cores with fp32 accumulation and one
rounding, like the reference's fp32-BLAS-then-round matmul (141-158).
Parameters are fp32 masters published as fp16 leaves every step; only the
logits cross to fp32, for the loss (203-217, 552-572).

Numerics modes (GraphBundle.numerics): "fast" runs the fp32-guarded SpMM;
"reference" runs the bit-exact reference-order SpMM for every aggregation.
SDDMM, scores and softmax are bit-exact in both modes.
"""
from __future__ import annotations

import csv
import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import device as D
from .kernels import Reduction
from .sparse import CooGraph

_DTYPES = {"half": torch.float16, "float32": torch.float32}
_MIRROR = {"none": "none", "left": "right", "right": "left", "both": "both"}

torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = False
torch.backends.cuda.matmul.allow_tf32 = False


class NanLossError(RuntimeError):
    """Training loss became non-finite; carries the epoch and overflow counters."""

    def __init__(self, epoch, counters):
        super().__init__(f"loss is NaN at epoch {epoch}")
        self.epoch = epoch
        self.counters = counters


@dataclass
class ConversionCounter:
    forward: int = 0
    backward: int = 0

    @property
    def total(self):
        return self.forward + self.backward

    def reset(self):
        self.forward = 0
        self.backward = 0


class OverflowCounters:
    """Non-finite output tallies per (layer, op) tag.  Counting runs on the
    device; the host copy is taken lazily (one sync when read)."""

    def __init__(self):
        self._pending = []
        self._inf = {}
        self._nan = {}

    def observe(self, tag, t):
        if isinstance(t, np.ndarray):
            t = torch.from_numpy(t)
        self._pending.append((tag, torch.isinf(t).sum(), torch.isnan(t).sum()))

    def _drain(self):
        for tag, ni, nn in self._pending:
            ni, nn = int(ni), int(nn)
            if ni:
                self._inf[tag] = self._inf.get(tag, 0) + ni
            if nn:
                self._nan[tag] = self._nan.get(tag, 0) + nn
        self._pending.clear()

    @property
    def inf(self):
        self._drain()
        return self._inf

    @property
    def nan(self):
        self._drain()
        return self._nan

    def totals(self):
        return sum(self.inf.values()), sum(self.nan.values())

    def reset(self):
        self._pending.clear()
        self._inf.clear()
        self._nan.clear()


# ── graph bundle ─────────────────────────────────────────────────────────


class GraphBundle:
    """Forward graph + transpose resident in HBM (models.py:246-264)."""

    def __init__(self, dg: D.DeviceGraph, warp_chunk=128, warps_per_cta=4, numerics="fast",
                 g: CooGraph | None = None):
        if numerics not in ("fast", "reference"):
            raise ValueError(f"unknown numerics {numerics!r}")
        self.dg = dg
        self.g = g
        self.warp_chunk = warp_chunk
        self.warps_per_cta = warps_per_cta
        self.numerics = numerics
        self._ones2 = {}

    @classmethod
    def build(cls, g, warp_chunk=128, warps_per_cta=4, numerics="fast"):
        if isinstance(g, D.DeviceGraph):
            return cls(g, warp_chunk, warps_per_cta, numerics)
        return cls(g.device(), warp_chunk, warps_per_cta, numerics, g)

    @property
    def n(self):
        return self.dg.n

    @property
    def num_edges(self):
        return self.dg.num_edges

    @property
    def fused_relu(self):
        """Aggregations may apply the following ReLU in their epilogue."""
        return self.numerics == "fast"

    def spmm(self, x, w=None, scaling="post", norm="none", transpose=False, heads=1,
             weight_via_perm=False, relu=False, combine=None):
        if self.numerics == "fast":
            return D.spmm(self.dg, x, w, scaling, norm, transpose, heads,
                          weight_via_perm=weight_via_perm, relu=relu, combine=combine)
        if combine is not None:
            raise ValueError("the combine epilogue needs numerics='fast'")
        if relu:
            raise ValueError("fused ReLU needs numerics='fast'")
        # reference order: one head at a time, weights materialised in CSC order
        if w is not None and weight_via_perm:
            w = w[self.dg.perm.long()]
        if heads == 1:
            w1 = None if w is None else w.reshape(-1)
            return D.spmm_edge_ref(self.dg, x, w1, scaling, norm, transpose, self.warp_chunk,
                                   self.warps_per_cta)
        fh = x.shape[1] // heads
        outs = [D.spmm_edge_ref(self.dg, x[:, h * fh:(h + 1) * fh].contiguous(),
                                w[:, h].contiguous(), scaling, norm, transpose,
                                self.warp_chunk, self.warps_per_cta) for h in range(heads)]
        return torch.cat(outs, dim=1)

    @property
    def fused_bias_agg(self):
        """GCN layers may fuse add_bias into the aggregation's input pass."""
        return self.numerics == "fast"

    def gcn_agg_tc(self, x, w, b, reduction, relu=False):
        """GCN layer forward: tcgen05 GEMM with bias + input scale fused, then
        the gather SpMM (optionally with the next ReLU in its epilogue)."""
        fin, fout = self.dg.norm_tables(reduction.norm, False, x.dtype)
        xs = D.gemm_tc(x, _wt(w), b, fin)
        return D.spmm_csr(self.dg.view(False), xs, None, None, 1, reduction.scaling, None, fout,
                          relu=relu)

    def bias_spmm(self, h, b, scaling, norm, relu=False):
        """spmm(add_bias(h, b)) with the bias add and the left-norm input
        scaling in one pass (hg_bias_scale_rows), then the gather kernel."""
        fin, fout = self.dg.norm_tables(norm, False, h.dtype)
        xs = D.bias_scale_rows(h, b, fin)
        return D.spmm_csr(self.dg.view(False), xs, None, None, 1, scaling, None, fout, relu=relu)

    @property
    def fused_gat(self):
        """GAT layers may run scores + leaky + softmax as one fp32-guarded pass."""
        return self.numerics == "fast"

    def gat_attention(self, s_l, s_r, slope):
        return D.gat_attention_fwd(self.dg.view(False), s_l, s_r, slope)

    def gat_attention_bwd(self, s_l, s_r, alpha, g, slope):
        """(ds_l, ds_r): row sums on the CSR, column sums through the CSC + perm."""
        de, ds_l = D.gat_attention_bwd(self.dg.view(False), s_l, s_r, alpha, g, slope)
        bwd = self.dg.view(True)
        return ds_l, D.edge_sums_fast(bwd, de, bwd.perm)

    def sddmm(self, x, y, heads=1):
        return D.sddmm(self.dg, x, y, heads=heads, fast=self.numerics == "fast")

    @staticmethod
    def head_dots(z, a_l, a_r, heads):
        return D.head_dots(z, a_l, a_r, heads)

    @staticmethod
    def scale(x, s):
        return D.scale_f64(x, s)

    @staticmethod
    def head_dots_bwd(z, a_l, a_r, g_l, g_r, heads):
        return D.head_dots_bwd(z, a_l, a_r, g_l, g_r, heads)

    def attn_logits(self, s_l, s_r, slope):
        return D.attention_logits(self.dg, s_l, s_r, slope)

    def softmax_fwd(self, e):
        return D.edge_softmax_fwd(self.dg, e)

    def softmax_bwd(self, alpha, g):
        return D.edge_softmax_bwd(self.dg, alpha, g)

    def edge_sums(self, v, transpose=False):
        """Row (or column) sums of per-edge values [E, H] -> [N, H]
        (attention_scores backward, models.py:329-337)."""
        if self.numerics == "fast":
            return D.edge_rowsum(self.dg, v, transpose)
        v2 = v.reshape(v.shape[0], -1)
        if transpose:
            v2 = v2[self.dg.perm.long()]
        ones = self._ones2.get(v.dtype)
        if ones is None:
            ones = torch.ones((self.n, 2), dtype=v.dtype, device=v.device)
            self._ones2[v.dtype] = ones
        cols = [D.spmm_edge_ref(self.dg, ones, v2[:, h].contiguous(), "post", "none", transpose,
                                self.warp_chunk, self.warps_per_cta)[:, :1]
                for h in range(v2.shape[1])]
        return torch.cat(cols, dim=1)


# ── sparse autograd ops ──────────────────────────────────────────────────


class _AggFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, bundle, reduction):
        ctx.bundle, ctx.reduction = bundle, reduction
        return bundle.spmm(x, None, reduction.scaling, reduction.norm)

    @staticmethod
    def backward(ctx, g):
        r = ctx.reduction
        gx = ctx.bundle.spmm(g.contiguous(), None, r.scaling, _MIRROR[r.norm], transpose=True)
        return gx, None, None


class _BiasAggFn(torch.autograd.Function):
    """spmm_agg(add_bias(h, b)) (models.py:161-173, 274-290) as one op: the
    forward fuses the bias add into the SpMM input pass; the backward is the
    mirrored-norm transposed SpMM, and the bias gradient is its column sum."""

    @staticmethod
    def forward(ctx, h, b, bundle, reduction, relu=False):
        ctx.bundle, ctx.reduction, ctx.relu = bundle, reduction, relu
        if relu:
            y = bundle.bias_spmm(h, b, reduction.scaling, reduction.norm, relu=True)
            ctx.save_for_backward(y)
            return y
        return bundle.bias_spmm(h, b, reduction.scaling, reduction.norm)

    @staticmethod
    def backward(ctx, g):
        r = ctx.reduction
        g = g.contiguous()
        if ctx.relu:
            g = D.relu_grad(ctx.saved_tensors[0], g)
        gh = ctx.bundle.spmm(g, None, r.scaling, _MIRROR[r.norm], transpose=True)
        return gh, D.col_sums(gh), None, None, None


class _GCNLayerFn(torch.autograd.Function):
    """GCNLayer (models.py:456-468) = spmm_agg(add_bias(matmul(x, W), b)) with
    the GEMM, the bias add and the aggregation's left-norm input scale in one
    tcgen05 kernel (hg_gemm_tc), then the gather SpMM.  Backward: transposed
    SpMM, then dW = x^T dh with the bias gradient (column sums of dh) in the
    same tcgen05 pass (hg_gemm_wgrad) and dx = dh W^T (hg_gemm_tc): fp32
    accumulation, one rounding (matmul's backward, 150-155)."""

    @staticmethod
    def forward(ctx, x, w, b, bundle, reduction, relu=False, link_out=None, link_in=None):
        ctx.bundle, ctx.reduction, ctx.relu = bundle, reduction, relu
        ctx.links = (link_out, link_in)
        ctx.leaves = (w, b)
        y = bundle.gcn_agg_tc(x, w, b, reduction, relu=True) if relu else \
            bundle.gcn_agg_tc(x, w, b, reduction)
        ctx.save_for_backward(x, w, y if relu else None)
        return y

    @staticmethod
    def backward(ctx, g):
        x, w, y = ctx.saved_tensors
        r = ctx.reduction
        link_out, link_in = ctx.links
        g = g.contiguous()
        if ctx.relu and not (link_out is not None and link_out.premasked):
            g = D.relu_grad(y, g)
        gh = ctx.bundle.spmm(g, None, r.scaling, _MIRROR[r.norm], transpose=True)
        gx = None
        if ctx.needs_input_grad[0]:
            if link_in is not None and FUSED_RELU_BWD and x.shape[1] % 16 == 0:
                gx = D.gemm_tc_masked(gh, w, x)   # x > 0: the previous layer's ReLU backward
                link_in.premasked = True
            else:
                gx = D.gemm_tc(gh, w)
        gw, gb = _weight_grads(x, gh, *ctx.leaves)
        return gx, gw, gb, None, None, None, None, None


def spmm_agg(bundle, x, reduction, width="half2", overflow=None, tag="agg"):
    """Y = norm-scaled aggregation of X; the adjoint runs the transposed graph."""
    y = _AggFn.apply(x, bundle, reduction)
    if overflow is not None:
        overflow.observe(tag, y.detach())
    return y


class _WeightedFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, w, x, bundle, heads, relu=False):
        ctx.bundle, ctx.heads, ctx.relu = bundle, heads, relu
        if relu:
            y = bundle.spmm(x, w, "post", "none", heads=heads, relu=True)
            ctx.save_for_backward(w, x, y)
            return y
        ctx.save_for_backward(w, x, None)
        return bundle.spmm(x, w, "post", "none", heads=heads)

    @staticmethod
    def backward(ctx, g):
        w, x, y = ctx.saved_tensors
        b, h = ctx.bundle, ctx.heads
        g = g.contiguous()
        if ctx.relu:
            g = D.relu_grad(y, g)
        gw = gx = None
        if ctx.needs_input_grad[0]:
            gw = b.sddmm(g, x, heads=h).reshape(w.shape)
        if ctx.needs_input_grad[1]:
            # w read through perm inside the kernel: materialising w[perm] first
            # (hg_gather_rows) costs the same random reads (measured: 5.5 ms
            # gather vs 4.4-5.3 ms saved in the SpMM on RMAT-24)
            gx = b.spmm(g, w, "post", "none", transpose=True, heads=h, weight_via_perm=True)
        return gw, gx, None, None, None


def spmm_weighted(bundle, w, x, width="half2", overflow=None, tag="agg", relu=False):
    """Y[r] = sum over edges (r, c) of w[e] * X[c] (per head when w is [E, H]);
    relu=True (bundles with fused_relu) applies the next ReLU in the epilogue."""
    heads = 1 if w.dim() == 1 else w.shape[1]
    y = _WeightedFn.apply(w, x, bundle, heads, relu)
    if overflow is not None:
        overflow.observe(tag, y.detach())
    return y


class _ScoresFn(torch.autograd.Function):
    """e = rnd(s_l[row] + s_r[col]), then leaky ReLU (slope None: no activation)."""

    @staticmethod
    def forward(ctx, s_l, s_r, bundle, slope):
        out = bundle.attn_logits(s_l, s_r, 1.0 if slope is None else slope)
        ctx.bundle, ctx.slope = bundle, slope
        ctx.save_for_backward(out)
        return out

    @staticmethod
    def backward(ctx, g):
        (out,) = ctx.saved_tensors
        g = g.contiguous()
        b = ctx.bundle
        if ctx.slope is not None:
            g = torch.where(out > 0, g, b.scale(g, ctx.slope))
        gl = b.edge_sums(g, transpose=False) if ctx.needs_input_grad[0] else None
        gr = b.edge_sums(g, transpose=True) if ctx.needs_input_grad[1] else None
        return gl, gr, None, None


class _GatAttnFn(torch.autograd.Function):
    """leaky(s_l[r] + s_r[c]) -> edge softmax in one fp32-guarded pass
    (models.py:188-200, 317-340, 382-412; numerics="fast")."""

    @staticmethod
    def forward(ctx, s_l, s_r, bundle, slope):
        ctx.bundle, ctx.slope = bundle, slope
        alpha = bundle.gat_attention(s_l, s_r, slope)
        ctx.save_for_backward(s_l, s_r, alpha)
        return alpha

    @staticmethod
    def backward(ctx, g):
        s_l, s_r, alpha = ctx.saved_tensors
        ds_l, ds_r = ctx.bundle.gat_attention_bwd(s_l, s_r, alpha, g, ctx.slope)
        return ds_l, ds_r, None, None


def attention_scores(bundle, s_l, s_r):
    """Per-edge s_l[row] + s_r[col] (models.py:317-340); [E] for one head."""
    one = s_l.dim() == 2 and s_l.shape[1] == 1
    e = _ScoresFn.apply(s_l, s_r, bundle, None)
    return e[:, 0] if one else e


def attention_logits(bundle, s_l, s_r, slope=0.2):
    """leaky_relu(attention_scores(s_l, s_r), slope), fused: [E, H]."""
    return _ScoresFn.apply(s_l, s_r, bundle, slope)


class _SoftmaxFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, e, bundle):
        alpha = bundle.softmax_fwd(e)
        ctx.bundle = bundle
        ctx.save_for_backward(alpha)
        return alpha

    @staticmethod
    def backward(ctx, g):
        (alpha,) = ctx.saved_tensors
        return ctx.bundle.softmax_bwd(alpha, g.contiguous()), None


def edge_softmax(bundle, e, overflow=None, tag="softmax"):
    """Row softmax over edge scores in the input precision, bit-exact."""
    alpha = _SoftmaxFn.apply(e, bundle)
    if overflow is not None:
        overflow.observe(tag + "/exp", alpha.detach())
        overflow.observe(tag + "/div", alpha.detach())
    return alpha


def shadow_exp(x, overflow=None, tag="exp"):
    """exp on non-positive inputs, one rounding (models.py:360-371)."""
    if bool((x > 0).any()):
        raise ValueError("shadow_exp expects non-positive inputs")
    y = torch.exp(x.double()).to(x.dtype)
    if overflow is not None:
        overflow.observe(tag, y)
    return y


def shadow_div(num, den, overflow=None, tag="div"):
    y = (num.double() / den.double()).to(num.dtype)
    if overflow is not None:
        overflow.observe(tag, y)
    return y


# ── dense / elementwise ops ──────────────────────────────────────────────


def _wt(w):
    """W^T [N, K] contiguous: the published transposed copy a ParamGroup keeps
    for its 2-D weights (written with the weights, no per-step transpose),
    else a copy."""
    t = getattr(w, "_hg_t", None)
    return t if t is not None else w.t().contiguous()


def _tc_shapes(x, w):
    """x @ w fits the tcgen05 kernels (hg_gemm_tc forward / dx, hg_gemm_wgrad
    dW): binary16 CUDA operands, widths multiples of 8 up to 256 (the input
    width only bounds dx, and only when x needs a gradient)."""
    return (x.is_cuda and x.dtype == torch.float16 and w.dtype == torch.float16
            and x.dim() == 2 and w.dim() == 2 and x.shape[1] == w.shape[0]
            and x.shape[1] % 8 == 0 and w.shape[1] % 8 == 0 and w.shape[1] <= 256
            and (not x.requires_grad or x.shape[1] <= 256))


def _weight_grads(x, g, w, b=None):
    """(dW, db) of y = x w (+ b): one hg_gemm_wgrad pass over x and g (fp32
    accumulation, one rounding each; matmul / add_bias backward, models.py:
    151-155, 168-170).  When the leaves own persistent gradient buffers (a
    ParamGroup), the kernel accumulates into them in place and autograd gets
    None -- no separate accumulate kernel."""
    if (w.is_leaf and w.grad is not None and w.grad.is_contiguous()
            and (b is None or (b.is_leaf and b.grad is not None))):
        D.gemm_wgrad(x, g, out=w.grad, bias_out=None if b is None else b.grad,
                     accumulate=True)
        return None, None
    if b is None:
        return D.gemm_wgrad(x, g), None
    return D.gemm_wgrad(x, g, bias=True)


class _MatmulTCFn(torch.autograd.Function):
    """matmul (models.py:141-158) on the tcgen05 tensor cores: y = x w with fp32
    accumulation and one rounding (hg_gemm_tc); backward dx = g w^T
    (hg_gemm_tc) and dW = x^T g (hg_gemm_wgrad, split over the vertices)."""

    @staticmethod
    def forward(ctx, x, w):
        ctx.w_leaf = w
        ctx.save_for_backward(x, w)
        return D.gemm_tc(x, _wt(w))

    @staticmethod
    def backward(ctx, g):
        x, w = ctx.saved_tensors
        g = g.contiguous()
        gx = D.gemm_tc(g, w) if ctx.needs_input_grad[0] else None
        gw = _weight_grads(x, g, ctx.w_leaf)[0] if ctx.needs_input_grad[1] else None
        return gx, gw


def matmul(a, b):
    """Tensor-core GEMM, fp32 accumulation, one rounding to the input dtype:
    the hand-written tcgen05 kernels for binary16 CUDA operands, torch for the
    float32 mode and host tensors."""
    if _tc_shapes(a, b):
        return _MatmulTCFn.apply(a, b)
    return a @ b


def add_bias(x, b):
    return x + b


def relu(x):
    return torch.relu(x)


class _LeakyFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, slope):
        ctx.slope = slope
        ctx.save_for_backward(x)
        return torch.where(x > 0, x, D.scale_f64(x, slope))

    @staticmethod
    def backward(ctx, g):
        (x,) = ctx.saved_tensors
        return torch.where(x > 0, g, D.scale_f64(g.contiguous(), ctx.slope)), None


def leaky_relu(x, slope=0.2):
    """where(x > 0, x, rnd(x * slope)), the product in fp64 (models.py:188-200)."""
    return _LeakyFn.apply(x, slope)


class _ConvertFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, dtype, counter):
        ctx.src, ctx.counter = x.dtype, counter
        if counter is not None:
            counter.forward += 1
        return x.to(dtype)

    @staticmethod
    def backward(ctx, g):
        if ctx.counter is not None:
            ctx.counter.backward += 1
        return g.to(ctx.src), None, None


def convert(x, mode, counter=None):
    """Precision crossing as a graph op; the only place conversions count."""
    return _ConvertFn.apply(x, _DTYPES[mode], counter)


class _ScaleCombineFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, a, ope, lam):
        ctx.lam = lam
        ctx.save_for_backward(x, ope)
        return D.scale_combine(x, a, ope, lam)

    @staticmethod
    def backward(ctx, g):
        x, ope = ctx.saved_tensors
        g = g.contiguous()
        gx, ga, gope = D.scale_combine_bwd(x, g, ope, ctx.lam, *ctx.needs_input_grad[:3])
        return gx, ga, gope, None


def scale_combine(x, a, one_plus_eps, lam):
    """(1 + eps) * x + lam * a with per-term rounding (GIN combine, models.py:220-240)."""
    return _ScaleCombineFn.apply(x, a, one_plus_eps, float(lam))


class _AggCombineFn(torch.autograd.Function):
    """GIN's scale_combine(x, spmm_agg(x)) (models.py:220-240, 274-290, 487) as
    one aggregation whose row store applies the combine (hg_spmm combine):
    the aggregate never goes to HBM.  Backward: the combine's backward (dx
    direct, d agg, d(1+eps)), the transposed aggregation of d agg with the
    direct dx added in its row store (the sum autograd would form)."""

    @staticmethod
    def forward(ctx, x, ope, bundle, reduction, lam):
        ctx.bundle, ctx.reduction, ctx.lam = bundle, reduction, lam
        ctx.save_for_backward(x, ope)
        return bundle.spmm(x, None, reduction.scaling, reduction.norm, combine=(x, ope, lam))

    @staticmethod
    def backward(ctx, g):
        x, ope = ctx.saved_tensors
        need_x, need_ope = ctx.needs_input_grad[0], ctx.needs_input_grad[1]
        g = g.contiguous()
        gx_d, ga, gope = D.scale_combine_bwd(x, g, ope, ctx.lam, need_x, need_x, need_ope)
        gx = None
        if need_x:
            r = ctx.reduction
            gx = ctx.bundle.spmm(ga, None, r.scaling, _MIRROR[r.norm], transpose=True,
                                 combine=(gx_d, None, 1.0))
        return gx, gope, None, None, None


# ── parameters and layers ────────────────────────────────────────────────


class Param:
    """fp32 master weight in HBM; publishes a compute-precision leaf each step.
    Inside a ParamGroup the master and the published leaf are views of the
    group's flat buffers, and publish() returns the persistent leaf."""

    def __init__(self, value, device="cuda", store_shape=None):
        v = torch.as_tensor(np.asarray(value, dtype=np.float32))
        if store_shape is not None and tuple(store_shape) != tuple(v.shape):
            padded = torch.zeros(store_shape, dtype=torch.float32)
            padded[tuple(slice(0, s) for s in v.shape)] = v
            v = padded
        self.master = v.to(device)
        self.published = None
        self.group = None

    def publish(self, mode):
        if self.group is not None and self.group.mode == mode:
            return self.published
        data = self.master if mode == "float32" else self.master.to(torch.float16)
        self.published = data.detach().requires_grad_(True)
        return self.published

    def grad32(self):
        if self.published is None or self.published.grad is None:
            return torch.zeros_like(self.master)
        return self.published.grad.to(torch.float32)


class ParamGroup:
    """All parameters of a model in flat buffers: fp32 masters, the published
    compute-precision copy (persistent autograd leaves viewing it) and their
    gradients.  A training step is one cast (publish), the backward pass
    accumulating straight into the flat gradient, and one fused Adam kernel."""

    def __init__(self, params, mode):
        self.params = list(params)
        self.mode = mode
        dev = self.params[0].master.device
        self.dtype = _DTYPES[mode]
        sizes = [p.master.numel() for p in self.params]
        offs = _offsets(self.params)
        total = offs[-1] + sizes[-1] if sizes else 0
        # parameters start on 8-element boundaries (16-byte aligned fp16 views for
        # the vectorised / TMA kernels); the gaps stay zero and take no updates
        self.master = torch.zeros(total, dtype=torch.float32, device=dev)
        self.pub = torch.empty(total, dtype=self.dtype, device=dev)
        self.grad = torch.zeros(total, dtype=self.dtype, device=dev)
        for p, sz, off in zip(self.params, sizes, offs):
            shape = p.master.shape
            self.master[off:off + sz].copy_(p.master.reshape(-1))
            p.master = self.master[off:off + sz].view(shape)
            leaf = self.pub[off:off + sz].view(shape)
            leaf.requires_grad_(True)
            leaf.grad = self.grad[off:off + sz].view(shape)
            p.published = leaf
            p.group = self
        self._ptrs = [p.published.grad.data_ptr() for p in self.params]
        self.fresh = False   # True: pub / grad already prepared by the fused Adam step
        # transposed published copies of the 2-D weights (the forward GEMMs' B^T
        # operand; written with the published copy, no per-step transpose)
        self.transposed = []
        toff = 0
        for p, off in zip(self.params, offs):
            if p.master.dim() == 2 and len(self.transposed) < 8:
                k, n = p.master.shape
                self.transposed.append((off, k, n, toff))
                toff += (k * n + 7) // 8 * 8
        self.pub_t = torch.empty(max(toff, 1), dtype=self.dtype, device=dev)
        for p, (off, k, n, t0) in zip([p for p in self.params if p.master.dim() == 2],
                                      self.transposed):
            p.published._hg_t = self.pub_t[t0:t0 + k * n].view(n, k)

    @torch.no_grad()
    def publish(self):
        self.pub.copy_(self.master)
        self.grad.zero_()
        for p in self.params:
            t = getattr(p.published, "_hg_t", None)
            if t is not None:
                t.copy_(p.published.t())
        self.fresh = False

    def publish_if_stale(self):
        """publish() unless the last fused Adam step already wrote the published
        copy and cleared the gradient; either way the state is consumed."""
        if not self.fresh:
            self.publish()
        self.fresh = False

    def check_grads(self):
        """True if autograd accumulated in place into the flat gradient."""
        return all(p.published.grad is not None and p.published.grad.data_ptr() == q
                   for p, q in zip(self.params, self._ptrs))


def _glorot(rng, fan_in, fan_out, shape=None):
    """models._glorot (models.py:436-438): same draws, same RNG order."""
    lim = np.sqrt(6.0 / (fan_in + fan_out))
    return rng.uniform(-lim, lim, size=shape or (fan_in, fan_out)).astype(np.float32)


def _round8(v):
    return (v + 7) // 8 * 8


def _round_store(v):
    """Stored input width: a multiple of 8 elements (16-byte rows); from 48 up,
    of 16 (32-byte rows), so the aggregation of raw inputs (GIN) takes the
    SpMM's 32-byte lanes (products' 100 features: 104 -> 112)."""
    return (v + 7) // 8 * 8 if v < 48 else (v + 15) // 16 * 16


def _placed(block, store_shape, in_rows=None):
    """Embed a logical (fan_in, fan_out) block in zero storage; logical input
    row i goes to storage row in_rows[i] (identity by default)."""
    out = np.zeros(store_shape, np.float32)
    rows = np.arange(block.shape[0]) if in_rows is None else np.asarray(in_rows)
    out[rows, : block.shape[1]] = block
    return out


class Linear:
    """x @ W (+ b).  Storage may be zero-padded beyond the logical (fan_in,
    fan_out) so rows stay 16-byte aligned; padded entries stay exactly zero."""

    def __init__(self, rng, fan_in, fan_out, bias=True, device="cuda", store_in=None,
                 store_out=None, in_rows=None):
        si, so = store_in or fan_in, store_out or fan_out
        self.w = Param(_placed(_glorot(rng, fan_in, fan_out), (si, so), in_rows), device)
        self.b = Param(np.zeros(fan_out, np.float32), device, (so,)) if bias else None

    def params(self):
        return [self.w] + ([self.b] if self.b is not None else [])

    def __call__(self, x, mode, tc=False, relu_out=False, link_out=None, link_in=None):
        """tc: run on the tcgen05 GEMM with the bias (and, with relu_out, the
        following ReLU) fused into its epilogue when the shapes allow.
        link_out / link_in (_ReluLink): this call's ReLU output feeds only the
        next Linear / x is such an output (the ReLU backward then runs in the
        consumer's dX GEMM)."""
        w = self.w.publish(mode)
        if tc and mode == "half" and self.b is not None and _tc_shapes(x, w):
            return _LinearTCFn.apply(x, w, self.b.publish(mode), relu_out,
                                     link_out if relu_out else None, link_in)
        out = matmul(x, w)
        if self.b is not None:
            out = add_bias(out, self.b.publish(mode))
        return relu(out) if relu_out else out


class _LinearTCFn(torch.autograd.Function):
    """[relu](add_bias(matmul(x, W), b)) (models.py:141-185) as one tcgen05 GEMM
    with the epilogue fused; backward on the tensor cores too: dx = g W^T
    (hg_gemm_tc), dW = x^T g and db = column sums of g from one hg_gemm_wgrad
    pass (fp32 accumulation, one rounding each), the ReLU mask taken from the
    output (y > 0 iff pre-activation > 0)."""

    @staticmethod
    def forward(ctx, x, w, b, relu_out, link_out=None, link_in=None):
        y = D.gemm_tc(x, _wt(w), b, None, relu=relu_out)
        ctx.relu_out = relu_out
        ctx.links = (link_out, link_in)
        ctx.leaves = (w, b)
        ctx.save_for_backward(x, w, y if relu_out else None)
        return y

    @staticmethod
    def backward(ctx, g):
        x, w, y = ctx.saved_tensors
        link_out, link_in = ctx.links
        g = g.contiguous()
        if ctx.relu_out and not (link_out is not None and link_out.premasked):
            g = D.relu_grad(y, g)
        # dx = g W^T: W is already the [K, N] "B transposed" operand of hg_gemm_tc
        gx = None
        if ctx.needs_input_grad[0]:
            if link_in is not None and FUSED_RELU_BWD and x.shape[1] % 16 == 0:
                gx = D.gemm_tc_masked(g, w, x)   # x > 0: the producer's ReLU backward
                link_in.premasked = True
            else:
                gx = D.gemm_tc(g, w)
        gw, gb = _weight_grads(x, g, *ctx.leaves)
        return gx, gw, gb, None, None, None


class GCNLayer:
    """norm-aggregate(X W + b) (models.py:456-468): bias before aggregation."""

    def __init__(self, rng, fan_in, fan_out, reduction, device="cuda", store_in=None,
                 store_out=None, in_rows=None):
        self.lin = Linear(rng, fan_in, fan_out, True, device, store_in, store_out, in_rows)
        self.reduction = reduction

    def params(self):
        return self.lin.params()

    fuses_relu_out = True
    takes_relu_link = True

    def __call__(self, bundle, x, mode, width, overflow, tag, relu_out=False, link_out=None,
                 link_in=None):
        """link_out / link_in (_ReluLink, Model.forward): this layer's fused
        ReLU output feeds only the next layer / x is such an output."""
        # fused ReLU only when no overflow counters watch the pre-activation
        fuse = relu_out and overflow is None and getattr(bundle, "fused_relu", False)
        if getattr(bundle, "fused_bias_agg", False) and self.lin.b is not None:
            w, b = self.lin.w.publish(mode), self.lin.b.publish(mode)
            if mode == "half" and _tc_shapes(x, w):
                # tensor-core GEMM with the bias / input-scale epilogue fused
                y = _GCNLayerFn.apply(x, w, b, bundle, self.reduction, fuse,
                                      link_out if fuse else None, link_in)
            else:
                y = _BiasAggFn.apply(matmul(x, w), b, bundle, self.reduction, fuse)
            if overflow is not None:
                overflow.observe(tag, y.detach())
            if relu_out and not fuse:
                y = relu(y)
            return y
        y = spmm_agg(bundle, self.lin(x, mode), self.reduction, width, overflow, tag)
        return relu(y) if relu_out else y


class GINLayer:
    """phi2(relu(phi1((1+eps) x + lam * mean-agg(x)))) (models.py:471-489)."""

    def __init__(self, rng, fan_in, fan_out, lam=0.1, scaling="discretized", device="cuda",
                 store_in=None, store_out=None, in_rows=None):
        if not 0.0 < lam <= 1.0:
            raise ValueError("lam must be in (0, 1]")
        self.lam = float(lam)
        self.reduction = Reduction(scaling, "right")
        self.one_plus_eps = Param(np.float32(1.0), device)
        self.phi1 = Linear(rng, fan_in, fan_out, True, device, store_in, store_out, in_rows)
        self.phi2 = Linear(rng, fan_out, fan_out, True, device, store_out, store_out)

    def params(self):
        return [self.one_plus_eps] + self.phi1.params() + self.phi2.params()

    fuses_relu_out = True

    def __call__(self, bundle, x, mode, width, overflow, tag, relu_out=False):
        ope = self.one_plus_eps.publish(mode)
        if (overflow is None and isinstance(bundle, GraphBundle) and bundle.numerics == "fast"
                and x.is_cuda and FUSED_GIN_COMBINE):
            mixed = _AggCombineFn.apply(x, ope, bundle, self.reduction, self.lam)
        else:
            agg = spmm_agg(bundle, x, self.reduction, width, overflow, tag)
            mixed = scale_combine(x, agg, ope, self.lam)
        tc = getattr(bundle, "fused_bias_agg", False)
        link = _ReluLink()   # phi1's ReLU output is consumed by phi2 alone
        return self.phi2(self.phi1(mixed, mode, tc=tc, relu_out=True, link_out=link), mode,
                         tc=tc, relu_out=relu_out, link_in=link)


class GATLayer:
    """Multi-head graph attention.  heads=1 is the reference layer
    (models.py:492-509); per-head parameters are drawn in head order exactly as
    `heads` separate reference GATLayers would draw them.  Output [N, heads*fo]
    (heads concatenated) or, with reduce="mean", the head mean [N, fo]."""

    def __init__(self, rng, fan_in, fan_out, heads=1, device="cuda", store_in=None,
                 store_out=None, reduce="concat", in_rows=None):
        self.heads, self.fan_out, self.reduce = heads, fan_out, reduce
        so = store_out or fan_out
        si = store_in or fan_in
        ws, al, ar = [], [], []
        for _ in range(heads):
            w = _placed(_glorot(rng, fan_in, fan_out), (si, so), in_rows)
            a_l = np.zeros(so, np.float32)
            a_l[:fan_out] = _glorot(rng, fan_out, 1)[:, 0]
            a_r = np.zeros(so, np.float32)
            a_r[:fan_out] = _glorot(rng, fan_out, 1)[:, 0]
            ws.append(w), al.append(a_l), ar.append(a_r)
        self.store_out = so
        self.w = Param(np.concatenate(ws, axis=1), device)
        self.a_l = Param(np.stack(al), device)
        self.a_r = Param(np.stack(ar), device)

    def params(self):
        return [self.w, self.a_l, self.a_r]

    fuses_relu_out = True
    takes_relu_link = True

    def __call__(self, bundle, x, mode, width, overflow, tag, relu_out=False, link_out=None,
                 link_in=None):
        """link_out / link_in (_ReluLink, Model.forward): this layer's fused
        ReLU output feeds only the next layer / x is such an output."""
        h, so = self.heads, self.store_out
        w = self.w.publish(mode)
        a_l, a_r = self.a_l.publish(mode), self.a_r.publish(mode)
        mean = self.reduce == "mean" and h > 1
        if (overflow is None and isinstance(bundle, GraphBundle) and bundle.fused_gat):
            fuse = relu_out and not mean
            if _dots_shapes(x, w, h) and a_l.dtype == torch.float16:
                z, s_l, s_r = _GATProjFn.apply(x, w, a_l, a_r, h, link_in)  # [N, H*so], [N, H] x 2
                out = _GATCoreFn.apply(z, a_l, a_r, bundle, h, fuse, s_l, s_r,
                                       link_out if fuse else None)
            else:
                z = matmul(x, w)                                      # [N, H*so]
                out = _GATCoreFn.apply(z, a_l, a_r, bundle, h, fuse, None, None,
                                       link_out if fuse else None)
            if mean:
                out = _HeadMeanFn.apply(out, h)
            return relu(out) if relu_out and not fuse else out
        z = matmul(x, w)                                          # [N, H*so]
        # s = z_h . a_h for every head (models.matmul semantics: fp32
        # accumulation of exact products, one rounding), one kernel
        s_l, s_r = _HeadDotsFn.apply(z, a_l, a_r, h, bundle)
        if getattr(bundle, "fused_gat", False):
            alpha = _GatAttnFn.apply(s_l, s_r, bundle, 0.2)       # [E, H]
            if overflow is not None:
                overflow.observe(tag + "/softmax", alpha.detach())
        else:
            e = attention_logits(bundle, s_l, s_r, 0.2)           # [E, H]
            alpha = edge_softmax(bundle, e, overflow, tag + "/softmax")
        fuse = (relu_out and overflow is None and not (self.reduce == "mean" and h > 1)
                and getattr(bundle, "fused_relu", False))
        out = spmm_weighted(bundle, alpha if h > 1 else alpha[:, 0], z, width, overflow, tag,
                            relu=fuse)
        if self.reduce == "mean" and h > 1:
            out = _HeadMeanFn.apply(out, h)
        return relu(out) if relu_out and not fuse else out


# GIN's combine folded into the aggregation's row store (and the backward's
# residual add into the transposed aggregation's); HG_FUSED_GIN=0: separate passes.
FUSED_GIN_COMBINE = os.environ.get("HG_FUSED_GIN", "1") != "0"

# GAT forward core as hg_gat_attention_stats + hg_gat_aggregate (SURVEY 8(f)1,
# bitwise the same result as hg_gat_attention_fwd + hg_spmm on alpha).  Off by
# default: measured on C5 (RMAT-24, 4 heads) the alpha math inside the gather
# loop lengthens each batch more than the saved alpha pass returns (119.6 ->
# 122.8 ms/epoch); equal on C2.  HG_FUSED_GAT=1 selects it.
FUSED_GAT_FWD = os.environ.get("HG_FUSED_GAT", "0") == "1"


# The GAT projection's head dots formed in the GEMM epilogue (hg_gemm_tc_dots)
# instead of a second read of z; HG_FUSED_GAT_DOTS=0: separate hg_head_dots.
FUSED_GAT_DOTS = os.environ.get("HG_FUSED_GAT_DOTS", "1") != "0"


# The head dots' dz term folded into the transposed aggregation's row store
# (hg_spmm hd_gl) instead of a read-modify-write pass over dz in
# hg_head_dots_bwd; HG_FUSED_GAT_DZ=0: the separate accumulate.
FUSED_GAT_DZ = os.environ.get("HG_FUSED_GAT_DZ", "1") != "0"


def _dots_shapes(x, w, heads):
    """hg_gemm_tc_dots takes the layer: <= 8 heads of a width that is a multiple
    of 16, an even head count unless the heads are 16 wide."""
    fh = w.shape[1] // heads
    return (FUSED_GAT_DOTS and _tc_shapes(x, w) and heads <= 8 and w.shape[1] % heads == 0
            and fh % 16 == 0 and (heads % 2 == 0 or fh == 16))


class _ReluLink:
    """Between a layer whose epilogue applied the inter-layer ReLU and the
    next layer, its ReLU output's only consumer (Model.forward): set when the
    consumer's dX GEMM already masked the gradient (hg_gemm_tc_masked), so the
    producer skips its relu_grad pass."""
    __slots__ = ("premasked",)

    def __init__(self):
        self.premasked = False


# The ReLU backward folded into the next GAT layer's dX GEMM (hg_gemm_tc_masked)
# instead of a relu_grad pass; HG_FUSED_RELU_BWD=0: the separate pass.
FUSED_RELU_BWD = os.environ.get("HG_FUSED_RELU_BWD", "1") != "0"


class _GATProjFn(torch.autograd.Function):
    """z = x W with the head dots s_l = z_h . a_l[h], s_r = z_h . a_r[h]
    (GATLayer, models.py:492-509) from one tcgen05 GEMM whose epilogue forms the
    dots from the accumulator tile (hg_gemm_tc_dots).  Backward: the head-dot
    gradient accumulates into dz in place (hg_head_dots_bwd, gz_acc), then
    dx = dz W^T (hg_gemm_tc) and dW = x^T dz (hg_gemm_wgrad)."""

    @staticmethod
    def forward(ctx, x, w, a_l, a_r, heads, link=None):
        ctx.set_materialize_grads(False)
        ctx.w_leaf, ctx.heads, ctx.link = w, heads, link
        z, s_l, s_r = D.gemm_tc_dots(x, _wt(w), a_l, a_r, heads)
        ctx.save_for_backward(x, w, z, a_l, a_r)
        return z, s_l, s_r

    @staticmethod
    def backward(ctx, gz, ds_l, ds_r):
        x, w, z, a_l, a_r = ctx.saved_tensors
        gz = gz.contiguous()
        ga_l = ga_r = None
        if ds_l is not None:  # (None: the consumer folded the head-dot backward in)
            gz, ga_l, ga_r = D.head_dots_bwd(z, a_l, a_r, ds_l.contiguous(), ds_r.contiguous(),
                                             ctx.heads, gz_acc=gz)
        gx = None
        if ctx.needs_input_grad[0]:
            if ctx.link is not None and FUSED_RELU_BWD and x.shape[1] % 16 == 0:
                # x is the previous layer's ReLU output, consumed only here:
                # mask dX by x > 0 in the GEMM epilogue (the ReLU's backward)
                gx = D.gemm_tc_masked(gz, w, x)
                ctx.link.premasked = True
            else:
                gx = D.gemm_tc(gz, w)
        gw = _weight_grads(x, gz, ctx.w_leaf)[0] if ctx.needs_input_grad[1] else None
        return gx, gw, ga_l, ga_r, None, None


class _GATCoreFn(torch.autograd.Function):
    """The multi-head GAT layer core (models.py:492-509) after z = x W as one
    autograd node, for single-GPU fast numerics: head dots s = z a -> fused
    attention (scores + leaky + softmax, fp32-guarded) -> weighted aggregation
    [-> the next ReLU].  Backward: SDDMM for d alpha, transposed weighted SpMM
    for dz, attention backward with row/column sums, then the head-dot
    backward accumulates its dz contribution into the SpMM's in the same pass
    (no separate add of the two N x H*F gradients)."""

    @staticmethod
    def forward(ctx, z, a_l, a_r, bundle, heads, relu, s_l=None, s_r=None, link=None):
        # s_l / s_r given: formed by the projection (_GATProjFn), whose backward
        # takes their gradients and the head-dot backward
        ctx.dots_in = s_l is not None
        if not ctx.dots_in:
            s_l, s_r = bundle.head_dots(z, a_l, a_r, heads)
        view = bundle.dg.view(False)
        if FUSED_GAT_FWD:
            # row statistics, then scores -> alpha -> weighted aggregation in
            # one gather pass (alpha written once for the backward, never re-read)
            stats = D.gat_attention_stats(view, s_l, s_r, 0.2)
            out, alpha = D.gat_aggregate(view, z, s_l, s_r, stats, heads, 0.2, relu=relu)
        else:
            alpha = D.gat_attention_fwd(view, s_l, s_r, 0.2)
            out = D.spmm_csr(view, z, alpha, None, heads, "post", relu=relu)
        ctx.bundle, ctx.heads, ctx.relu, ctx.link = bundle, heads, relu, link
        ctx.save_for_backward(z, a_l, a_r, s_l, s_r, alpha, out if relu else None)
        return out

    @staticmethod
    def backward(ctx, g):
        z, a_l, a_r, s_l, s_r, alpha, y = ctx.saved_tensors
        b, h = ctx.bundle, ctx.heads
        g = g.contiguous()
        if ctx.relu and not (ctx.link is not None and ctx.link.premasked):
            g = D.relu_grad(y, g)
        dalpha = b.sddmm(g, z, heads=h).reshape(-1, h)
        bwd = b.dg.view(True)
        de, ds_l = D.gat_attention_bwd(b.dg.view(False), s_l, s_r, alpha, dalpha, 0.2)
        # (fusing these column sums into the transposed aggregation through
        # interleaved (alpha | d_e) rows -- hg_spmm out2 -- measured slower on
        # RMAT-24: +14.7 ms in the aggregation and +3 ms in the strided
        # attention kernels against the 10.6 ms sum pass it replaces)
        ds_r = D.edge_sums_fast(bwd, de, bwd.perm)
        if FUSED_GAT_DZ:
            # the head dots' dz term added in the transposed aggregation's row
            # store (bitwise the separate accumulate), then only da = z^T ds
            gz = D.spmm_csr(bwd, g, alpha, bwd.perm, h, "post",
                            head_dots=(ds_l, ds_r, a_l, a_r))
            _, ga_l, ga_r = D.head_dots_bwd(z, a_l, a_r, ds_l, ds_r, h, dz=False)
            return gz, ga_l, ga_r, None, None, None, None, None, None
        gz = D.spmm_csr(bwd, g, alpha, bwd.perm, h, "post")
        if ctx.dots_in:
            return gz, None, None, None, None, None, ds_l, ds_r, None
        gz, ga_l, ga_r = D.head_dots_bwd(z, a_l, a_r, ds_l, ds_r, h, gz_acc=gz)
        return gz, ga_l, ga_r, None, None, None, None, None, None


class _HeadDotsFn(torch.autograd.Function):
    """(s_l, s_r)[n, h] = z[n, h, :] . (a_l, a_r)[h, :] (hg_head_dots).
    Backward: dz = rnd(g_l a_l) + rnd(g_r a_r) (each an exact product rounded
    once, as the reference's N x 1 by 1 x F matmul gradient), da = z_h^T g."""

    @staticmethod
    def forward(ctx, z, a_l, a_r, heads, bundle):
        ctx.heads, ctx.bundle = heads, bundle
        ctx.save_for_backward(z, a_l, a_r)
        return bundle.head_dots(z, a_l, a_r, heads)

    @staticmethod
    def backward(ctx, g_l, g_r):
        z, a_l, a_r = ctx.saved_tensors
        gz, ga_l, ga_r = ctx.bundle.head_dots_bwd(z, a_l, a_r, g_l, g_r, ctx.heads)
        return gz, ga_l, ga_r, None, None


class _HeadMeanFn(torch.autograd.Function):
    """Mean over heads: fp64 sum / H, one rounding; backward rnd(g / H)."""

    @staticmethod
    def forward(ctx, y, heads):
        ctx.heads = heads
        if y.is_cuda:
            return D.head_mean(y, heads)
        n, f = y.shape
        return (y.view(n, heads, f // heads).double().sum(1) / heads).to(y.dtype)

    @staticmethod
    def backward(ctx, g):
        if g.is_cuda:
            return D.head_mean_bwd(g, ctx.heads), None
        gg = (g.double() / ctx.heads).to(g.dtype)
        return gg.repeat(1, ctx.heads), None


_LAYER_KINDS = ("gcn", "gin", "gat")


class Model:
    """Stack of `layers` layers of one kind with ReLU between (models.py:515-546).
    Defaults reproduce the reference (2 layers, 1 head).  Storage widths are
    padded to multiples of 8 (zero, inert) for 128-bit feature rows."""

    def __init__(self, kind, rng, dims, reduction=None, lam=0.1, heads=1, layers=2,
                 device="cuda", in_store=None):
        if kind not in _LAYER_KINDS:
            raise ValueError(f"unknown model kind {kind!r}")
        if layers < 1:
            raise ValueError("need at least one layer")
        self.kind, self.heads = kind, heads
        fan_in, hidden, n_cls = dims
        red = reduction or Reduction("discretized", "both")
        self.n_cls = n_cls
        self.out_store = _round8(n_cls)
        fi, si = fan_in, in_store or fan_in
        in_rows = None
        self.layers = []
        for li in range(layers):
            last = li == layers - 1
            fo = n_cls if last else hidden
            so = self.out_store if last else _round8(hidden)
            if kind == "gcn":
                layer = GCNLayer(rng, fi, fo, red, device, si, so, in_rows)
            elif kind == "gin":
                layer = GINLayer(rng, fi, fo, lam, red.scaling, device, si, so, in_rows)
            else:
                layer = GATLayer(rng, fi, fo, heads, device, si, so,
                                 reduce="mean" if last else "concat", in_rows=in_rows)
            self.layers.append(layer)
            if kind == "gat" and not last:
                # concatenated heads: logical feature (h, j) lives at storage h*so + j
                fi, si = fo * heads, so * heads
                in_rows = (np.arange(heads)[:, None] * so + np.arange(fo)[None, :]).reshape(-1)
            else:
                fi, si, in_rows = fo, so, None

    def params(self):
        return [p for layer in self.layers for p in layer.params()]

    def forward(self, bundle, x, mode, width="half2", overflow=None):
        h = x
        link = None   # the previous GAT layer's fused ReLU output, consumed only by this layer
        for i, layer in enumerate(self.layers):
            inner = i + 1 < len(self.layers)
            linked = getattr(layer, "takes_relu_link", False)
            kw = {"link_in": link} if linked and link is not None else {}
            link = None
            if inner and getattr(layer, "fuses_relu_out", False):
                # the layer applies the inter-layer ReLU in its own epilogue
                if linked and getattr(self.layers[i + 1], "takes_relu_link", False):
                    link = kw["link_out"] = _ReluLink()
                h = layer(bundle, h, mode, width, overflow, f"{self.kind}{i}", relu_out=True,
                          **kw)
                continue
            h = layer(bundle, h, mode, width, overflow, f"{self.kind}{i}", **kw)
            if inner:
                h = relu(h)
        return h


# ── loss, optimiser, training loop ───────────────────────────────────────


class _CrossEntropyFn(torch.autograd.Function):
    """Forward and backward of the softmax cross-entropy in one fused fp64 pass
    (hg_softmax_xent); the saved gradient is scaled by the upstream grad."""

    @staticmethod
    def forward(ctx, logits, labels, n_active, denom, impl):
        nll, grad = impl(logits, labels, n_active, denom)
        ctx.save_for_backward(grad)
        return (nll.sum() / denom).float()

    @staticmethod
    def backward(ctx, g):
        (grad,) = ctx.saved_tensors
        return grad * g, None, None, None, None


def cross_entropy(logits, labels, n_active=None, denom=None, impl=None):
    """Mean CE over all nodes on fp32 logits (models.py:552-572); columns at or
    beyond n_active (storage padding) take no part.  denom: the global node
    count when the rows are one partition of the graph."""
    if logits.dtype != torch.float32:
        raise ValueError("cross-entropy expects float32 logits")
    return _CrossEntropyFn.apply(logits, labels, n_active or logits.shape[1],
                                 denom or logits.shape[0], impl or D.softmax_xent)


class Adam:
    """models.Adam (models.py:575-592) on device fp32 masters.  The step count
    lives on the device (fp64) so a step can be captured in a CUDA graph; with
    a ParamGroup the update is one fused kernel over the flat buffers."""

    def __init__(self, params, lr=1e-2, betas=(0.9, 0.999), eps=1e-8, group=None,
                 grad_unscale=1.0):
        self.params = list(params)
        self.lr, self.betas, self.eps = lr, betas, eps
        self.grad_unscale = float(grad_unscale)
        self.group = group
        if group is not None:
            self.m = torch.zeros_like(group.master)
            self.v = torch.zeros_like(group.master)
        else:
            self.m = [torch.zeros_like(p.master) for p in self.params]
            self.v = [torch.zeros_like(p.master) for p in self.params]
        dev = self.params[0].master.device if self.params else "cpu"
        self._t = torch.zeros((), dtype=torch.float64, device=dev)
        self._done = None
        self.t = 0

    @torch.no_grad()
    def step(self, flat_grad=None):
        """flat_grad: optional gradient for the whole group (e.g. all-reduced fp32)."""
        self.t += 1
        b1, b2 = self.betas
        g = self.group
        if g is not None and g.master.is_cuda and (flat_grad is not None or g.check_grads()):
            grad = g.grad if flat_grad is None else flat_grad
            # the kernel also advances the device step count, publishes the next
            # step's weights (and their transposed copies) and clears the
            # gradient (ParamGroup.publish fused away: g.fresh)
            if self._done is None:
                self._done = torch.zeros(1, dtype=torch.int32, device=g.master.device)
            D.adam_step(g.master, self.m, self.v, grad, self.lr, b1, b2, self.eps, self._t,
                        self.grad_unscale, pub=g.pub, grad_zero=g.grad, step_done=self._done,
                        transposed=g.transposed, pub_t=g.pub_t)
            g.fresh = True
            return
        self._t.add_(1.0)
        if flat_grad is not None:
            for o, p in zip(_offsets(self.params), self.params):
                p.published.grad = flat_grad[o:o + p.master.numel()].view(p.master.shape)
        c1 = (1.0 - torch.pow(b1, self._t)).float()
        c2 = (1.0 - torch.pow(b2, self._t)).float()
        ms = self.m if g is None else [self.m[o:o + p.master.numel()]
                                       for o, p in zip(_offsets(self.params), self.params)]
        vs = self.v if g is None else [self.v[o:o + p.master.numel()]
                                       for o, p in zip(_offsets(self.params), self.params)]
        for p, m, v in zip(self.params, ms, vs):
            grad = p.grad32().reshape(m.shape)
            if self.grad_unscale != 1.0:
                grad = grad * self.grad_unscale
            m.add_((1 - b1) * (grad - m))
            v.add_((1 - b2) * (grad * grad - v))
            p.master.sub_((self.lr * (m / c1) / (torch.sqrt(v / c2) + self.eps)).view(p.master.shape))


def _offsets(params):
    """Start of each parameter in a ParamGroup's flat buffers (8-element aligned)."""
    out, o = [], 0
    for p in params:
        out.append(o)
        o += (p.master.numel() + 7) // 8 * 8
    return out


@dataclass
class TrainConfig:
    kind: str = "gcn"
    mode: str = "half"
    epochs: int = 200
    hidden: int = 16
    lr: float = 1e-2
    seed: int = 0
    width: str = "half2"
    scaling: str = "discretized"
    norm: str = "both"
    lam: float = 0.1
    val_fraction: float = 0.2
    # builder extensions
    numerics: str = "fast"
    # static power-of-two loss scale (1 = the reference; "auto" = the largest
    # power of two <= N/64).  The reference's mean-over-N loss gradient
    # (p - y)/N lands in fp16 subnormals for N ~ 1e5 (models.py:566-570);
    # scaling it by 2^k keeps it normal and Adam unscales exactly in fp32.
    grad_scale: float | str = 1.0
    heads: int = 1
    layers: int = 2
    device: str = "cuda"


@dataclass
class TrainResult:
    train_acc: float
    val_acc: float
    losses: list
    trace: list
    conversions: ConversionCounter
    overflow: OverflowCounters
    logits: torch.Tensor | None = field(default=None, repr=False)

    def write_trace(self, path):
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["epoch", "loss", "train_acc", "val_acc", "inf_count", "nan_count"])
            w.writerows(self.trace)


def accuracy(logits, labels, mask, n_active=None):
    if isinstance(logits, torch.Tensor):
        if not bool(mask.any()):
            return 0.0
        pred = logits[mask][:, : n_active or logits.shape[1]].argmax(dim=1)
        return float((pred == labels[mask]).float().mean())
    if not mask.any():
        return 0.0
    pred = logits[mask][:, : n_active or logits.shape[1]].argmax(axis=1)
    return float((pred == labels[mask]).mean())


def resolve_grad_scale(spec, n):
    """grad_scale value: a power of two >= 1, or "auto" -> largest 2^k <= n/64."""
    if spec == "auto":
        return float(2 ** max(0, int(math.floor(math.log2(max(n, 1) / 64.0)))))
    s = float(spec)
    if s < 1.0 or math.frexp(s)[0] != 0.5:
        raise ValueError(f"grad_scale must be a power of two >= 1 or 'auto', got {spec!r}")
    return s


class Trainer:
    """Full-batch node classification state (models.train, models.py:633-684):
    model, optimiser, masks and device-resident inputs.  `step()` is one epoch
    (forward, loss, backward, Adam) with no host synchronisation."""

    def __init__(self, bundle, features, labels, config: TrainConfig, row_slice=None,
                 node_order=None):
        """node_order (new -> old vertex id, e.g. device.locality_order): the
        bundle's graph is the relabelled one (DeviceGraph.relabel); features and
        labels are given in the original ids and the train / validation split
        is drawn over the original ids, so every original vertex keeps its
        features, label and split."""
        self.cfg = config
        self.bundle = bundle
        dev = config.device
        rng = np.random.default_rng(config.seed)
        feats = features if isinstance(features, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(features))
        n, fan_in = feats.shape
        labels_t = labels if isinstance(labels, torch.Tensor) else torch.from_numpy(
            np.asarray(labels, dtype=np.int64))
        self.node_order = node_order
        if node_order is not None:
            order = torch.as_tensor(node_order, dtype=torch.int64)
            feats = feats[order.to(feats.device)]
            labels_t = labels_t[order.to(labels_t.device)]
        c = int(labels_t.max()) + 1
        self.n_cls = c + c % 2   # the reference harness pads odd class counts to even
        self.in_store = _round_store(fan_in)
        red = Reduction(config.scaling, config.norm)
        self.model = Model(config.kind, rng, (fan_in, config.hidden, self.n_cls), red,
                           config.lam, config.heads, config.layers, dev, self.in_store)
        self.group = ParamGroup(self.model.params(), config.mode)
        self.grad_scale = resolve_grad_scale(config.grad_scale, n)
        self.opt = Adam(self.model.params(), lr=config.lr, group=self.group,
                        grad_unscale=1.0 / self.grad_scale)
        perm = rng.permutation(n)
        val = np.zeros(n, dtype=bool)
        val[perm[: int(n * config.val_fraction)]] = True
        if node_order is not None:
            val = val[torch.as_tensor(node_order).cpu().numpy()]
        lo, hi = row_slice or (0, n)
        self.val_mask = torch.from_numpy(val[lo:hi]).to(dev)
        self.train_mask = ~self.val_mask
        self.labels = labels_t[lo:hi].to(dev).long()
        self.dtype = _DTYPES[config.mode]
        self.x = self.load_features(feats[lo:hi])
        self.conversions = ConversionCounter()
        self._graph = None
        self._graph_out = None

    def load_features(self, feats, out=None):
        """Round to the compute dtype (via fp32, as models.train does) and pad
        columns to the 8-aligned storage width; `out` reuses a buffer."""
        n, f = feats.shape
        if out is None:
            out = torch.zeros((n, self.in_store), dtype=self.dtype, device=self.cfg.device)
        src = feats.to(self.cfg.device, non_blocking=True)
        out[:, :f] = src.to(torch.float32).to(self.dtype) if src.dtype != self.dtype else src
        return out

    def step(self, overflow=None):
        if self._graph is not None and overflow is None:
            self._graph.replay()
            return self._graph_out
        return self._step_eager(overflow)

    def _step_eager(self, overflow=None):
        cfg = self.cfg
        self.group.publish_if_stale()
        logits = self.model.forward(self.bundle, self.x, cfg.mode, cfg.width, overflow)
        loss = self.loss_backward(logits, D.softmax_xent, logits.shape[0])
        self.opt.step()
        return loss, logits.detach()

    def loss_backward(self, logits, xent, denom):
        """convert(logits, "float32") -> cross_entropy -> backward, fused: one
        kernel reads the compute-dtype logits, returns the per-row nll and the
        loss gradient already in the logits' dtype (the rounding convert's
        backward applies), scaled by grad_scale; autograd continues from the
        logits.  Counts the two conversions the reference performs."""
        nll, grad = xent(logits.detach(), self.labels, self.n_cls, denom,
                         scale=self.grad_scale, grad_dtype=logits.dtype)
        if self.cfg.mode == "half":
            self.conversions.forward += 1
            self.conversions.backward += 1
        loss = D.loss_mean(nll, denom) if nll.is_cuda else (nll.sum() / denom).float()
        torch.autograd.backward(logits, grad)
        return loss

    def capture(self, warmup=0, double_buffer=True):
        """Record one training step (forward, backward, Adam) as a CUDA graph;
        later step() calls replay it (one launch per epoch).  Call after at
        least one eager step (schedules, workspaces and cuBLAS state exist);
        capturing does not advance training, `warmup` extra side-stream steps
        do.  With double_buffer a second graph reads a second input buffer, so
        run_epochs can copy the next epoch's features while one computes."""
        if warmup:
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                for _ in range(warmup):
                    self._step_eager()
            torch.cuda.current_stream().wait_stream(side)
        bufs = [self.x] + ([torch.empty_like(self.x)] if double_buffer else [])
        graphs = []
        pool = None
        for b in bufs:
            self.x = b
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, pool=pool):
                out = self._step_eager()
            pool = graph.pool()
            graphs.append((graph, out, b))
        self.x = bufs[0]
        self._graphs = graphs
        self._graph, self._graph_out = graphs[0][0], graphs[0][1]
        return graphs[0][0]

    def host_features(self, feats):
        """Pinned host copy of the features in the device storage layout
        (compute dtype, columns padded to the 8-aligned width)."""
        f = feats if isinstance(feats, torch.Tensor) else torch.from_numpy(np.asarray(feats))
        n, w = f.shape
        host = torch.zeros((n, self.in_store), dtype=self.dtype).pin_memory()
        host[:, :w] = f.to(torch.float32).to(self.dtype) if f.dtype != self.dtype else f
        return host

    def run_epochs(self, host_x, epochs, check_loss=True):
        """Train `epochs` epochs feeding the inputs from pinned host memory every
        epoch: the next epoch's host->device copy runs on a side stream while
        the current epoch computes (double-buffered), and the loss is read back
        and checked every epoch like models.train.  Uses the captured graphs
        when capture(double_buffer=True) was called.  Returns the losses."""
        cur_stream = torch.cuda.current_stream()
        copy_stream = torch.cuda.Stream()
        graphs = getattr(self, "_graphs", None)
        if graphs is not None and len(graphs) == 2:
            bufs = [graphs[0][2], graphs[1][2]]
        else:
            graphs = None
            bufs = [self.x, torch.empty_like(self.x)]
        copied = [torch.cuda.Event(), torch.cuda.Event()]
        used = [torch.cuda.Event(), torch.cuda.Event()]
        copy_stream.wait_stream(cur_stream)
        with torch.cuda.stream(copy_stream):
            bufs[0].copy_(host_x, non_blocking=True)
            copied[0].record()
        losses = []
        for i in range(epochs):
            cur, nxt = i % 2, 1 - i % 2
            if i + 1 < epochs:
                with torch.cuda.stream(copy_stream):
                    if i >= 1:
                        copy_stream.wait_event(used[nxt])
                    bufs[nxt].copy_(host_x, non_blocking=True)
                    copied[nxt].record()
            cur_stream.wait_event(copied[cur])
            if graphs is not None:
                graphs[cur][0].replay()
                loss = graphs[cur][1][0]
            else:
                self.x = bufs[cur]
                loss, _ = self._step_eager()
            used[cur].record()
            if check_loss:
                lv = float(loss)
                if not math.isfinite(lv):
                    raise NanLossError(i, OverflowCounters())
                losses.append(lv)
        self.x = bufs[0]
        return losses


def train(g, features, labels, config: TrainConfig) -> TrainResult:
    """Full-batch node classification; raises NanLossError on a non-finite loss."""
    bundle = g if isinstance(g, GraphBundle) else GraphBundle.build(g, numerics=config.numerics)
    tr = Trainer(bundle, features, labels, config)
    overflow = OverflowCounters()
    trace, losses = [], []
    train_acc = val_acc = 0.0
    if config.epochs == 0:
        with torch.no_grad():
            logits = tr.model.forward(bundle, tr.x, config.mode, config.width, overflow)
            if config.mode == "half":
                logits = convert(logits, "float32", tr.conversions)
        return TrainResult(accuracy(logits, tr.labels, tr.train_mask, tr.n_cls),
                           accuracy(logits, tr.labels, tr.val_mask, tr.n_cls), [], [],
                           tr.conversions, overflow, logits)
    logits = None
    for epoch in range(config.epochs):
        overflow.reset()
        loss, logits = tr.step(overflow)
        lv = float(loss)
        if not math.isfinite(lv):
            raise NanLossError(epoch, overflow)
        train_acc = accuracy(logits, tr.labels, tr.train_mask, tr.n_cls)
        val_acc = accuracy(logits, tr.labels, tr.val_mask, tr.n_cls)
        n_inf, n_nan = overflow.totals()
        losses.append(lv)
        trace.append([epoch, lv, train_acc, val_acc, n_inf, n_nan])
    if logits is not None:
        logits = logits.float()  # the fp32 logits the reference's convert produced
    return TrainResult(train_acc, val_acc, losses, trace, tr.conversions, overflow, logits)
