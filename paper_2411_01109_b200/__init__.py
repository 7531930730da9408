"""B200-native (sm_100a) half-precision GNN hot path of HalfGNN (arXiv 2411.01109).

Drop-in for the hot-path subset of the reference package `halfsparse`: the same
names for graphs, schedules, sparse kernels, sparse autograd ops, layers and
the training loop, computed by hand-written CUDA in libhalfgnn.so (C ABI,
include/halfgnn.h).  The package imports without a GPU (host containers and
validation work everywhere); every operator raises if the CUDA library or the
device is missing -- there is no CPU fallback.
"""
from __future__ import annotations

__version__ = "0.1.0"

from .simt import (  # noqa: F401
    KernelMetrics,
    Schedule,
    SubWarpLayout,
    check_spmm_rules,
    feature_transactions,
    intra_cta_rounds,
    plan_edge_parallel,
    plan_vertex_grouped,
    sddmm_reduction_rounds,
    subwarp_layout,
    warp_load_bytes,
)
from .sparse import (  # noqa: F401
    CooGraph,
    CsrGraph,
    DenseTensor,
    add_self_loops,
    col_degrees,
    coo_to_csr,
    csr_to_coo,
    load_edge_list,
    load_tensor,
    pad_features,
    save_tensor,
    symmetrize,
    synth_sbm,
    transpose,
)
from .kernels import (  # noqa: F401
    Reduction,
    StagingBuffer,
    scalar_reference,
    sddmm,
    spmm_v,
    spmm_ve,
    spmm_vertex_grouped,
)

_MODELS = ("Adam", "ConversionCounter", "GraphBundle", "Model", "NanLossError",
           "OverflowCounters", "TrainConfig", "TrainResult", "Trainer", "accuracy",
           "cross_entropy", "edge_softmax", "shadow_div", "shadow_exp", "train",
           "spmm_agg", "spmm_weighted", "attention_scores", "attention_logits",
           "GCNLayer", "GINLayer", "GATLayer", "Linear", "Param")


def __getattr__(name):
    # models imports torch at module import; keep `import paper_2411_01109_b200` light
    if name in _MODELS:
        from . import models

        return getattr(models, name)
    raise AttributeError(name)


__all__ = [
    "KernelMetrics", "Schedule", "SubWarpLayout", "check_spmm_rules", "feature_transactions",
    "intra_cta_rounds", "plan_edge_parallel", "plan_vertex_grouped", "sddmm_reduction_rounds",
    "subwarp_layout", "warp_load_bytes", "CooGraph", "CsrGraph", "DenseTensor",
    "add_self_loops", "col_degrees", "coo_to_csr", "csr_to_coo", "load_edge_list",
    "load_tensor", "pad_features", "save_tensor", "symmetrize", "synth_sbm", "transpose",
    "Reduction", "StagingBuffer", "scalar_reference", "sddmm", "spmm_v", "spmm_ve",
    "spmm_vertex_grouped", *_MODELS,
]
