"""ctypes binding of libhalfgnn.so (the C ABI declared in include/halfgnn.h).

There is no fallback: if the library is missing or fails to load, every
operator raises.  Status codes map to Python exceptions the way the reference
raises them: HG_EINVAL -> ValueError (message from hg_last_error()),
HG_ECUDA -> RuntimeError.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import (POINTER, c_char_p, c_double, c_float, c_int, c_int32, c_int64, c_size_t,
                    c_void_p)
from pathlib import Path

# HG_LIB: an alternative build of the same library (A/B measurements of
# compile-time kernel variants, tools/exp/variants); default the in-tree build
LIB_PATH = Path(os.environ.get("HG_LIB") or Path(__file__).resolve().with_name("libhalfgnn.so"))

HG_OK, HG_EINVAL, HG_ECUDA = 0, 1, 2
ABI_VERSION = 6
HG_F16, HG_F32 = 0, 1
SCALING_CODES = {"post": 0, "pre": 1, "discretized": 2}
FACTOR_INV, FACTOR_INV_SQRT = 1, 2

_P = c_void_p
_I64 = c_int64
_I32 = c_int32
_PSZ = POINTER(c_size_t)
_PI64 = POINTER(c_int64)

# name -> argtypes (restype int unless listed in _RESTYPES)
SIGNATURES = {
    "hg_last_error": [],
    "hg_abi_version": [],
    "hg_build_csr_workspace": [_I64, _I64, _PSZ],
    "hg_build_csr": [_P, _P, _I64, _I64, _P, _P, _P, _PI64, _P, c_size_t, _P],
    "hg_transpose_workspace": [_I64, _I64, _PSZ],
    "hg_transpose": [_P, _P, _I64, _I64, _P, _P, _P, _P, c_size_t, _P],
    "hg_degree_factors": [_P, _I64, c_int, c_int, _P, _P],
    "hg_schedule_workspace": [_I64, _I64, _I32, _PSZ],
    "hg_schedule_build": [_P, _I64, _I32, _I32, _I32, _P, _I64, _P, _I64, _P, _I64, _PI64, _P,
                          c_size_t, _P],
    "hg_spmm_workspace": [_I64, _I32, _I64, c_int, _I32, c_int, _PSZ],
    "hg_spmm": [_P, _P, _I64, _I64, _I64, _P, _I64, _P, _I64, _I64, _P, _I64, _P, _P, _P, _I32,
                _P, _P,
                _I32, _I64, _I64, _I32, _I32, _P, _P, _I64, _I32, _P, c_int, _P, c_size_t, _P,
                _P, _P, _P, _I64, _P, c_double, _P, _P, _P, _P],
    "hg_spmm_edge_ref_workspace": [_I64, _I64, _I32, _I32, _I32, c_int, c_int, _PSZ],
    "hg_spmm_edge_ref": [_P, _P, _I64, _I64, _I64, _I32, _I32, _P, _P, _P, _I32, _I32, _P, _P,
                         _P, _P, c_int, _P, c_size_t, _P],
    "hg_spmm_vertex_ref_workspace": [_I64, _I32, c_int, c_int, _PSZ],
    "hg_spmm_vertex_ref": [_P, _P, _I64, _I64, _P, _P, _I32, _I32, _P, _P, _P, _P, _P, c_int,
                           _P, c_size_t, _P],
    "hg_gather_probe": [_P, _I64, _P, _I32, _I64, _P, _P],
    "hg_sddmm": [_P, _P, _I64, _I64, _P, _I64, _P, _P, _P, _I32, _I32, c_int, _P],
    "hg_sddmm_fast": [_P, _P, _I64, _I64, _P, _I64, _P, _I64, _P, _P, _P, _P, _I32, _I32, c_int,
                      _P],
    "hg_attn_scores": [_P, _P, _I64, _I64, _P, _P, _I32, c_double, _P, c_int, _P],
    "hg_edge_softmax_fwd": [_P, _I64, _I64, _P, _P, _I32, _P, _I64, _I64, c_int, _P],
    "hg_edge_softmax_bwd": [_P, _I64, _I64, _P, _P, _P, _I32, _P, _I64, _I64, c_int, _P],
    "hg_edge_rowsum": [_P, _I64, _I64, _P, _P, _I32, _P, _P, _I64, _I64, c_int, _P],
    "hg_scale_f64": [_P, c_double, _P, _I64, c_int, _P],
    "hg_softmax_xent": [_P, c_int, _I64, _P, _I64, _I32, c_double, c_float, _P, c_int, _P, _P],
    "hg_head_dots": [_P, _P, _P, _I64, _I32, _I32, _P, _P, c_int, _P],
    "hg_head_dots_bwd_workspace": [_I32, _I32, _PSZ],
    "hg_head_dots_bwd": [_P, _P, _P, _P, _P, _I64, _I32, _I32, _P, _P, _P, _P, c_int, _P, c_size_t,
                         _P],
    "hg_gemm_tc": [_P, _I64, _I64, _I64, _P, _I32, _I64, _P, _P, _I32, _P, _I64, _P],
    "hg_gemm_tc_dots": [_P, _I64, _I64, _I64, _P, _I32, _I64, _P, _I64, _P, _P, _I32, _P, _P,
                        _P],
    "hg_gemm_tc_masked": [_P, _I64, _I64, _I64, _P, _I32, _I64, _P, _I64, _P, _I64, _P],
    "hg_gemm_wgrad_workspace": [_I64, _I64, _I32, _PSZ],
    "hg_gemm_wgrad": [_P, _I64, _I64, _I64, _P, _I32, _I64, _P, _I64, _P, _I32, _P, c_size_t, _P],
    "hg_count_lines_workspace": [_I64, _PSZ],
    "hg_count_lines": [_P, _I64, _PI64, _P, c_size_t, _P],
    "hg_parse_edges_workspace": [_I64, _I64, _PSZ],
    "hg_parse_edges": [_P, _I64, _I64, _P, _P, _PI64, _P, c_size_t, _P],
    "hg_gat_attention_fwd": [_P, _P, _I64, _P, _P, _I32, c_float, _P, _I64, _P, _I64, _P, _I64,
                             _I32, c_int, _P],
    "hg_nccl_available": [],
    "hg_nccl_unique_id": [_P],
    "hg_nccl_comm_init": [_P, _I32, _P, _I32],
    "hg_nccl_comm_destroy": [_P],
    "hg_allgather_features": [_P, _P, _P, _P, _I32, _I32, _I64, _P],
    "hg_spmm_acc": [_P, _P, _I64, _I64, _I64, _P, _I64, _P, _I64, _I64, _P, _I64, _P, _P, _P,
                    _I32, _I64, _P, _P, _I32, _I64, _I64, _I32, _I32, _P, _P, _P, c_int, _P,
                    c_size_t, _P],
    "hg_gat_attention_stats": [_P, _P, _I64, _P, _P, _I32, c_float, _P, _P, _I64, _P, _I64,
                               _I32, c_int, _P],
    "hg_gat_aggregate": [_P, _P, _I64, _I64, _I64, _P, _I64, _P, _I64, _I64, _P, _I64, _P,
                         _P, _P, _P, c_float, _P, _I32, _P, _P, _I32, _I64, _I64, _I32, c_int,
                         _P, c_size_t, _P],
    "hg_gat_attention_bwd": [_P, _P, _I64, _P, _P, _I32, c_float, _P, _P, _P, _I64, _P, _P, _I64,
                             _P, _I64, _I32, c_int, _P],
    "hg_edge_sums_fast": [_P, _I64, _P, _P, _I32, _P, _P, _I64, _P, _I64, _I32, c_int, _P],
    "hg_head_mean": [_P, _I64, _I32, _I32, _P, c_int, _P],
    "hg_head_mean_bwd": [_P, _I64, _I32, _I32, _P, c_int, _P],
    "hg_scale_combine": [_P, _P, _P, c_double, _I64, _P, c_int, _P],
    "hg_scale_combine_bwd_workspace": [_PSZ],
    "hg_scale_combine_bwd": [_P, _P, _P, c_double, _I64, _P, _P, _P, c_int, _P, c_size_t, _P],
    "hg_relu_grad": [_P, _P, _I64, _P, c_int, _P],
    "hg_gather_rows": [_P, _P, _I64, _I32, _P, _P],
    "hg_bias_scale_rows": [_P, _P, _P, _I64, _I32, _P, c_int, _P],
    "hg_col_sums_workspace": [_I64, _I32, _PSZ],
    "hg_col_sums": [_P, _I64, _I32, _P, c_int, _P, c_size_t, _P],
    "hg_adam_step": [_P, _P, _P, _P, c_int, _I64, c_float, c_float, c_float, c_double, c_double,
                     c_float, _P, c_float, _P, _P, c_int, _P, _P, _I32, _P, _P],
    "hg_loss_mean_workspace": [_PSZ],
    "hg_loss_mean": [_P, _I64, c_double, _P, _P, c_size_t, _P],
}
_RESTYPES = {"hg_last_error": c_char_p}

_lib = None


class NativeLibraryMissing(ImportError):
    pass


def lib():
    """Load libhalfgnn.so once; raise loudly if it is absent."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise NativeLibraryMissing(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        handle = ctypes.CDLL(str(LIB_PATH))
        for name, argtypes in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.argtypes = argtypes
            fn.restype = _RESTYPES.get(name, c_int)
        if handle.hg_abi_version() != ABI_VERSION:
            raise NativeLibraryMissing("libhalfgnn.so ABI version mismatch")
        _lib = handle
    return _lib


def check(rc: int) -> None:
    if rc == HG_OK:
        return
    msg = (lib().hg_last_error() or b"").decode()
    if rc == HG_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"halfgnn CUDA failure: {msg}")


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def size_query(name: str, *args) -> int:
    out = c_size_t(0)
    check(getattr(lib(), name)(*args, ctypes.byref(out)))
    return int(out.value)
