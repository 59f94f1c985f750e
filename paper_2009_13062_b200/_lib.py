"""ctypes binding of the C-ABI kernel library (include/netfuse_b200.h).

The library is built in-tree by :mod:`paper_2009_13062_b200.build`. There is
no fallback: if the shared object is missing or a CUDA device is absent, any
compute call raises. :func:`load` only opens the library (no device work), so
symbol checks run on CPU-only machines.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import ExecutionError, ShapeError, UnsupportedOpError

LIB_PATH = Path(__file__).resolve().parent / "libnetfuse_b200.so"
if os.environ.get("NF_LIB_PATH"):  # A/B experiments with alternative builds (tools/)
    LIB_PATH = Path(os.environ["NF_LIB_PATH"]).resolve()
HEADER_PATH = Path(__file__).resolve().parent.parent / "include" / "netfuse_b200.h"

NF_OK, NF_ERR_SHAPE, NF_ERR_UNSUPPORTED, NF_ERR_LAUNCH = 0, 1, 2, 3
NF_F32, NF_BF16 = 0, 1
NF_ACT_NONE, NF_ACT_RELU, NF_ACT_GELU, NF_ACT_TANH = 0, 1, 2, 3
NF_MODE_FAST, NF_MODE_EXACT = 0, 1
NF_W_NK, NF_W_KN = 0, 1
NF_EW_ADD, NF_EW_MUL, NF_EW_RELU, NF_EW_TANH, NF_EW_GELU = 0, 1, 2, 3, 4
NF_POOL_MAX, NF_POOL_MEAN = 0, 1
NF_CHAIN_KEEP_COUNTERS = 1
NF_MAX_RANK = 8

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i = ctypes.c_int
_f = ctypes.c_float

# name -> argtypes; must mirror include/netfuse_b200.h exactly.
SIGNATURES: dict[str, list] = {
    "nf_abi_version": [],
    "nf_status_string": [_i],
    "nf_grouped_linear": [_p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i, _i, _i, _i, _p],
    "nf_grouped_linear_strided": [_p, _i64, _i64, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64,
                                  _i64, _i, _i, _i, _i, _p],
    "nf_linear_workspace_bytes": [_i64, _i64, _i64, _i64],
    "nf_grouped_linear_ws": [_p, _i64, _i64, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64,
                             _i64, _i, _i, _i, _i, _p, _i64, _p],
    "nf_im2col_nhwc": [_p, _p] + [_i] * 10 + [_p],
    "nf_conv_nhwc_direct": [_p, _p, _p, _p, _p] + [_i] * 11 + [_p],
    "nf_pool2d_nhwc": [_p, _p] + [_i] * 9 + [_p],
    "nf_grouped_conv_tc": [_p, _p, _p, _p, _p] + [_i] * 11 + [_p, _i64, _p],
    "nf_conv_workspace_bytes": [_i] * 10,
    "nf_grouped_conv_tf32": [_p, _p, _p, _p, _p] + [_i] * 11 + [_p, _i64, _p],
    "nf_conv_tf32_workspace_bytes": [_i] * 10,
    "nf_qkv_attention": [_p, _i64, _i64, _p, _p, _p, _i64, _i64, _i64, _i64, _f, _p],
    "nf_linear_fold_supported": [_i64, _i64, _i64, _i64],
    "nf_grouped_linear_fold": [_p, _i64, _i64, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64,
                               _i64, _i, _p, _i64, _p, _i, _p, _f, _p, _i, _p, _p, _f, _p, _p],
    "nf_qkv_attention_fold": [_p, _i64, _i64, _p, _p, _p, _i64, _i64, _i64, _i64, _f,
                              _p, _i, _p, _f, _p],
    "nf_space_to_depth_stem": [_p, _p, _i, _i, _i, _i, _i, _p],
    "nf_linear_chain_supported": [_i64, _i64, _i64, _i64],
    "nf_linear_chain_counter_bytes": [_i, _i64],
    "nf_grouped_linear_chain": [_i, _p, _i64, _p, _p],
    "nf_linear_link_units": [_i64, _i64, _i64, _i64],
    "nf_conv_link_units": [_i] * 9,
    "nf_grouped_linear_linked": [_p, _i64, _i64, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64,
                                 _i64, _i, _p, _i64, _p, ctypes.c_uint32, _p, ctypes.c_uint32,
                                 _p, _i, _p],
    "nf_grouped_conv_tc_linked": [_p, _p, _p, _p, _p] + [_i] * 11 + [_p, _i64, _p,
                                  ctypes.c_uint32, _p, ctypes.c_uint32, _p, _i, _p],
    "nf_grouped_linear_chain_ex": [_i, _p, _i64, _p, _i, _p, ctypes.c_uint32, _p],
    "nf_qkv_attention_after": [_p, _i64, _i64, _p, _p, _p, _i64, _i64, _i64, _i64, _f,
                               _p, _i, _p, _f, _p, ctypes.c_uint32, _p, _p],
    "nf_grouped_conv2d": [_p, _p, _p, _p, _p, _p] + [_i64] * 5 + [_i] * 7 + [_p],
    "nf_elementwise": [_i, _p, _p, _p, _i64, _i, _p],
    "nf_copy_strided": [_p, _p, _i, _p, _p, _p, _i, _p],
    "nf_counters_rearm": [_p, _i64, _p],
    "nf_group_norm": [_p, _p, _p, _p, _p] + [_i64] * 9 + [_f, _i, _p],
    "nf_softmax": [_p, _p] + [_i64] * 6 + [_i, _p],
    "nf_attention": [_p, _p, _i64, _i64, _i64, _i64, _f, _i, _i, _p],
    "nf_rel_attention": [_p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64, _i64, _f, _i, _i,
                         _p],
    "nf_batch_norm": [_p, _p, _p, _p, _p, _p, _i64, _i64, _i64, _f, _i, _p],
    "nf_pool2d": [_p, _p, _i64, _i64, _i, _i, _i, _i, _i, _i, _i, _p],
}

_RESTYPES = {"nf_status_string": ctypes.c_char_p, "nf_linear_workspace_bytes": ctypes.c_int64,
             "nf_conv_workspace_bytes": ctypes.c_int64,
             "nf_conv_tf32_workspace_bytes": ctypes.c_int64,
             "nf_linear_chain_counter_bytes": ctypes.c_int64}


class LinearOp(ctypes.Structure):
    """`nf_linear_op` (include/netfuse_b200.h): one op of a chained launch."""
    _fields_ = [
        ("x", _p), ("x_ld", _i64), ("x_gs", _i64), ("w", _p), ("bias", _p), ("residual", _p),
        ("y", _p), ("y_ld", _i64), ("y_gs", _i64), ("rows", _i64), ("k", _i64), ("n", _i64),
        ("act", _i), ("workspace", _p), ("workspace_bytes", _i64),
        ("in_stats", _p), ("in_parts", _i), ("in_colsum", _p), ("in_eps", _f),
        ("res_stats", _p), ("res_parts", _i), ("res_gamma", _p), ("res_beta", _p),
        ("res_eps", _f), ("out_stats", _p),
    ]

_lib: ctypes.CDLL | None = None


def load() -> ctypes.CDLL:
    """Open the kernel library, building nothing; raise if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH.name} is not built; run `python -m paper_2009_13062_b200.build` "
            "(there is no CPU fallback for the merged operators)")
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, argtypes in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = _RESTYPES.get(name, ctypes.c_int)
    _lib = lib
    return lib


def check(status: int, what: str) -> None:
    """Map a C-ABI status to the reference's exception types."""
    if status == NF_OK:
        return
    lib = load()
    msg = f"{what}: {lib.nf_status_string(status).decode()}"
    if status == NF_ERR_SHAPE:
        raise ShapeError(msg)
    if status == NF_ERR_UNSUPPORTED:
        raise UnsupportedOpError(msg)
    raise ExecutionError(what, RuntimeError(msg))


def call(name: str, *args) -> None:
    """Invoke one C-ABI entry point and raise on a non-OK status."""
    check(getattr(load(), name)(*args), name)
