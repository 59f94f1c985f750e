"""Per-op kernel API on CUDA tensors — the reference's kernel functions
(pkg/src/modelmerge/engine.py:122-420), same names, keyword attributes and
error behaviour (ShapeError on bad operands), each one call into the sm_100a
C-ABI library. Outputs are fresh contiguous tensors; inputs are never
mutated (engine.py:554 contract). No CPU fallback: a host tensor raises.

``mode`` selects arithmetic: "fast" (tensor cores / FMA) or "exact" (the
reference's accumulation order, bit-identical for matmul / conv / BN / pools
/ add / mul in f32).
"""

from __future__ import annotations

import ctypes
import math

import torch

from . import _lib
from .errors import ShapeError, UnsupportedOpError
from .ir import MergeDim, channel_axis, conv_output_extent, pool_output_extent

_DT = {torch.float32: _lib.NF_F32, torch.bfloat16: _lib.NF_BF16}
_MODES = {"fast": _lib.NF_MODE_FAST, "exact": _lib.NF_MODE_EXACT}
_ACTS = {None: _lib.NF_ACT_NONE, "relu": _lib.NF_ACT_RELU, "gelu": _lib.NF_ACT_GELU,
         "tanh": _lib.NF_ACT_TANH}


def dtype_code(t: torch.Tensor) -> int:
    code = _DT.get(t.dtype)
    if code is None:
        raise UnsupportedOpError(f"no sm_100a kernel for dtype {t.dtype}")
    return code


def _cuda(*ts: torch.Tensor | None) -> None:
    for t in ts:
        if t is not None and not t.is_cuda:
            raise UnsupportedOpError("merged-operator kernels run on CUDA tensors only "
                                     "(no CPU fallback)")


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: torch.Tensor | None):
    return None if t is None else t.data_ptr()


def _f32(v: torch.Tensor | None) -> torch.Tensor | None:
    return None if v is None else v.to(torch.float32).contiguous()


# ---------------------------------------------------------------------------
# Linear
# ---------------------------------------------------------------------------

def linear_launch(x: torch.Tensor, w: torch.Tensor, bias: torch.Tensor | None,
                  residual: torch.Tensor | None, y: torch.Tensor, groups: int, rows: int,
                  k: int, n: int, w_layout: int, act: int, mode: int, stream: int) -> None:
    _lib.call("nf_grouped_linear", x.data_ptr(), w.data_ptr(), _ptr(bias), _ptr(residual),
              y.data_ptr(), groups, rows, k, n, dtype_code(x), w_layout, act, mode, stream)


def batch_matmul(x: torch.Tensor, w: torch.Tensor, bias: torch.Tensor | None = None, *,
                 act: str | None = None, mode: str = "fast") -> torch.Tensor:
    """Merged Linear (engine.py:215-235): x (B, ..., D_in), w (B, D_in, D_out)."""
    _cuda(x, w, bias)
    if w.dim() != 3 or x.dim() < 2 or x.shape[0] != w.shape[0] or x.shape[-1] != w.shape[1]:
        raise ShapeError(f"batch matmul operands incompatible: {tuple(x.shape)} vs "
                         f"{tuple(w.shape)}")
    if x.dtype != w.dtype:
        raise ShapeError(f"dtype mismatch: input {x.dtype} vs weight {w.dtype}")
    g, d_in, d_out = w.shape
    if bias is not None and tuple(bias.shape) != (g, d_out):
        raise ShapeError(f"bias {tuple(bias.shape)} != ({g}, {d_out})")
    rows = x[0].numel() // d_in
    y = torch.empty(x.shape[:-1] + (d_out,), dtype=x.dtype, device=x.device)
    xc = x.contiguous()
    m = _MODES[mode]
    if m == _lib.NF_MODE_FAST and x.dtype == torch.bfloat16:
        wk, layout = w.transpose(1, 2).contiguous(), _lib.NF_W_NK
    else:
        wk, layout = w.contiguous(), _lib.NF_W_KN
    linear_launch(xc, wk, _f32(bias), None, y, g, rows, d_in, d_out, layout, _ACTS[act], m,
                  stream_ptr())
    return y


def matmul(x: torch.Tensor, w: torch.Tensor, bias: torch.Tensor | None = None, *,
           act: str | None = None, mode: str = "fast") -> torch.Tensor:
    """Dense layer (engine.py:194-212): contract x's last axis with w (D_in, D_out)."""
    _cuda(x, w, bias)
    if w.dim() != 2 or x.shape[-1] != w.shape[0]:
        raise ShapeError(f"matmul operands incompatible: {tuple(x.shape)} vs {tuple(w.shape)}")
    if bias is not None and tuple(bias.shape) != (w.shape[1],):
        raise ShapeError(f"bias {tuple(bias.shape)} != ({w.shape[1]},)")
    y = batch_matmul(x.reshape(1, -1, x.shape[-1]), w.unsqueeze(0),
                     None if bias is None else bias.unsqueeze(0), act=act, mode=mode)
    return y.reshape(x.shape[:-1] + (w.shape[1],))


# ---------------------------------------------------------------------------
# Norms and softmax
# ---------------------------------------------------------------------------

def _row_geometry(t: torch.Tensor, ca: int) -> tuple[int, int, int, int]:
    """(R1, R2, s1, s2) covering every index of ``t`` except axis ``ca``,
    for a contiguous tensor: rows before the channel axis x rows after."""
    shape = list(t.shape)
    before = math.prod(shape[:ca])
    after = math.prod(shape[ca + 1:])
    return before, after, shape[ca] * after, 1


def group_norm(x: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor, *, groups: int,
               eps: float, residual: torch.Tensor | None = None) -> torch.Tensor:
    """Merged LayerNorm (engine.py:263-284) over the channel axis."""
    _cuda(x, gamma, beta, residual)
    ca = channel_axis(x.dim())
    c = x.shape[ca]
    if groups < 1 or c % groups:
        raise ShapeError(f"groups {groups} does not divide channels {c}")
    if tuple(gamma.shape) != (c,) or tuple(beta.shape) != (c,):
        raise ShapeError(f"gamma/beta must be ({c},), got {tuple(gamma.shape)} and "
                         f"{tuple(beta.shape)}")
    if residual is not None and (tuple(residual.shape) != tuple(x.shape)
                                 or residual.dtype != x.dtype or residual.device != x.device):
        raise ShapeError(f"residual {tuple(residual.shape)}/{residual.dtype}/{residual.device} "
                         f"must match x {tuple(x.shape)}/{x.dtype}/{x.device}")
    xc = x.contiguous()
    rc = None if residual is None else residual.contiguous()
    y = torch.empty_like(xc)
    r1, r2, s1, s2 = _row_geometry(xc, ca)
    inner = math.prod(xc.shape[ca + 1:])
    cg = c // groups
    _lib.call("nf_group_norm", xc.data_ptr(), _ptr(rc), _f32(gamma).data_ptr(),
              _f32(beta).data_ptr(), y.data_ptr(), r1, r2, s1, s2, groups, cg, cg * inner, inner,
              0, float(eps), dtype_code(xc), stream_ptr())
    return y


def layer_norm(x: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor, *, eps: float,
               residual: torch.Tensor | None = None) -> torch.Tensor:
    """engine.py:246-260 (== group_norm with one group)."""
    return group_norm(x, gamma, beta, groups=1, eps=eps, residual=residual)


def softmax(x: torch.Tensor, *, axis: int) -> torch.Tensor:
    """engine.py:313-319."""
    _cuda(x)
    if not -x.dim() <= axis < x.dim():
        raise ShapeError(f"softmax axis {axis} out of range for rank {x.dim()}")
    ax = axis % x.dim()
    xc = x.contiguous()
    y = torch.empty_like(xc)
    outer = math.prod(xc.shape[:ax])
    inner = math.prod(xc.shape[ax + 1:])
    L = xc.shape[ax]
    _lib.call("nf_softmax", xc.data_ptr(), y.data_ptr(), outer, L, inner, L * inner, inner, 1,
              dtype_code(xc), stream_ptr())
    return y


def batch_norm_inference(x: torch.Tensor, gamma, beta, running_mean, running_var, *,
                         eps: float) -> torch.Tensor:
    """engine.py:287-302."""
    _cuda(x, gamma, beta, running_mean, running_var)
    ca = channel_axis(x.dim())
    c = x.shape[ca]
    for name, v in (("gamma", gamma), ("beta", beta), ("running_mean", running_mean),
                    ("running_var", running_var)):
        if tuple(v.shape) != (c,):
            raise ShapeError(f"{name} must be ({c},), got {tuple(v.shape)}")
    if bool((running_var < 0).any()):
        raise ShapeError("running_var has negative entries")
    xc = x.contiguous()
    y = torch.empty_like(xc)
    _lib.call("nf_batch_norm", xc.data_ptr(), _f32(gamma).data_ptr(), _f32(beta).data_ptr(),
              _f32(running_mean).data_ptr(), _f32(running_var).data_ptr(), y.data_ptr(),
              math.prod(xc.shape[:ca]), c, math.prod(xc.shape[ca + 1:]), float(eps),
              dtype_code(xc), stream_ptr())
    return y


# ---------------------------------------------------------------------------
# Elementwise, pooling, attention
# ---------------------------------------------------------------------------

def _ew(op: int, a: torch.Tensor, b: torch.Tensor | None = None) -> torch.Tensor:
    _cuda(a, b)
    ac = a.contiguous()
    bc = None if b is None else b.contiguous()
    y = torch.empty_like(ac)
    _lib.call("nf_elementwise", op, ac.data_ptr(), _ptr(bc), y.data_ptr(), ac.numel(),
              dtype_code(ac), stream_ptr())
    return y


def add(x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
    """engine.py:322-325."""
    if x.shape != y.shape or x.dtype != y.dtype:
        raise ShapeError(f"add operands differ: {tuple(x.shape)}/{x.dtype} vs "
                         f"{tuple(y.shape)}/{y.dtype}")
    return _ew(_lib.NF_EW_ADD, x, y)


def mul(x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
    """engine.py:328-331."""
    if x.shape != y.shape or x.dtype != y.dtype:
        raise ShapeError(f"mul operands differ: {tuple(x.shape)}/{x.dtype} vs "
                         f"{tuple(y.shape)}/{y.dtype}")
    return _ew(_lib.NF_EW_MUL, x, y)


def relu(x: torch.Tensor) -> torch.Tensor:
    return _ew(_lib.NF_EW_RELU, x)


def tanh(x: torch.Tensor) -> torch.Tensor:
    return _ew(_lib.NF_EW_TANH, x)


def gelu(x: torch.Tensor) -> torch.Tensor:
    return _ew(_lib.NF_EW_GELU, x)


def _pool(kind: int, x: torch.Tensor, kernel: int, stride: int, padding: int) -> torch.Tensor:
    _cuda(x)
    if x.dim() != 4:
        raise ShapeError(f"pool wants rank 4, got {tuple(x.shape)}")
    n, c, h, w = x.shape
    ho, wo = pool_output_extent(h, kernel, stride, padding), \
        pool_output_extent(w, kernel, stride, padding)
    xc = x.contiguous()
    y = torch.empty((n, c, ho, wo), dtype=x.dtype, device=x.device)
    _lib.call("nf_pool2d", xc.data_ptr(), y.data_ptr(), n, c, h, w, kind, kernel, stride,
              padding, dtype_code(xc), stream_ptr())
    return y


def max_pool2d(x: torch.Tensor, *, kernel: int, stride: int, padding: int = 0) -> torch.Tensor:
    """engine.py:334-349 (+ padding extension)."""
    return _pool(_lib.NF_POOL_MAX, x, kernel, stride, padding)


def mean_pool2d(x: torch.Tensor, *, kernel: int, stride: int, padding: int = 0) -> torch.Tensor:
    """engine.py:352-365 (+ padding extension)."""
    return _pool(_lib.NF_POOL_MEAN, x, kernel, stride, padding)


def attention(qkv: torch.Tensor, *, heads: int, scale: float | None = None,
              mode: str = "fast") -> torch.Tensor:
    """Merged self-attention over a fused QKV tensor (..., S, 3*D)."""
    _cuda(qkv)
    if qkv.dim() < 3 or qkv.shape[-1] % 3:
        raise ShapeError(f"attention wants (..., S, 3*D), got {tuple(qkv.shape)}")
    d = qkv.shape[-1] // 3
    if d % heads:
        raise ShapeError(f"heads {heads} does not divide width {d}")
    dh = d // heads
    s = qkv.shape[-2]
    bt = qkv.numel() // (s * 3 * d)
    xc = qkv.contiguous()
    y = torch.empty(qkv.shape[:-1] + (d,), dtype=qkv.dtype, device=qkv.device)
    sc = 1.0 / math.sqrt(dh) if scale is None else scale
    _lib.call("nf_attention", xc.data_ptr(), y.data_ptr(), bt, s, heads, dh, float(sc),
              dtype_code(xc), _MODES[mode], stream_ptr())
    return y


def rel_attention(qkv: torch.Tensor, r: torch.Tensor, r_w_bias: torch.Tensor,
                  r_r_bias: torch.Tensor, *, heads: int, scale: float | None = None,
                  mode: str = "fast") -> torch.Tensor:
    """XLNet relative attention; biases (H, dh) or per instance (M, H, dh)
    with qkv (M, ..., S, 3D)."""
    _cuda(qkv, r, r_w_bias, r_r_bias)
    d = qkv.shape[-1] // 3
    s = qkv.shape[-2]
    dh = d // heads
    if qkv.shape[-1] != 3 * d or r.shape[-1] != d or r.shape[-2] != 2 * s or d % heads:
        raise ShapeError(f"rel attention operands {tuple(qkv.shape)} / {tuple(r.shape)}")
    bt = qkv.numel() // (s * 3 * d)
    br = r.numel() // (2 * s * d)  # positional-key blocks, each shared by bt // br sequences
    if br < 1 or bt % br:
        raise ShapeError(f"positional keys {tuple(r.shape)} do not tile qkv {tuple(qkv.shape)}")
    rw = _f32(r_w_bias).reshape(-1, heads, dh)
    rr = _f32(r_r_bias).reshape(-1, heads, dh)
    if bt % rw.shape[0]:
        raise ShapeError("bias instances do not divide the sequences")
    y = torch.empty(qkv.shape[:-1] + (d,), dtype=qkv.dtype, device=qkv.device)
    sc = 1.0 / math.sqrt(dh) if scale is None else scale
    _lib.call("nf_rel_attention", qkv.contiguous().data_ptr(), r.contiguous().data_ptr(),
              rw.data_ptr(), rr.data_ptr(), y.data_ptr(), bt, s, heads, dh, bt // rw.shape[0],
              bt // br, float(sc), dtype_code(qkv), _MODES[mode], stream_ptr())
    return y


# ---------------------------------------------------------------------------
# Layout
# ---------------------------------------------------------------------------

def copy_strided(src: torch.Tensor, dst: torch.Tensor, stream: int | None = None) -> None:
    """dst[...] = src[...] for same-shape views with arbitrary strides."""
    if src.shape != dst.shape or src.dtype != dst.dtype:
        raise ShapeError("copy operands differ")
    if src.dim() > _lib.NF_MAX_RANK:
        raise UnsupportedOpError(f"rank {src.dim()} exceeds {_lib.NF_MAX_RANK}")
    rank = max(src.dim(), 1)
    arr = ctypes.c_int64 * rank
    dims = arr(*(src.shape or (1,)))
    ss = arr(*(src.stride() or (1,)))
    ds = arr(*(dst.stride() or (1,)))
    _lib.call("nf_copy_strided", src.data_ptr(), dst.data_ptr(), rank, dims, ss, ds,
              src.element_size(), stream_ptr() if stream is None else stream)


def contiguous(t: torch.Tensor) -> torch.Tensor:
    if t.is_contiguous():
        return t
    out = torch.empty(t.shape, dtype=t.dtype, device=t.device)
    copy_strided(t, out)
    return out


def pack(parts: list[torch.Tensor], *, dim: MergeDim) -> torch.Tensor:
    """engine.py:380-397: model-major packing (channel concat / batch stack)."""
    first = parts[0]
    for p in parts[1:]:
        if p.shape != first.shape or p.dtype != first.dtype:
            raise ShapeError("pack operands must agree in shape and dtype")
    _cuda(*parts)
    m = len(parts)
    if dim is MergeDim.CHANNEL:
        ca = channel_axis(first.dim())
        shape = list(first.shape)
        shape[ca] *= m
        out = torch.empty(shape, dtype=first.dtype, device=first.device)
        for j, p in enumerate(parts):
            copy_strided(p, out.narrow(ca, j * first.shape[ca], first.shape[ca]))
        return out
    if first.dim() == 4:
        out = torch.empty((m * first.shape[0],) + tuple(first.shape[1:]), dtype=first.dtype,
                          device=first.device)
        for j, p in enumerate(parts):
            copy_strided(p, out.narrow(0, j * first.shape[0], first.shape[0]))
        return out
    out = torch.empty((m,) + tuple(first.shape), dtype=first.dtype, device=first.device)
    for j, p in enumerate(parts):
        copy_strided(p, out[j])
    return out


def unpack(x: torch.Tensor, count: int, *, dim: MergeDim, stacked: bool) -> list[torch.Tensor]:
    """engine.py:400-420: pack's inverse, fresh contiguous slices."""
    if dim is MergeDim.CHANNEL:
        ca = channel_axis(x.dim())
        if x.shape[ca] % count:
            raise ShapeError(f"count {count} does not divide channels {x.shape[ca]}")
        c = x.shape[ca] // count
        return [contiguous(x.narrow(ca, j * c, c)) for j in range(count)]
    if stacked:
        if x.shape[0] != count:
            raise ShapeError(f"model axis {x.shape[0]} != count {count}")
        return [contiguous(x[j]) for j in range(count)]
    if x.shape[0] % count:
        raise ShapeError(f"count {count} does not divide batch {x.shape[0]}")
    b = x.shape[0] // count
    return [contiguous(x.narrow(0, j * b, b)) for j in range(count)]


# ---------------------------------------------------------------------------
# Convolution
# ---------------------------------------------------------------------------

def grouped_conv2d(x: torch.Tensor, w: torch.Tensor, bias: torch.Tensor | None = None, *,
                   groups: int, stride: int = 1, padding: int = 0,
                   mode: str = "fast") -> torch.Tensor:
    """Merged Conv2d (engine.py:155-191): NCHW, w (C_out, C_in/G, k, k)."""
    _cuda(x, w, bias)
    if x.dim() != 4 or w.dim() != 4:
        raise ShapeError(f"grouped_conv2d wants rank-4 operands, got {tuple(x.shape)} and "
                         f"{tuple(w.shape)}")
    if x.dtype != w.dtype:
        raise ShapeError(f"dtype mismatch: input {x.dtype} vs kernel {w.dtype}")
    n, c_in, h, wd = x.shape
    c_out, cg, k, k2 = w.shape
    if groups < 1 or c_in % groups or c_out % groups:
        raise ShapeError(f"groups {groups} does not divide channels ({c_in} in, {c_out} out)")
    if cg != c_in // groups or k != k2:
        raise ShapeError(f"kernel {tuple(w.shape)} incompatible with {c_in} channels in "
                         f"{groups} groups")
    if bias is not None and tuple(bias.shape) != (c_out,):
        raise ShapeError(f"bias {tuple(bias.shape)} != ({c_out},)")
    ho, wo = conv_output_extent(h, k, stride, padding), conv_output_extent(wd, k, stride, padding)
    xc, wc = x.contiguous(), w.contiguous()
    y = torch.empty((n, c_out, ho, wo), dtype=x.dtype, device=x.device)
    _lib.call("nf_grouped_conv2d", xc.data_ptr(), wc.data_ptr(), _ptr(_f32(bias)), None, None,
              y.data_ptr(), n, c_in, h, wd, c_out, k, stride, padding, groups, 0,
              dtype_code(xc), _MODES[mode], stream_ptr())
    return y


def conv2d(x: torch.Tensor, w: torch.Tensor, bias: torch.Tensor | None = None, *,
           stride: int = 1, padding: int = 0, mode: str = "fast") -> torch.Tensor:
    """engine.py:122-152 (== grouped_conv2d with one group)."""
    if x.dim() == 4 and w.dim() == 4 and w.shape[1] != x.shape[1]:
        raise ShapeError(f"kernel {tuple(w.shape)} incompatible with input {tuple(x.shape)}")
    return grouped_conv2d(x, w, bias, groups=1, stride=stride, padding=padding, mode=mode)
