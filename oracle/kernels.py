"""CPU oracle kernels — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
arm may import this package, and only as the checker or the timed reference
CPU path — never as part of the GPU product path.

Each function restates one reference kernel of pkg/src/modelmerge/engine.py
(cited per function) with the same numpy arithmetic in the same order, so
results are bit-identical to the reference (pinned by tests/test_oracle.py
against the reference itself and the committed golden fixtures in
tests/golden/). Ops the reference cannot express (GELU, attention, padded
max-pool, XLNet relative attention) are restatements of their published
definitions; those are marked "parity unpinned by reference tests".
"""

from __future__ import annotations

import math

import numpy as np

try:  # scipy's erf for the exact-erf GELU; numpy fallback via math.erf
    from scipy.special import erf as _erf
except Exception:  # pragma: no cover
    _erf = np.vectorize(math.erf)

CHANNEL_AXIS = {2: 1, 3: 2, 4: 1}


class OracleShapeError(ValueError):
    pass


def _conv_extent(extent, k, stride, pad):
    padded = extent + 2 * pad
    if padded < k:
        raise OracleShapeError("kernel larger than padded extent")
    return (padded - k) // stride + 1


def _zero_pad(x, pad):
    if pad == 0:
        return x
    n, c, h, w = x.shape
    out = np.zeros((n, c, h + 2 * pad, w + 2 * pad), x.dtype)
    out[:, :, pad:pad + h, pad:pad + w] = x
    return out


def conv2d(x, w, bias=None, *, stride=1, padding=0):
    """engine.py:122-152. Accumulate c_in outer, then kernel row, kernel col;
    each term is one rounded multiply then one rounded add; bias after."""
    n, c_in, h, wd = x.shape
    c_out, kc, k, k2 = w.shape
    if kc != c_in or k != k2 or x.dtype != w.dtype:
        raise OracleShapeError(f"conv operands {x.shape} {w.shape}")
    ho, wo = _conv_extent(h, k, stride, padding), _conv_extent(wd, k, stride, padding)
    xp = _zero_pad(x, padding)
    y = np.zeros((n, c_out, ho, wo), x.dtype)
    for ci in range(c_in):
        for r in range(k):
            rows = slice(r, r + (ho - 1) * stride + 1, stride)
            for s in range(k):
                cols = slice(s, s + (wo - 1) * stride + 1, stride)
                y += w[:, ci, r, s].reshape(1, c_out, 1, 1) * xp[:, ci:ci + 1, rows, cols]
    if bias is not None:
        y = y + bias.reshape(1, c_out, 1, 1)
    return y


def grouped_conv2d(x, w, bias=None, *, groups, stride=1, padding=0):
    """engine.py:155-191. Output channel c reads input channels
    base(c) + [0, c_in/G) with base(c) = (c // (c_out/G)) * c_in/G; same
    (ci, kh, kw) term order as conv2d."""
    n, c_in, h, wd = x.shape
    c_out, cg, k, _ = w.shape
    if groups < 1 or c_in % groups or c_out % groups or cg != c_in // groups:
        raise OracleShapeError(f"grouped conv {x.shape} {w.shape} G={groups}")
    ho, wo = _conv_extent(h, k, stride, padding), _conv_extent(wd, k, stride, padding)
    xp = _zero_pad(x, padding)
    first = (np.arange(c_out) // (c_out // groups)) * cg
    y = np.zeros((n, c_out, ho, wo), x.dtype)
    for ci in range(cg):
        gathered = xp[:, first + ci, :, :]
        for r in range(k):
            rows = slice(r, r + (ho - 1) * stride + 1, stride)
            for s in range(k):
                cols = slice(s, s + (wo - 1) * stride + 1, stride)
                y += w[:, ci, r, s].reshape(1, c_out, 1, 1) * gathered[:, :, rows, cols]
    if bias is not None:
        y = y + bias.reshape(1, c_out, 1, 1)
    return y


def matmul(x, w, bias=None):
    """engine.py:194-212: contraction index ascending, bias added after."""
    if w.ndim != 2 or x.shape[-1] != w.shape[0] or x.dtype != w.dtype:
        raise OracleShapeError(f"matmul {x.shape} {w.shape}")
    y = np.zeros(x.shape[:-1] + (w.shape[1],), x.dtype)
    for kk in range(w.shape[0]):
        y += x[..., kk:kk + 1] * w[kk]
    return y if bias is None else y + bias


def batch_matmul(x, w, bias=None):
    """engine.py:215-235: per-leading-slice matmul, same contraction order."""
    if w.ndim != 3 or x.shape[0] != w.shape[0] or x.shape[-1] != w.shape[1]:
        raise OracleShapeError(f"batch matmul {x.shape} {w.shape}")
    b, d_in, d_out = w.shape
    bshape = (b,) + (1,) * (x.ndim - 2) + (d_out,)
    y = np.zeros(x.shape[:-1] + (d_out,), x.dtype)
    for kk in range(d_in):
        y += x[..., kk:kk + 1] * w[:, kk, :].reshape(bshape)
    return y if bias is None else y + bias.reshape(bshape)


def _per_channel(v, rank):
    shape = [1] * rank
    shape[CHANNEL_AXIS[rank]] = v.shape[0]
    return v.reshape(shape)


def layer_norm(x, gamma, beta, *, eps):
    """engine.py:246-260: population mean/var over the channel axis,
    d / sqrt(var + eps), then gamma * . + beta."""
    ax = CHANNEL_AXIS[x.ndim]
    c = x.dtype.type(x.shape[ax])
    mu = np.sum(x, axis=ax, keepdims=True) / c
    d = x - mu
    var = np.sum(d * d, axis=ax, keepdims=True) / c
    return _per_channel(gamma, x.ndim) * (d / np.sqrt(var + x.dtype.type(eps))) \
        + _per_channel(beta, x.ndim)


def group_norm(x, gamma, beta, *, groups, eps):
    """engine.py:263-284: statistics per contiguous channel group."""
    ax = CHANNEL_AXIS[x.ndim]
    c = x.shape[ax]
    if groups < 1 or c % groups:
        raise OracleShapeError(f"groups {groups} vs channels {c}")
    cg = c // groups
    xg = x.reshape(x.shape[:ax] + (groups, cg) + x.shape[ax + 1:])
    n = x.dtype.type(cg)
    mu = np.sum(xg, axis=ax + 1, keepdims=True) / n
    d = xg - mu
    var = np.sum(d * d, axis=ax + 1, keepdims=True) / n
    normed = (d / np.sqrt(var + x.dtype.type(eps))).reshape(x.shape)
    return _per_channel(gamma, x.ndim) * normed + _per_channel(beta, x.ndim)


def batch_norm_inference(x, gamma, beta, mean, var, *, eps):
    """engine.py:287-302: gamma * ((x - mean) / sqrt(var + eps)) + beta."""
    if np.any(var < 0):
        raise OracleShapeError("negative running variance")
    r = x.ndim
    den = np.sqrt(var + x.dtype.type(eps))
    return _per_channel(gamma, r) * ((x - _per_channel(mean, r)) / _per_channel(den, r)) \
        + _per_channel(beta, r)


def relu(x):
    """engine.py:305-306."""
    return np.maximum(x, x.dtype.type(0))


def tanh(x):
    """engine.py:309-310."""
    return np.tanh(x)


def gelu(x):
    """Restatement (not in the reference): 0.5 x (1 + erf(x / sqrt 2)), the
    transformers `hidden_act="gelu"`. Parity unpinned by reference tests."""
    xd = x.astype(np.float64)
    return (0.5 * xd * (1.0 + _erf(xd / math.sqrt(2.0)))).astype(x.dtype)


def softmax(x, *, axis):
    """engine.py:313-319: max-shifted exp, normalised by the sum."""
    e = np.exp(x - np.max(x, axis=axis, keepdims=True))
    return e / np.sum(e, axis=axis, keepdims=True)


def add(x, y):
    """engine.py:322-325."""
    if x.shape != y.shape or x.dtype != y.dtype:
        raise OracleShapeError("add operands differ")
    return x + y


def mul(x, y):
    """engine.py:328-331."""
    if x.shape != y.shape or x.dtype != y.dtype:
        raise OracleShapeError("mul operands differ")
    return x * y


def _pool_windows(x, kernel, stride, padding, fill):
    n, c, h, w = x.shape
    if padding:
        # Extension: torch MaxPool2d/AvgPool2d padding. Pads with `fill` on
        # every side; the output extent is the floor rule.
        xp = np.full((n, c, h + 2 * padding, w + 2 * padding), fill, x.dtype)
        xp[:, :, padding:padding + h, padding:padding + w] = x
        x = xp
        ho = (h + 2 * padding - kernel) // stride + 1
        wo = (w + 2 * padding - kernel) // stride + 1
    else:
        if h < kernel or w < kernel or (h - kernel) % stride or (w - kernel) % stride:
            raise OracleShapeError("pool windows overhang")  # ir.py:254-262
        ho, wo = (h - kernel) // stride + 1, (w - kernel) // stride + 1
    for r in range(kernel):
        for s in range(kernel):
            yield x[:, :, r:r + (ho - 1) * stride + 1:stride, s:s + (wo - 1) * stride + 1:stride]


def max_pool2d(x, *, kernel, stride, padding=0):
    """engine.py:334-349: running max over row-major window offsets. The
    padded variant (-inf pad) is a restatement of torch.nn.MaxPool2d for the
    ResNet stem; parity unpinned by reference tests."""
    y = None
    for win in _pool_windows(x, kernel, stride, padding, -np.inf):
        y = win.copy() if y is None else np.maximum(y, win)
    return y


def mean_pool2d(x, *, kernel, stride, padding=0):
    """engine.py:352-365: window sum in row-major offset order, then / k^2."""
    y = None
    for win in _pool_windows(x, kernel, stride, padding, 0.0):
        y = np.zeros(win.shape, x.dtype) + win if y is None else y + win
    return y / x.dtype.type(kernel * kernel)


def pack(parts, *, dim, stacked=None):
    """engine.py:380-397: model-major; channel -> concat on the channel axis;
    batch -> stack (rank < 4) or concat on axis 0 (rank 4)."""
    first = parts[0]
    if any(p.shape != first.shape or p.dtype != first.dtype for p in parts):
        raise OracleShapeError("pack operands differ")
    if dim == "channel":
        return np.concatenate(parts, axis=CHANNEL_AXIS[first.ndim])
    return np.concatenate(parts, 0) if first.ndim == 4 else np.stack(parts, 0)


def unpack(x, count, *, dim, stacked):
    """engine.py:400-420: pack's inverse."""
    if dim == "channel":
        return [np.ascontiguousarray(p) for p in np.split(x, count, axis=CHANNEL_AXIS[x.ndim])]
    if stacked:
        return [np.ascontiguousarray(x[m]) for m in range(count)]
    return [np.ascontiguousarray(p) for p in np.split(x, count, axis=0)]


def _heads(t, heads):
    """(..., S, D) -> (..., H, S, D/H)."""
    *lead, s, d = t.shape
    return np.swapaxes(t.reshape(*lead, s, heads, d // heads), -2, -3)


def _contract_last(a, b):
    """out[..., i, j] = sum_k a[..., i, k] * b[..., j, k], k ascending, one
    rounded multiply and add per term: the reference batch_matmul order with
    an activation as the weight operand."""
    out = np.zeros(a.shape[:-1] + (b.shape[-2],), a.dtype)
    for kk in range(a.shape[-1]):
        out += a[..., :, kk:kk + 1] * np.expand_dims(b[..., :, kk], -2)
    return out


def attention(qkv, *, heads, scale=None):
    """Restatement of BERT self-attention over a fused QKV projection
    (transformers BertSelfAttention, eager path): per head,
    softmax(Q K^T * scale) V with scale = 1/sqrt(d_head), composed from the
    reference's contraction order and `softmax` (engine.py:313-319).
    Parity unpinned by reference tests (the reference IR has no attention)."""
    d = qkv.shape[-1] // 3
    q, k, v = (_heads(qkv[..., i * d:(i + 1) * d], heads) for i in range(3))
    dh = d // heads
    sc = qkv.dtype.type(1.0 / math.sqrt(dh) if scale is None else scale)
    p = softmax(_contract_last(q, k) * sc, axis=-1)
    ctx = _contract_last(p, np.swapaxes(v, -1, -2))
    ctx = np.swapaxes(ctx, -2, -3)
    return np.ascontiguousarray(ctx.reshape(qkv.shape[:-1] + (d,)))


def rel_shift(bd, klen):
    """XLNet rel_shift_bnij (transformers modeling_xlnet.py:81-93) for
    qlen = klen: out[i, j] = raw[i, qlen - i + j]."""
    qlen = bd.shape[-2]
    idx = qlen - np.arange(qlen)[:, None] + np.arange(klen)[None, :]
    return np.take_along_axis(bd, np.broadcast_to(idx, bd.shape[:-2] + idx.shape), axis=-1)


def rel_attention(qkv, r, r_w_bias, r_r_bias, *, heads, scale=None):
    """Restatement of XLNet relative attention (modeling_xlnet.py:95-140,
    attn_type="bi", no segment term, no mask): AC = (q + r_w_bias) k^T,
    BD = rel_shift((q + r_r_bias) r^T), P = softmax((AC + BD) * scale), P v.
    qkv (..., S, 3D); r (..., 2S, D) are the projected positional keys.
    Parity unpinned by reference tests."""
    d = qkv.shape[-1] // 3
    s = qkv.shape[-2]
    q, k, v = (_heads(qkv[..., i * d:(i + 1) * d], heads) for i in range(3))
    kr = _heads(r, heads)
    dh = d // heads
    sc = qkv.dtype.type(1.0 / math.sqrt(dh) if scale is None else scale)
    rw = r_w_bias.reshape(r_w_bias.shape[:-2] + (heads, 1, dh)).astype(qkv.dtype)
    rr = r_r_bias.reshape(r_r_bias.shape[:-2] + (heads, 1, dh)).astype(qkv.dtype)
    ac = _contract_last(q + rw, k)
    bd = rel_shift(_contract_last(q + rr, kr), s)
    p = softmax((ac + bd) * sc, axis=-1)
    ctx = np.swapaxes(_contract_last(p, np.swapaxes(v, -1, -2)), -2, -3)
    return np.ascontiguousarray(ctx.reshape(qkv.shape[:-1] + (d,)))


def bf16_round(a):
    """Round fp32 values to the nearest bf16 (RNE), returned as fp32."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    rounded = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    out = rounded.astype(np.uint32).view(np.float32)
    return np.where(np.isnan(a), a, out)
