"""Folded LayerNorm entry points (nf_grouped_linear_fold, nf_qkv_attention_fold)
against the oracle's unfused composition: producer Linear + residual writing
the norm's partial sums, consumers rebuilding LN(x) from the raw sum (as GEMM
activations, as a residual, and in the fused QKV + attention launch).
Tolerance: bf16 normwise 2e-2 (the fold skips one bf16 rounding of LN(x)).

Statistics are per 128-feature part (sum, centred M2) merged with Chan's
update, so the fold must stay accurate when the LayerNorm input has a large
mean relative to its spread (offset-mean stress: residual + c, c/std up to
~100): E[x^2] - mean^2 would lose the variance to cancellation there."""

import numpy as np
import pytest
import torch

from oracle import kernels as OK
from paper_2009_13062_b200 import _lib

pytestmark = pytest.mark.gpu


def normwise(got, want):
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-30))


def cuda(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)


def host(t):
    return t.float().cpu().numpy()


def _ln(x, gam, bet, eps):
    mu = x.mean(-1, keepdims=True)
    var = ((x - mu) ** 2).mean(-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps) * gam + bet


def _fold_w(w_nk, gam, bet, b):
    """W' = W * gamma over K (bf16), b' = b + W beta, colsum = sum_k W' (fp32)."""
    w2 = OK.bf16_round(w_nk * gam[:, None, :])
    b2 = b + np.einsum("gnk,gk->gn", w_nk, bet)
    return w2, b2.astype(np.float32), w2.sum(-1).astype(np.float32)


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _part_stats(y, parts):
    """(G, parts, T, 2): per 128-feature part, (sum, sum of (y - part mean)^2)."""
    g, t, n = y.shape
    yp = y.reshape(g, t, parts, n // parts).astype(np.float64)
    s = yp.sum(-1)
    m2 = ((yp - yp.mean(-1, keepdims=True)) ** 2).sum(-1)
    return np.stack([s, m2], -1).transpose(0, 2, 1, 3)


@pytest.mark.parametrize("G,T,K,N", [(3, 128, 256, 384), (2, 100, 768, 768), (1, 128, 3072, 768)])
@pytest.mark.parametrize("offset", [0.3, 10.0, 100.0])
def test_linear_fold_chain(G, T, K, N, offset):
    lib = _lib.load()
    assert lib.nf_linear_fold_supported(G, T, K, N) == 1
    rng = np.random.default_rng(G * 1000 + K)
    eps = 1e-12
    x = OK.bf16_round(rng.uniform(-1, 1, (G, T, K)).astype(np.float32))
    w1 = OK.bf16_round((rng.uniform(-1, 1, (G, N, K)) / np.sqrt(K)).astype(np.float32))
    b1 = rng.uniform(-.1, .1, (G, N)).astype(np.float32)
    r = OK.bf16_round(rng.uniform(-1, 1, (G, T, N)).astype(np.float32) + np.float32(offset))
    ws_need = int(lib.nf_linear_workspace_bytes(G, T, K, N))
    ws = torch.zeros(max(ws_need, 1), dtype=torch.uint8, device="cuda")
    wsp = ws.data_ptr() if ws_need > 0 else None
    parts = N // 128

    # 1) producer: y = x W1^T + b1 + r, with the per-token partial sums of y
    xt, w1t, b1t, rt = cuda(x, torch.bfloat16), cuda(w1, torch.bfloat16), cuda(b1), \
        cuda(r, torch.bfloat16)
    y = torch.empty(G, T, N, dtype=torch.bfloat16, device="cuda")
    stats = torch.zeros(G, parts, T, 2, device="cuda")
    for _ in range(2):  # split-K semaphores re-arm
        _lib.call("nf_grouped_linear_fold", xt.data_ptr(), K, T * K, w1t.data_ptr(),
                  b1t.data_ptr(), rt.data_ptr(), y.data_ptr(), N, T * N, G, T, K, N, 0, wsp,
                  ws_need, None, 0, None, 0.0, None, 0, None, None, 0.0, stats.data_ptr(),
                  _stream())
    torch.cuda.synchronize()
    want_y = np.einsum("gtk,gnk->gtn", x, w1) + b1[:, None, :] + r
    yh = host(y)
    assert normwise(yh, want_y) < 1e-2
    want_st = _part_stats(yh, parts)
    got_st = host(stats)
    np.testing.assert_allclose(got_st[..., 0], want_st[..., 0], rtol=1e-4,
                               atol=1e-3 * max(1.0, offset))
    np.testing.assert_allclose(got_st[..., 1], want_st[..., 1], rtol=1e-3, atol=1e-2)

    # 2) consumer of LN(y) as activations: z = LN(y) W2^T + b2
    N2 = 256
    gam = rng.uniform(.5, 1.5, (G, N)).astype(np.float32)
    bet = rng.uniform(-.5, .5, (G, N)).astype(np.float32)
    w2 = OK.bf16_round((rng.uniform(-1, 1, (G, N2, N)) / np.sqrt(N)).astype(np.float32))
    b2 = rng.uniform(-.1, .1, (G, N2)).astype(np.float32)
    wf, bf, cs = _fold_w(w2, gam, bet, b2)
    z = torch.empty(G, T, N2, dtype=torch.bfloat16, device="cuda")
    wft, bft, cst = cuda(wf, torch.bfloat16), cuda(bf), cuda(cs)
    _lib.call("nf_grouped_linear_fold", y.data_ptr(), N, T * N, wft.data_ptr(), bft.data_ptr(),
              None, z.data_ptr(), N2, T * N2, G, T, N, N2, 0, None, 0, stats.data_ptr(), parts,
              cst.data_ptr(), eps, None, 0, None, None, 0.0, None, _stream())
    torch.cuda.synchronize()
    h = _ln(yh, gam[:, None, :], bet[:, None, :], eps)
    want_z = np.einsum("gtk,gnk->gtn", OK.bf16_round(h), w2) + b2[:, None, :]
    assert normwise(host(z), want_z) < 2e-2

    # 3) LN(y) as the residual of another producer: u = x W1^T + b1 + LN(y)
    u = torch.empty_like(y)
    st2 = torch.zeros_like(stats)
    gt, bt = cuda(gam), cuda(bet)
    _lib.call("nf_grouped_linear_fold", xt.data_ptr(), K, T * K, w1t.data_ptr(), b1t.data_ptr(),
              y.data_ptr(), u.data_ptr(), N, T * N, G, T, K, N, 0, wsp, ws_need, None, 0, None,
              0.0, stats.data_ptr(), parts, gt.data_ptr(), bt.data_ptr(), eps, st2.data_ptr(),
              _stream())
    torch.cuda.synchronize()
    want_u = np.einsum("gtk,gnk->gtn", x, w1) + b1[:, None, :] + h
    assert normwise(host(u), want_u) < 2e-2


@pytest.mark.parametrize("offset", [0.2, 20.0])
def test_qkv_attention_fold(offset):
    rng = np.random.default_rng(5)
    g, heads = 2, 4
    d = 64 * heads
    eps = 1e-12
    x = OK.bf16_round(rng.uniform(-1, 1, (g, 128, d)).astype(np.float32) + np.float32(offset))
    gam = rng.uniform(.5, 1.5, (g, d)).astype(np.float32)
    bet = rng.uniform(-.5, .5, (g, d)).astype(np.float32)
    w = OK.bf16_round((rng.uniform(-1, 1, (g, 3 * d, d)) / np.sqrt(d)).astype(np.float32))
    b = rng.uniform(-.1, .1, (g, 3 * d)).astype(np.float32)
    h = OK.bf16_round(_ln(x, gam[:, None, :], bet[:, None, :], eps))
    qkv = OK.bf16_round(np.einsum("gtk,gnk->gtn", h, w) + b[:, None, :])
    want = np.stack([OK.attention(qkv[j], heads=heads) for j in range(g)])
    wf, bf, cs = _fold_w(w, gam, bet, b)
    stats = _part_stats(x, d // 128).astype(np.float32)  # (g, parts, 128, 2)
    wf = wf.reshape(g, 3, heads, 64, d).transpose(0, 2, 1, 3, 4).reshape(g, 3 * d, d)  # head-major
    xt, wt, bt, ct, stt = cuda(x, torch.bfloat16), cuda(wf, torch.bfloat16), cuda(bf), \
        cuda(cs), cuda(stats)
    y = torch.empty(g, 128, d, dtype=torch.bfloat16, device="cuda")
    _lib.call("nf_qkv_attention_fold", xt.data_ptr(), d, 128 * d, wt.data_ptr(), bt.data_ptr(),
              y.data_ptr(), g, 128, d, heads, 1.0 / 8.0, stt.data_ptr(), d // 128, ct.data_ptr(), eps,
              _stream())
    torch.cuda.synchronize()
    assert normwise(host(y), want) < 2e-2


def test_fold_rejected_where_not_implemented():
    lib = _lib.load()
    assert lib.nf_linear_fold_supported(2, 1024, 768, 200) == 0  # token-row tiles (large T)
    assert lib.nf_linear_fold_supported(2, 1024, 768, 768) == 0  # (separate TMA-ring norm)
    assert lib.nf_linear_fold_supported(2, 200, 768, 768) == 0   # swapped 256-token tiles
    assert lib.nf_linear_fold_supported(2, 128, 768, 200) == 0   # N not whole 128-feature parts
    stats = torch.zeros(2, 2, 1024, 2, device="cuda")
    x = torch.zeros(2, 1024, 768, dtype=torch.bfloat16, device="cuda")
    w = torch.zeros(2, 200, 768, dtype=torch.bfloat16, device="cuda")
    y = torch.empty(2, 1024, 200, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(Exception):
        _lib.call("nf_grouped_linear_fold", x.data_ptr(), 768, 1024 * 768, w.data_ptr(), None,
                  None, y.data_ptr(), 200, 1024 * 200, 2, 1024, 768, 200, 0, None, 0, None, 0,
                  None, 0.0, None, 0, None, None, 0.0, stats.data_ptr(), _stream())
