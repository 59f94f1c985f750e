"""First-contact GPU checks of the merged-Linear C-ABI entry point against a
plain fp32 torch reference (bf16 tensor-core path) and the exact SIMT path."""

import pytest
import torch

from paper_2009_13062_b200 import _lib

pytestmark = pytest.mark.gpu


def _call_linear(x, w_nk, bias, residual, y, act, mode, dtype_code, w_layout=_lib.NF_W_NK):
    G, T, K = x.shape
    N = y.shape[-1]
    _lib.call("nf_grouped_linear", x.data_ptr(), w_nk.data_ptr(),
              bias.data_ptr() if bias is not None else None,
              residual.data_ptr() if residual is not None else None,
              y.data_ptr(), G, T, K, N, dtype_code, w_layout, act, mode,
              torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("G,T,K,N", [(2, 128, 768, 768), (3, 64, 256, 384), (2, 512, 512, 1024),
                                     (1, 200, 320, 200), (4, 16, 128, 96), (2, 300, 192, 130),
                                     # CTA-pair tiles: persistent loop, partial pair tiles
                                     (8, 1024, 768, 1024), (3, 700, 256, 512),
                                     (8, 128, 3072, 768), (5, 100, 512, 1000),
                                     # N = 768 CTA-pair tiles, partial pair tiles
                                     (4, 512, 768, 768), (3, 700, 384, 1152),
                                     (32, 1024, 3072, 768)])
@pytest.mark.parametrize("act", [_lib.NF_ACT_NONE, _lib.NF_ACT_GELU])
def test_tc_linear_bf16_vs_torch(G, T, K, N, act):
    torch.manual_seed(0)
    dev = "cuda"
    x = (torch.rand(G, T, K, device=dev) * 2 - 1).bfloat16()
    w = ((torch.rand(G, N, K, device=dev) * 2 - 1) / K ** 0.5).bfloat16()
    b = (torch.rand(G, N, device=dev) - 0.5).float()
    r = (torch.rand(G, T, N, device=dev) - 0.5).bfloat16()
    y = torch.empty(G, T, N, device=dev, dtype=torch.bfloat16)
    _call_linear(x, w, b, r, y, act, _lib.NF_MODE_FAST, _lib.NF_BF16)
    torch.cuda.synchronize()
    # epilogue contract: y = act(x @ W + bias + residual)
    ref = torch.einsum("gtk,gnk->gtn", x.float(), w.float()) + b[:, None, :] + r.float()
    if act == _lib.NF_ACT_GELU:
        ref = torch.nn.functional.gelu(ref)
    err = (y.float() - ref).abs().max().item() / ref.abs().max().item()
    assert err < 2e-2, err


def test_exact_linear_f32_matches_sequential_order():
    torch.manual_seed(1)
    G, T, K, N = 2, 5, 37, 11
    x = torch.rand(G, T, K, device="cuda") * 2 - 1
    w_kn = torch.rand(G, K, N, device="cuda") - 0.5
    b = torch.rand(G, N, device="cuda") - 0.5
    y = torch.empty(G, T, N, device="cuda")
    _call_linear(x, w_kn, b, None, y, _lib.NF_ACT_NONE, _lib.NF_MODE_EXACT, _lib.NF_F32,
                 w_layout=_lib.NF_W_KN)
    torch.cuda.synchronize()
    import numpy as np
    xn, wn, bn = x.cpu().numpy(), w_kn.cpu().numpy(), b.cpu().numpy()
    ref = np.zeros((G, T, N), np.float32)
    for kk in range(K):  # engine.batch_matmul order (engine.py:229-230)
        ref += xn[..., kk:kk + 1] * wn[:, kk, :].reshape(G, 1, N)
    ref = ref + bn.reshape(G, 1, N)
    assert y.cpu().numpy().tobytes() == ref.tobytes()
