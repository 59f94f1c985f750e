"""nf_grouped_conv_tf32 (fp32 merged conv, 3xTF32 on tcgen05) against an
fp64 PyTorch conv of the same fp32 operands: normwise <= 2e-5 (one fp32
rounding of the folded result is ~6e-8; 3xTF32 products are ~2^-20)."""

import pytest
import torch
import torch.nn.functional as F

from paper_2009_13062_b200 import _lib

pytestmark = pytest.mark.gpu

CASES = [
    # N, H, W, G, cg, coutg, k, stride, pad, residual, relu
    (1, 224, 224, 2, 4, 64, 7, 2, 3, False, True),     # merged stem (RGB padded to 4)
    (1, 56, 56, 2, 64, 64, 3, 1, 1, False, True),      # layer1 3x3
    (1, 56, 56, 2, 64, 256, 1, 1, 0, True, True),      # 1x1 + residual
    (1, 28, 28, 2, 256, 128, 1, 2, 0, False, False),   # strided 1x1 downsample
    (1, 7, 7, 2, 512, 512, 3, 1, 1, False, True),      # layer4: split-K
    (1, 7, 7, 2, 512, 2048, 1, 1, 0, True, True),      # layer4 1x1 + residual, split-K
    (2, 9, 11, 3, 8, 20, 3, 2, 1, True, False),        # ragged, coutg % 32 != 0
]


def _run(N, H, W, G, cg, coutg, k, stride, pad, residual, relu, seed=0):
    gen = torch.Generator().manual_seed(seed)
    C, Cout = G * cg, G * coutg
    x = torch.rand(N, C, H, W, generator=gen) * 2 - 1
    w = (torch.rand(Cout, cg, k, k, generator=gen) * 2 - 1) / (cg * k * k) ** 0.5
    b = torch.rand(Cout, generator=gen) - 0.5
    ref = F.conv2d(x.double(), w.double(), b.double(), stride=stride, padding=pad, groups=G)
    r = None
    if residual:
        r = torch.rand(ref.shape, generator=gen) * 2 - 1
        ref = ref + r.double()
    if relu:
        ref = ref.clamp_min(0)
    kk = k * k * cg
    kpad = -(-kk // 32) * 32
    wg = F.pad(w.permute(0, 2, 3, 1).reshape(G, coutg, kk), (0, kpad - kk)).contiguous()
    hi = (wg.view(torch.int32) & -8192).view(torch.float32)
    wcat = torch.cat([hi, wg - hi], 0).contiguous().cuda()
    xn = x.permute(0, 2, 3, 1).contiguous().cuda()
    ho, wo = ref.shape[2], ref.shape[3]
    y = torch.full((N, ho, wo, Cout), float("nan"), device="cuda")
    rn = r.permute(0, 2, 3, 1).contiguous().cuda() if r is not None else None
    lib = _lib.load()
    need = int(lib.nf_conv_tf32_workspace_bytes(N, H, W, C, Cout, G, k, stride, pad, kpad))
    ws = torch.zeros(max(need, 256), dtype=torch.uint8, device="cuda")
    for _ in range(2):  # split-K semaphores re-arm between launches
        _lib.call("nf_grouped_conv_tf32", xn.data_ptr(), wcat.data_ptr(), b.cuda().data_ptr(),
                  rn.data_ptr() if rn is not None else None, y.data_ptr(), N, H, W, C, Cout, G,
                  k, stride, pad, kpad, int(relu), ws.data_ptr() if need else None, need,
                  torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    got = y.permute(0, 3, 1, 2).double().cpu()
    return got, ref, need


@pytest.mark.parametrize("case", CASES)
def test_conv_tf32x3_matches_fp64(case):
    got, ref, _ = _run(*case)
    assert not torch.isnan(got).any()
    err = ((got - ref).abs().max() / ref.abs().max()).item()
    assert err < 2e-5, err


def test_conv_tf32x3_split_k_is_deterministic():
    a, _, need = _run(1, 7, 7, 2, 512, 512, 3, 1, 1, False, True)
    b, _, _ = _run(1, 7, 7, 2, 512, 512, 3, 1, 1, False, True)
    assert need > 0 and torch.equal(a, b)


def test_conv_tf32x3_rejects_unaligned_channels():
    y = torch.empty(16, device="cuda")
    with pytest.raises(Exception):
        _lib.call("nf_grouped_conv_tf32", y.data_ptr(), y.data_ptr(), None, None, y.data_ptr(),
                  1, 4, 4, 6, 8, 2, 1, 1, 0, 32, 0, None, 0,
                  torch.cuda.current_stream().cuda_stream)
