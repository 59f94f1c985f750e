"""Implicit-GEMM conv (nf_grouped_conv_tc) vs a plain fp32 PyTorch conv of
the same bf16-rounded operands: every orientation / tile width / gather
chunk / split-K path the merged CNN plans use."""

import pytest
import torch
import torch.nn.functional as F

from paper_2009_13062_b200 import _lib

pytestmark = pytest.mark.gpu

CASES = [
    # N, H, W, G, cg, coutg, k, stride, pad, residual, relu
    (1, 56, 56, 32, 4, 4, 3, 1, 1, False, True),      # ResNeXt layer1 merged (8-byte gather, BN=16)
    (1, 56, 56, 64, 8, 8, 3, 2, 1, False, True),      # ResNeXt layer2 first block (stride 2)
    (1, 14, 14, 64, 16, 16, 3, 1, 1, False, True),    # ResNeXt layer3
    (1, 7, 7, 32, 32, 32, 3, 1, 1, False, True),      # ResNeXt layer4
    (1, 224, 224, 2, 4, 64, 7, 2, 3, False, True),    # stem, channels padded 3 -> 4
    (1, 56, 56, 2, 64, 64, 3, 1, 1, False, True),     # ResNet layer1 3x3
    (1, 28, 28, 2, 128, 128, 3, 1, 1, True, True),    # ResNet layer2 (+ residual)
    (1, 14, 14, 2, 256, 256, 3, 1, 1, False, True),   # swapped, split-K
    (1, 7, 7, 2, 512, 512, 3, 1, 1, True, False),     # swapped, split-K, residual
    (2, 56, 56, 2, 256, 512, 1, 2, 0, False, False),  # 1x1 stride-2 downsample
    (3, 9, 11, 3, 24, 40, 3, 2, 1, True, True),       # ragged: odd sizes, coutg % 8 != 0
    # halo gather (one image, 16..64-channel groups)
    (1, 56, 56, 128, 32, 32, 3, 1, 1, False, True),   # ResNeXt layer1 32-channel super-groups
    (1, 56, 56, 64, 32, 32, 3, 2, 1, False, True),    # stride 2: 13-row halo
    (1, 9, 11, 4, 16, 16, 3, 1, 1, True, True),       # ragged rows, residual
    (1, 20, 20, 3, 64, 48, 3, 1, 1, False, False),    # 64-channel groups, coutg 48
    (1, 30, 30, 3, 4, 16, 7, 2, 3, False, True),      # 4-channel stem-like groups
]


def _run(N, H, W, G, cg, coutg, k, stride, pad, residual, relu, seed=0):
    gen = torch.Generator().manual_seed(seed)
    C, Cout = G * cg, G * coutg
    x = (torch.rand(N, C, H, W, generator=gen) * 2 - 1).bfloat16()
    w = ((torch.rand(Cout, cg, k, k, generator=gen) * 2 - 1) / (cg * k * k) ** 0.5).bfloat16()
    b = torch.rand(Cout, generator=gen) - 0.5
    ref = F.conv2d(x.float(), w.float(), b, stride=stride, padding=pad, groups=G)
    r = None
    if residual:
        r = (torch.rand(ref.shape, generator=gen) * 2 - 1).bfloat16()
        ref = ref + r.float()
    if relu:
        ref = ref.clamp_min(0)
    kk = k * k * cg
    kpad = -(-kk // 8) * 8
    wg = w.permute(0, 2, 3, 1).reshape(G, coutg, kk)
    wg = F.pad(wg, (0, kpad - kk)).contiguous().cuda()
    xn = x.permute(0, 2, 3, 1).contiguous().cuda()
    ho, wo = ref.shape[2], ref.shape[3]
    y = torch.empty(N, ho, wo, Cout, dtype=torch.bfloat16, device="cuda")
    rn = r.permute(0, 2, 3, 1).contiguous().cuda() if r is not None else None
    bc = b.cuda()
    lib = _lib.load()
    need = int(lib.nf_conv_workspace_bytes(N, H, W, C, Cout, G, k, stride, pad, kpad))
    ws = torch.zeros(max(need, 1), dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    for _ in range(2):  # twice: split-K semaphores must re-arm
        _lib.call("nf_grouped_conv_tc", xn.data_ptr(), wg.data_ptr(), bc.data_ptr(),
                  rn.data_ptr() if rn is not None else None, y.data_ptr(), N, H, W, C, Cout, G,
                  k, stride, pad, kpad, int(relu), ws.data_ptr() if need > 0 else None, need,
                  stream)
    torch.cuda.synchronize()
    got = y.permute(0, 3, 1, 2).float().cpu()
    return got, ref, need


@pytest.mark.parametrize("case", CASES, ids=[str(c[:9]) for c in CASES])
def test_conv_igemm_vs_torch_fp32(case):
    got, ref, _ = _run(*case)
    err = (got - ref).abs().max() / ref.abs().max()
    assert err < 1e-2, f"normwise error {err:.3e}"


def test_conv_igemm_split_k_is_used_and_deterministic():
    case = (1, 7, 7, 2, 512, 512, 3, 1, 1, True, False)
    a, _, need = _run(*case)
    b, _, _ = _run(*case)
    assert need > 0
    assert torch.equal(a, b)
