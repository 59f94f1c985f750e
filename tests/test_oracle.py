"""The CPU oracle is pinned before it is trusted: every restated reference
kernel must reproduce the reference's own outputs bit for bit on the golden
vectors (tests/golden/kernels.npz, produced by the real reference via
oracle/gen_golden.py), and the oracle executor must reproduce the
reference's merged-execution outputs for the zoo verify matrix."""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import executor as OX
from oracle import kernels as OK
from paper_2009_13062_b200 import build_zoo, merge, model_inputs

GOLD = Path(__file__).parent / "golden"
VEC = np.load(GOLD / "kernels.npz")
META = json.loads((GOLD / "kernels.json").read_text())
ZOO = np.load(GOLD / "zoo_outputs.npz")

_FN = {
    "conv2d": OK.conv2d, "grouped_conv2d": OK.grouped_conv2d, "matmul": OK.matmul,
    "batch_matmul": OK.batch_matmul, "layer_norm": OK.layer_norm, "group_norm": OK.group_norm,
    "batch_norm_inference": OK.batch_norm_inference, "relu": OK.relu, "tanh": OK.tanh,
    "softmax": OK.softmax, "add": OK.add, "mul": OK.mul, "max_pool2d": OK.max_pool2d,
    "mean_pool2d": OK.mean_pool2d,
}


@pytest.mark.parametrize("case", META, ids=[c["name"] for c in META])
def test_oracle_kernel_bit_exact_vs_reference(case):
    name = case["name"]
    ins = [VEC[f"{name}/in{i}"] for i in range(case["n_in"])]
    if name.startswith("pack_"):
        dim = name.split("_")[1]
        got = OK.pack(ins, dim=dim)
        want = VEC[f"{name}/out0"]
        assert got.tobytes() == want.tobytes()
        stacked = dim == "batch" and ins[0].ndim < 4
        for a, b in zip(OK.unpack(got, len(ins), dim=dim, stacked=stacked), ins):
            assert a.tobytes() == b.tobytes()
        return
    fn = _FN[case["fn"]]
    got = fn(*ins, **case["kwargs"])
    want = VEC[f"{name}/out0"]
    assert got.dtype == want.dtype and got.shape == want.shape
    assert got.tobytes() == want.tobytes(), name


def test_pool_known_answers():
    x = np.arange(16, dtype=np.float32).reshape(1, 1, 4, 4)
    assert OK.max_pool2d(x, kernel=2, stride=2).ravel().tolist() == [5, 7, 13, 15]
    assert OK.mean_pool2d(x, kernel=2, stride=2).ravel().tolist() == [2.5, 4.5, 10.5, 12.5]


def test_spec_kats():
    ones = np.ones((1, 1, 3, 3), np.float32)
    assert OK.conv2d(ones, ones).item() == 9.0
    x = np.arange(9, dtype=np.float32).reshape(1, 1, 3, 3)
    ident = np.zeros((1, 1, 3, 3), np.float32)
    ident[0, 0, 1, 1] = 1
    assert (OK.conv2d(x, ident, padding=1) == x).all()
    row = np.full((2, 4), 3.0, np.float32)
    beta = np.array([1, 2, 3, 4], np.float32)
    assert (OK.layer_norm(row, np.ones(4, np.float32), beta, eps=1e-5) == beta).all()


@pytest.mark.parametrize("name", ["ffnn", "cnnblock", "attnblock"])
@pytest.mark.parametrize("m", [1, 2, 4])
@pytest.mark.parametrize("batch", [1, 4])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_oracle_merged_zoo_matches_reference(name, m, batch, dtype):
    graph, stores = build_zoo(name, num_models=m, batch=batch, dtype=dtype)
    key = f"{name}/m{m}/b{batch}/{dtype}"
    wsum = [sum(float(np.sum(t.numpy(), dtype=np.float64)) for t in s.tensors.values())
            for s in stores]
    np.testing.assert_array_equal(np.array(wsum), ZOO[f"{key}/wsum"])  # same seeded weights
    merged, mstore = merge(graph, stores)
    inputs = [model_inputs(graph, seed=0, model=j) for j in range(m)]
    outs = OX.execute(merged.graph, mstore.tensors, merged.bind_inputs(inputs))
    for j in range(m):
        assert outs[j].tobytes() == ZOO[f"{key}/out{j}"].tobytes()


def test_bf16_rounding_is_rne():
    import torch
    x = np.random.default_rng(0).standard_normal(4096).astype(np.float32)
    want = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    assert OK.bf16_round(x).tobytes() == want.tobytes()


def test_attention_oracle_matches_torch_sdpa():
    import torch
    rng = np.random.default_rng(3)
    qkv = rng.uniform(-1, 1, (2, 3, 17, 3 * 32)).astype(np.float32)
    got = OK.attention(qkv, heads=4)
    t = torch.from_numpy(qkv).double()
    q, k, v = (t[..., i * 32:(i + 1) * 32].reshape(2, 3, 17, 4, 8).transpose(-2, -3)
               for i in range(3))
    ref = torch.nn.functional.scaled_dot_product_attention(q, k, v)
    ref = ref.transpose(-2, -3).reshape(2, 3, 17, 32).numpy()
    np.testing.assert_allclose(got, ref, rtol=1e-5, atol=1e-6)


def test_gelu_oracle_matches_torch():
    import torch
    x = np.linspace(-6, 6, 1001, dtype=np.float32)
    ref = torch.nn.functional.gelu(torch.from_numpy(x).double()).numpy()
    np.testing.assert_allclose(OK.gelu(x), ref, rtol=1e-6, atol=1e-7)


@pytest.mark.skipif(not Path("/root/reference/pkg/src/modelmerge").exists(),
                    reason="reference tree not mounted (GPU box)")
def test_oracle_vs_live_reference_random():
    """Where the reference is importable, compare on fresh random draws too."""
    import importlib
    import sys
    import types
    sys.dont_write_bytecode = True
    if "modelmerge" not in sys.modules:
        pkg = types.ModuleType("modelmerge")
        pkg.__path__ = ["/root/reference/pkg/src/modelmerge"]
        sys.modules["modelmerge"] = pkg
    E = importlib.import_module("modelmerge.engine")
    rng = np.random.default_rng(99)
    for _ in range(20):
        g = int(rng.integers(1, 5))
        cin, cout = g * int(rng.integers(1, 4)), g * int(rng.integers(1, 4))
        x = rng.uniform(-1, 1, (2, cin, 7, 7)).astype(np.float32)
        w = rng.uniform(-.5, .5, (cout, cin // g, 3, 3)).astype(np.float32)
        s = int(rng.integers(1, 3))
        a = OK.grouped_conv2d(x, w, groups=g, stride=s, padding=1)
        b = E.grouped_conv2d(x, w, groups=g, stride=s, padding=1)
        assert a.tobytes() == b.tobytes()
        xm = rng.uniform(-1, 1, (g, 5, 33)).astype(np.float32)
        wm = rng.uniform(-.5, .5, (g, 33, 9)).astype(np.float32)
        assert OK.batch_matmul(xm, wm).tobytes() == E.batch_matmul(xm, wm).tobytes()


def test_rel_attention_oracle_matches_transformers_xlnet():
    """The unpinned XLNet restatement vs transformers' rel_attn_core (f64)."""
    import torch
    from transformers import XLNetConfig
    from transformers.models.xlnet import modeling_xlnet as X
    torch.manual_seed(0)
    att = X.XLNetRelativeAttention(XLNetConfig(d_model=64, n_head=4, d_inner=128)).eval().double()
    for p in att.parameters():
        torch.nn.init.uniform_(p, -0.5, 0.5)
    S, B, H, dh = 9, 2, 4, 16
    q, k, v = (torch.rand(S, B, H, dh, dtype=torch.float64) - .5 for _ in range(3))
    kr = torch.rand(2 * S, B, H, dh, dtype=torch.float64) - .5
    with torch.no_grad():
        ref = att.rel_attn_core(q, k, v, kr)
    ref = ref[0] if isinstance(ref, tuple) else ref
    D = H * dh
    qkv = torch.cat([t.permute(1, 0, 2, 3).reshape(B, S, D) for t in (q, k, v)], -1).numpy()
    r = kr.permute(1, 0, 2, 3).reshape(B, 2 * S, D).numpy()
    got = OK.rel_attention(qkv, r, att.r_w_bias.detach().numpy(), att.r_r_bias.detach().numpy(),
                           heads=H)
    np.testing.assert_allclose(got, ref.permute(1, 0, 2, 3).reshape(B, S, D).numpy(),
                               rtol=1e-12, atol=1e-12)


def test_relative_positional_embedding_matches_transformers():
    import torch
    from transformers import XLNetConfig, XLNetModel
    from paper_2009_13062_b200.workloads import relative_positional_embedding
    m = XLNetModel(XLNetConfig(d_model=32, n_head=2, d_inner=64, n_layer=1, attn_type="bi"))
    ref = m.relative_positional_encoding(7, 7, bsz=1)[:, 0, :].numpy()
    np.testing.assert_allclose(relative_positional_embedding(7, 32), ref, rtol=1e-6, atol=1e-6)
