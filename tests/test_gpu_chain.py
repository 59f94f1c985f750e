"""Chained batch-1 merged Linears (nf_grouped_linear_chain, csrc/gemm_chain.cuh).

The chained launch must be bit-identical to launching the same ops one by
one (same tiles, same split-K order, same folded-LayerNorm arithmetic), stay
identical across CUDA-graph replays (its per-instance counters re-arm), and
meet the reference gates end to end (test_gpu_execute / test_gpu_configs run
the default, chained plans).
"""

import pytest
import torch

from paper_2009_13062_b200 import _lib, compile_plan, merge, model_inputs
from paper_2009_13062_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _run(plan, bound, replays=1):
    plan.load_inputs(bound)
    g = plan.capture()
    outs = []
    for _ in range(replays):
        g.replay()
        torch.cuda.synchronize()
        outs.append([o.clone() for o in plan.outputs()])
    return outs


@pytest.mark.parametrize("m", [1, 3, 8])
@pytest.mark.parametrize("fold_ln", [True, False])
def test_chain_bit_identical_to_separate_launches(m, fold_ln):
    graph, stores = W.build_zoo("bert-2l", num_models=m, dtype="bf16")
    merged, mstore = merge(graph, stores)
    inputs = [model_inputs(graph, seed=3, model=j) for j in range(m)]
    bound = merged.bind_inputs(inputs)
    chained = compile_plan(merged.graph, mstore, fold_ln=fold_ln)
    assert any(nid.startswith("chain:merged") for nid, _, _ in chained.steps)
    ref = compile_plan(merged.graph, mstore, fold_ln=fold_ln, chain=False)
    assert not any(nid.startswith("chain:") for nid, _, _ in ref.steps)
    got = _run(chained, bound, replays=3)
    want = _run(ref, bound)[0]
    for rep in got:  # every replay (counters re-armed by the kernel)
        for a, b in zip(rep, want):
            assert torch.equal(a, b)


def test_chain_full_depth_bert_base():
    graph, stores = W.build_zoo("bert-base", num_models=2, dtype="bf16")
    merged, mstore = merge(graph, stores)
    bound = merged.bind_inputs([model_inputs(graph, seed=1, model=j) for j in range(2)])
    chained = compile_plan(merged.graph, mstore)
    assert sum(nid.startswith("chain:merged") for nid, _, _ in chained.steps) == 12
    # layers 1..11 start their QKV+attention per instance after the previous
    # chain, and every chain starts instance g once g's attention heads are in
    kinds = [(type(fn).__name__, getattr(fn, "dep", None) is not None)
             for _, fn, _ in chained.steps]
    assert kinds.count(("_QKVStep", True)) == 11 and kinds.count(("_ChainStep", True)) == 12
    ref = compile_plan(merged.graph, mstore, chain=False)
    for a, b in zip(_run(chained, bound)[0], _run(ref, bound)[0]):
        assert torch.equal(a, b)


def _op(x, w, b, y, rows, k, n, act=_lib.NF_ACT_NONE, residual=None, ws=None):
    o = _lib.LinearOp()
    o.x, o.x_ld, o.x_gs = x.data_ptr(), k, rows * k
    o.w, o.bias = w.data_ptr(), b.data_ptr()
    o.residual = residual.data_ptr() if residual is not None else None
    o.y, o.y_ld, o.y_gs = y.data_ptr(), n, rows * n
    o.rows, o.k, o.n, o.act = rows, k, n, act
    if ws is not None:
        o.workspace, o.workspace_bytes = ws.data_ptr(), ws.numel()
    return o


@pytest.mark.parametrize("G", [1, 5])
def test_chain_c_abi_vs_fp32_torch(G):
    """Two unfused ops through the C ABI (split-K on the second) against a
    plain fp32 PyTorch reference of the same bf16 operands."""
    torch.manual_seed(0)
    T, K, N1, N2 = 128, 512, 2048, 384  # K2 = 2048: split-K on op 2
    dev = "cuda"
    x = (torch.rand(G, T, K, device=dev) - 0.5).bfloat16()
    w1 = ((torch.rand(G, N1, K, device=dev) - 0.5) / K ** 0.5).bfloat16()
    w2 = ((torch.rand(G, N2, N1, device=dev) - 0.5) / N1 ** 0.5).bfloat16()
    b1 = torch.rand(G, N1, device=dev) - 0.5
    b2 = torch.rand(G, N2, device=dev) - 0.5
    res = (torch.rand(G, T, N2, device=dev) - 0.5).bfloat16()
    h = torch.empty(G, T, N1, device=dev, dtype=torch.bfloat16)
    y = torch.empty(G, T, N2, device=dev, dtype=torch.bfloat16)
    lib = _lib.load()
    wsb = int(lib.nf_linear_workspace_bytes(G, T, N1, N2))
    ws = torch.zeros(max(wsb, 256), dtype=torch.uint8, device=dev) if wsb else None
    ops = (_lib.LinearOp * 2)(_op(x, w1, b1, h, T, K, N1, _lib.NF_ACT_GELU),
                              _op(h, w2, b2, y, T, N1, N2, residual=res, ws=ws))
    ctr = torch.zeros(int(lib.nf_linear_chain_counter_bytes(2, G)) // 4, dtype=torch.int32,
                      device=dev)
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(2):  # a second launch reuses the re-armed counters
        _lib.call("nf_grouped_linear_chain", 2, ops, G, ctr.data_ptr(), st)
        torch.cuda.synchronize()
        assert int(ctr.abs().sum()) == 0
        h_ref = torch.nn.functional.gelu(torch.einsum("gtk,gnk->gtn", x.float(), w1.float())
                                         + b1[:, None], approximate="tanh")
        assert (h.float() - h_ref).abs().max() / h_ref.abs().max() < 2e-2
        y_ref = torch.einsum("gtk,gnk->gtn", h.float(), w2.float()) + b2[:, None] + res.float()
        assert (y.float() - y_ref).abs().max() / y_ref.abs().max() < 2e-2


def test_chain_rejects_unsupported_shapes():
    lib = _lib.load()
    assert lib.nf_linear_chain_supported(8, 128, 768, 3072) == 1
    assert lib.nf_linear_chain_supported(8, 1024, 768, 3072) == 0  # token-row tiles
    assert lib.nf_linear_chain_supported(8, 128, 768, 200) == 0    # n % 128
    assert lib.nf_grouped_linear_chain(0, None, 1, None, None) == _lib.NF_ERR_SHAPE


@pytest.mark.parametrize("name,m", [("resnext50_32x4d", 4), ("resnet50", 2)])
def test_linked_conv_launches_bit_identical(name, m):
    """Merged CNN plans link conv launches per instance (a conv starts
    instance k once its input / residual producers stored k's tiles): the
    outputs are bit-identical to the unlinked plan, on every replay."""
    graph, stores = W.build_zoo(name, num_models=m, dtype="bf16")
    merged, mstore = merge(graph, stores)
    bound = merged.bind_inputs([model_inputs(graph, seed=2, model=j) for j in range(m)])
    linked = compile_plan(merged.graph, mstore)
    kinds = [type(fn).__name__ for _, fn, _ in linked.steps]
    assert sum(getattr(fn, "dep_x", None) is not None for _, fn, _ in linked.steps) >= 40
    ref = compile_plan(merged.graph, mstore, chain=False)
    assert not any(getattr(fn, "dep_x", None) for _, fn, _ in ref.steps)
    got = _run(linked, bound, replays=3)
    want = _run(ref, bound)[0]
    for rep in got:
        for a, b in zip(rep, want):
            assert torch.equal(a, b)
    assert "rearm" == linked.steps[0][0] and "_LinkedStep" in kinds


def test_eager_forwards_back_to_back_on_the_default_stream():
    """Three eager forwards of the linked BERT-base N=8 B=1 plan issued back
    to back on the legacy default stream (no sync in between) -- the pattern
    that faulted while the per-forward counter re-arm was a torch fill under
    an ExternalStream(0) context (now a memset on the launch stream,
    nf_counters_rearm) -- complete and match a CUDA-graph replay bit for bit."""
    graph, stores = W.build_zoo("bert-base", num_models=8, dtype="bf16")
    merged, mstore = merge(graph, stores)
    bound = merged.bind_inputs([model_inputs(graph, seed=2, model=j) for j in range(8)])
    plan = compile_plan(merged.graph, mstore)
    assert any(getattr(fn, "dep", None) is not None for _, fn, _ in plan.steps)
    want = _run(plan, bound)[0]
    assert torch.cuda.current_stream().cuda_stream == 0
    for _ in range(3):
        plan.launch()
    torch.cuda.synchronize()
    for a, b in zip(plan.outputs(), want):
        assert torch.equal(a, b)
