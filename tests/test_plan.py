"""Host-side executor logic without a GPU: plans built on the CPU device
(structure only, nothing launches) must lower the merger's glue to views."""

import pytest
import torch

from paper_2009_13062_b200 import OpKind, Plan, UnsupportedOpError, build_zoo, merge
from paper_2009_13062_b200 import workloads as W


def _copies(plan):
    return sum(1 for nid, fn, _ in plan.steps
               if hasattr(fn, "__code__") and fn.__code__.co_consts
               and "nf_copy_strided" in fn.__code__.co_consts)


def test_bert_glue_is_zero_copy():
    graph, stores = W.build_zoo("bert-2l", num_models=3, dtype="bf16")
    merged, mstore = merge(graph, stores)
    plan = Plan(merged.graph, mstore, device="cpu")
    kinds = [merged.graph.node_map()[nid].kind for nid, _, _ in plan.steps
             if nid in merged.graph.node_map()]
    assert OpKind.TRANSPOSE not in kinds and OpKind.RESHAPE not in kinds
    # outputs are views of plan-owned buffers: no copy launch at all
    assert _copies(plan) == 0
    # per layer at batch 1: qkv+attn (fused), then proj(+residual) ->
    # ff1(+gelu) -> ff2(+residual) chained in one persistent launch; the
    # LayerNorms are folded into those launches, only the last one (a graph
    # output) runs as a norm kernel
    assert plan.kernel_launches == 2 * 2 + 1
    ids = [nid for nid, _, _ in plan.steps]
    assert "merged::l00.attn" in ids and "merged::l00.qkv" not in ids
    assert "chain:merged::l00.proj+merged::l00.ff1+merged::l00.ff2" in ids
    # the chains' counters are re-armed by one memset at the start (layer 1's
    # attention waits on layer 0's chain per instance)
    assert ids[0] == "rearm"
    unchained = Plan(merged.graph, mstore, device="cpu", chain=False)
    assert len(unchained.steps) == unchained.kernel_launches == 2 * 4 + 1
    assert not any("res" in nid for nid, _, _ in plan.steps)
    with pytest.raises(UnsupportedOpError):
        plan.launch()


def _consts(fn):
    return [c for c in getattr(fn, "__code__", None).co_consts if isinstance(c, str)] \
        if hasattr(fn, "__code__") else []


def test_layernorms_fold_into_neighbouring_linears():
    graph, stores = W.build_zoo("bert-2l", num_models=3, dtype="bf16")
    merged, mstore = merge(graph, stores)
    plan = Plan(merged.graph, mstore, device="cpu")
    st = dict((nid, fn) for nid, fn, _ in plan.steps)
    st.update(plan.linear_steps())
    # producers add the residual and write the norm statistics
    for nid in ("merged::l00.proj", "merged::l00.ff2", "merged::l01.proj", "merged::l01.ff2"):
        assert st[nid].residual is not None and st[nid].out_stats is not None
    # the first layer's residual is the graph input; later ones are folded norms
    assert st["merged::l00.proj"].fres is None and st["merged::l01.proj"].fres is not None
    assert st["merged::l00.ff2"].fres is not None
    # consumers rebuild LN(x) from the raw sum + statistics
    assert st["merged::l00.ff1"].fin is not None and st["merged::l01.ff1"].fin is not None
    assert st["merged::l01.attn"].fold is not None and st["merged::l00.attn"].fold is None
    # layer 1's QKV+attention starts per instance after layer 0's chain
    assert st["merged::l01.attn"].dep is not None and st["merged::l00.attn"].dep is None
    assert [nid for nid in st if ".ln" in nid] == ["merged::l01.ln2"]


def test_batch1_linears_chain_only_when_consecutive_and_supported():
    graph, stores = W.build_zoo("bert-2l", num_models=3, dtype="bf16")
    merged, mstore = merge(graph, stores)
    plan = Plan(merged.graph, mstore, device="cpu")
    chains = [fn for _, fn, _ in plan.steps if type(fn).__name__ == "_ChainStep"]
    assert len(chains) == 2
    for ch in chains:
        names = [n.split(".")[-1] for n, _ in ch.members]
        assert names == ["proj", "ff1", "ff2"]
        # each op reads the previous op's output
        for (_, a), (_, b) in zip(ch.members, ch.members[1:]):
            assert b.x == a.y
        # the ctypes op table mirrors the launch descriptions
        assert [o.n for o in ch.ops] == [m.n for _, m in ch.members]
    # batch 4 (token-row tiles): nothing chains
    graph, stores = W.build_zoo("bert-2l", num_models=2, batch=4, dtype="bf16")
    merged, mstore = merge(graph, stores)
    plan = Plan(merged.graph, mstore, device="cpu")
    assert not any(nid.startswith("chain:") for nid, _, _ in plan.steps)


def test_layernorm_fold_opt_out():
    graph, stores = W.build_zoo("bert-2l", num_models=3, dtype="bf16")
    merged, mstore = merge(graph, stores)
    plan = Plan(merged.graph, mstore, device="cpu", fold_ln=False, chain=False)
    assert len(plan.steps) == 2 * 6
    # unfolded norms split the layer: only ff1 -> ff2 stays consecutive
    plan = Plan(merged.graph, mstore, device="cpu", fold_ln=False)
    assert plan.kernel_launches == 2 * 5


def test_qkv_attention_fusion_needs_batch_one():
    graph, stores = W.build_zoo("bert-2l", num_models=2, batch=2, dtype="bf16")
    merged, mstore = merge(graph, stores)
    plan = Plan(merged.graph, mstore, device="cpu")
    ids = [nid for nid, _, _ in plan.steps]
    assert "merged::l00.qkv" in ids and "merged::l00.attn" in ids


def test_gelu_fused_into_linear_epilogue():
    graph, stores = W.build_zoo("bert-2l", num_models=2, dtype="bf16")
    merged, mstore = merge(graph, stores)
    plan = Plan(merged.graph, mstore, device="cpu")
    ids = list(plan.linear_steps())
    assert "merged::l00.gelu" not in ids and "merged::l00.ff1" in ids
    assert plan.vals["merged::l00.gelu"] is plan.vals["merged::l00.ff1"]


def test_split_values_reach_the_norm():
    graph, stores = build_zoo("ffnn", num_models=2, batch=4)
    merged, mstore = merge(graph, stores)
    plan = Plan(merged.graph, mstore, device="cpu")
    v = plan.vals["reshape::0"]
    assert v.split == 1 and tuple(v.t.shape) == (4, 2, 8)
    assert plan.vals["merged::ln1"].split == 1


def test_dispatch_count_matches_reference_semantics():
    for name in ("ffnn", "cnnblock", "attnblock"):
        graph, stores = build_zoo(name, num_models=3)
        merged, mstore = merge(graph, stores)
        plan = Plan(merged.graph, mstore, device="cpu")
        assert plan.dispatch_count == merged.dispatch_count


def test_sibling_heads_batch_into_grouped_launches():
    from paper_2009_13062_b200 import merge_backbone
    graph, stores = W.build_zoo("bert-2l", num_models=3, dtype="bf16")
    out = graph.node_map()["l01.ln2"].output_spec
    heads = [W.classifier_head(out, w, seed=j) for j, w in enumerate((2, 3, 5))]
    merged, mstore = merge_backbone(graph, {n.id for n in graph.nodes}, stores, heads)
    plan = Plan(merged.graph, mstore, device="cpu")
    head_steps = [nid for nid, _, _ in plan.steps if nid.startswith("head")]
    # pooler (tanh fused) and classifier: one launch each for all 3 models
    assert head_steps == ["head0::pool", "head0::logits"]
    assert [plan.vals[f"head{j}::logits"].dims for j in range(3)] == [(1, 2), (1, 3), (1, 5)]


def test_cnn_conv_launches_link_per_instance():
    """Merged CNN plans: every conv whose input and residual come from conv
    launches waits on those launches' per-instance tile counters (targets =
    producer tiles per group x groups per instance); linked launches with
    split-K own their workspace; one memset step re-arms the counters."""
    graph, stores = W.build_zoo("resnext50_32x4d", num_models=4, dtype="bf16")
    merged, mstore = merge(graph, stores)
    plan = Plan(merged.graph, mstore, device="cpu")
    steps = [fn for _, fn, _ in plan.steps if type(fn).__name__ == "_LinkedStep"]
    assert plan.steps[0][0] == "rearm" and plan.steps[0][2] == 0  # a memset, not a kernel
    by_y = {fn.y: fn for fn in steps}
    consumers = [fn for fn in steps if fn.dep_x is not None]
    assert len(consumers) >= 48
    for fn in consumers:
        px = by_y[fn.x]
        assert px.done is not None and fn.dep_x == (px.done, px.units * px.gpi)
        assert (fn.residual is None) == (fn.dep_r is None)
        if fn.residual is not None:
            pr = by_y[fn.residual]
            assert fn.dep_r == (pr.done, pr.units * pr.gpi)
        assert fn.gpi * 4 == fn.groups
    shared = getattr(plan, "_ws", None)
    for fn in steps:
        if (fn.dep_x is not None or fn.done is not None) and fn.ws_need > 0:
            assert shared is None or fn.args[-2] != shared.data_ptr()
    # without chaining / linking nothing waits per instance
    ref = Plan(merged.graph, mstore, device="cpu", chain=False)
    assert not any(getattr(fn, "dep_x", None) for _, fn, _ in ref.steps)
