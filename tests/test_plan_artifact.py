"""Pre-tiled plan artifacts (serialize.save_plan / load_plan): the device
layouts a compiled Plan holds (K-major / head-major / LayerNorm-folded
Linear weights, BN-folded NHWC conv slabs, TF32 hi/lo splits, stacked heads)
written as TNSR blobs (reference serialize.py:168-207 format + bf16) and
loaded without any conversion. CPU: structure-only plans round-trip every
layout bit-exactly; GPU: a loaded plan's outputs are bit-identical."""
import pytest
import torch

from paper_2009_13062_b200 import GraphFormatError, Plan, compile_plan
import importlib

S = importlib.import_module("paper_2009_13062_b200.serialize")
from paper_2009_13062_b200 import workloads as W

CASES = [("bert-2l", 3, 1, "bf16"), ("xlnet-2l", 2, 1, "bf16"),
         ("resnext-mini", 4, 1, "bf16"), ("resnet-mini", 2, 1, "f32")]


def _flat(v):
    if isinstance(v, tuple):
        return [x for e in v for x in _flat(e)]
    return [v]


def _same_cache(a: dict, b: dict):
    assert set(a) == set(b)
    for k in a:
        xa, xb = _flat(a[k]), _flat(b[k])
        assert len(xa) == len(xb)
        for ta, tb in zip(xa, xb):
            if ta is None:
                assert tb is None
                continue
            assert ta.dtype == tb.dtype and ta.shape == tb.shape, k
            assert torch.equal(ta.cpu().view(torch.uint8), tb.cpu().view(torch.uint8)), k


def test_key_codec_roundtrip():
    for k in [("w", "linear_nk", torch.bfloat16), ("convchain", "c1", "igemm", 8),
              ("qkv_hm", "l0.qkv.w", None, "l0.ln.g"), ("siblings", "h", 16, True)]:
        assert S._dec_key(S._enc_key(k)) == k


@pytest.mark.parametrize("model,n,batch,dtype", CASES)
def test_plan_artifact_roundtrip_cpu(tmp_path, model, n, batch, dtype):
    _, _, _, merged, mstore, _ = W.merged_workload(model, n, batch, dtype)
    plan = Plan(merged.graph, mstore, device="cpu")
    assert not any(k[0] == "convchain" and len(k) == 2 for k in plan._wcache)
    S.save_plan(plan, tmp_path)
    got = S.load_plan(tmp_path, device="cpu")
    assert [s[0] for s in got.steps] == [s[0] for s in plan.steps]
    assert got.kernel_launches == plan.kernel_launches
    _same_cache(plan._wcache, got._wcache)


def test_plan_artifact_missing_layout_fails_loudly(tmp_path):
    _, _, _, merged, mstore, _ = W.merged_workload("bert-2l", 2, 1, "bf16")
    S.save_plan(Plan(merged.graph, mstore, device="cpu"), tmp_path)
    doc = (tmp_path / "plan.json").read_text()
    import json
    d = json.loads(doc)
    d["layouts"] = [e for e in d["layouts"] if e["key"]["tuple"][0] != "qkv_hm"]
    (tmp_path / "plan.json").write_text(json.dumps(d))
    with pytest.raises(GraphFormatError):
        S.load_plan(tmp_path, device="cpu")


@pytest.mark.gpu
@pytest.mark.parametrize("model,n,batch,dtype", CASES)
def test_plan_artifact_outputs_bit_identical(tmp_path, model, n, batch, dtype):
    _, _, inputs, merged, mstore, _ = W.merged_workload(model, n, batch, dtype)
    bound = merged.bind_inputs(inputs)
    plan = compile_plan(merged.graph, mstore)
    plan.load_inputs(bound)
    plan.launch()
    want = [o.clone() for o in plan.outputs()]
    S.save_plan(plan, tmp_path)
    got = S.load_plan(tmp_path)
    got.load_inputs(bound)
    got.launch()
    torch.cuda.synchronize()
    for a, b in zip(want, got.outputs()):
        assert torch.equal(a.view(torch.uint8) if a.dtype != torch.float32 else a,
                           b.view(torch.uint8) if b.dtype != torch.float32 else b)
