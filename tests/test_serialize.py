"""Artifact formats (paper_2009_13062_b200/serialize.py) against fixtures
written by the REAL reference serializer (oracle/gen_artifacts.py): TNSR
blobs byte-identical for f32/f64, reference graph JSON and store
directories readable, merged models round-tripping with their merge record,
and the bf16 extension. CPU only."""

import json
from pathlib import Path

import numpy as np
import pytest
import torch

import importlib

from paper_2009_13062_b200 import build_zoo, merge, model_inputs
from paper_2009_13062_b200.errors import GraphFormatError, UnsupportedOpError
from paper_2009_13062_b200.ir import TensorSpec
from paper_2009_13062_b200.tensors import TensorValue

S = importlib.import_module("paper_2009_13062_b200.serialize")  # the module, not the function
ART = Path(__file__).parent / "golden" / "artifacts"
CASES = json.loads((ART / "tensors.json").read_text())


@pytest.mark.parametrize("name", sorted(CASES))
def test_tnsr_blobs_byte_identical_to_reference(name):
    arr = np.load(ART / f"{name}.npy")
    ref = (ART / f"{name}.tnsr").read_bytes()
    tv = TensorValue(TensorSpec(CASES[name]["dtype"], tuple(CASES[name]["dims"])), arr)
    assert S.tensor_to_bytes(tv) == ref
    back = S.tensor_from_bytes(ref)
    assert back.spec.dims == tuple(CASES[name]["dims"]) and back.spec.dtype == CASES[name]["dtype"]
    assert np.array_equal(back.numpy(), arr)


@pytest.mark.parametrize("fname,model,m", [("ffnn_m2.json", "ffnn", 2),
                                           ("cnnblock_m3.json", "cnnblock", 3)])
def test_reference_merged_graph_json_matches_our_merge(fname, model, m):
    ref_graph = S.deserialize((ART / fname).read_bytes())
    graph, stores = build_zoo(model, num_models=m)
    merged, _ = merge(graph, stores)
    merged.embed_metadata()
    ours = merged.graph
    assert [n.id for n in ref_graph.nodes] == [n.id for n in ours.nodes]
    assert [n.kind for n in ref_graph.nodes] == [n.kind for n in ours.nodes]
    assert [n.output_spec.dims for n in ref_graph.nodes] == [n.output_spec.dims for n in ours.nodes]
    assert ref_graph.graph_outputs == ours.graph_outputs
    # our writer emits the same document (parsed) as the reference's
    assert json.loads(S.serialize(ours)) == json.loads((ART / fname).read_bytes())


def test_reference_store_directory_loads_and_round_trips(tmp_path):
    store = S.load_weight_store(ART / "ffnn_m2_store")
    graph, stores = build_zoo("ffnn", num_models=2)
    _, mstore = merge(graph, stores)
    assert store.names() == mstore.names()
    for n in store.names():
        assert store[n].bit_equal(mstore[n]), n
    S.save_weight_store(store, tmp_path / "again")
    for f in sorted((ART / "ffnn_m2_store").iterdir()):
        assert (tmp_path / "again" / f.name).read_bytes() == f.read_bytes(), f.name


def test_bf16_blobs_and_merged_model_round_trip(tmp_path):
    t = torch.randn(4, 3, 5).bfloat16()
    tv = TensorValue(TensorSpec("bf16", (4, 3, 5)), t)
    blob = S.tensor_to_bytes(tv)
    assert blob[6] == 2 and len(blob) == 8 + 3 * 8 + t.numel() * 2
    assert S.tensor_from_bytes(blob).bit_equal(tv)
    graph, stores = build_zoo("attnblock", num_models=3, dtype="bf16")
    merged, mstore = merge(graph, stores)
    S.save_merged(merged, mstore, tmp_path / "m")
    m2, s2 = S.load_merged(tmp_path / "m")
    assert m2.num_models == 3 and m2.input_plan == merged.input_plan
    assert [n.id for n in m2.graph.nodes] == [n.id for n in merged.graph.nodes]
    assert all(s2[n].bit_equal(mstore[n]) for n in mstore.names())
    inputs = [model_inputs(graph, model=j) for j in range(3)]
    assert set(m2.bind_inputs(inputs)) == set(merged.bind_inputs(inputs))


def test_malformed_artifacts_raise_with_offsets():
    good = (ART / "t0.tnsr").read_bytes()
    with pytest.raises(GraphFormatError, match="magic"):
        S.tensor_from_bytes(b"XXXX" + good[4:])
    with pytest.raises(GraphFormatError, match="payload length"):
        S.tensor_from_bytes(good[:-4])
    with pytest.raises(GraphFormatError, match="dtype code"):
        S.tensor_from_bytes(good[:6] + bytes([9]) + good[7:])
    with pytest.raises(GraphFormatError, match="byte offset"):
        S.deserialize(b"{not json")
    doc = json.loads((ART / "ffnn_m2.json").read_bytes())
    doc["nodes"][1]["kind"] = "FancyOp"
    with pytest.raises(UnsupportedOpError):
        S.deserialize(json.dumps(doc))
    doc = json.loads((ART / "ffnn_m2.json").read_bytes())
    doc["extra"] = 1
    with pytest.raises(GraphFormatError, match="unknown"):
        S.deserialize(json.dumps(doc))


def test_blob_name_double_collision_chains_prefix(tmp_path):
    """Sanitisation collisions chain the numeric prefix like the reference
    (serialize.py:227-230): '2_a_b', 'a/b', 'a_b' -> '2_2_a_b.tnsr'."""
    import json

    import numpy as np

    from paper_2009_13062_b200.serialize import load_weight_store, save_weight_store
    from paper_2009_13062_b200.tensors import TensorValue, WeightStore

    store = WeightStore({n: TensorValue.from_array(np.full(3, i, np.float32))
                         for i, n in enumerate(["2_a_b", "a/b", "a_b"])})
    save_weight_store(store, tmp_path)
    files = json.loads((tmp_path / "manifest.json").read_text())["tensors"]
    assert files == {"2_a_b": "2_a_b.tnsr", "a/b": "a_b.tnsr", "a_b": "2_2_a_b.tnsr"}
    back = load_weight_store(tmp_path)
    for n in store.tensors:
        assert back[n].bit_equal(store[n])
