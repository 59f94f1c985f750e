"""Merged-model artifacts on disk: graph JSON, TNSR tensor blobs and
weight-store directories in the reference's formats (pkg/src/modelmerge/
serialize.py:25-255), so merged models saved by either implementation load
in the other, extended for the B200 path with:

* bf16 blobs (dtype code 2, payload = the raw little-endian 16-bit words);
* ``save_merged`` / ``load_merged``: a merged graph (with its embedded merge
  record, merger.py:130-170) plus its fused weight store in one directory, so
  a serving process skips ``merge`` and goes straight to ``compile_plan``.

Blob layout (reference serialize.py:168-175): ``TNSR`` magic, u16 version
(1), u8 dtype code, u8 rank, rank x u64 dims, row-major payload, all
little-endian. Malformed input raises ``GraphFormatError`` with a byte
offset; unknown op kinds raise ``UnsupportedOpError``.
"""

from __future__ import annotations

import json
import struct
from pathlib import Path

import numpy as np
import torch

from .errors import GraphFormatError, UnsupportedOpError, ValidationError
from .ir import Graph, Layout, OpKind, OpNode, TensorSpec, validate
from .tensors import TORCH_DTYPES, TensorValue, WeightStore

TNSR_MAGIC = b"TNSR"
TNSR_VERSION = 1
# name -> (code, little-endian storage dtype of the payload words)
TNSR_DTYPES = {"f32": (0, "<f4"), "f64": (1, "<f8"), "bf16": (2, "<u2")}
_BY_CODE = {code: (name, store) for name, (code, store) in TNSR_DTYPES.items()}

GRAPH_KEYS = ("nodes", "graph_inputs", "graph_outputs", "metadata")
NODE_KEYS = ("id", "kind", "attrs", "inputs", "weights", "output")


# ----------------------------------------------------------------------------
# Tensor blobs
# ----------------------------------------------------------------------------

def _payload(value: TensorValue) -> bytes:
    t = value.data.detach().cpu().contiguous()
    if value.spec.dtype == "bf16":
        return t.view(torch.int16).numpy().astype("<u2", copy=False).tobytes()
    return t.numpy().astype(TNSR_DTYPES[value.spec.dtype][1], copy=False).tobytes()


def tensor_to_bytes(value: TensorValue) -> bytes:
    """One TNSR blob: header, dims, row-major little-endian payload."""
    code = TNSR_DTYPES[value.spec.dtype][0]
    dims = value.spec.dims
    return (TNSR_MAGIC + struct.pack("<HBB", TNSR_VERSION, code, len(dims))
            + struct.pack(f"<{len(dims)}Q", *dims) + _payload(value))


def tensor_from_bytes(data: bytes) -> TensorValue:
    """Decode a TNSR blob (f32 / f64 as the reference writes them, or bf16)."""
    data = bytes(data)
    if len(data) < 8:
        raise GraphFormatError("blob shorter than header", offset=len(data))
    if data[:4] != TNSR_MAGIC:
        raise GraphFormatError(f"bad magic {data[:4]!r}", offset=0)
    version, code, rank = struct.unpack_from("<HBB", data, 4)
    if version != TNSR_VERSION:
        raise GraphFormatError(f"unsupported blob version {version}", offset=4)
    if code not in _BY_CODE:
        raise GraphFormatError(f"unknown dtype code {code}", offset=6)
    if rank < 1:
        raise GraphFormatError("rank must be >= 1", offset=7)
    start = 8 + 8 * rank
    if len(data) < start:
        raise GraphFormatError("blob truncated inside dims", offset=len(data))
    dims = struct.unpack_from(f"<{rank}Q", data, 8)
    if any(d < 1 for d in dims):
        raise GraphFormatError(f"bad dims {dims}", offset=8)
    name, store = _BY_CODE[code]
    count = int(np.prod(dims))
    if len(data) - start != count * np.dtype(store).itemsize:
        raise GraphFormatError(f"payload length {len(data) - start} does not match dims {dims}",
                               offset=start)
    words = np.frombuffer(data, dtype=store, offset=start).reshape(dims)
    if name == "bf16":
        t = torch.from_numpy(words.astype(np.int16)).view(torch.bfloat16)
    else:
        t = torch.from_numpy(words.astype(store.lstrip("<")))  # native-endian copy
    return TensorValue(TensorSpec(name, tuple(dims)), t.to(TORCH_DTYPES[name]).clone())


# ----------------------------------------------------------------------------
# Graph JSON
# ----------------------------------------------------------------------------

def _spec_json(spec: TensorSpec) -> dict:
    return {"dtype": spec.dtype, "dims": list(spec.dims), "layout": spec.layout.value}


def _spec_of(obj, where: str) -> TensorSpec:
    if not isinstance(obj, dict):
        raise GraphFormatError(f"{where}: tensor spec must be an object")
    try:
        return TensorSpec(obj["dtype"], tuple(obj["dims"]), Layout(obj.get("layout", "unlaid")))
    except (KeyError, TypeError, ValueError) as exc:
        raise GraphFormatError(f"{where}: bad tensor spec: {exc}") from exc


def serialize(graph: Graph) -> bytes:
    """Canonical JSON (indent 2, trailing newline) of a validated graph."""
    diags = validate(graph)
    if diags:
        raise ValidationError(diags)
    doc = {
        "nodes": [dict(zip(NODE_KEYS, (n.id, n.kind.value, n.attrs, list(n.inputs),
                                       list(n.weights), _spec_json(n.output_spec))))
                  for n in graph.nodes],
        "graph_inputs": [{"name": k, **_spec_json(v)} for k, v in graph.graph_inputs.items()],
        "graph_outputs": list(graph.graph_outputs),
        "metadata": graph.metadata,
    }
    return (json.dumps(doc, indent=2) + "\n").encode("utf-8")


def _node_of(obj, i: int) -> OpNode:
    where = f"nodes[{i}]"
    if not isinstance(obj, dict):
        raise GraphFormatError(f"{where}: must be an object")
    extra = sorted(set(obj) - set(NODE_KEYS))
    if extra:
        raise GraphFormatError(f"{where}: unknown keys: {extra}")
    if "kind" not in obj:
        raise GraphFormatError(f"{where}: missing 'kind'")
    try:
        kind = OpKind(obj["kind"])
    except ValueError:
        raise UnsupportedOpError(f"{where}: unknown op kind {obj['kind']!r}") from None
    attrs = obj.get("attrs", {})
    if not isinstance(attrs, dict):
        raise GraphFormatError(f"{where}: 'attrs' must be an object")
    try:
        return OpNode(id=obj["id"], kind=kind, inputs=tuple(obj.get("inputs", ())),
                      output_spec=_spec_of(obj.get("output"), where),
                      weights=tuple(obj.get("weights", ())), attrs=attrs)
    except (KeyError, TypeError, ValueError) as exc:
        raise GraphFormatError(f"{where}: {exc}") from exc


def deserialize(data: bytes | str) -> Graph:
    """Parse graph JSON written by :func:`serialize` (or the reference's)."""
    text = data.decode("utf-8", errors="replace") if isinstance(data, bytes) else data
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as exc:
        raise GraphFormatError(f"not valid JSON: {exc.msg}", offset=exc.pos) from exc
    if not isinstance(doc, dict):
        raise GraphFormatError("top level must be a JSON object")
    if set(doc) != set(GRAPH_KEYS):
        extra, missing = sorted(set(doc) - set(GRAPH_KEYS)), sorted(set(GRAPH_KEYS) - set(doc))
        raise GraphFormatError(f"top-level keys: unknown {extra}, missing {missing}")
    if not isinstance(doc["nodes"], list):
        raise GraphFormatError("'nodes' must be a list")
    nodes = tuple(_node_of(obj, i) for i, obj in enumerate(doc["nodes"]))
    if not isinstance(doc["graph_inputs"], list):
        raise GraphFormatError("'graph_inputs' must be a list")
    inputs: dict[str, TensorSpec] = {}
    for i, obj in enumerate(doc["graph_inputs"]):
        if not isinstance(obj, dict) or "name" not in obj:
            raise GraphFormatError(f"graph_inputs[{i}]: must be an object with a 'name'")
        if obj["name"] in inputs:
            raise GraphFormatError(f"graph_inputs[{i}]: duplicate input name {obj['name']!r}")
        inputs[obj["name"]] = _spec_of({k: v for k, v in obj.items() if k != "name"},
                                       f"graph_inputs[{i}]")
    outs = doc["graph_outputs"]
    if not isinstance(outs, list) or not all(isinstance(r, str) for r in outs):
        raise GraphFormatError("'graph_outputs' must be a list of edge references")
    if not isinstance(doc["metadata"], dict):
        raise GraphFormatError("'metadata' must be an object")
    return Graph(nodes, inputs, tuple(outs), doc["metadata"])


def save_graph(graph: Graph, path: str | Path) -> None:
    Path(path).write_bytes(serialize(graph))


def load_graph(path: str | Path) -> Graph:
    return deserialize(Path(path).read_bytes())


# ----------------------------------------------------------------------------
# Weight-store directories (manifest.json + one blob per tensor)
# ----------------------------------------------------------------------------

def _blob_name(name: str, taken: set[str]) -> str:
    base = "".join(c if c.isalnum() or c in "._-" else "_" for c in name) + ".tnsr"
    fname = base
    while fname in taken:  # sanitisation collisions chain a numeric prefix
        fname = f"{len(taken)}_{fname}"
    taken.add(fname)
    return fname


def save_weight_store(store: WeightStore, directory: str | Path) -> None:
    directory = Path(directory)
    directory.mkdir(parents=True, exist_ok=True)
    taken: set[str] = set()
    files = {}
    for name in sorted(store.tensors):
        files[name] = _blob_name(name, taken)
        (directory / files[name]).write_bytes(tensor_to_bytes(store.tensors[name]))
    manifest = {"schema": 1, "model_index": store.model_index, "tensors": files}
    (directory / "manifest.json").write_text(json.dumps(manifest, indent=2, sort_keys=True) + "\n")


def load_weight_store(path: str | Path) -> WeightStore:
    path = Path(path)
    manifest = path / "manifest.json" if path.is_dir() else path
    try:
        doc = json.loads(manifest.read_text())
    except json.JSONDecodeError as exc:
        raise GraphFormatError(f"{manifest}: not valid JSON: {exc.msg}", offset=exc.pos) from exc
    if not isinstance(doc, dict) or doc.get("schema") != 1:
        raise GraphFormatError(f"{manifest}: unsupported manifest schema")
    tensors = {}
    for name, fname in doc.get("tensors", {}).items():
        try:
            blob = (manifest.parent / fname).read_bytes()
        except OSError as exc:
            raise GraphFormatError(f"cannot read blob for {name!r}: {exc}") from exc
        tensors[name] = tensor_from_bytes(blob)
    return WeightStore(tensors, model_index=int(doc.get("model_index", 0)))


# ----------------------------------------------------------------------------
# Merged models (graph + merge record + fused weights)
# ----------------------------------------------------------------------------

def save_merged(merged, store: WeightStore, directory: str | Path) -> None:
    """Write ``merged`` (a MergedGraph) and its fused store: graph.json with
    the embedded merge record, weights/ as a store directory."""
    directory = Path(directory)
    directory.mkdir(parents=True, exist_ok=True)
    merged.embed_metadata()
    save_graph(merged.graph, directory / "graph.json")
    save_weight_store(store, directory / "weights")


def load_merged(directory: str | Path):
    """Inverse of :func:`save_merged`: (MergedGraph, WeightStore)."""
    from .merger import MergedGraph
    directory = Path(directory)
    graph = load_graph(directory / "graph.json")
    return MergedGraph.from_graph(graph), load_weight_store(directory / "weights")


# ----------------------------------------------------------------------------
# Pre-tiled plan artifacts (device layouts, loaded without conversion)
# ----------------------------------------------------------------------------
# A compiled Plan holds every weight in its kernel layout: Linear weights
# K-major (G, N, K) bf16, the fused QKV weights head-major, LayerNorm-folded
# weights with their column sums, conv weights NHWC (G, Cout/G, kh*kw*Cg)
# with BatchNorm folded in (ResNeXt super-group slabs block-diagonal; fp32
# convs split into TF32 hi/lo halves), per-task heads stacked. save_plan
# writes exactly those tensors (TNSR blobs, reference serialize.py:168-207
# format + bf16) beside the graph, keyed by the plan's layout keys; load_plan
# copies them straight to the device and compiles the graph against a
# spec-only store, so no transpose / fold / einsum runs at load time — and a
# layout the artifact lacks fails loudly (the spec-only store has no data).

PLAN_SCHEMA = 1


def _enc_key(k):
    if isinstance(k, tuple):
        return {"tuple": [_enc_key(x) for x in k]}
    if isinstance(k, torch.dtype):
        return {"dtype": str(k).removeprefix("torch.")}
    if k is None or isinstance(k, (str, int, float, bool)):
        return k
    raise GraphFormatError(f"cannot encode plan layout key element {k!r}")


def _dec_key(obj):
    if isinstance(obj, dict):
        if "tuple" in obj:
            return tuple(_dec_key(x) for x in obj["tuple"])
        if "dtype" in obj:
            return getattr(torch, obj["dtype"])
        raise GraphFormatError(f"bad plan layout key {obj!r}")
    return obj


def save_plan(plan, directory: str | Path) -> None:
    """Write ``plan``'s graph and its device-layout weights (see above)."""
    from .tensors import DTYPE_NAMES
    directory = Path(directory)
    (directory / "tiled").mkdir(parents=True, exist_ok=True)
    save_graph(plan.graph, directory / "graph.json")
    taken: set[str] = set()
    entries = []

    def enc_val(v, stem):
        if v is None:
            return None
        if isinstance(v, tuple):
            return {"tuple": [enc_val(x, f"{stem}.{i}") for i, x in enumerate(v)]}
        if not isinstance(v, torch.Tensor) or v.dtype not in DTYPE_NAMES:
            raise GraphFormatError(f"plan layout {stem!r}: unsupported value {type(v)}")
        fname = _blob_name(stem, taken)
        tv = TensorValue(TensorSpec(DTYPE_NAMES[v.dtype], tuple(v.shape)), v.detach().cpu())
        (directory / "tiled" / fname).write_bytes(tensor_to_bytes(tv))
        return fname

    for i, (key, val) in enumerate(plan._wcache.items()):
        stem = "_".join(str(x) for x in (key if isinstance(key, tuple) else (key,)))
        entries.append({"key": _enc_key(key), "value": enc_val(val, stem)})
    doc = {"schema": PLAN_SCHEMA, "mode": plan.mode, "fuse": plan.fuse, "fold_ln": plan.fold_ln,
           "weights": {n: _spec_json(s) for n, s in sorted(plan.weight_specs.items())},
           "layouts": entries}
    (directory / "plan.json").write_text(json.dumps(doc, indent=1) + "\n")


def load_plan(directory: str | Path, device: str = "cuda"):
    """Compile the artifact written by :func:`save_plan` into a Plan on
    ``device``; the weights go host -> device once, already tiled."""
    from .engine import Plan
    directory = Path(directory)
    try:
        doc = json.loads((directory / "plan.json").read_text())
    except json.JSONDecodeError as exc:
        raise GraphFormatError(f"plan.json: not valid JSON: {exc.msg}", offset=exc.pos) from exc
    if not isinstance(doc, dict) or doc.get("schema") != PLAN_SCHEMA:
        raise GraphFormatError("plan.json: unsupported schema")
    graph = load_graph(directory / "graph.json")
    dev = torch.device(device)

    def dec_val(obj):
        if obj is None:
            return None
        if isinstance(obj, dict):
            return tuple(dec_val(x) for x in obj["tuple"])
        try:
            blob = (directory / "tiled" / obj).read_bytes()
        except OSError as exc:
            raise GraphFormatError(f"cannot read layout blob {obj!r}: {exc}") from exc
        return tensor_from_bytes(blob).data.to(dev)

    cache = {_dec_key(e["key"]): dec_val(e["value"]) for e in doc["layouts"]}
    specs = {n: _spec_of(s, f"weights[{n!r}]") for n, s in doc["weights"].items()}
    store = WeightStore({n: TensorValue(s, torch.empty(s.dims, dtype=TORCH_DTYPES[s.dtype],
                                                       device="meta"))
                         for n, s in specs.items()})
    try:
        return Plan(graph, store, mode=doc["mode"], device=dev, fuse=doc["fuse"],
                    fold_ln=doc["fold_ln"], weight_cache=cache)
    except NotImplementedError as exc:  # a meta tensor was read: layout missing
        raise GraphFormatError(f"plan artifact lacks a weight layout the graph needs: {exc}") \
            from exc
