"""Workloads: the reference zoo (pkg/src/modelmerge/zoo.py) and the BASELINE
model families, as IR graphs with deterministic synthetic weights and inputs.

Zoo models (ffnn, cnnblock, attnblock) reproduce the reference graphs and its
seeding exactly: weights draw from ``default_rng([seed, 0, model])`` in
declaration order, U[-0.5, 0.5] (BN running variance U[0.5, 1.5]); inputs from
``default_rng([seed, 1, model])``, U[-1, 1] (zoo.py:146-184).

BASELINE families (BERT-base, XLNet-base, ResNet-50, ResNeXt-50 32x4d) keep
the same seeding keys but scale linear / conv weights by fan-in,
U(+-1/sqrt(fan_in)), with gamma ~ U[0.5, 1.5], beta / BN mean ~ U[-0.5, 0.5],
BN var ~ U[0.5, 1.5] (SURVEY §8d "documented deviation": unscaled weights
drive ResNet-50 logits to ~1e11). bf16 models round the fp32 draws (RNE).
Heads are per-instance and unmerged (merge_backbone), as in the paper
(PAPER.md:382-389).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np
import torch

from .ir import Graph, OpKind, OpNode, TensorSpec
from .tensors import NUMPY_DTYPES, TORCH_DTYPES, TensorValue, WeightStore

ZOO_NAMES = ("ffnn", "cnnblock", "attnblock")

# (name, dims, draw) in generation order. draws: "std" U[-.5,.5]; "var"
# U[.5,1.5]; "fan:<n>" U(+-1/sqrt(n)); "gamma" U[.5,1.5]; "beta" U[-.5,.5].
WeightPlan = list[tuple[str, tuple[int, ...], str]]


def _spec(dtype, *dims) -> TensorSpec:
    return TensorSpec(dtype, tuple(dims))


# ----------------------------------------------------------------------------
# Reference zoo (zoo.py:39-132)
# ----------------------------------------------------------------------------

def _ffnn(batch: int, dtype: str) -> tuple[Graph, WeightPlan]:
    act = _spec(dtype, batch, 8)
    nodes = (
        OpNode("mm1", OpKind.MATMUL, ("x:0",), act, weights=("mm1.w", "mm1.b")),
        OpNode("ln1", OpKind.LAYER_NORM, ("mm1:0",), act, weights=("ln1.gamma", "ln1.beta"),
               attrs={"eps": 1e-5}),
        OpNode("act1", OpKind.RELU, ("ln1:0",), act),
    )
    g = Graph(nodes, {"x": _spec(dtype, batch, 6)}, ("act1:0",),
              metadata={"zoo": "ffnn", "batch": batch, "dtype": dtype})
    return g, [("mm1.w", (6, 8), "std"), ("mm1.b", (8,), "std"),
               ("ln1.gamma", (8,), "std"), ("ln1.beta", (8,), "std")]


def _cnnblock(batch: int, dtype: str) -> tuple[Graph, WeightPlan]:
    c, hw = 8, 8
    img = _spec(dtype, batch, c, hw, hw)
    conv = {"kernel": 3, "stride": 1, "padding": 1}

    def bn(p):
        return tuple(f"{p}.{s}" for s in ("gamma", "beta", "mean", "var"))

    nodes = (
        OpNode("conv1", OpKind.CONV2D, ("x:0",), img, weights=("conv1.w", "conv1.b"),
               attrs=dict(conv)),
        OpNode("bn1", OpKind.BATCH_NORM, ("conv1:0",), img, weights=bn("bn1"),
               attrs={"eps": 1e-5}),
        OpNode("relu1", OpKind.RELU, ("bn1:0",), img),
        OpNode("gconv1", OpKind.GROUPED_CONV2D, ("relu1:0",), img,
               weights=("gconv1.w", "gconv1.b"), attrs=dict(conv, groups=2)),
        OpNode("bn2", OpKind.BATCH_NORM, ("gconv1:0",), img, weights=bn("bn2"),
               attrs={"eps": 1e-5}),
        OpNode("add1", OpKind.ADD, ("bn2:0", "x:0"), img),
        OpNode("pool1", OpKind.MAX_POOL2D, ("add1:0",), _spec(dtype, batch, c, hw // 2, hw // 2),
               attrs={"kernel": 2, "stride": 2}),
    )
    g = Graph(nodes, {"x": img}, ("pool1:0",),
              metadata={"zoo": "cnnblock", "batch": batch, "dtype": dtype})
    v = (c,)
    plan: WeightPlan = [("conv1.w", (c, c, 3, 3), "std"), ("conv1.b", v, "std")]
    plan += [(f"bn1.{s}", v, "var" if s == "var" else "std") for s in ("gamma", "beta", "mean", "var")]
    plan += [("gconv1.w", (c, c // 2, 3, 3), "std"), ("gconv1.b", v, "std")]
    plan += [(f"bn2.{s}", v, "var" if s == "var" else "std") for s in ("gamma", "beta", "mean", "var")]
    return g, plan


def _attnblock(batch: int, dtype: str) -> tuple[Graph, WeightPlan]:
    seq, d, dff = 6, 8, 16
    tok, wide = _spec(dtype, batch, seq, d), _spec(dtype, batch, seq, dff)
    ln = {"eps": 1e-5}
    nodes = (
        OpNode("qkv", OpKind.MATMUL, ("x:0",), tok, weights=("qkv.w", "qkv.b")),
        OpNode("attn", OpKind.SOFTMAX, ("qkv:0",), tok, attrs={"axis": -2}),
        OpNode("proj", OpKind.MATMUL, ("attn:0",), tok, weights=("proj.w", "proj.b")),
        OpNode("ln1", OpKind.LAYER_NORM, ("proj:0",), tok, weights=("ln1.gamma", "ln1.beta"),
               attrs=dict(ln)),
        OpNode("ff1", OpKind.MATMUL, ("ln1:0",), wide, weights=("ff1.w", "ff1.b")),
        OpNode("act", OpKind.RELU, ("ff1:0",), wide),
        OpNode("ff2", OpKind.MATMUL, ("act:0",), tok, weights=("ff2.w", "ff2.b")),
        OpNode("ln2", OpKind.LAYER_NORM, ("ff2:0",), tok, weights=("ln2.gamma", "ln2.beta"),
               attrs=dict(ln)),
    )
    g = Graph(nodes, {"x": tok}, ("ln2:0",),
              metadata={"zoo": "attnblock", "batch": batch, "dtype": dtype})
    plan: WeightPlan = []
    for name, (a, b) in (("qkv", (d, d)), ("proj", (d, d))):
        plan += [(f"{name}.w", (a, b), "std"), (f"{name}.b", (b,), "std")]
    plan += [("ln1.gamma", (d,), "std"), ("ln1.beta", (d,), "std"),
             ("ff1.w", (d, dff), "std"), ("ff1.b", (dff,), "std"),
             ("ff2.w", (dff, d), "std"), ("ff2.b", (d,), "std"),
             ("ln2.gamma", (d,), "std"), ("ln2.beta", (d,), "std")]
    return g, plan


# ----------------------------------------------------------------------------
# BASELINE families
# ----------------------------------------------------------------------------

@dataclass(frozen=True)
class BertConfig:
    layers: int = 12
    hidden: int = 768
    heads: int = 12
    ffn: int = 3072
    seq: int = 128
    eps: float = 1e-12


BERT_BASE = BertConfig()


def _bert(batch: int, dtype: str, cfg: BertConfig = BERT_BASE) -> tuple[Graph, WeightPlan]:
    """BERT-base encoder on (B, S, 768) embeddings (no lookup).
    Per layer: fused QKV MatMul -> Attention -> proj MatMul -> Add(residual)
    -> LayerNorm -> FF1 MatMul -> GELU -> FF2 MatMul -> Add -> LayerNorm."""
    b, s, d, f = batch, cfg.seq, cfg.hidden, cfg.ffn
    tok, qkv, wide = _spec(dtype, b, s, d), _spec(dtype, b, s, 3 * d), _spec(dtype, b, s, f)
    nodes: list[OpNode] = []
    plan: WeightPlan = []
    x = "x:0"
    for i in range(cfg.layers):
        p = f"l{i:02d}"
        nodes += [
            OpNode(f"{p}.qkv", OpKind.MATMUL, (x,), qkv, weights=(f"{p}.qkv.w", f"{p}.qkv.b")),
            OpNode(f"{p}.attn", OpKind.ATTENTION, (f"{p}.qkv:0",), tok,
                   attrs={"heads": cfg.heads}),
            OpNode(f"{p}.proj", OpKind.MATMUL, (f"{p}.attn:0",), tok,
                   weights=(f"{p}.proj.w", f"{p}.proj.b")),
            OpNode(f"{p}.res1", OpKind.ADD, (f"{p}.proj:0", x), tok),
            OpNode(f"{p}.ln1", OpKind.LAYER_NORM, (f"{p}.res1:0",), tok,
                   weights=(f"{p}.ln1.g", f"{p}.ln1.b"), attrs={"eps": cfg.eps}),
            OpNode(f"{p}.ff1", OpKind.MATMUL, (f"{p}.ln1:0",), wide,
                   weights=(f"{p}.ff1.w", f"{p}.ff1.b")),
            OpNode(f"{p}.gelu", OpKind.GELU, (f"{p}.ff1:0",), wide),
            OpNode(f"{p}.ff2", OpKind.MATMUL, (f"{p}.gelu:0",), tok,
                   weights=(f"{p}.ff2.w", f"{p}.ff2.b")),
            OpNode(f"{p}.res2", OpKind.ADD, (f"{p}.ff2:0", f"{p}.ln1:0"), tok),
            OpNode(f"{p}.ln2", OpKind.LAYER_NORM, (f"{p}.res2:0",), tok,
                   weights=(f"{p}.ln2.g", f"{p}.ln2.b"), attrs={"eps": cfg.eps}),
        ]
        plan += [(f"{p}.qkv.w", (d, 3 * d), f"fan:{d}"), (f"{p}.qkv.b", (3 * d,), f"fan:{d}"),
                 (f"{p}.proj.w", (d, d), f"fan:{d}"), (f"{p}.proj.b", (d,), f"fan:{d}"),
                 (f"{p}.ln1.g", (d,), "gamma"), (f"{p}.ln1.b", (d,), "beta"),
                 (f"{p}.ff1.w", (d, f), f"fan:{d}"), (f"{p}.ff1.b", (f,), f"fan:{d}"),
                 (f"{p}.ff2.w", (f, d), f"fan:{f}"), (f"{p}.ff2.b", (d,), f"fan:{f}"),
                 (f"{p}.ln2.g", (d,), "gamma"), (f"{p}.ln2.b", (d,), "beta")]
        x = f"{p}.ln2:0"
    g = Graph(tuple(nodes), {"x": tok}, (x,),
              metadata={"model": "bert-base", "batch": batch, "dtype": dtype,
                        "layers": cfg.layers})
    return g, plan


@dataclass(frozen=True)
class XLNetConfig:
    layers: int = 12
    hidden: int = 768
    heads: int = 12
    ffn: int = 3072
    seq: int = 128
    eps: float = 1e-12


XLNET_BASE = XLNetConfig()


def _xlnet(batch: int, dtype: str, cfg: XLNetConfig = XLNET_BASE) -> tuple[Graph, WeightPlan]:
    """XLNet-base encoder (attn_type "bi", no memory / segments / masks) on
    (B, S, 768) embeddings plus the sinusoidal relative positional embedding
    input ``pos`` (1, 2S, 768), projected once per instance and shared by its
    B sequences (transformers expands the same pos_emb over the batch). Per layer (transformers XLNetLayer): fused
    q|k|v projection (no bias), positional-key projection r, relative
    attention with per-instance r_w_bias / r_r_bias, output projection o (no
    bias), Add + LayerNorm, FF1 + GELU + FF2, Add + LayerNorm."""
    b, s, d, f, h = batch, cfg.seq, cfg.hidden, cfg.ffn, cfg.heads
    dh = d // h
    tok, qkv, wide = _spec(dtype, b, s, d), _spec(dtype, b, s, 3 * d), _spec(dtype, b, s, f)
    rsp = _spec(dtype, 1, 2 * s, d)  # shared by the batch: r projected once per instance
    nodes: list[OpNode] = []
    plan: WeightPlan = []
    x = "x:0"
    for i in range(cfg.layers):
        p = f"l{i:02d}"
        nodes += [
            OpNode(f"{p}.qkv", OpKind.MATMUL, (x,), qkv, weights=(f"{p}.qkv.w",)),
            OpNode(f"{p}.r", OpKind.MATMUL, ("pos:0",), rsp, weights=(f"{p}.r.w",)),
            OpNode(f"{p}.attn", OpKind.REL_ATTENTION, (f"{p}.qkv:0", f"{p}.r:0"), tok,
                   weights=(f"{p}.rwb", f"{p}.rrb"), attrs={"heads": h}),
            OpNode(f"{p}.proj", OpKind.MATMUL, (f"{p}.attn:0",), tok, weights=(f"{p}.o.w",)),
            OpNode(f"{p}.res1", OpKind.ADD, (f"{p}.proj:0", x), tok),
            OpNode(f"{p}.ln1", OpKind.LAYER_NORM, (f"{p}.res1:0",), tok,
                   weights=(f"{p}.ln1.g", f"{p}.ln1.b"), attrs={"eps": cfg.eps}),
            OpNode(f"{p}.ff1", OpKind.MATMUL, (f"{p}.ln1:0",), wide,
                   weights=(f"{p}.ff1.w", f"{p}.ff1.b")),
            OpNode(f"{p}.gelu", OpKind.GELU, (f"{p}.ff1:0",), wide),
            OpNode(f"{p}.ff2", OpKind.MATMUL, (f"{p}.gelu:0",), tok,
                   weights=(f"{p}.ff2.w", f"{p}.ff2.b")),
            OpNode(f"{p}.res2", OpKind.ADD, (f"{p}.ff2:0", f"{p}.ln1:0"), tok),
            OpNode(f"{p}.ln2", OpKind.LAYER_NORM, (f"{p}.res2:0",), tok,
                   weights=(f"{p}.ln2.g", f"{p}.ln2.b"), attrs={"eps": cfg.eps}),
        ]
        plan += [(f"{p}.qkv.w", (d, 3 * d), f"fan:{d}"), (f"{p}.r.w", (d, d), f"fan:{d}"),
                 (f"{p}.rwb", (h, dh), f"fan:{dh}"), (f"{p}.rrb", (h, dh), f"fan:{dh}"),
                 (f"{p}.o.w", (d, d), f"fan:{d}"),
                 (f"{p}.ln1.g", (d,), "gamma"), (f"{p}.ln1.b", (d,), "beta"),
                 (f"{p}.ff1.w", (d, f), f"fan:{d}"), (f"{p}.ff1.b", (f,), f"fan:{d}"),
                 (f"{p}.ff2.w", (f, d), f"fan:{f}"), (f"{p}.ff2.b", (d,), f"fan:{f}"),
                 (f"{p}.ln2.g", (d,), "gamma"), (f"{p}.ln2.b", (d,), "beta")]
        x = f"{p}.ln2:0"
    g = Graph(tuple(nodes), {"x": tok, "pos": rsp}, (x,),
              metadata={"model": "xlnet-base", "batch": batch, "dtype": dtype,
                        "layers": cfg.layers, "sinusoid_inputs": ["pos"]})
    return g, plan


def relative_positional_embedding(seq: int, d_model: int) -> np.ndarray:
    """transformers XLNetModel.relative_positional_encoding, attn_type "bi",
    klen = qlen = seq: positions seq, seq-1, ..., -seq+1; [sin | cos]."""
    inv_freq = 1.0 / np.power(10000.0, np.arange(0, d_model, 2.0) / d_model)
    pos_seq = np.arange(seq, -seq, -1.0)
    inp = np.outer(pos_seq, inv_freq)
    return np.concatenate([np.sin(inp), np.cos(inp)], axis=-1)


def bert_layers(n: int) -> Callable[[int, str], tuple[Graph, WeightPlan]]:
    """BERT builder truncated to ``n`` layers (tests; oracle sampling)."""
    cfg = BertConfig(layers=n)
    return lambda batch, dtype: _bert(batch, dtype, cfg)


def _resnet(batch: int, dtype: str, *, groups: int = 1, width_per_group: int = 64,
            layers=(3, 4, 6, 3), image: int = 224, stages: int = 4) -> tuple[Graph, WeightPlan]:
    """torchvision ResNet-50 (groups=1) / ResNeXt-50 32x4d (groups=32,
    width_per_group=4) backbone, v1.5 (stride on the 3x3), up to the global
    average pool: (B, 3, 224, 224) -> (B, 2048, 1, 1). Convs have no bias
    (BatchNorm follows every conv); the stem max-pool is padded (3x3 s2 p1)."""
    nodes: list[OpNode] = []
    plan: WeightPlan = []
    img = lambda c, h: _spec(dtype, batch, c, h, h)  # noqa: E731

    def conv(nid, src, cin, cout, k, stride, pad, h_in, g=1):
        h = (h_in + 2 * pad - k) // stride + 1
        kind = OpKind.GROUPED_CONV2D if g > 1 else OpKind.CONV2D
        attrs = {"kernel": k, "stride": stride, "padding": pad}
        if g > 1:
            attrs["groups"] = g
        nodes.append(OpNode(nid, kind, (src,), img(cout, h), weights=(f"{nid}.w",), attrs=attrs))
        plan.append((f"{nid}.w", (cout, cin // g, k, k), f"fan:{cin // g * k * k}"))
        return f"{nid}:0", h

    def bn(nid, src, c, h):
        nodes.append(OpNode(nid, OpKind.BATCH_NORM, (src,), img(c, h),
                            weights=tuple(f"{nid}.{s}" for s in ("g", "b", "m", "v")),
                            attrs={"eps": 1e-5}))
        plan.extend([(f"{nid}.g", (c,), "gamma"), (f"{nid}.b", (c,), "beta"),
                     (f"{nid}.m", (c,), "beta"), (f"{nid}.v", (c,), "var")])
        return f"{nid}:0"

    def relu(nid, src, c, h):
        nodes.append(OpNode(nid, OpKind.RELU, (src,), img(c, h)))
        return f"{nid}:0"

    x, h = conv("stem.conv", "x:0", 3, 64, 7, 2, 3, image)
    x = relu("stem.relu", bn("stem.bn", x, 64, h), 64, h)
    hp = (h + 2 - 3) // 2 + 1
    nodes.append(OpNode("stem.pool", OpKind.MAX_POOL2D, (x,), img(64, hp),
                        attrs={"kernel": 3, "stride": 2, "padding": 1}))
    x, h, cin = "stem.pool:0", hp, 64
    for li, (nblocks, planes) in enumerate(zip(layers[:stages], (64, 128, 256, 512))):
        width = planes * width_per_group // 64 * groups
        cout = planes * 4
        for bi in range(nblocks):
            p = f"l{li + 1}.b{bi}"
            stride = 2 if (bi == 0 and li > 0) else 1
            y, h1 = conv(f"{p}.conv1", x, cin, width, 1, 1, 0, h)
            y = relu(f"{p}.relu1", bn(f"{p}.bn1", y, width, h1), width, h1)
            y, h2 = conv(f"{p}.conv2", y, width, width, 3, stride, 1, h1, g=groups)
            y = relu(f"{p}.relu2", bn(f"{p}.bn2", y, width, h2), width, h2)
            y, h3 = conv(f"{p}.conv3", y, width, cout, 1, 1, 0, h2)
            y = bn(f"{p}.bn3", y, cout, h3)
            if bi == 0:
                sc, _ = conv(f"{p}.down", x, cin, cout, 1, stride, 0, h)
                sc = bn(f"{p}.down_bn", sc, cout, h3)
            else:
                sc = x
            nodes.append(OpNode(f"{p}.add", OpKind.ADD, (y, sc), img(cout, h3)))
            x = relu(f"{p}.relu3", f"{p}.add:0", cout, h3)
            h, cin = h3, cout
    nodes.append(OpNode("pool", OpKind.MEAN_POOL2D, (x,), img(cin, 1),
                        attrs={"kernel": h, "stride": h}))
    g = Graph(tuple(nodes), {"x": img(3, image)}, ("pool:0",),
              metadata={"model": "resnext50_32x4d" if groups > 1 else "resnet50",
                        "batch": batch, "dtype": dtype})
    return g, plan


def fc_head(in_spec: TensorSpec, width: int, *, seed: int) -> tuple[Graph, WeightStore]:
    """Per-task CNN classifier: (B, C, 1, 1) -> Reshape (B, C) -> Linear."""
    dt = in_spec.dtype
    b, c = in_spec.dims[0], in_spec.dims[1]
    nodes = (OpNode("flat", OpKind.RESHAPE, ("feat:0",), _spec(dt, b, c), attrs={"dims": [b, c]}),
             OpNode("fc", OpKind.MATMUL, ("flat:0",), _spec(dt, b, width),
                    weights=("fc.w", "fc.b")))
    plan = [("fc.w", (c, width), f"fan:{c}"), ("fc.b", (width,), f"fan:{c}")]
    rng = np.random.default_rng([seed, 2, width])
    store = WeightStore({n: TensorValue(TensorSpec(dt, dims), _materialize(
        _draw(rng, dims, draw, False), dt)) for n, dims, draw in plan})
    return Graph(nodes, {"feat": in_spec}, ("fc:0",)), store


_BUILDERS: dict[str, Callable[[int, str], tuple[Graph, WeightPlan]]] = {
    "resnet50": lambda b, d: _resnet(b, d),
    "resnext50_32x4d": lambda b, d: _resnet(b, d, groups=32, width_per_group=4),
    # reduced variants for fast tests: one bottleneck per stage at 64x64
    "resnet-mini": lambda b, d: _resnet(b, d, layers=(1, 1, 1, 1), image=64),
    "resnext-mini": lambda b, d: _resnet(b, d, groups=32, width_per_group=4, layers=(1, 1, 1, 1),
                                         image=64),
    "ffnn": _ffnn,
    "cnnblock": _cnnblock,
    "attnblock": _attnblock,
    "bert-base": _bert,
    "bert-2l": bert_layers(2),
    "xlnet-base": _xlnet,
    "xlnet-2l": lambda b, d: _xlnet(b, d, XLNetConfig(layers=2)),
    # one encoder layer: the reference CPU path's bounded timing sample
    "bert-1l": bert_layers(1),
    "xlnet-1l": lambda b, d: _xlnet(b, d, XLNetConfig(layers=1)),
}

MODEL_NAMES = tuple(_BUILDERS)


def register(name: str, builder: Callable[[int, str], tuple[Graph, WeightPlan]]) -> None:
    _BUILDERS[name] = builder


# ----------------------------------------------------------------------------
# Seeded weights and inputs
# ----------------------------------------------------------------------------

def _draw(rng: np.random.Generator, dims, draw: str, zoo_exact: bool) -> np.ndarray:
    if zoo_exact:  # reference zoo.py:152-158 draws float64 then casts
        lo, hi = (0.5, 1.5) if draw == "var" else (-0.5, 0.5)
        return rng.uniform(lo, hi, size=dims)
    if draw.startswith("fan:"):
        bound = 1.0 / np.sqrt(float(draw[4:]))
        lo, hi = -bound, bound
    elif draw in ("var", "gamma"):
        lo, hi = 0.5, 1.5
    else:
        lo, hi = -0.5, 0.5
    u = rng.random(size=dims, dtype=np.float32)
    return (u * np.float32(hi - lo) + np.float32(lo)).astype(np.float32)


def _materialize(arr: np.ndarray, dtype: str) -> torch.Tensor:
    if dtype == "bf16":
        return torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32)).to(torch.bfloat16)
    return torch.from_numpy(np.ascontiguousarray(arr.astype(NUMPY_DTYPES[dtype])))


def build_graph(name: str, *, batch: int = 1, dtype: str = "f32") -> Graph:
    if name not in _BUILDERS:
        raise ValueError(f"unknown model {name!r}; choose from {tuple(_BUILDERS)}")
    if batch < 1:
        raise ValueError("batch must be >= 1")
    if dtype not in TORCH_DTYPES:
        raise ValueError(f"unknown dtype {dtype!r}")
    return _BUILDERS[name](batch, dtype)[0]


def build_weights(name: str, *, dtype: str = "f32", seed: int = 0, model: int = 0) -> WeightStore:
    """One model's parameters, deterministic in (name, dtype, seed, model)."""
    if name not in _BUILDERS:
        raise ValueError(f"unknown model {name!r}; choose from {tuple(_BUILDERS)}")
    _, plan = _BUILDERS[name](1, dtype)
    rng = np.random.default_rng([seed, 0, model])
    zoo_exact = name in ZOO_NAMES
    tensors = {}
    for wname, dims, draw in plan:
        arr = _draw(rng, dims, draw, zoo_exact)
        tensors[wname] = TensorValue(TensorSpec(dtype, dims), _materialize(arr, dtype))
    return WeightStore(tensors, model_index=model)


def build_zoo(name: str, *, batch: int = 1, dtype: str = "f32", seed: int = 0,
              num_models: int = 1) -> tuple[Graph, list[WeightStore]]:
    if num_models < 1:
        raise ValueError("num_models must be >= 1")
    graph = build_graph(name, batch=batch, dtype=dtype)
    return graph, [build_weights(name, dtype=dtype, seed=seed, model=m)
                   for m in range(num_models)]


def model_inputs(graph: Graph, *, seed: int = 0, model: int = 0) -> dict[str, TensorValue]:
    """Seeded inputs for one model, U[-1, 1] (zoo.py:173-184)."""
    rng = np.random.default_rng([seed, 1, model])
    fixed = set(graph.metadata.get("sinusoid_inputs", ()))
    out = {}
    for name, spec in graph.graph_inputs.items():
        if name in fixed:  # deterministic positional input, same for every model
            emb = relative_positional_embedding(spec.dims[-2] // 2, spec.dims[-1])
            arr = np.broadcast_to(emb, spec.dims)
        else:
            arr = rng.uniform(-1.0, 1.0, size=spec.dims)
        out[name] = TensorValue(spec, _materialize(arr, spec.dtype))
    return out


# ----------------------------------------------------------------------------
# Per-task heads (unmerged, attached with merge_backbone)
# ----------------------------------------------------------------------------

def classifier_head(in_spec: TensorSpec, width: int, *, seed: int,
                    pooler: bool = True) -> tuple[Graph, WeightStore]:
    """First-token classifier for encoder outputs (B, S, D): Slice token 0 ->
    [pooler dense + tanh] -> Linear(D -> width)."""
    dt = in_spec.dtype
    b, s, d = in_spec.dims
    nodes = [OpNode("cls", OpKind.SLICE, ("feat:0",), _spec(dt, b, d),
                    attrs={"axis": 1, "start": 0, "stop": 1, "squeeze": True})]
    plan: WeightPlan = []
    x = "cls:0"
    if pooler:
        nodes += [OpNode("pool", OpKind.MATMUL, (x,), _spec(dt, b, d), weights=("pool.w", "pool.b")),
                  OpNode("pool_act", OpKind.TANH, ("pool:0",), _spec(dt, b, d))]
        plan += [("pool.w", (d, d), f"fan:{d}"), ("pool.b", (d,), f"fan:{d}")]
        x = "pool_act:0"
    nodes.append(OpNode("logits", OpKind.MATMUL, (x,), _spec(dt, b, width),
                        weights=("logits.w", "logits.b")))
    plan += [("logits.w", (d, width), f"fan:{d}"), ("logits.b", (width,), f"fan:{d}")]
    g = Graph(tuple(nodes), {"feat": in_spec}, ("logits:0",))
    rng = np.random.default_rng([seed, 2, width])
    store = WeightStore({n: TensorValue(TensorSpec(dt, dims), _materialize(
        _draw(rng, dims, draw, False), dt)) for n, dims, draw in plan})
    return g, store


def head_widths(n: int) -> list[int]:
    """Deterministic per-task class counts (GLUE-like: 2, 3, ... )."""
    return [2 + (m % 4) for m in range(n)]


# ----------------------------------------------------------------------------
# BASELINE configurations as merged workloads (bench.py and the config parity
# tests build the exact same plan through this one function)
# ----------------------------------------------------------------------------

def merged_workload(model: str, instances: int, batch: int, dtype: str = "bf16",
                    first_instance: int = 0, heads: bool = True):
    """Instances ``first_instance .. first_instance+instances-1`` of ``model``
    merged into one graph: every instance its own seeded weights and inputs,
    plus (``heads``) its own unmerged per-task head attached with
    ``merge_backbone``: FC 2048->1000 for the CNNs, a
    first-token pooler + classifier (``head_widths``) for the encoders.

    Returns (graph, stores, inputs, merged, merged_store, heads)."""
    from .merger import merge, merge_backbone

    graph = build_graph(model, batch=batch, dtype=dtype)
    ids = list(range(first_instance, first_instance + instances))
    stores = [build_weights(model, dtype=dtype, seed=0, model=m) for m in ids]
    inputs = [model_inputs(graph, seed=0, model=m) for m in ids]
    head_list = None
    if heads:
        out = graph.node_map()[graph.graph_outputs[0].rsplit(":", 1)[0]].output_spec
        if len(out.dims) == 4:  # CNN: per-task FC 2048 -> 1000 on the pooled features
            head_list = [fc_head(out, 1000, seed=100 + m) for m in ids]
        else:
            widths = head_widths(first_instance + instances)[first_instance:]
            head_list = [classifier_head(out, w, seed=100 + m) for m, w in zip(ids, widths)]
        merged, mstore = merge_backbone(graph, {n.id for n in graph.nodes}, stores, head_list)
    else:
        merged, mstore = merge(graph, stores)
    return graph, stores, inputs, merged, mstore, head_list


def instance_workload(model: str, m: int, batch: int, dtype: str = "bf16",
                      heads: bool = True, total: int | None = None):
    """Instance ``m`` of ``merged_workload`` on its own (unmerged serving
    strategies): the same seeded weights, inputs and per-task head.
    ``total`` = the instance count the head widths are drawn for.

    Returns (graph, store, inputs, head or None)."""
    graph = build_graph(model, batch=batch, dtype=dtype)
    store = build_weights(model, dtype=dtype, seed=0, model=m)
    inputs = model_inputs(graph, seed=0, model=m)
    head = None
    if heads:
        out = graph.node_map()[graph.graph_outputs[0].rsplit(":", 1)[0]].output_spec
        if len(out.dims) == 4:
            head = fc_head(out, 1000, seed=100 + m)
        else:
            head = classifier_head(out, head_widths(max(total or 0, m + 1))[m], seed=100 + m)
    return graph, store, inputs, head


def layer_count(model: str) -> int | None:
    """Encoder layers of a transformer family member (None for CNNs)."""
    if model.startswith("bert"):
        return BERT_BASE.layers if model == "bert-base" else int(model.split("-")[1][:-1])
    if model.startswith("xlnet"):
        return XLNET_BASE.layers if model == "xlnet-base" else int(model.split("-")[1][:-1])
    return None


def one_layer_model(model: str) -> str | None:
    """The one-layer member of a transformer family (timing samples)."""
    if model.startswith("bert"):
        return "bert-1l"
    if model.startswith("xlnet"):
        return "xlnet-1l"
    return None


# BASELINE.json configs (name -> model, instances, batch, dtype)
BASELINE_CONFIGS = {
    "C1": ("resnet50", 2, 1, "f32"),
    "C2": ("bert-base", 8, 1, "bf16"),
    "C3": ("resnext50_32x4d", 32, 1, "bf16"),
    "C4": ("xlnet-base", 32, 4, "bf16"),
    "C5": ("bert-base", 32, 8, "bf16"),  # per-GPU shard of N=256 over 8 GPUs
}
