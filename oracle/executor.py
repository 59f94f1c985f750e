"""Oracle graph executor — TEST INFRASTRUCTURE ONLY (see oracle/kernels.py).

Runs an IR graph node by node on the CPU with the oracle kernels, in the
reference's deterministic topological order (engine.py:516-573 semantics).
bf16 graphs execute in fp32 on operands pre-rounded to bf16 (RNE), the
oracle convention of SURVEY §8c.
"""

from __future__ import annotations

import numpy as np

from . import kernels as K


def _np(t) -> np.ndarray:
    import torch
    if isinstance(t, torch.Tensor):
        t = t.detach()
        if t.dtype == torch.bfloat16:
            t = t.float()
        return t.cpu().numpy()
    return np.asarray(t)


def _compute_dtype(dtype: str):
    return np.float64 if dtype == "f64" else np.float32


def run_node(node, xs, ws):
    """Dispatch one node to its oracle kernel (mirrors engine._run_node,
    engine.py:456-510, plus the extension kinds)."""
    kind = node.kind.value
    a = node.attrs
    x = xs[0] if xs else None
    bias = ws[1] if len(ws) > 1 else None
    if kind == "Conv2D":
        return K.conv2d(x, ws[0], bias, stride=a["stride"], padding=a["padding"])
    if kind == "GroupedConv2D":
        return K.grouped_conv2d(x, ws[0], bias, groups=a["groups"], stride=a["stride"],
                                padding=a["padding"])
    if kind == "MatMul":
        return K.matmul(x, ws[0], bias)
    if kind == "BatchMatMul":
        return K.batch_matmul(x, ws[0], bias)
    if kind == "LayerNorm":
        return K.layer_norm(x, ws[0], ws[1], eps=a["eps"])
    if kind == "GroupNorm":
        return K.group_norm(x, ws[0], ws[1], groups=a["groups"], eps=a["eps"])
    if kind == "BatchNorm":
        return K.batch_norm_inference(x, *ws, eps=a["eps"])
    if kind == "ReLU":
        return K.relu(x)
    if kind == "Tanh":
        return K.tanh(x)
    if kind == "GELU":
        return K.gelu(x)
    if kind == "Softmax":
        return K.softmax(x, axis=a["axis"])
    if kind == "MaxPool2D":
        return K.max_pool2d(x, kernel=a["kernel"], stride=a["stride"], padding=a.get("padding", 0))
    if kind == "MeanPool2D":
        return K.mean_pool2d(x, kernel=a["kernel"], stride=a["stride"],
                             padding=a.get("padding", 0))
    if kind == "Add":
        return K.add(x, xs[1])
    if kind == "Mul":
        return K.mul(x, xs[1])
    if kind == "Concat":
        return np.concatenate(xs, axis=a["axis"])
    if kind == "Reshape":
        return np.ascontiguousarray(x.reshape(tuple(a["dims"])))
    if kind == "Transpose":
        return np.ascontiguousarray(np.transpose(x, tuple(a["perm"])))
    if kind == "Pack":
        return K.pack(xs, dim=a["dim"])
    if kind == "Unpack":
        return K.unpack(x, a["count"], dim=a["dim"], stacked=a["stacked"])[a["index"]]
    if kind == "Attention":
        return K.attention(x, heads=a["heads"], scale=a.get("scale"))
    if kind == "RelAttention":
        return K.rel_attention(x, xs[1], ws[0], ws[1], heads=a["heads"], scale=a.get("scale"))
    if kind == "Slice":
        ax = a["axis"] % x.ndim
        sl = [slice(None)] * x.ndim
        sl[ax] = slice(a["start"], a["stop"])
        out = x[tuple(sl)]
        if a.get("squeeze", False):
            out = np.squeeze(out, axis=ax)
        return np.ascontiguousarray(out)
    raise NotImplementedError(f"oracle has no kernel for {kind}")


def execute(graph, weights, inputs, *, keep=False):
    """Run ``graph`` with ``weights`` (name -> array or TensorValue) and
    ``inputs`` (name -> array or TensorValue). Returns the list of outputs
    (and every node value when ``keep``)."""
    from paper_2009_13062_b200.ir import parse_ref, topological_order

    def arr(v, dtype):
        v = _np(getattr(v, "data", v))
        if dtype == "bf16":
            return K.bf16_round(v)
        return np.ascontiguousarray(v, dtype=_compute_dtype(dtype))

    vals = {name: arr(inputs[name], spec.dtype) for name, spec in graph.graph_inputs.items()}
    wcache = {}
    for node in topological_order(graph):
        xs = [vals[parse_ref(r)[0]] for r in node.inputs]
        ws = []
        for w in node.weights:
            if w not in wcache:
                wcache[w] = arr(weights[w], node.output_spec.dtype)
            ws.append(wcache[w])
        out = run_node(node, xs, ws)
        if tuple(out.shape) != node.output_spec.dims:
            raise K.OracleShapeError(f"{node.id}: produced {out.shape}, "
                                     f"declared {node.output_spec.dims}")
        vals[node.id] = np.ascontiguousarray(out)
    outs = [vals[parse_ref(r)[0]] for r in graph.graph_outputs]
    return (outs, vals) if keep else outs
