"""PyTorch (cuBLAS / cuDNN / SDPA) executor for IR graphs — the "N separate
runs" baseline of the BASELINE metric (speedup vs N unmerged
per-instance runs on the same GPU, measured with PyTorch eager and with this
framework's own kernels at M=1).

Not part of the product: bench.py times it beside the merged plan. Each node
maps to the stock PyTorch op a user of the paper's PyTorch 1.3 setup would
call: F.linear, F.scaled_dot_product_attention, the
transformers XLNet relative attention (einsum + rel_shift_bnij), F.conv2d in
channels_last, F.batch_norm, F.layer_norm, pools and pointwise ops.
"""

from __future__ import annotations

import math

import torch
import torch.nn.functional as F

from paper_2009_13062_b200.ir import channel_axis, parse_ref, topological_order
from paper_2009_13062_b200.tensors import TORCH_DTYPES


class TorchModel:
    """One (unmerged) graph with its own weights, resident on ``device``."""

    def __init__(self, graph, store, device="cuda"):
        self.graph = graph
        self.order = topological_order(graph)
        self.dev = torch.device(device)
        self.w: dict[str, torch.Tensor] = {}
        for node in self.order:
            kind = node.kind.value
            for i, name in enumerate(node.weights):
                if name in self.w:
                    continue
                t = store[name].data.to(self.dev)
                if kind in ("MatMul", "BatchMatMul") and i == 0:
                    t = t.transpose(-1, -2).contiguous()  # (…, N, K) for F.linear
                elif kind in ("Conv2D", "GroupedConv2D") and i == 0:
                    t = t.contiguous(memory_format=torch.channels_last)
                elif kind == "BatchNorm":
                    t = t.float()
                self.w[name] = t
        self.inputs = {n: torch.empty(s.dims, dtype=TORCH_DTYPES[s.dtype], device=self.dev)
                       for n, s in graph.graph_inputs.items()}

    def load(self, inputs: dict, non_blocking=True):
        for n, v in inputs.items():
            data = getattr(v, "data", v)
            self.inputs[n].copy_(data, non_blocking=non_blocking)

    def forward(self) -> list[torch.Tensor]:
        vals = dict(self.inputs)
        for node in self.order:
            xs = [vals[parse_ref(r)[0]] for r in node.inputs]
            ws = [self.w[n] for n in node.weights]
            vals[node.id] = _run(node, xs, ws)
        return [vals[parse_ref(r)[0]] for r in self.graph.graph_outputs]


def _run(node, xs, ws):
    k = node.kind.value
    a = node.attrs
    x = xs[0] if xs else None
    b = ws[1] if len(ws) > 1 else None
    if k == "MatMul":
        return F.linear(x, ws[0], b)
    if k == "BatchMatMul":
        y = torch.matmul(x, ws[0].transpose(-1, -2).unsqueeze(1) if x.dim() == 4
                         else ws[0].transpose(-1, -2))
        return y if b is None else y + b.view(b.shape[0], *([1] * (y.dim() - 2)), b.shape[-1])
    if k in ("Conv2D", "GroupedConv2D"):
        x = x.contiguous(memory_format=torch.channels_last)
        return F.conv2d(x, ws[0], b, stride=a["stride"], padding=a["padding"],
                        groups=a.get("groups", 1))
    if k == "BatchNorm":
        return F.batch_norm(x, ws[2], ws[3], ws[0], ws[1], False, 0.0, a["eps"])
    if k == "LayerNorm":
        return F.layer_norm(x, (x.shape[-1],), ws[0].to(x.dtype), ws[1].to(x.dtype), a["eps"])
    if k == "GroupNorm":
        ca = channel_axis(x.dim())
        xt = x.movedim(ca, 1)
        y = F.group_norm(xt, a["groups"], ws[0].to(x.dtype), ws[1].to(x.dtype), a["eps"])
        return y.movedim(1, ca)
    if k == "ReLU":
        return F.relu(x)
    if k == "Tanh":
        return torch.tanh(x)
    if k == "GELU":
        return F.gelu(x)
    if k == "Add":
        return x + xs[1]
    if k == "Mul":
        return x * xs[1]
    if k == "Softmax":
        return torch.softmax(x, dim=a["axis"])
    if k == "MaxPool2D":
        return F.max_pool2d(x, a["kernel"], a["stride"], a.get("padding", 0))
    if k == "MeanPool2D":
        return F.avg_pool2d(x, a["kernel"], a["stride"], a.get("padding", 0))
    if k == "Slice":
        ax = a["axis"] % x.dim()
        y = x.narrow(ax, a["start"], a["stop"] - a["start"])
        return y.squeeze(ax) if a.get("squeeze", False) else y
    if k == "Reshape":
        return x.reshape(tuple(a["dims"]))
    if k == "Transpose":
        return x.permute(tuple(a["perm"]))
    if k == "Concat":
        return torch.cat(xs, dim=a["axis"])
    if k == "Attention":
        return _attention(x, a["heads"], a.get("scale"))
    if k == "RelAttention":
        return _rel_attention(x, xs[1], ws[0], ws[1], a["heads"], a.get("scale"))
    raise NotImplementedError(f"torch baseline has no lowering for {k}")


def _attention(qkv, heads, scale):
    *lead, s, d3 = qkv.shape
    d = d3 // 3
    dh = d // heads
    q, k, v = qkv.reshape(-1, s, 3, heads, dh).permute(2, 0, 3, 1, 4)
    o = F.scaled_dot_product_attention(q, k, v, scale=scale)
    return o.transpose(1, 2).reshape(*lead, s, d)


def _rel_attention(qkv, r, rwb, rrb, heads, scale):
    """transformers XLNetRelativeAttention.rel_attn_core (attn_type "bi", no
    segments / mask) with rel_shift_bnij, in the input dtype."""
    *lead, s, d3 = qkv.shape
    d = d3 // 3
    dh = d // heads
    q, k, v = qkv.reshape(-1, s, 3, heads, dh).unbind(2)
    kr = r.reshape(-1, 2 * s, heads, dh)
    if kr.shape[0] != q.shape[0]:  # positional keys shared by an instance's sequences
        kr = kr.repeat_interleave(q.shape[0] // kr.shape[0], dim=0)
    rw = rwb.reshape(heads, dh).to(qkv.dtype)
    rr = rrb.reshape(heads, dh).to(qkv.dtype)
    ac = torch.einsum("bihd,bjhd->bhij", q + rw, k)
    bd = torch.einsum("bihd,bjhd->bhij", q + rr, kr)
    bsz, h, i_len, j_len = bd.shape
    bd = bd.reshape(bsz, h, j_len, i_len)[:, :, 1:, :].reshape(bsz, h, i_len, j_len - 1)
    bd = bd[..., :s]
    sc = 1.0 / math.sqrt(dh) if scale is None else scale
    prob = torch.softmax((ac + bd) * sc, dim=-1)
    ctx = torch.einsum("bhij,bjhd->bihd", prob, v)
    return ctx.reshape(*lead, s, d)
