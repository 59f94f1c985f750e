"""GPU executor for (merged) graphs — the drop-in for the reference's
``execute`` (pkg/src/modelmerge/engine.py:516-573) and its ``_run_node``
dispatch seam (engine.py:456-510).

A graph is compiled once into a :class:`Plan`: a list of launch closures
over preallocated device buffers, each one C-ABI call into the sm_100a
library, so a forward is replayable as a single CUDA graph (no host work per
node). Compilation does three B200-specific things the reference cannot:

* **kernel-native weights**: merged Linear weights are transposed once to
  K-major (G, N, K) bf16 for the tcgen05 GEMM; biases / norm affines become
  fp32; everything lives in HBM for the life of the plan;
* **zero-copy glue**: the merger's Pack / Transpose / Reshape / Unpack
  junctions (merger.py:237-301, 418-513) become tensor views. A reshape that
  merges a model axis into the channel axis is kept *unmaterialised* (a
  "split" value: logical (..., M*C), physical (M, ..., C) model-major) and
  the grouped norm / pointwise kernels consume it directly, so the BERT
  plan's per-LayerNorm transposes cost nothing;
* **epilogue fusion**: an activation whose only consumer is a Linear's output
  is folded into the GEMM epilogue.

Arithmetic ``mode``: "fast" (tensor cores, FMA) or "exact" (reference
accumulation order, f32).
"""

from __future__ import annotations

import math
import threading
import time
from dataclasses import dataclass, field
from typing import Callable

import torch

from . import _lib
from . import kernels as K
from .errors import ExecutionError, ShapeError, UnsupportedOpError
from .ir import (
    Graph,
    MergeDim,
    OpKind,
    OpNode,
    TensorSpec,
    channel_axis,
    parse_ref,
    topological_order,
)
from .tensors import TORCH_DTYPES, TensorValue, WeightStore

_BOUNDARY = (OpKind.PACK, OpKind.UNPACK)
_ACT_OF = {OpKind.RELU: _lib.NF_ACT_RELU, OpKind.GELU: _lib.NF_ACT_GELU,
           OpKind.TANH: _lib.NF_ACT_TANH}
_EW_OF = {OpKind.ADD: _lib.NF_EW_ADD, OpKind.MUL: _lib.NF_EW_MUL, OpKind.RELU: _lib.NF_EW_RELU,
          OpKind.TANH: _lib.NF_EW_TANH, OpKind.GELU: _lib.NF_EW_GELU}
_MODES = {"fast": _lib.NF_MODE_FAST, "exact": _lib.NF_MODE_EXACT}
# Channels per densified super-group for narrow grouped convs (ResNeXt).
_SUPER_GROUP = 64


class _LinearStep:
    """One merged-Linear launch. A later norm lowering may attach a residual
    and folded-LayerNorm operands to it (it is emitted before the norm that
    absorbs its output is seen)."""

    def __init__(self, x, k, w, b, y, n, groups, rows, dcode, layout, act, mcode, ws, wsb,
                 fold_ok):
        self.x, self.k, self.w, self.b, self.y, self.n = x, k, w, b, y, n
        self.groups, self.rows, self.dcode, self.layout = groups, rows, dcode, layout
        self.act, self.mcode, self.ws, self.wsb = act, mcode, ws, wsb
        self.fold_ok = fold_ok
        self.residual = None
        self.fin = None   # (stats, parts, colsum, eps)
        self.fres = None  # (stats, parts, gamma, beta, eps)
        self.out_stats = None

    def __call__(self, st):
        k, n, rows = self.k, self.n, self.rows
        if self.fin is None and self.fres is None and self.out_stats is None:
            _lib.call("nf_grouped_linear_ws", self.x, k, rows * k, self.w, self.b, self.residual,
                      self.y, n, rows * n, self.groups, rows, k, n, self.dcode, self.layout,
                      self.act, self.mcode, self.ws, self.wsb, st)
            return
        fin = self.fin or (None, 0, None, 0.0)
        fres = self.fres or (None, 0, None, None, 0.0)
        _lib.call("nf_grouped_linear_fold", self.x, k, rows * k, self.w, self.b, self.residual,
                  self.y, n, rows * n, self.groups, rows, k, n, self.act, self.ws, self.wsb,
                  *fin, *fres, self.out_stats, st)


class _ChainStep:
    """Consecutive batch-1 merged Linears of one model run as ONE persistent
    launch (``nf_grouped_linear_chain``): weight tiles of op j+1 stream while
    op j finishes, units wait on per-instance completion counters. Built by
    :meth:`Plan._chain_linears` from finished :class:`_LinearStep` s."""

    def __init__(self, members: list[tuple[str, "_LinearStep"]], counters: torch.Tensor):
        self.members = members
        self.counters = counters
        self.groups = members[0][1].groups
        ops = (_lib.LinearOp * len(members))()
        for o, (_, ls) in zip(ops, members):
            k, n, rows = ls.k, ls.n, ls.rows
            o.x, o.x_ld, o.x_gs, o.w, o.bias = ls.x, k, rows * k, ls.w, ls.b
            o.residual, o.y, o.y_ld, o.y_gs = ls.residual, ls.y, n, rows * n
            o.rows, o.k, o.n, o.act = rows, k, n, ls.act
            o.workspace, o.workspace_bytes = ls.ws, ls.wsb
            if ls.fin is not None:
                o.in_stats, o.in_parts, o.in_colsum, o.in_eps = ls.fin
            if ls.fres is not None:
                o.res_stats, o.res_parts, o.res_gamma, o.res_beta, o.res_eps = ls.fres
            o.out_stats = ls.out_stats
        self.ops = ops

        self.keep = False  # a later launch reads the counters (Plan._link_chains)
        self.dep = None    # (ptr, target): per-instance completion of op 0's producer

    def __call__(self, st):
        if not self.keep and self.dep is None:
            _lib.call("nf_grouped_linear_chain", len(self.members), self.ops, self.groups,
                      self.counters.data_ptr(), st)
            return
        dp, dt = self.dep if self.dep is not None else (None, 0)
        _lib.call("nf_grouped_linear_chain_ex", len(self.members), self.ops, self.groups,
                  self.counters.data_ptr(), _lib.NF_CHAIN_KEEP_COUNTERS if self.keep else 0,
                  dp, dt, st)


class _QKVStep:
    """One fused QKV-projection + attention launch at batch 1. When its input
    is the last output of a chained launch, :meth:`Plan._link_chains` points
    ``dep`` at that chain's per-instance completion counters: instance g's
    heads start once the chain stored g's tiles (nf_qkv_attention_after)."""

    def __init__(self, x, d, w, b, y, groups, heads, scale, fold):
        self.x, self.d, self.w, self.b, self.y = x, d, w, b, y
        self.groups, self.heads, self.scale = groups, heads, scale
        self.fold = fold  # (stats, parts, colsum, eps) or None
        self.dep = None   # (counters ptr, target) or None
        self.done = None  # [groups] counters this launch bumps per stored head

    def __call__(self, st):
        x, d, g, h, sc = self.x, self.d, self.groups, self.heads, float(self.scale)
        if self.dep is not None or self.done is not None:
            sp, parts, cp, eps = self.fold if self.fold else (None, 0, None, 0.0)
            dp, dt = self.dep if self.dep is not None else (None, 0)
            _lib.call("nf_qkv_attention_after", x, d, 128 * d, self.w, self.b, self.y, g, 128, d,
                      h, sc, sp, parts, cp, eps, dp, dt, self.done, st)
        elif self.fold is not None:
            _lib.call("nf_qkv_attention_fold", x, d, 128 * d, self.w, self.b, self.y, g, 128, d,
                      h, sc, *self.fold, st)
        else:
            _lib.call("nf_qkv_attention", x, d, 128 * d, self.w, self.b, self.y, g, 128, d, h,
                      sc, st)


class _LinkedStep:
    """A merged conv launch (implicit GEMM, or a 1x1 conv as a grouped GEMM)
    that :meth:`Plan._link_convs` may link per instance: its units of
    instance m start once the launches producing its input / residual stored
    m's tiles, and it counts its own stored tiles per instance."""

    def __init__(self, kind, args, x, residual, y, groups, gpi, units, ws_need):
        self.kind, self.args = kind, args  # "gemm" | "conv", plain-call arguments
        self.x, self.residual, self.y = x, residual, y
        self.groups, self.gpi, self.units = groups, gpi, units  # units: tiles per group
        self.ws_need = ws_need
        self.dep_x = self.dep_r = None  # (counters ptr, target)
        self.done = None                 # counters ptr

    def set_workspace(self, ptr, nbytes):
        self.args = self.args[:-2] + (ptr, nbytes)  # both call forms end (ws, ws_bytes)

    def __call__(self, st):
        if self.dep_x is None and self.done is None:
            name = "nf_grouped_linear_ws" if self.kind == "gemm" else "nf_grouped_conv_tc"
            _lib.call(name, *self.args, st)
            return
        dx, tx = self.dep_x if self.dep_x else (None, 0)
        dr, tr = self.dep_r if self.dep_r else (None, 0)
        if self.kind == "gemm":
            a = self.args  # nf_grouped_linear_ws arguments
            _lib.call("nf_grouped_linear_linked", *a[:13], a[15], a[17], a[18], dx, tx, dr, tr,
                      self.done, self.gpi, st)
        else:
            _lib.call("nf_grouped_conv_tc_linked", *self.args, dx, tx, dr, tr, self.done,
                      self.gpi, st)


@dataclass
class _FoldedNorm:
    """A per-instance LayerNorm that is not launched: ``raw`` (G, T, D) holds
    its input, ``stats`` the producer's per-token partial sums; ``out`` is
    only written if some consumer cannot fold it (``emit``)."""

    node_id: str
    raw: torch.Tensor
    out: torch.Tensor
    stats: torch.Tensor
    parts: int
    gamma: torch.Tensor
    beta: torch.Tensor
    gamma_name: str
    eps: float
    m: int
    rows: int
    d: int
    emit: Callable[[int], None]


@dataclass
class ExecTrace:
    """What one execute() did (reference engine.py:428-443), plus the number
    of sm_100a kernel launches the plan issued."""

    node_outputs: dict[str, TensorValue] = field(default_factory=dict)
    node_times_ns: dict[str, int] = field(default_factory=dict)
    op_invocations: int = 0
    dispatch_count: int = 0
    kernel_launches: int = 0
    total_ns: int = 0


@dataclass
class DVal:
    """A device value. ``t`` is a (possibly strided) view; when ``split`` is
    set, logical axis ``split`` is the merge of ``t``'s axes split, split+1
    (model-major storage of a channel-packed tensor, never materialised)."""

    t: torch.Tensor
    dims: tuple[int, ...]
    split: int | None = None

    @property
    def dtype(self):
        return self.t.dtype


def _dense_block(t: torch.Tensor) -> bool:
    """True when ``t`` is a permutation of one contiguous storage block."""
    if t.numel() == 0:
        return False
    pairs = sorted((s, d) for s, d in zip(t.stride(), t.shape) if d != 1)
    expect = 1
    for s, d in pairs:
        if s != expect:
            return False
        expect *= d
    return True


def _same_physical(a: DVal, b: DVal) -> bool:
    return (a.split == b.split and a.t.shape == b.t.shape and a.t.stride() == b.t.stride()
            and a.dims == b.dims)


def _flatten_rows(shape, strides) -> tuple[int, int] | None:
    """Collapse dims into one (count, stride) if they are uniformly strided."""
    dims = [(d, s) for d, s in zip(shape, strides) if d != 1]
    if not dims:
        return 1, 0
    count = 1
    for i in range(len(dims) - 1):
        if dims[i][1] != dims[i + 1][0] * dims[i + 1][1]:
            return None
    for d, _ in dims:
        count *= d
    return count, dims[-1][1]


class Plan:
    """A compiled graph: preallocated buffers plus one launch closure per
    kernel. ``run`` executes eagerly; ``capture`` records a CUDA graph."""

    def __init__(self, graph: Graph, weights: WeightStore, *, mode: str = "fast",
                 device: str | torch.device = "cuda", fuse: bool = True,
                 fold_ln: bool = True, chain: bool = True, weight_cache: dict | None = None):
        if mode not in _MODES:
            raise ValueError(f"mode must be one of {sorted(_MODES)}")
        if torch.device(device).type == "cuda" and not torch.cuda.is_available():
            raise UnsupportedOpError("a CUDA (sm_100a) device is required; there is no CPU "
                                     "fallback for the merged operators")
        _lib.load()
        self.graph = graph
        self.mode = mode
        self.mcode = _MODES[mode]
        self.device = torch.device(device)
        self.fuse = fuse
        # the store's specs (a pre-tiled artifact rebuilds a spec-only store)
        self.weight_specs = {name: tv.spec for name, tv in weights.tensors.items()}
        self.steps: list[tuple[str, Callable[[int], None], int]] = []  # (node, fn, launches)
        self.vals: dict[str, DVal] = {}
        self.input_views: dict[str, torch.Tensor] = {}
        self.out_buffers: list[torch.Tensor] = []
        self.out_sources: list[DVal] = []
        # converted device weights; plans of one (graph, store) may share it
        self._wcache: dict[tuple, torch.Tensor] = {} if weight_cache is None else weight_cache
        self._buffers: list[torch.Tensor] = []
        # Adds whose launch is deferred so the consuming norm can fuse them:
        # output data_ptr -> (node id, a, b, out, launch closure)
        self._deferred: dict[int, tuple] = {}
        # Batch-1 LayerNorms folded into their producing / consuming GEMMs (no
        # norm launch; include/netfuse_b200.h "Folded LayerNorm")
        self.fold_ln = fold_ln
        self.chain = chain
        self._add_into_norm: dict[str, str] = {}
        self._lin_out: dict[int, _LinearStep] = {}  # output data_ptr -> its launch
        self._folded: dict[int, _FoldedNorm] = {}   # out data_ptr -> folded norm (not launched)
        self._cuda_graph: torch.cuda.CUDAGraph | None = None
        self.dispatch_count = 0
        self.op_invocations = 0
        self._build(weights)

    # ----------------------------------------------------------------- weights
    def _w(self, weights: WeightStore, name: str, kind: str, dtype: torch.dtype,
           cache: bool = True) -> torch.Tensor:
        """``name`` converted to a kernel layout on the device; ``cache=False``
        for intermediates of a derived layout (not kept in HBM)."""
        key = (name, kind, dtype)
        if key in self._wcache:
            return self._wcache[key]
        src = weights[name].data
        if kind == "linear_nk":  # (G, K, N) or (K, N) -> (G, N, K) K-major
            w = src if src.dim() == 3 else src.unsqueeze(0)
            out = w.to(self.device, dtype).transpose(1, 2).contiguous()
        elif kind == "linear_kn":
            w = src if src.dim() == 3 else src.unsqueeze(0)
            out = w.to(self.device, dtype).contiguous()
        elif kind == "vec_f32":
            out = src.to(self.device, torch.float32).contiguous()
        elif kind == "same":
            out = src.to(self.device, dtype).contiguous()
        else:  # pragma: no cover
            raise AssertionError(kind)
        if cache:
            self._wcache[key] = out
        return out

    # ---------------------------------------------------------------- helpers
    def _workspace(self, groups, rows, k, n) -> torch.Tensor | None:
        """One zero-initialised split-K workspace shared by every GEMM of the
        plan (launches are stream-ordered; the kernel re-arms semaphores)."""
        need = int(_lib.load().nf_linear_workspace_bytes(groups, rows, k, n))
        if need <= 0:
            return None
        return self._ws_buffer(need)

    def _ws_buffer(self, need: int) -> torch.Tensor:
        cur = getattr(self, "_ws", None)
        if cur is None or cur.numel() < need:
            # A larger shape gets a fresh buffer; earlier launches keep theirs.
            self._ws = self._own(torch.zeros(need, dtype=torch.uint8, device=self.device))
        return self._ws

    def _alloc(self, dims, dtype) -> torch.Tensor:
        return self._own(torch.empty(tuple(dims), dtype=dtype, device=self.device))

    def _own(self, t: torch.Tensor) -> torch.Tensor:
        """Launch closures capture raw device pointers, so the plan must own
        every buffer it hands to a kernel for its whole lifetime (otherwise
        the caching allocator would recycle a temporary's memory)."""
        self._buffers.append(t)
        return t

    def _emit(self, node_id: str, fn: Callable[[int], None], launches: int = 1) -> None:
        self.steps.append((node_id, fn, launches))

    def _copy_step(self, node_id: str, src: torch.Tensor, dst: torch.Tensor) -> None:
        import ctypes
        self._flush_deferred(src)
        rank = max(src.dim(), 1)
        arr = ctypes.c_int64 * rank
        dims = arr(*(src.shape or (1,)))
        ss = arr(*(src.stride() or (1,)))
        ds = arr(*(dst.stride() or (1,)))
        sp, dp, es = src.data_ptr(), dst.data_ptr(), src.element_size()
        self._emit(node_id, lambda st: _lib.call("nf_copy_strided", sp, dp, rank, dims, ss, ds,
                                                 es, st))

    def _materialize(self, node_id: str, v: DVal) -> torch.Tensor:
        """Contiguous tensor with the logical dims of ``v`` (copy if needed)."""
        if v.split is None and v.t.is_contiguous():
            return v.t
        out = self._alloc(v.dims, v.dtype)
        if v.split is None:
            self._copy_step(node_id, v.t, out)
        else:
            a = v.split
            m, c = v.t.shape[a], v.t.shape[a + 1]
            self._copy_step(node_id, v.t, out.view(v.dims[:a] + (m, c) + v.dims[a + 1:]))
        return out

    # ------------------------------------------------------------------ build
    def _build(self, weights: WeightStore) -> None:
        g = self.graph
        order = topological_order(g)
        users: dict[str, list[OpNode]] = {}
        for n in order:
            for r in n.inputs:
                users.setdefault(parse_ref(r)[0], []).append(n)
        outputs = {parse_ref(r)[0] for r in g.graph_outputs}
        self._users, self._outputs = users, outputs

        # Graph inputs: Pack-only inputs alias their slice of the packed buffer.
        packs = [n for n in order if n.kind is OpKind.PACK]
        for p in packs:
            dt = TORCH_DTYPES[p.output_spec.dtype]
            buf = self._alloc(p.output_spec.dims, dt)
            count, dim = p.attrs["count"], MergeDim(p.attrs["dim"])
            for j, ref in enumerate(p.inputs):
                name = parse_ref(ref)[0]
                per = g.graph_inputs.get(name)
                if per is None:
                    continue
                if dim is MergeDim.CHANNEL:
                    ca = channel_axis(len(per.dims))
                    view = buf.narrow(ca, j * per.dims[ca], per.dims[ca])
                elif p.attrs["stacked"]:
                    view = buf[j]
                else:
                    view = buf.narrow(0, j * per.dims[0], per.dims[0])
                only_pack = all(u.kind is OpKind.PACK for u in users.get(name, []))
                if only_pack and name not in self.input_views:
                    self.input_views[name] = view
            self.vals[p.id] = DVal(buf, p.output_spec.dims)
        for name, spec in g.graph_inputs.items():
            if name not in self.input_views:
                t = self._alloc(spec.dims, TORCH_DTYPES[spec.dtype])
                self.input_views[name] = t
            self.vals[name] = DVal(self.input_views[name], spec.dims)
        # Packs whose inputs are not pure graph inputs copy at run time.
        for p in packs:
            count, dim = p.attrs["count"], MergeDim(p.attrs["dim"])
            buf = self.vals[p.id].t
            for j, ref in enumerate(p.inputs):
                name = parse_ref(ref)[0]
                if name in g.graph_inputs and self._aliases(buf, self.input_views[name]):
                    continue
                src = self.vals[name]
                per = src.dims
                if dim is MergeDim.CHANNEL:
                    ca = channel_axis(len(per))
                    view = buf.narrow(ca, j * per[ca], per[ca])
                elif p.attrs["stacked"]:
                    view = buf[j]
                else:
                    view = buf.narrow(0, j * per[0], per[0])
                self._copy_step(p.id, self._materialize(p.id, src), view)

        fused_into: dict[str, str] = {}
        self._add_into_norm = self._fusable_adds(order, users, outputs) if self.fuse else {}
        groups = self._sibling_groups(order) if self.fuse else {}
        chains = self._conv_chains(order, users, outputs) \
            if self.fuse and self.mcode == _lib.NF_MODE_FAST else {}
        groups.update({cid: ch["nodes"] for cid, ch in chains.items()})
        done: set[str] = set()
        for node in self._grouped_order(order, groups):
            if node.id in done:
                continue
            if node.kind is OpKind.PACK:
                self.op_invocations += 1
                continue
            if node.id in fused_into:
                self.vals[node.id] = self.vals[fused_into[node.id]]
                self.op_invocations += 1
                self.dispatch_count += 1
                continue
            if node.id in chains:
                ch = chains[node.id]
                self._flush_members(ch["nodes"])
                try:
                    out = self._lower_conv_chain(ch, weights)
                except (ShapeError, UnsupportedOpError) as exc:
                    raise ExecutionError(node.id, exc) from exc
                last = ch["nodes"][-1]
                if tuple(out.dims) != last.output_spec.dims:
                    raise ExecutionError(node.id, ShapeError(
                        f"kernel produced {out.dims}, node declares {last.output_spec.dims}"))
                self.vals[last.id] = out
                for mem in ch["nodes"]:
                    done.add(mem.id)
                    self.op_invocations += 1
                    self.dispatch_count += 1
                continue
            members = groups.get(node.id)
            if members is not None:
                self._flush_members(members)
                try:
                    batched = self._lower_siblings(members, weights, users, outputs, fused_into)
                except (ShapeError, UnsupportedOpError) as exc:
                    raise ExecutionError(node.id, exc) from exc
                if batched:
                    for mem in members:
                        done.add(mem.id)
                        self.op_invocations += 1
                        self.dispatch_count += 1
                    continue
            ins = [self.vals[parse_ref(r)[0]] for r in node.inputs]
            for v in ins:
                self._flush_deferred(v.t, keep_for=node)
            attn = self._qkv_attention_pair(node, ins, weights, users, outputs)
            if attn is not None:
                try:
                    out = self._lower_qkv_attention(node, attn, ins[0], weights)
                except (ShapeError, UnsupportedOpError) as exc:
                    raise ExecutionError(node.id, exc) from exc
                self.vals[attn.id] = out
                done.add(attn.id)
                self.op_invocations += 2
                self.dispatch_count += 2
                continue
            try:
                act_user = None
                if self.fuse and node.kind in (OpKind.MATMUL, OpKind.BATCH_MATMUL):
                    us = users.get(node.id, [])
                    exact_ok = self.mcode == _lib.NF_MODE_FAST or (
                        us and us[0].kind is OpKind.RELU)
                    if len(us) == 1 and us[0].kind in _ACT_OF and node.id not in outputs \
                            and exact_ok:
                        act_user = us[0]
                        fused_into[act_user.id] = node.id
                out = self._lower(node, ins, weights, act_user)
            except (ShapeError, UnsupportedOpError) as exc:
                raise ExecutionError(node.id, exc) from exc
            if tuple(out.dims) != node.output_spec.dims:
                raise ExecutionError(node.id, ShapeError(
                    f"kernel produced {out.dims}, node declares {node.output_spec.dims}"))
            self.vals[node.id] = out
            self.op_invocations += 1
            if node.kind not in _BOUNDARY:
                self.dispatch_count += 1
        out_ts = [self.vals[parse_ref(r)[0]].t for r in g.graph_outputs]
        for key in list(self._deferred):
            if key not in self._deferred:
                continue
            fo = self._folded.get(key)
            if fo is not None and not any(self._aliases(fo.out, t) for t in out_ts):
                del self._deferred[key]  # every consumer folded it: never launched
                del self._folded[key]
                continue
            self._emit_deferred(key)

        for ref in g.graph_outputs:
            v = self.vals[parse_ref(ref)[0]]
            if v.split is None and tuple(v.t.shape) == tuple(v.dims):
                # a plan-owned buffer (or a view of one) is stable across
                # replays: hand it out as is, no copy launch
                self.out_buffers.append(v.t)
                continue
            buf = self._alloc(v.dims, v.dtype)
            if v.split is None:
                self._copy_step("output", v.t, buf)
            else:
                a = v.split
                m, c = v.t.shape[a], v.t.shape[a + 1]
                self._copy_step("output", v.t, buf.view(v.dims[:a] + (m, c) + v.dims[a + 1:]))
            self.out_buffers.append(buf)
        # the BN-folded fp32 conv weights only fed the kernel layouts above
        for key in [k for k in self._wcache if k[0] == "convchain" and len(k) == 2]:
            del self._wcache[key]
        if self.fuse and self.chain and self.mcode == _lib.NF_MODE_FAST:
            self._chain_linears()
            self._link_convs()

    def _gpi(self, groups: int) -> int:
        """Kernel groups per merged instance (0: unknown / not instance-aligned)."""
        m = (getattr(self.graph, "metadata", None) or {}).get("merge", {}).get("num_models")
        return groups // m if m and groups % m == 0 else 0

    def _link_convs(self) -> None:
        """Per-instance linking of merged conv launches (CNN plans): a conv
        whose input and residual both come from linked conv launches starts
        instance m's units once those stored m's tiles, instead of waiting for
        the whole previous launch -- each launch's tail overlaps the next
        launch's first instances. Linked launches with split-K get their own
        workspace (they may overlap other launches); the counters live in one
        buffer that a memset re-arms at the start of every forward."""
        linked = [fn for _, fn, _ in self.steps if isinstance(fn, _LinkedStep) and fn.gpi > 0]
        if not linked:
            return
        producers: dict[int, _LinkedStep] = {}
        consumers = []
        for fn in linked:
            px = producers.get(fn.x)
            pr = producers.get(fn.residual) if fn.residual else None
            if px is not None and (fn.residual is None or pr is not None):
                consumers.append((fn, px, pr))
            producers[fn.y] = fn
        if not consumers:
            return
        publishers = {id(p): p for _, px, pr in consumers for p in (px, pr) if p is not None}
        m = self.graph.metadata["merge"]["num_models"]
        buf = self._own(torch.zeros(-(-m * len(publishers) // 64) * 64, dtype=torch.int32,
                                    device=self.device))
        for i, p in enumerate(publishers.values()):
            p.done = buf[i * m:].data_ptr()
        for fn, px, pr in consumers:
            fn.dep_x = (px.done, px.units * px.gpi)
            if pr is not None:
                fn.dep_r = (pr.done, pr.units * pr.gpi)
        for fn in {id(f): f for f in [c[0] for c in consumers] + list(publishers.values())}.values():
            if fn.ws_need > 0:
                ws = self._own(torch.zeros(fn.ws_need, dtype=torch.uint8, device=self.device))
                fn.set_workspace(ws.data_ptr(), ws.numel())
        self._add_rearm(buf)

    def _add_rearm(self, buf: torch.Tensor) -> None:
        """Zero ``buf`` (per-instance counters) at the start of every forward."""
        if getattr(self, "_rearm_bufs", None) is None:
            self._rearm_bufs = []

            # A memset on the launch stream itself (nf_counters_rearm), not a
            # torch fill under an ExternalStream context: on the legacy default
            # stream (handle 0) that fill was measured racing the next
            # forward's linked launches (a counter spin trapped).
            def rearm(st, bufs=self._rearm_bufs):
                for b in bufs:
                    _lib.call("nf_counters_rearm", b.data_ptr(), b.numel() * b.element_size(), st)
            self.steps.insert(0, ("rearm", rearm, 0))
        self._rearm_bufs.append(buf)

    def _chainable(self, ls, run) -> bool:
        if not isinstance(ls, _LinearStep) or ls.dcode != _lib.NF_BF16 \
                or ls.layout != _lib.NF_W_NK or ls.mcode != _lib.NF_MODE_FAST:
            return False
        if ls.fin is not None and ls.fres is not None:
            return False
        if not _lib.load().nf_linear_chain_supported(ls.groups, ls.rows, ls.k, ls.n):
            return False
        if not run:
            return True
        head = run[0][1]
        # consumes the previous op's output; at most one op uses split-K
        # (they would share the plan's workspace)
        return (ls.groups == head.groups and ls.rows == head.rows and ls.x == run[-1][1].y
                and not (ls.wsb and any(m.wsb for _, m in run)))

    def _chain_linears(self) -> None:
        """Merge runs of 2-3 consecutive chainable merged-Linear launches
        (e.g. attention projection -> FF1 -> FF2 of a batch-1 encoder layer)
        into one persistent launch each."""
        out, i, steps, runs = [], 0, self.steps, []
        while i < len(steps):
            run = []
            while i + len(run) < len(steps) and len(run) < 3:
                nid, fn, _ = steps[i + len(run)]
                if not self._chainable(fn, run):
                    break
                run.append((nid, fn))
            if len(run) >= 2:
                runs.append((len(out), run))
                out.append(None)
                i += len(run)
            else:
                out.append(steps[i])
                i += 1
        if runs:
            # every chain's counters in one buffer (one memset re-arms them all)
            lib = _lib.load()
            sizes = [int(lib.nf_linear_chain_counter_bytes(len(r), r[0][1].groups)) // 4
                     for _, r in runs]
            sizes = [-(-n // 64) * 64 for n in sizes]  # 256-byte aligned slices
            buf = self._own(torch.zeros(sum(sizes), dtype=torch.int32, device=self.device))
            self._chain_counters = buf
            off = 0
            for (pos, run), n in zip(runs, sizes):
                out[pos] = ("chain:" + "+".join(m for m, _ in run),
                            _ChainStep(run, buf[off:off + n]), 1)
                off += n
        self.steps = out
        self._link_chains()

    def _link_chains(self) -> None:
        """A fused QKV+attention launch whose input is a chain's last output
        waits on that chain's per-instance counters instead of the whole
        launch; those chains keep their counters set, so one memset at the
        start of the forward re-arms them."""
        # Linked launches of consecutive layers overlap instance by instance,
        # and every split-K GEMM of the plan shares one workspace indexed by
        # (instance, tile): only safe when those GEMMs all tile alike (work on
        # the same (instance, tile) is ordered through the counters).
        splitk = {(m.groups, m.rows, m.k, m.n) for _, fn, _ in self.steps
                  if isinstance(fn, _ChainStep) for _, m in fn.members if m.wsb}
        splitk |= {(fn.groups, fn.rows, fn.k, fn.n) for _, fn, _ in self.steps
                   if isinstance(fn, _LinearStep) and fn.wsb}
        if len(splitk) > 1:
            return
        linked = False
        # attention -> chain: op 0 (proj) of instance g starts once g's heads
        # are stored (the QKV launch counts them in a slice of the same buffer)
        qkv_links = []
        for i in range(len(self.steps) - 1):
            fn, nxt = self.steps[i][1], self.steps[i + 1][1]
            if isinstance(fn, _QKVStep) and isinstance(nxt, _ChainStep) and \
                    nxt.members[0][1].x == fn.y and nxt.groups == fn.groups:
                qkv_links.append((fn, nxt))
        for i in range(1, len(self.steps)):
            fn, prev = self.steps[i][1], self.steps[i - 1][1]
            if not (isinstance(fn, _QKVStep) and isinstance(prev, _ChainStep)):
                continue
            last = prev.members[-1][1]
            if fn.x != last.y or fn.groups != prev.groups or \
                    (fn.fold is not None and fn.fold[0] != last.out_stats):
                continue
            j = len(prev.members) - 1
            ptr = prev.counters.data_ptr() + 4 * j * prev.groups
            fn.dep = (ptr, (last.n + 127) // 128)
            prev.keep = True
            linked = True
        if qkv_links:
            n = -(-sum(q.groups for q, _ in qkv_links) // 64) * 64
            done = self._own(torch.zeros(n, dtype=torch.int32, device=self.device))
            off = 0
            for q, ch in qkv_links:
                q.done = done[off:].data_ptr()
                ch.dep = (q.done, q.heads)
                off += q.groups
            self._qkv_done = done
            linked = True
        if linked:
            self._add_rearm(self._chain_counters)
            if qkv_links:
                self._add_rearm(self._qkv_done)

    def linear_steps(self) -> dict[str, "_LinearStep"]:
        """node id -> its merged-Linear launch description (chained or not)."""
        got = {}
        for nid, fn, _ in self.steps:
            if isinstance(fn, _ChainStep):
                got.update(dict(fn.members))
            elif isinstance(fn, _LinearStep):
                got[nid] = fn
        return got

    # ------------------------------------------------------- fusion helpers
    @staticmethod
    def _fusable_adds(order, users, outputs) -> dict[str, str]:
        """Add nodes whose only effective consumer (looking through glue
        Reshape/Transpose views) is a Layer/GroupNorm: add_id -> norm_id."""
        glue = (OpKind.RESHAPE, OpKind.TRANSPOSE)
        out = {}
        for n in order:
            if n.kind is not OpKind.ADD or n.id in outputs:
                continue
            frontier, seen_norm, ok = [n.id], None, True
            while frontier and ok:
                cur = frontier.pop()
                for u in users.get(cur, []):
                    if u.kind in glue and u.id not in outputs:
                        frontier.append(u.id)
                    elif u.kind in (OpKind.LAYER_NORM, OpKind.GROUP_NORM) and seen_norm is None:
                        seen_norm = u.id
                    else:
                        ok = False
            if ok and seen_norm is not None:
                out[n.id] = seen_norm
        return out

    def _deferred_for(self, t: torch.Tensor):
        p = t.data_ptr()
        for key, entry in self._deferred.items():
            o = entry[3]
            if key <= p < key + o.numel() * o.element_size():
                return key, entry
        return None, None

    def _emit_deferred(self, key: int) -> None:
        nid, a, b, _, fn = self._deferred.pop(key)
        self._folded.pop(key, None)
        for t in (a, b):  # a deferred Add reading a folded norm's output
            if t is not None:
                self._flush_folded(t)
        self._emit(nid, fn)

    def _flush_folded(self, t: torch.Tensor) -> None:
        key, _ = self._deferred_for(t)
        if key is not None and key in self._folded:
            self._emit_deferred(key)

    def _flush_members(self, members) -> None:
        for mem in members:
            for r in mem.inputs:
                v = self.vals.get(parse_ref(r)[0])
                if v is not None:
                    self._flush_deferred(v.t)

    def _folded_exact(self, x: torch.Tensor) -> _FoldedNorm | None:
        """The folded norm whose whole output ``x`` is (same storage, dense)."""
        fo = self._folded.get(x.data_ptr())
        if fo is None or x.numel() != fo.out.numel() or not x.is_contiguous():
            return None
        return fo

    def _fold_aware(self, node: OpNode) -> bool:
        if node.kind in (OpKind.MATMUL, OpKind.BATCH_MATMUL):
            return True
        return node.kind is OpKind.ADD and node.id in self._add_into_norm and \
            self.mcode == _lib.NF_MODE_FAST

    def _flush_deferred(self, t: torch.Tensor, keep_for: OpNode | None = None) -> None:
        key, entry = self._deferred_for(t)
        if key is None:
            return
        if key in self._folded and keep_for is not None and self._fold_aware(keep_for):
            return  # the consumer's lowering folds it or flushes it itself
        if keep_for is not None and self._add_into_norm.get(entry[0]) == keep_for.id:
            return
        if keep_for is not None and keep_for.kind in (OpKind.RESHAPE, OpKind.TRANSPOSE):
            return  # views; a materialising copy flushes through _copy_step
        self._emit_deferred(key)

    # ------------------------------------------------------ conv chains
    @staticmethod
    def _conv_chains(order, users, outputs) -> dict[str, dict]:
        """Conv -> [BatchNorm] -> (ReLU | Add(other) -> [ReLU]) chains whose
        interior values have exactly one consumer: lowered as one conv launch
        with BN folded into weights/bias and the residual + ReLU in the
        epilogue (the CNN plans' only inter-op traffic is then conv outputs)."""
        out = {}
        claimed: set[str] = set()

        def single(nid):
            us = users.get(nid, [])
            u = us[0] if len(us) == 1 and nid not in outputs else None
            return None if u is None or u.id in claimed else u

        for n in order:
            if n.kind not in (OpKind.CONV2D, OpKind.GROUPED_CONV2D):
                continue
            nodes, bn, add, other, relu = [n], None, None, None, False
            cur = n
            u = single(cur.id)
            if u is not None and u.kind is OpKind.BATCH_NORM:
                bn, cur = u, u
                nodes.append(u)
                u = single(cur.id)
            if u is not None and u.kind is OpKind.RELU:
                nodes.append(u)
                relu = True
            elif u is not None and u.kind is OpKind.ADD and len(u.inputs) == 2:
                refs = [parse_ref(r)[0] for r in u.inputs]
                if refs.count(cur.id) == 1:
                    add, other = u, refs[1] if refs[0] == cur.id else refs[0]
                    nodes.append(u)
                    u2 = single(u.id)
                    if u2 is not None and u2.kind is OpKind.RELU:
                        nodes.append(u2)
                        relu = True
            if len(nodes) > 1:
                out[n.id] = {"nodes": nodes, "conv": n, "bn": bn, "add": add, "other": other,
                             "relu": relu}
                claimed.update(m.id for m in nodes)
        return out

    def _nhwc(self, node_id: str, v: DVal) -> torch.Tensor:
        """Contiguous NHWC storage of a logical NCHW value (copy if needed)."""
        if v.split is None and v.t.dim() == 4:
            p = v.t.permute(0, 2, 3, 1)
            if p.is_contiguous():
                return p
        src = v.t if v.split is None else self._materialize(node_id, v)
        n, c, h, w = v.dims
        out = self._alloc((n, h, w, c), v.dtype)
        self._copy_step(node_id, src, out.permute(0, 3, 1, 2))
        return out

    def _nhwc_padded(self, node_id: str, v: DVal, groups: int, cg: int, cg_pad: int):
        """NHWC copy of a logical NCHW value with each group's channels
        zero-padded from cg to cg_pad (16-byte-friendly gather rows)."""
        src = v.t if v.split is None else self._materialize(node_id, v)
        n, c, h, w = v.dims
        out = self._own(torch.zeros((n, h, w, groups * cg_pad), dtype=v.dtype,
                                    device=self.device))
        dst = out.view(n, h, w, groups, cg_pad)[..., :cg].permute(0, 3, 4, 1, 2)
        self._copy_step(node_id, src.reshape(n, groups, cg, h, w), dst)
        return out

    def _folded_conv(self, ch, weights, dt):
        """Conv weights with BatchNorm folded in: returns (w (Cout, k, k, Cg)
        fp32 scaled, bias (Cout,) fp32)."""
        conv, bn = ch["conv"], ch["bn"]
        w = weights[conv.weights[0]].data.to(self.device, torch.float32)
        cout = w.shape[0]
        bias = weights[conv.weights[1]].data.to(self.device, torch.float32) \
            if len(conv.weights) > 1 else torch.zeros(cout, device=self.device)
        if bn is not None:
            g, b, m, v = (weights[x].data.to(self.device, torch.float32) for x in bn.weights)
            if bool((v < 0).any()):
                raise ShapeError("running_var has negative entries")
            scale = g / torch.sqrt(v + float(bn.attrs["eps"]))
            w = w * scale.view(-1, 1, 1, 1)
            bias = (bias - m) * scale + b
        return w.permute(0, 2, 3, 1).contiguous(), bias.contiguous()

    def _lower_conv_chain(self, ch, weights) -> DVal:
        conv = ch["conv"]
        a = conv.attrs
        v = self.vals[parse_ref(conv.inputs[0])[0]]
        dt = v.dtype
        groups = a.get("groups", 1)
        k, s, pad = a["kernel"], a["stride"], a["padding"]
        n, c, h, wd = v.dims
        last = ch["nodes"][-1]
        _, cout, ho, wo = last.output_spec.dims
        if c % groups or cout % groups:
            raise ShapeError(f"groups {groups} does not divide channels ({c} in, {cout} out)")
        cg, coutg = c // groups, cout // groups
        wsrc = weights[conv.weights[0]]
        if wsrc.spec.dims != (cout, cg, k, k):
            raise ShapeError(f"kernel {wsrc.spec.dims} incompatible with {c} channels in "
                             f"{groups} group(s)")
        key = ("convchain", conv.id)

        def folded():
            # BN-folded fp32 weights: only an intermediate of the kernel
            # layouts below (dropped from the cache once the plan is built)
            if key not in self._wcache:
                self._wcache[key] = self._folded_conv(ch, weights, dt)
            return self._wcache[key]

        relu = 1 if ch["relu"] else 0
        other = self.vals[ch["other"]] if ch["add"] is not None else None
        if dt == torch.float32 and coutg % 4 == 0:
            return self._lower_conv_tf32(ch, v, key, folded, other, relu, groups, cg, coutg,
                                         k, s, pad, (n, c, h, wd), (cout, ho, wo))
        if dt != torch.bfloat16:
            # fp32: NCHW direct conv with the fused scale-free folded epilogue
            x = self._materialize(conv.id, v)
            wkey = key + ("nchw",)
            if wkey not in self._wcache:
                wf, bias = folded()
                self._wcache[wkey] = (wf.permute(0, 3, 1, 2).contiguous().to(dt), bias)
            wn, bias = self._wcache[wkey]
            r = self._materialize(conv.id, other) if other is not None else None
            y = self._alloc((n, cout, ho, wo), dt)
            xp, wp, bp, yp = x.data_ptr(), wn.data_ptr(), bias.data_ptr(), y.data_ptr()
            rp = r.data_ptr() if r is not None else None
            dcode = K.dtype_code(x)
            self._emit(conv.id, lambda st: _lib.call(
                "nf_grouped_conv2d", xp, wp, bp, None, rp, yp, n, c, h, wd, cout, k, s, pad,
                groups, relu, dcode, _lib.NF_MODE_FAST, st))
            return DVal(y, (n, cout, ho, wo))
        if (k, s, pad) == (7, 2, 3) and cg <= 4 and h % 2 == 0 and wd % 2 == 0 \
                and coutg % 4 == 0 and ho == h // 2 and wo == wd // 2:
            return self._lower_stem_s2d(ch, v, key, folded, other, relu, groups, cg, coutg,
                                        (n, c, h, wd), (cout, ho, wo))
        cg_pad = cg if cg % 4 == 0 else -(-cg // 4) * 4  # stem: 3 -> 4 channels
        if coutg % 4:
            cg_pad = cg  # direct kernel below reads the unpadded layout
        if cg_pad != cg:
            xn = self._nhwc_padded(conv.id, v, groups, cg, cg_pad)
        else:
            xn = self._nhwc(conv.id, v)
        c_in = groups * cg_pad
        yn = self._alloc((n, ho, wo, cout), dt)
        rn = self._nhwc(conv.id, other) if other is not None else None
        rp = rn.data_ptr() if rn is not None else None
        pix = n * ho * wo
        act = _lib.NF_ACT_RELU if relu else _lib.NF_ACT_NONE
        if k == 1 and s == 1 and pad == 0 and cg % 8 == 0 and coutg % 8 == 0:
            # 1x1 conv == grouped GEMM over the pixel matrix: TMA reads the
            # NHWC rows in place (row stride C, group stride C/G).
            wkey = key + ("gemm",)
            if wkey not in self._wcache:
                wf, bias = folded()
                self._wcache[wkey] = (wf.reshape(groups, coutg, cg).to(dt).contiguous(),
                                      bias.view(groups, coutg).contiguous())
            wg, bg = self._wcache[wkey]
            xp, wp, bp, yp = xn.data_ptr(), wg.data_ptr(), bg.data_ptr(), yn.data_ptr()
            ws = self._workspace(groups, pix, cg, coutg)
            wsp, wsb = (ws.data_ptr(), ws.numel()) if ws is not None else (None, 0)
            args = (xp, c, cg, wp, bp, rp, yp, cout, coutg, groups, pix, cg, coutg, _lib.NF_BF16,
                    _lib.NF_W_NK, act, _lib.NF_MODE_FAST, wsp, wsb)
            lib = _lib.load()
            self._emit(conv.id, _LinkedStep(
                "gemm", args, xp, rp, yp, groups, self._gpi(groups),
                int(lib.nf_linear_link_units(groups, pix, cg, coutg)),
                int(lib.nf_linear_workspace_bytes(groups, pix, cg, coutg))))
        elif coutg % 4 == 0:
            # implicit GEMM: im2col rows gathered on chip (cp.async), never in HBM.
            # Narrow groups (ResNeXt: 4..16 channels) are densified into
            # super-groups of 32 channels with block-diagonal weights: 16-byte
            # gather rows and a 32-wide MMA tile instead of many tiny units
            # (at most 8x the FLOPs of a conv that is HBM-bound anyway).
            sup = 1
            sg = _SUPER_GROUP
            if cg_pad == cg and cg < sg and sg % cg == 0 and groups % (sg // cg) == 0:
                sup = sg // cg
            g_eff, cg_eff, coutg_eff = groups // sup, cg_pad * sup, coutg * sup
            kk = k * k * cg_eff
            kpad = -(-kk // 8) * 8
            wkey = key + ("igemm", sup)
            if wkey not in self._wcache:
                wf, bias = folded()
                w4 = wf
                if cg_pad != cg:
                    w4 = torch.nn.functional.pad(wf, (0, cg_pad - cg))
                if sup > 1:
                    blk = w4.reshape(g_eff, sup, coutg, k, k, cg)
                    dense = torch.zeros((g_eff, sup, coutg, k, k, sup, cg), dtype=w4.dtype,
                                        device=w4.device)
                    for q in range(sup):
                        dense[:, q, :, :, :, q, :] = blk[:, q]
                    w4 = dense.reshape(cout, k, k, cg_eff)
                wg = w4.reshape(g_eff, coutg_eff, kk)
                if kpad != kk:
                    wg = torch.nn.functional.pad(wg, (0, kpad - kk))
                self._wcache[wkey] = (wg.to(dt).contiguous(), bias.contiguous())
            wg, bg = self._wcache[wkey]
            groups = g_eff
            need = int(_lib.load().nf_conv_workspace_bytes(n, h, wd, c_in, cout, groups, k, s,
                                                           pad, kpad))
            ws = self._ws_buffer(need) if need > 0 else None
            wsp, wsb = (ws.data_ptr(), ws.numel()) if ws is not None else (None, 0)
            xp, wp, bp, yp = xn.data_ptr(), wg.data_ptr(), bg.data_ptr(), yn.data_ptr()
            args = (xp, wp, bp, rp, yp, n, h, wd, c_in, cout, groups, k, s, pad, kpad, relu,
                    wsp, wsb)
            self._emit(conv.id, _LinkedStep(
                "conv", args, xp, rp, yp, groups, self._gpi(groups),
                int(_lib.load().nf_conv_link_units(n, h, wd, c_in, cout, groups, k, s, pad)),
                need))
        else:
            wkey = key + ("direct",)
            if wkey not in self._wcache:
                wf, bias = folded()
                self._wcache[wkey] = (wf.to(dt).contiguous(), bias)
            wd_t, bias = self._wcache[wkey]
            xp, wp, bp, yp = xn.data_ptr(), wd_t.data_ptr(), bias.data_ptr(), yn.data_ptr()
            self._emit(conv.id, lambda st: _lib.call(
                "nf_conv_nhwc_direct", xp, wp, bp, rp, yp, n, h, wd, c, cout, groups, k, s, pad,
                relu, _lib.NF_BF16, st))
        return DVal(yn.permute(0, 3, 1, 2), (n, cout, ho, wo))

    def _lower_stem_s2d(self, ch, v, key, folded, other, relu, groups, cg, coutg, in_dims,
                        out_dims) -> DVal:
        """The 7x7 / stride-2 / pad-3 stem (RGB, 3 channels per instance) as a
        4x4 / stride-1 conv over a space-to-depth input: s2d pixel (i, j) of
        group g holds channels [(bh*2 + bw)*4 + c] = x[2i + bh, 2j + bw, c]
        (c < 3, 16 per group: 16-byte gather rows and the halo-box path
        instead of 8-byte per-tap gathers of 4-channel pixels), behind one
        explicit zero row / column so the kernel's symmetric pad 1 gives the
        stem's top/left pad of 3 input pixels. Weights: W'[o][a][a'][(bh, bw,
        c)] = W[o][2a+bh-1][2a'+bw-1][c] (zero where that tap is outside the
        7x7 window). Same products as the direct stem, summed in another order."""
        conv = ch["conv"]
        n, c, h, wd = in_dims
        cout, ho, wo = out_dims
        dt = v.dtype
        hs, ws_ = h // 2 + 1, wd // 2 + 1
        src = v.t if v.split is None else self._materialize(conv.id, v)
        if not src.is_contiguous():
            src = self._materialize(conv.id, v)
        xs = self._own(torch.zeros((n, hs, ws_, groups * 16), dtype=dt, device=self.device))
        # (n, g, c, i, bh, j, bw) -> s2d channel (bh*2 + bw)*4 + c at pixel (i+1, j+1)
        gs = groups * 16
        self._flush_deferred(src)
        sp, xsp = src.data_ptr(), xs.data_ptr()
        self._emit(conv.id, lambda st: _lib.call(
            "nf_space_to_depth_stem", sp, xsp, n, groups, cg, h, wd, st))
        wkey = key + ("s2d",)
        if wkey not in self._wcache:
            wf, bias = folded()  # (Cout, 7, 7, cg) fp32
            wp = torch.zeros((cout, 8, 8, 4), dtype=torch.float32, device=self.device)
            wp[:, 1:, 1:, :cg] = wf
            w4 = wp.view(cout, 4, 2, 4, 2, 4).permute(0, 1, 3, 2, 4, 5).reshape(cout, 256)
            self._wcache[wkey] = (w4.reshape(groups, coutg, 256).to(dt).contiguous(),
                                  bias.contiguous())
        wg, bg = self._wcache[wkey]
        yn = self._alloc((n, ho, wo, cout), dt)
        rn = self._nhwc(conv.id, other) if other is not None else None
        rp = rn.data_ptr() if rn is not None else None
        need = int(_lib.load().nf_conv_workspace_bytes(n, hs, ws_, gs, cout, groups, 4, 1, 1,
                                                       256))
        wsb = self._ws_buffer(need) if need > 0 else None
        wsp, wsn = (wsb.data_ptr(), wsb.numel()) if wsb is not None else (None, 0)
        xp, wp_, bp, yp = xs.data_ptr(), wg.data_ptr(), bg.data_ptr(), yn.data_ptr()
        self._emit(conv.id, lambda st: _lib.call(
            "nf_grouped_conv_tc", xp, wp_, bp, rp, yp, n, hs, ws_, gs, cout, groups, 4, 1, 1,
            256, relu, wsp, wsn, st))
        return DVal(yn.permute(0, 3, 1, 2), (n, cout, ho, wo))

    def _lower_conv_tf32(self, ch, v, key, folded, other, relu, groups, cg, coutg, k, s, pad,
                         in_dims, out_dims) -> DVal:
        """fp32 conv chain on the tensor cores (nf_grouped_conv_tf32, 3xTF32):
        NHWC fp32 activations (channels per group padded to a multiple of 4,
        e.g. the RGB stem 3 -> 4), BN-folded weights (G, Cout/G, (kh, kw, c))
        split once into TF32 hi / lo halves, residual + ReLU in the epilogue."""
        conv = ch["conv"]
        n, c, h, wd = in_dims
        cout, ho, wo = out_dims
        cg_pad = -(-cg // 4) * 4
        xn = self._nhwc_padded(conv.id, v, groups, cg, cg_pad) if cg_pad != cg \
            else self._nhwc(conv.id, v)
        kk = k * k * cg_pad
        kpad = -(-kk // 32) * 32
        wkey = key + ("tf32",)
        if wkey not in self._wcache:
            wf, bias = folded()
            w4 = wf if cg_pad == cg else torch.nn.functional.pad(wf, (0, cg_pad - cg))
            wg = torch.nn.functional.pad(w4.reshape(groups, coutg, kk), (0, kpad - kk))
            wg = wg.to(torch.float32).contiguous()
            hi = (wg.view(torch.int32) & -8192).view(torch.float32)  # clear 13 low bits
            self._wcache[wkey] = (torch.cat([hi, wg - hi], 0).contiguous(), bias.contiguous())
        wt, bt = self._wcache[wkey]
        yn = self._alloc((n, ho, wo, cout), torch.float32)
        rn = self._nhwc(conv.id, other) if other is not None else None
        c_in = groups * cg_pad
        need = int(_lib.load().nf_conv_tf32_workspace_bytes(n, h, wd, c_in, cout, groups, k, s,
                                                            pad, kpad))
        ws = self._ws_buffer(need) if need > 0 else None
        wsp, wsb = (ws.data_ptr(), ws.numel()) if ws is not None else (None, 0)
        xp, wp, bp, yp = xn.data_ptr(), wt.data_ptr(), bt.data_ptr(), yn.data_ptr()
        rp = rn.data_ptr() if rn is not None else None
        self._emit(conv.id, lambda st: _lib.call(
            "nf_grouped_conv_tf32", xp, wp, bp, rp, yp, n, h, wd, c_in, cout, groups, k, s, pad,
            kpad, relu, wsp, wsb, st))
        return DVal(yn.permute(0, 3, 1, 2), (n, cout, ho, wo))

    # ------------------------------------------------------ sibling heads
    @staticmethod
    def _sibling_groups(order) -> dict[str, list[OpNode]]:
        """Per-model head nodes ``head<m>::<id>`` present for every model with
        the same kind and attributes: first member id -> all members."""
        import re
        pat = re.compile(r"^head(\d+)::(.+)$")
        by_suffix: dict[str, dict[int, OpNode]] = {}
        for n in order:
            mt = pat.match(n.id)
            if mt:
                by_suffix.setdefault(mt.group(2), {})[int(mt.group(1))] = n
        out = {}
        for suffix, members in by_suffix.items():
            if len(members) < 2 or sorted(members) != list(range(len(members))):
                continue
            ms = [members[i] for i in range(len(members))]
            k0 = ms[0]
            if any(m.kind is not k0.kind or m.attrs != k0.attrs or
                   len(m.inputs) != len(k0.inputs) for m in ms):
                continue
            out[ms[0].id] = ms
        return out

    @staticmethod
    def _grouped_order(order, groups):
        """Topological order in which every sibling group is contiguous: a
        Kahn sort over super-nodes (a group = the union of its members'
        dependencies), ties broken by position in ``order``."""
        if not groups:
            return order
        import heapq
        unit_of = {}
        units: dict[str, list[OpNode]] = {}
        for first, ms in groups.items():
            units[first] = ms
            for m in ms:
                unit_of[m.id] = first
        for n in order:
            if n.id not in unit_of:
                unit_of[n.id] = n.id
                units[n.id] = [n]
        rank = {n.id: i for i, n in enumerate(order)}
        deps: dict[str, set[str]] = {u: set() for u in units}
        users: dict[str, set[str]] = {u: set() for u in units}
        for u, ms in units.items():
            for m in ms:
                for r in m.inputs:
                    p = parse_ref(r)[0]
                    if p in unit_of and unit_of[p] != u:
                        deps[u].add(unit_of[p])
                        users[unit_of[p]].add(u)
        key = {u: min(rank[m.id] for m in ms) for u, ms in units.items()}
        heap = [(key[u], u) for u in units if not deps[u]]
        heapq.heapify(heap)
        out = []
        while heap:
            _, u = heapq.heappop(heap)
            out.extend(units[u])
            for v in users[u]:
                deps[v].discard(u)
                if not deps[v]:
                    heapq.heappush(heap, (key[v], v))
        assert len(out) == len(order), "sibling grouping broke the dependency order"
        return out

    def _lower_siblings(self, members, weights, users, outputs, fused_into) -> bool:
        """One grouped launch for M same-shape per-model MatMuls (different
        weights, possibly different output widths): inputs read in place
        through a uniformly strided view, weights stacked (zero-padded to a
        common width) once at compile time."""
        first = members[0]
        if first.kind is not OpKind.MATMUL or self.mcode != _lib.NF_MODE_FAST:
            return False
        ins = [self.vals[parse_ref(m.inputs[0])[0]] for m in members]
        if any(v.split is not None for v in ins):
            return False
        t0 = ins[0].t
        if t0.dtype not in (torch.bfloat16, torch.float32) or any(
                v.t.shape != t0.shape or v.t.stride() != t0.stride() for v in ins):
            return False
        # bf16: K-major (G, N, K) for the tensor-core GEMM; fp32 heads (few
        # rows): (G, K, N) for the weight-streaming GEMV
        f32 = t0.dtype == torch.float32
        esz = t0.element_size()
        ptrs = [v.t.data_ptr() for v in ins]
        gaps = {(b - a) for a, b in zip(ptrs, ptrs[1:])}
        if len(gaps) != 1 or next(iter(gaps)) <= 0 or next(iter(gaps)) % esz:
            return False
        gstride = next(iter(gaps)) // esz
        if t0.stride(-1) != 1:
            return False
        lead = _flatten_rows(t0.shape[:-1], t0.stride()[:-1])
        if lead is None:
            return False
        rows, xld = lead
        k_in = t0.shape[-1]
        xld = xld or k_in
        widths = [weights[m.weights[0]].spec.dims[1] for m in members]
        if any(weights[m.weights[0]].spec.dims[0] != k_in for m in members):
            return False
        npad = -(-max(widths) // 8) * 8
        G = len(members)
        dev, dt = self.device, t0.dtype
        has_bias = all(len(m.weights) > 1 for m in members)
        skey = ("siblings", first.id, npad, has_bias, f32)
        if skey not in self._wcache:
            w = torch.zeros((G, k_in, npad) if f32 else (G, npad, k_in), dtype=dt, device=dev)
            bias = torch.zeros((G, npad), dtype=torch.float32, device=dev)
            for j, m in enumerate(members):
                wj = weights[m.weights[0]].data.to(dev, dt)
                if f32:
                    w[j, :, :widths[j]] = wj
                else:
                    w[j, :widths[j]] = wj.t()
                if has_bias:
                    bias[j, :widths[j]] = weights[m.weights[1]].data.to(dev, torch.float32)
            self._wcache[skey] = (w, bias)
        w, bias = self._wcache[skey]
        act, act_users = _lib.NF_ACT_NONE, []
        us = [users.get(m.id, []) for m in members]
        if all(len(u) == 1 and u[0].kind in _ACT_OF and m.id not in outputs
               for u, m in zip(us, members)) and len({u[0].kind for u in us}) == 1:
            act = _ACT_OF[us[0][0].kind]
            act_users = [u[0] for u in us]
        y = self._alloc((G,) + tuple(t0.shape[:-1]) + (npad,), dt)
        xp, wp, bp, yp = t0.data_ptr(), w.data_ptr(), bias.data_ptr() if has_bias else None, \
            y.data_ptr()
        yld, ygs = npad, rows * npad
        mcode = self.mcode
        dcode, layout = (_lib.NF_F32, _lib.NF_W_KN) if f32 else (_lib.NF_BF16, _lib.NF_W_NK)
        self._emit(first.id, lambda st: _lib.call(
            "nf_grouped_linear_strided", xp, xld, gstride, wp, bp, None, yp, yld, ygs, G, rows,
            k_in, npad, dcode, layout, act, mcode, st))
        for j, m in enumerate(members):
            view = y[j].narrow(-1, 0, widths[j])
            self.vals[m.id] = DVal(view, m.output_spec.dims)
            if act_users:
                fused_into[act_users[j].id] = m.id
        return True

    @staticmethod
    def _aliases(buf: torch.Tensor, view: torch.Tensor) -> bool:
        lo = buf.data_ptr()
        hi = lo + buf.numel() * buf.element_size()
        return lo <= view.data_ptr() < hi

    # ------------------------------------------------------------------ nodes
    def _lower(self, node: OpNode, ins: list[DVal], weights: WeightStore,
               act_user: OpNode | None) -> DVal:
        k = node.kind
        a = node.attrs
        spec = node.output_spec
        if k in (OpKind.MATMUL, OpKind.BATCH_MATMUL):
            return self._linear(node, ins[0], weights, act_user)
        if k is OpKind.ATTENTION:
            return self._attention(node, ins[0])
        if k is OpKind.REL_ATTENTION:
            return self._rel_attention(node, ins[0], ins[1], weights)
        if k in (OpKind.LAYER_NORM, OpKind.GROUP_NORM):
            return self._norm(node, ins[0], weights)
        if k in (OpKind.ADD, OpKind.MUL, OpKind.RELU, OpKind.TANH, OpKind.GELU):
            return self._pointwise(node, ins)
        if k is OpKind.RESHAPE:
            return self._reshape(node, ins[0], tuple(a["dims"]))
        if k is OpKind.TRANSPOSE:
            v = ins[0]
            if v.split is not None:
                v = DVal(self._materialize(node.id, v), v.dims)
            perm = tuple(a["perm"])
            return DVal(v.t.permute(perm), tuple(v.dims[p] for p in perm))
        if k is OpKind.UNPACK:
            return self._unpack(node, ins[0])
        if k is OpKind.SOFTMAX:
            return self._softmax(node, ins[0])
        if k is OpKind.BATCH_NORM:
            return self._batch_norm(node, ins[0], weights)
        if k in (OpKind.CONV2D, OpKind.GROUPED_CONV2D):
            return self._conv(node, ins[0], weights)
        if k in (OpKind.MAX_POOL2D, OpKind.MEAN_POOL2D):
            return self._pool(node, ins[0])
        if k is OpKind.SLICE:
            v = ins[0]
            x = v.t if v.split is None else self._materialize(node.id, v)
            ax = a["axis"] % len(v.dims)
            t = x.narrow(ax, a["start"], a["stop"] - a["start"])
            if a.get("squeeze", False):
                t = t.squeeze(ax)
            return DVal(t, spec.dims)
        if k is OpKind.CONCAT:
            out = self._alloc(spec.dims, ins[0].dtype)
            ax = a["axis"] % len(spec.dims)
            off = 0
            for v in ins:
                x = v.t if v.split is None else self._materialize(node.id, v)
                self._copy_step(node.id, x, out.narrow(ax, off, v.dims[ax]))
                off += v.dims[ax]
            return DVal(out, spec.dims)
        raise UnsupportedOpError(f"no sm_100a lowering for kind {k.value}")

    def _linear(self, node, v, weights, act_user):
        x = self._materialize(node.id, v)
        wname = node.weights[0]
        wsrc = weights[wname]
        dt = x.dtype
        if wsrc.data.dtype != dt:
            raise ShapeError(f"weight {wname!r} dtype {wsrc.spec.dtype} does not match input")
        if node.kind is OpKind.BATCH_MATMUL:
            groups, k_in, n_out = wsrc.spec.dims
            if groups != node.attrs["batch_count"] or x.shape[0] != groups:
                raise ShapeError(f"weight batch {groups} != batch_count "
                                 f"{node.attrs['batch_count']}")
        else:
            groups = 1
            k_in, n_out = wsrc.spec.dims
        if x.shape[-1] != k_in:
            raise ShapeError(f"operands incompatible: {tuple(x.shape)} vs {wsrc.spec.dims}")
        rows = x.numel() // (groups * k_in)
        fast_tc = self.mcode == _lib.NF_MODE_FAST and dt == torch.bfloat16
        # Folded norms: swapped 128-token tiles (batch 1); the kernel says
        # where it implements them (nf_linear_fold_supported).
        fold_ok = fast_tc and self.fuse and self.fold_ln and bool(
            _lib.load().nf_linear_fold_supported(groups, rows, k_in, n_out))
        # an output that may take the residual must have no other reader
        feeds_add = fold_ok and act_user is None and self._only_feeds_add(node.id)
        fo = self._folded_exact(x)
        if fo is not None and not (fold_ok and fo.m == groups and fo.rows == rows
                                   and fo.d == k_in):
            fo = None
        if fo is None:
            self._flush_deferred(x)  # x must be materialised before this launch
        layout = _lib.NF_W_NK if fast_tc else _lib.NF_W_KN
        bname = node.weights[1] if len(node.weights) > 1 else None
        if fo is not None:
            w, bias, colsum = self._folded_weights(weights, wname, bname, fo, dt)
        else:
            w = self._w(weights, wname, "linear_nk" if fast_tc else "linear_kn", dt)
            bias = self._w(weights, bname, "vec_f32", dt) if bname else None
        y = self._alloc(node.output_spec.dims, dt)
        act = _ACT_OF[act_user.kind] if act_user is not None else _lib.NF_ACT_NONE
        xp = fo.raw.data_ptr() if fo is not None else x.data_ptr()
        wp, bp, yp = w.data_ptr(), bias.data_ptr() if bias is not None else None, y.data_ptr()
        dcode, mcode = K.dtype_code(x), self.mcode
        ws = self._workspace(groups, rows, k_in, n_out) if fast_tc else None
        wsp, wsb = (ws.data_ptr(), ws.numel()) if ws is not None else (None, 0)
        step = _LinearStep(xp, k_in, wp, bp, yp, n_out, groups, rows, dcode, layout, act, mcode,
                           wsp, wsb, fold_ok)
        if fo is not None:
            step.fin = (fo.stats.data_ptr(), fo.parts, colsum.data_ptr(), fo.eps)
        if feeds_add and y.is_contiguous():
            self._lin_out[yp] = step
        self._emit(node.id, step)
        return DVal(y, node.output_spec.dims)

    def _only_feeds_add(self, nid: str) -> bool:
        """``nid``'s value reaches exactly one consumer, an Add, through glue views."""
        cur = nid
        while True:
            us = self._users.get(cur, [])
            if len(us) != 1 or cur in self._outputs:
                return False
            if us[0].kind in (OpKind.RESHAPE, OpKind.TRANSPOSE):
                cur = us[0].id
                continue
            return us[0].kind is OpKind.ADD

    def _folded_weights(self, weights, wname, bname, fo: _FoldedNorm, dt, cache: bool = True):
        """Weights / bias / column sums of a Linear consuming a folded norm:
        W' = W * gamma (over K), b' = b + W beta, colsum = sum_k W'."""
        key = ("fold", wname, bname, fo.gamma_name)
        if key not in self._wcache:
            w = self._w(weights, wname, "linear_nk", dt, cache=False)  # (G, N, K)
            g, n, k = w.shape
            wf = w.float()
            w2 = (wf * fo.gamma.reshape(g, 1, k)).to(dt).contiguous()
            b = torch.einsum("gnk,gk->gn", wf, fo.beta.reshape(g, k))
            if bname:
                b = b + self._w(weights, bname, "vec_f32", dt).reshape(g, n)
            out = (w2, b.contiguous(), w2.float().sum(-1).contiguous())
            if not cache:
                return out
            self._wcache[key] = out
        return self._wcache[key]

    def _qkv_attention_pair(self, node, ins, weights, users, outputs):
        """A batch-1 QKV projection whose only consumer is an Attention over
        128-token sequences of 64-wide heads: run both as one fused launch
        (nf_qkv_attention) so the per-head Q/K/V stay on chip."""
        if not self.fuse or self.mcode != _lib.NF_MODE_FAST:
            return None
        if node.kind not in (OpKind.MATMUL, OpKind.BATCH_MATMUL) or node.id in outputs:
            return None
        us = users.get(node.id, [])
        if len(us) != 1 or us[0].kind is not OpKind.ATTENTION or us[0].attrs.get("scale"):
            return None
        attn = us[0]
        v = ins[0]
        if v.split is not None or v.dtype != torch.bfloat16:
            return None
        wsrc = weights[node.weights[0]]
        if wsrc.data.dtype != torch.bfloat16:
            return None
        groups = wsrc.spec.dims[0] if node.kind is OpKind.BATCH_MATMUL else 1
        d = wsrc.spec.dims[-2]
        heads = attn.attrs["heads"]
        x = v.t
        if (wsrc.spec.dims[-1] != 3 * d or d != 64 * heads or x.shape[-1] != d
                or x.numel() != groups * 128 * d or x.shape[-2] != 128):
            return None
        return attn

    def _lower_qkv_attention(self, node, attn, v, weights):
        x = self._materialize(node.id, v)
        wname = node.weights[0]
        groups = weights[wname].spec.dims[0] if node.kind is OpKind.BATCH_MATMUL else 1
        d = weights[wname].spec.dims[-2]
        heads = attn.attrs["heads"]
        fo = self._folded_exact(x)
        if fo is not None and not (self.fold_ln and fo.m == groups and fo.rows == 128
                                   and fo.d == d):
            fo = None
        if fo is None:
            self._flush_deferred(x)
        bname = node.weights[1] if len(node.weights) > 1 else None
        key = ("qkv_hm", wname, bname, fo.gamma_name if fo else None)
        if key not in self._wcache:
            if fo is not None:
                w, bias, colsum = self._folded_weights(weights, wname, bname, fo, x.dtype,
                                                       cache=False)
            else:
                w = self._w(weights, wname, "linear_nk", x.dtype, cache=False)
                bias = self._w(weights, bname, "vec_f32", x.dtype) if bname else None
                colsum = None
            self._wcache[key] = (self._head_major(w, heads), bias, colsum)
        w, bias, colsum = self._wcache[key]
        y = self._alloc(attn.output_spec.dims, x.dtype)
        scale = 1.0 / math.sqrt(d // heads)
        xp = fo.raw.data_ptr() if fo is not None else x.data_ptr()
        wp, bp, yp = w.data_ptr(), bias.data_ptr() if bias is not None else None, y.data_ptr()
        fold = ((fo.stats.data_ptr(), fo.parts, colsum.data_ptr(), fo.eps)
                if fo is not None else None)
        self._emit(attn.id, _QKVStep(xp, d, wp, bp, yp, groups, heads, scale, fold))
        return DVal(y, attn.output_spec.dims)

    @staticmethod
    def _head_major(w: torch.Tensor, heads: int) -> torch.Tensor:
        """(G, 3D, D) q|k|v rows -> head-major rows (G, H, 3, 64, D) for the
        fused QKV+attention kernel (one TMA box per head)."""
        g, n3, k = w.shape
        dh = n3 // (3 * heads)
        return w.reshape(g, 3, heads, dh, k).permute(0, 2, 1, 3, 4).reshape(g, n3, k).contiguous()

    def _attention(self, node, v):
        x = self._materialize(node.id, v)
        heads = node.attrs["heads"]
        d = x.shape[-1] // 3
        dh = d // heads
        s = x.shape[-2]
        bt = x.numel() // (s * 3 * d)
        y = self._alloc(node.output_spec.dims, x.dtype)
        scale = node.attrs.get("scale") or 1.0 / math.sqrt(dh)
        xp, yp, dcode, mcode = x.data_ptr(), y.data_ptr(), K.dtype_code(x), self.mcode
        self._emit(node.id, lambda st: _lib.call("nf_attention", xp, yp, bt, s, heads, dh,
                                                 float(scale), dcode, mcode, st))
        return DVal(y, node.output_spec.dims)

    def _rel_attention(self, node, v, rv, weights):
        x = self._materialize(node.id, v)
        r = self._materialize(node.id, rv)
        heads = node.attrs["heads"]
        d = x.shape[-1] // 3
        dh = d // heads
        s = x.shape[-2]
        bt = x.numel() // (s * 3 * d)
        rw = self._w(weights, node.weights[0], "vec_f32", x.dtype).reshape(-1, heads, dh)
        rr = self._w(weights, node.weights[1], "vec_f32", x.dtype).reshape(-1, heads, dh)
        if bt % rw.shape[0]:
            raise ShapeError("bias instances do not divide the sequences")
        br = r.numel() // (2 * s * d)  # positional-key blocks (one per instance when shared)
        if br < 1 or bt % br:
            raise ShapeError("positional keys do not tile the sequences")
        y = self._alloc(node.output_spec.dims, x.dtype)
        scale = node.attrs.get("scale") or 1.0 / math.sqrt(dh)
        xp, rp, yp = x.data_ptr(), r.data_ptr(), y.data_ptr()
        wp, bp, spb, spr = rw.data_ptr(), rr.data_ptr(), bt // rw.shape[0], bt // br
        dcode, mcode = K.dtype_code(x), self.mcode
        self._emit(node.id, lambda st: _lib.call("nf_rel_attention", xp, rp, wp, bp, yp, bt, s,
                                                 heads, dh, spb, spr, float(scale), dcode, mcode,
                                                 st))
        return DVal(y, node.output_spec.dims)

    def _norm(self, node, v, weights):
        groups = node.attrs.get("groups", 1)
        eps = float(node.attrs["eps"])
        gam = self._w(weights, node.weights[0], "vec_f32", v.dtype)
        bet = self._w(weights, node.weights[1], "vec_f32", v.dtype)
        rank = len(v.dims)
        ca = channel_axis(rank)
        c = v.dims[ca]
        if c % groups:
            raise ShapeError(f"groups {groups} does not divide channels {c}")
        geom = None
        if v.split is not None and v.split == ca and rank in (2, 3):
            # model-major storage (..., M, C): rows = (M, leading rows)
            t = v.t
            m, cm = t.shape[ca], t.shape[ca + 1]
            if groups % m == 0 and t.stride(ca + 1) == 1:
                lead = _flatten_rows(t.shape[:ca], t.stride()[:ca])
                if lead is not None:
                    rows, srow = lead
                    g_per = groups // m
                    cg = cm // g_per
                    geom = (m, rows, t.stride(ca), srow, g_per, cg, cg, 1, rows)
                    out = self._own(torch.empty_strided(t.shape, t.stride(), dtype=t.dtype,
                                                        device=self.device))
                    base_t = t
        if geom is None:
            x = self._materialize(node.id, v)
            before = math.prod(x.shape[:ca])
            after = math.prod(x.shape[ca + 1:])
            cg = c // groups
            geom = (before, after, c * after, 1, groups, cg, cg * after, after, 0)
            out = self._own(torch.empty_like(x))
            base_t = x
            result = DVal(out, v.dims)
        else:
            result = DVal(out, v.dims, split=v.split)
        xp, yp = base_t.data_ptr(), out.data_ptr()
        rp = None
        gp, bp = gam.data_ptr(), bet.data_ptr()
        dcode = K.dtype_code(base_t)
        key, entry = self._deferred_for(base_t)
        if key is not None and self._add_into_norm.get(entry[0]) == node.id:
            if result.split is not None and self._fold_norm(node, entry, geom, out, gam, bet, eps):
                del self._deferred[key]
                return result
            off = xp - key
            a_t, b_t = entry[1], entry[2]
            self._flush_folded(a_t)
            self._flush_folded(b_t)
            xp, rp = a_t.data_ptr() + off, b_t.data_ptr() + off
            del self._deferred[key]
        elif key is not None:
            self._emit_deferred(key)
        self._emit(node.id, lambda st: _lib.call("nf_group_norm", xp, rp, gp, bp, yp, *geom,
                                                 eps, dcode, st))
        return result

    def _fold_norm(self, node, entry, geom, out, gam, bet, eps) -> bool:
        """Add(Linear output, residual) -> per-instance LayerNorm at batch 1:
        the Linear adds the residual in its epilogue and writes the norm's
        per-token partial sums; the norm itself is not launched (its
        consumers fold it, or it is emitted on first non-folding use)."""
        if not (self.fuse and self.fold_ln) or self.mcode != _lib.NF_MODE_FAST:
            return False
        m, rows, s_inst, s_row, g_per, cg = geom[:6]
        if g_per != 1 or out.dtype != torch.bfloat16:
            return False
        _, a_t, b_t, _, _ = entry
        lin, other = self._lin_out.get(a_t.data_ptr()), b_t
        if lin is None or a_t.numel() != m * rows * cg:
            lin, other = self._lin_out.get(b_t.data_ptr()), a_t
        if lin is None or other.numel() != m * rows * cg or not _dense_block(other):
            return False
        if (lin.residual is not None or lin.out_stats is not None or not lin.fold_ok
                or lin.groups != m or lin.rows != rows or lin.n != cg
                or s_inst != rows * cg or s_row != cg):
            return False
        # same physical layout as the Linear's (G, T, N) output (the Add's
        # operands are the same view of equal storage blocks)
        fo_res = self._folded.get(other.data_ptr())
        if fo_res is not None and (other.numel() != fo_res.out.numel()
                                   or (fo_res.m, fo_res.rows, fo_res.d) != (m, rows, cg)):
            fo_res = None
        if fo_res is None:
            self._flush_deferred(other)  # plain residual: must be in memory
            lin.residual = other.data_ptr()
        else:
            lin.residual = fo_res.raw.data_ptr()
            lin.fres = (fo_res.stats.data_ptr(), fo_res.parts, fo_res.gamma.data_ptr(),
                        fo_res.beta.data_ptr(), fo_res.eps)
        parts = -(-cg // 128)
        stats = self._own(torch.zeros((m, parts, rows, 2), dtype=torch.float32,
                                      device=self.device))
        lin.out_stats = stats.data_ptr()
        raw = self._lin_raw(lin, a_t if other is b_t else b_t)
        xp, yp, gp, bp = raw.data_ptr(), out.data_ptr(), gam.data_ptr(), bet.data_ptr()
        dcode = K.dtype_code(out)
        fn = lambda st: _lib.call("nf_group_norm", xp, None, gp, bp, yp, *geom, eps, dcode, st)
        fo = _FoldedNorm(node.id, raw, out, stats, parts, gam, bet, node.weights[0], eps, m,
                         rows, cg, fn)
        self._deferred[out.data_ptr()] = (node.id, None, None, out, fn)
        self._folded[out.data_ptr()] = fo
        return True

    @staticmethod
    def _lin_raw(lin: _LinearStep, view: torch.Tensor) -> torch.Tensor:
        """The Linear's output buffer as a dense (G, T, N) view."""
        return view.as_strided((lin.groups, lin.rows, lin.n), (lin.rows * lin.n, lin.n, 1))

    def _pointwise(self, node, ins):
        op = _EW_OF[node.kind]
        if len(ins) == 2 and not _same_physical(ins[0], ins[1]):
            ins = [DVal(self._materialize(node.id, v), v.dims) for v in ins]
        v0 = ins[0]
        if _dense_block(v0.t):
            out = self._own(torch.empty_strided(v0.t.shape, v0.t.stride(), dtype=v0.dtype,
                                                device=self.device))
            srcs = [v.t for v in ins]
            result = DVal(out, v0.dims, v0.split)
        else:
            srcs = [self._materialize(node.id, v) for v in ins]
            out = self._alloc(v0.dims, v0.dtype)
            result = DVal(out, v0.dims)
        n = out.numel()
        ap = srcs[0].data_ptr()
        bp = srcs[1].data_ptr() if len(srcs) > 1 else None
        # storage start of a permuted dense block is the min-offset element,
        # which for non-negative strides is data_ptr() itself.
        yp, dcode = out.data_ptr(), K.dtype_code(out)
        fn = lambda st: _lib.call("nf_elementwise", op, ap, bp, yp, n, dcode, st)
        if node.id in self._add_into_norm and srcs[0] is ins[0].t and \
                srcs[1] is ins[1].t and self.mcode == _lib.NF_MODE_FAST:
            self._deferred[yp] = (node.id, srcs[0], srcs[1], out, fn)
        else:
            for t in srcs:
                self._flush_deferred(t)
            self._emit(node.id, fn)
        return result

    def _reshape(self, node, v, dims):
        if v.split is not None:
            a = v.split
            unsplit = v.dims[:a] + (v.t.shape[a], v.t.shape[a + 1]) + v.dims[a + 1:]
            if dims == unsplit:
                return DVal(v.t, dims)
            v = DVal(self._materialize(node.id, v), v.dims)
        try:
            return DVal(v.t.view(dims), dims)
        except RuntimeError:
            pass
        src = tuple(v.t.shape)
        for a in range(len(src) - 1):
            if src[:a] + (src[a] * src[a + 1],) + src[a + 2:] == dims and v.t.stride(a + 1) == 1:
                return DVal(v.t, dims, split=a)
        return DVal(self._materialize(node.id, v).view(dims), dims)

    def _unpack(self, node, v):
        count, dim, stacked, j = node.attrs["count"], MergeDim(node.attrs["dim"]), \
            node.attrs["stacked"], node.attrs["index"]
        if dim is MergeDim.CHANNEL:
            ca = channel_axis(len(v.dims))
            if v.split is not None and v.split == ca and v.t.shape[ca] == count:
                return DVal(v.t.select(ca, j), node.output_spec.dims)
            x = v.t if v.split is None else self._materialize(node.id, v)
            c = v.dims[ca] // count
            return DVal(x.narrow(ca, j * c, c), node.output_spec.dims)
        x = v.t if v.split is None else self._materialize(node.id, v)
        if stacked:
            return DVal(x.select(0, j), node.output_spec.dims)
        b = v.dims[0] // count
        return DVal(x.narrow(0, j * b, b), node.output_spec.dims)

    def _softmax(self, node, v):
        x = self._materialize(node.id, v)
        ax = node.attrs["axis"] % x.dim()
        outer = math.prod(x.shape[:ax])
        inner = math.prod(x.shape[ax + 1:])
        L = x.shape[ax]
        y = self._own(torch.empty_like(x))
        xp, yp, dcode = x.data_ptr(), y.data_ptr(), K.dtype_code(x)
        self._emit(node.id, lambda st: _lib.call("nf_softmax", xp, yp, outer, L, inner,
                                                 L * inner, inner, 1, dcode, st))
        return DVal(y, v.dims)

    def _batch_norm(self, node, v, weights):
        x = self._materialize(node.id, v)
        ca = channel_axis(x.dim())
        c = x.shape[ca]
        vecs = [self._w(weights, w, "vec_f32", x.dtype) for w in node.weights]
        for name, t in zip(("gamma", "beta", "running_mean", "running_var"), vecs):
            if tuple(t.shape) != (c,):
                raise ShapeError(f"{name} must be ({c},), got {tuple(t.shape)}")
        if bool((vecs[3] < 0).any()):
            raise ShapeError("running_var has negative entries")
        y = self._own(torch.empty_like(x))
        n, inner = math.prod(x.shape[:ca]), math.prod(x.shape[ca + 1:])
        ptrs = [t.data_ptr() for t in vecs]
        xp, yp, dcode, eps = x.data_ptr(), y.data_ptr(), K.dtype_code(x), float(node.attrs["eps"])
        self._emit(node.id, lambda st: _lib.call("nf_batch_norm", xp, *ptrs, yp, n, c, inner,
                                                 eps, dcode, st))
        return DVal(y, v.dims)

    def _conv(self, node, v, weights):
        x = self._materialize(node.id, v)
        w = self._w(weights, node.weights[0], "same", x.dtype)
        if weights[node.weights[0]].data.dtype != x.dtype:
            raise ShapeError(f"weight {node.weights[0]!r} dtype does not match input")
        bias = self._w(weights, node.weights[1], "vec_f32", x.dtype) if len(node.weights) > 1 \
            else None
        groups = node.attrs.get("groups", 1)
        n, cin, h, wd = x.shape
        cout, cg, k, _ = w.shape
        if cg != cin // groups or cin % groups or cout % groups:
            raise ShapeError(f"kernel {tuple(w.shape)} incompatible with {cin} channels in "
                             f"{groups} group(s)")
        y = self._alloc(node.output_spec.dims, x.dtype)
        s, p = node.attrs["stride"], node.attrs["padding"]
        xp, wp, bp, yp = x.data_ptr(), w.data_ptr(), None if bias is None else bias.data_ptr(), \
            y.data_ptr()
        dcode, mcode = K.dtype_code(x), self.mcode
        self._emit(node.id, lambda st: _lib.call("nf_grouped_conv2d", xp, wp, bp, None, None, yp,
                                                 n, cin, h, wd, cout, k, s, p, groups, 0, dcode,
                                                 mcode, st))
        return DVal(y, node.output_spec.dims)

    def _pool(self, node, v):
        kind = _lib.NF_POOL_MAX if node.kind is OpKind.MAX_POOL2D else _lib.NF_POOL_MEAN
        k, s, p = node.attrs["kernel"], node.attrs["stride"], node.attrs.get("padding", 0)
        if v.split is None and v.t.dim() == 4 and v.t.permute(0, 2, 3, 1).is_contiguous() \
                and not v.t.is_contiguous():
            xn = v.t.permute(0, 2, 3, 1)
            n, h, w, c = xn.shape
            _, _, ho, wo = node.output_spec.dims
            yn = self._alloc((n, ho, wo, c), xn.dtype)
            xp, yp, dcode = xn.data_ptr(), yn.data_ptr(), K.dtype_code(xn)
            self._emit(node.id, lambda st: _lib.call("nf_pool2d_nhwc", xp, yp, n, h, w, c, kind,
                                                     k, s, p, dcode, st))
            return DVal(yn.permute(0, 3, 1, 2), node.output_spec.dims)
        x = self._materialize(node.id, v)
        n, c, h, w = x.shape
        y = self._alloc(node.output_spec.dims, x.dtype)
        kind = _lib.NF_POOL_MAX if node.kind is OpKind.MAX_POOL2D else _lib.NF_POOL_MEAN
        k, s, p = node.attrs["kernel"], node.attrs["stride"], node.attrs.get("padding", 0)
        xp, yp, dcode = x.data_ptr(), y.data_ptr(), K.dtype_code(x)
        self._emit(node.id, lambda st: _lib.call("nf_pool2d", xp, yp, n, c, h, w, kind, k, s, p,
                                                 dcode, st))
        return DVal(y, node.output_spec.dims)

    # -------------------------------------------------------------- running
    @property
    def kernel_launches(self) -> int:
        return sum(n for _, _, n in self.steps)

    def load_inputs(self, inputs: dict, non_blocking: bool = True) -> None:
        """Copy graph inputs into the plan's static input buffers."""
        for name, spec in self.graph.graph_inputs.items():
            if name not in inputs:
                raise ExecutionError(name, KeyError(f"graph input {name!r} not provided"))
            val = inputs[name]
            data = val.data if isinstance(val, TensorValue) else val
            if not isinstance(data, torch.Tensor):
                data = torch.as_tensor(data)
            if tuple(data.shape) != spec.dims or data.dtype != TORCH_DTYPES[spec.dtype]:
                raise ExecutionError(name, ShapeError(
                    f"input {name!r}: got {tuple(data.shape)} ({data.dtype}), graph wants "
                    f"{spec.dims} ({spec.dtype})"))
            self.input_views[name].copy_(data, non_blocking=non_blocking)

    def launch(self, stream: int | None = None, events: list | None = None) -> None:
        if self.device.type != "cuda":
            raise UnsupportedOpError("plan was built for structure inspection only (no device)")
        st = torch.cuda.current_stream().cuda_stream if stream is None else stream
        if events is None:
            for _, fn, _ in self.steps:
                fn(st)
            return
        for _, fn, _ in self.steps:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record()
            fn(st)
            events.append(e0)
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        events.append(e)

    def capture(self) -> torch.cuda.CUDAGraph:
        """Record every launch into one CUDA graph (after one warm-up run)."""
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.launch()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.launch()
        self._cuda_graph = g
        return g

    def replay(self) -> None:
        if self._cuda_graph is None:
            self.capture()
        self._cuda_graph.replay()

    def outputs(self) -> list[torch.Tensor]:
        return self.out_buffers


class PipelinedRunner:
    """Serve a stream of host batches through one plan with the host->device
    copy of batch i+1 (pinned host -> device staging, on a copy stream)
    overlapping the forward of batch i. Each forward starts with one
    device-side copy per plan input buffer from the staging mirror (so the
    captured CUDA graph keeps its pointers), and ends with the device->host
    read of its outputs; the next batch's staging copy waits only for the
    device copy that consumed the buffer two batches earlier."""

    def __init__(self, plan: Plan):
        if plan.device.type != "cuda":
            raise UnsupportedOpError("PipelinedRunner needs a CUDA plan")
        self.plan = plan
        bases: dict[int, torch.Tensor] = {}
        for v in plan.input_views.values():
            b = v._base if v._base is not None else v
            bases.setdefault(b.data_ptr(), b)
        self._bases = list(bases.values())
        self._mirrors = [[torch.empty_like(b) for b in self._bases] for _ in range(2)]
        self._views = []
        for mir in self._mirrors:
            views = {}
            for name, v in plan.input_views.items():
                b = v._base if v._base is not None else v
                j = next(i for i, bb in enumerate(self._bases) if bb.data_ptr() == b.data_ptr())
                views[name] = mir[j].as_strided(v.shape, v.stride(),
                                                v.storage_offset() - b.storage_offset())
            self._views.append(views)
        self.copy_stream = torch.cuda.Stream(device=plan.device)
        self._h2d_done = [torch.cuda.Event(), torch.cuda.Event()]
        self._staged_free = [torch.cuda.Event(), torch.cuda.Event()]
        # outputs that are views of one plan buffer (e.g. the stacked heads)
        # come back with one device->host copy per buffer
        obases: dict[int, torch.Tensor] = {}
        for o in plan.outputs():
            b = o._base if o._base is not None else o
            obases.setdefault(b.data_ptr(), b)
        self._out_bases = list(obases.values())
        self._host_sets: dict[int, list[torch.Tensor]] = {}  # id(output list) -> pinned bases

    def alloc_host_outputs(self, count: int = 1) -> list[list[torch.Tensor]]:
        """``count`` sets of pinned host outputs laid out like the plan's
        output buffers; ``run`` fills each set with one copy per buffer."""
        sets = []
        for _ in range(count):
            # same physical layout as each buffer (views index it by stride)
            mir = [torch.empty_strided(b.shape, b.stride(), dtype=b.dtype, pin_memory=True)
                   for b in self._out_bases]
            outs = []
            for o in self.plan.outputs():
                b = o._base if o._base is not None else o
                j = next(i for i, bb in enumerate(self._out_bases)
                         if bb.data_ptr() == b.data_ptr())
                outs.append(mir[j].as_strided(o.shape, o.stride(),
                                              o.storage_offset() - b.storage_offset()))
            self._host_sets[id(outs)] = mir
            sets.append(outs)
        return sets

    def d2h_bytes(self, outputs_host) -> int:
        mir = self._host_sets.get(id(outputs_host))
        ts = mir if mir is not None else outputs_host
        return sum(t.numel() * t.element_size() for t in ts)

    def _stage(self, i: int, inputs: dict) -> None:
        k = i % 2
        with torch.cuda.stream(self.copy_stream):
            self.copy_stream.wait_event(self._staged_free[k])
            for name in self.plan.graph.graph_inputs:
                if name not in inputs:
                    raise ExecutionError(name, KeyError(f"graph input {name!r} not provided"))
                val = inputs[name]
                data = val.data if isinstance(val, TensorValue) else val
                dst = self._views[k][name]
                if tuple(data.shape) != tuple(dst.shape) or data.dtype != dst.dtype:
                    raise ExecutionError(name, ShapeError(
                        f"input {name!r}: got {tuple(data.shape)} ({data.dtype}), graph wants "
                        f"{tuple(dst.shape)} ({dst.dtype})"))
                dst.copy_(data, non_blocking=True)
            self._h2d_done[k].record(self.copy_stream)

    def run(self, batches, outputs_host) -> None:
        """``batches``: sequence of input dicts (pinned host tensors for
        overlap); ``outputs_host``: one list of host tensors per batch (or a
        single list reused by every batch) receiving the plan outputs."""
        main = torch.cuda.current_stream()
        n = len(batches)
        if n == 0:
            return
        per_batch = len(outputs_host) == n and isinstance(outputs_host[0], (list, tuple))
        self.copy_stream.wait_stream(main)  # staging starts after work already queued
        self._stage(0, batches[0])
        for i in range(n):
            if i + 1 < n:
                self._stage(i + 1, batches[i + 1])
            k = i % 2
            main.wait_event(self._h2d_done[k])
            for dst, src in zip(self._bases, self._mirrors[k]):
                dst.copy_(src, non_blocking=True)
            self._staged_free[k].record(main)
            self.plan.replay()
            outs = outputs_host[i] if per_batch else outputs_host
            mir = self._host_sets.get(id(outs))
            if mir is not None:
                for h, b in zip(mir, self._out_bases):
                    h.copy_(b, non_blocking=True)
            else:
                for h, o in zip(outs, self.plan.outputs()):
                    h.copy_(o, non_blocking=True)


# ----------------------------------------------------------------------------
# Reference-compatible entry point
# ----------------------------------------------------------------------------

class _PlanEntry:
    """Compiled plans of one (graph, weight store, mode, fuse): the graph and
    store are held weakly and re-identified with ``is``; the fingerprint pins
    the exact TensorValue objects (and their in-place version counters) the
    plans were built from, so a replaced or mutated weight is never served
    from a stale plan. Plans share the converted device weights but each
    owns its activations, I/O buffers and split-K workspace; a plan is used
    by one execute() call at a time."""

    def __init__(self, graph, weights, mode, fuse):
        import weakref
        self.graph_ref = weakref.ref(graph)
        self.store_ref = weakref.ref(weights)
        self.fingerprint = _weights_fingerprint(graph, weights)
        self.mode, self.fuse = mode, fuse
        self.wcache: dict = {}
        self.free: list[Plan] = []
        self.lock = threading.Lock()

    def valid_for(self, graph, weights) -> bool:
        return (self.graph_ref() is graph and self.store_ref() is weights
                and self.fingerprint == _weights_fingerprint(graph, weights))


def _weights_fingerprint(graph: Graph, weights: WeightStore) -> tuple:
    tvs = tuple((name, id(tv), tv.data._version) for name, tv in weights.tensors.items())
    return (id(graph.nodes), graph.graph_outputs, tuple(graph.graph_inputs.items()), tvs)


class _PlanCache:
    """Bounded LRU of plan entries behind the stateless ``execute`` entry
    point (reference contract: pure and reentrant). Entries die
    with their graph or weight store (weakref finalizers: ids recycle) and
    past ``capacity``."""

    def __init__(self, capacity: int = 4):
        from collections import OrderedDict
        self.capacity = capacity
        self._lock = threading.Lock()
        self._entries: "OrderedDict[tuple, _PlanEntry]" = OrderedDict()

    def _drop(self, key, entry) -> None:
        with self._lock:
            if self._entries.get(key) is entry:
                del self._entries[key]

    def checkout(self, graph, weights, mode, fuse) -> tuple[_PlanEntry, Plan]:
        import weakref
        key = (id(graph), id(weights), mode, fuse)
        with self._lock:
            entry = self._entries.get(key)
            if entry is not None and not entry.valid_for(graph, weights):
                del self._entries[key]
                entry = None
            if entry is None:
                entry = _PlanEntry(graph, weights, mode, fuse)
                self._entries[key] = entry
                weakref.finalize(graph, self._drop, key, entry)
                weakref.finalize(weights, self._drop, key, entry)
                while len(self._entries) > self.capacity:
                    self._entries.popitem(last=False)
            else:
                self._entries.move_to_end(key)
        with entry.lock:
            if entry.free:
                return entry, entry.free.pop()
            # A new plan (first call, or other threads hold every free one).
            # Built under the entry lock and synchronised before release: the
            # converted weights it adds to the shared cache are produced on
            # this thread's stream, and another thread's plan will read them
            # from its own stream.
            plan = Plan(graph, weights, mode=mode, fuse=fuse, weight_cache=entry.wcache)
            if plan.device.type == "cuda":
                torch.cuda.current_stream(plan.device).synchronize()
            return entry, plan

    @staticmethod
    def checkin(entry: _PlanEntry, plan: Plan) -> None:
        with entry.lock:
            entry.free.append(plan)

    def clear(self) -> None:
        with self._lock:
            self._entries.clear()

    def __len__(self) -> int:
        return len(self._entries)


_PLANS = _PlanCache()


def compile_plan(graph: Graph, weights: WeightStore, *, mode: str = "fast",
                 fuse: bool = True, fold_ln: bool = True, chain: bool = True) -> Plan:
    """Compile ``graph`` with ``weights`` into a caller-owned :class:`Plan`
    (weights converted to kernel layouts in HBM, buffers preallocated).
    Every call builds a new plan: the handle is the cache."""
    return Plan(graph, weights, mode=mode, fuse=fuse, fold_ln=fold_ln, chain=chain)


def execute(graph: Graph, weights: WeightStore, inputs: dict[str, TensorValue], *,
            mode: str = "fast", trace_nodes: bool = False,
            fuse: bool = True) -> tuple[list[TensorValue], ExecTrace]:
    """Run a graph on the GPU (reference engine.py:516-573 contract).

    Inputs may live on the host or the device; outputs are fresh device
    tensors in ``graph_outputs`` order. Missing inputs / shape errors /
    kernel failures raise ExecutionError naming the node.
    """
    for name, spec in graph.graph_inputs.items():
        tv = inputs.get(name)
        if tv is None:
            raise ExecutionError(name, KeyError(f"graph input {name!r} not provided"))
        if tv.spec.dims != spec.dims or tv.spec.dtype != spec.dtype:
            raise ExecutionError(name, ShapeError(
                f"input {name!r}: got {tv.spec.dims} ({tv.spec.dtype}), graph wants "
                f"{spec.dims} ({spec.dtype})"))
    entry, plan = _PLANS.checkout(graph, weights, mode, fuse)
    trace = ExecTrace(op_invocations=plan.op_invocations, dispatch_count=plan.dispatch_count,
                      kernel_launches=plan.kernel_launches)
    t0 = time.perf_counter_ns()
    plan.load_inputs(inputs)
    events: list | None = [] if trace_nodes else None
    plan.launch(events=events)
    outs = [b.clone() for b in plan.outputs()]
    torch.cuda.current_stream(plan.device).synchronize()
    trace.total_ns = time.perf_counter_ns() - t0
    if events:
        for i, (nid, _, _) in enumerate(plan.steps):
            ms = events[i].elapsed_time(events[i + 1])
            trace.node_times_ns[nid] = trace.node_times_ns.get(nid, 0) + int(ms * 1e6)
    # nothing in flight reads the plan's buffers after the stream sync: it
    # may serve the next call (a call that raised never returns its plan)
    _PLANS.checkin(entry, plan)
    result = []
    for ref, t in zip(graph.graph_outputs, outs):
        prod = parse_ref(ref)[0]
        spec = graph.graph_inputs.get(prod) or graph.node_map()[prod].output_spec
        tv = TensorValue(spec, t)
        trace.node_outputs[prod] = tv
        result.append(tv)
    return result, trace
