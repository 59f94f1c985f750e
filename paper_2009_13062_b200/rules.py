"""Merge rules: which input-weight-local counterpart absorbs M instances.

Paper Table 1 as implemented by the reference catalog
(pkg/src/modelmerge/rules.py:75-116). A weight only ever meets activations of
its own model, so M instances become one op once their operands are packed
along an axis the op treats independently:

* channel-wise weight binding (conv, norms) -> pack on channels, grouped op
  with M x the groups;
* matmuls -> pack on a model axis, batched matmul;
* weightless pointwise / spatial ops -> either packing (DontCare);
* reductions (softmax) -> any packing that leaves the reduced axis alone.

Extensions for the BASELINE models (not in the reference):
GELU (DontCare), Attention and RelAttention (batch-packed: heads and the
sequence axis stay per instance), padded pools (DontCare), Slice (structural).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .errors import ArchitectureMismatchError, UnsupportedOpError
from .ir import MergeDim, OpKind, TensorSpec, channel_axis
from .tensors import TensorValue

BATCH_STACK = "batch-stack"
CHANNEL_CONCAT = "channel-concat"


@dataclass(frozen=True)
class WeightRecipe:
    """How one weight slot is assembled from M per-model tensors (model-major).
    ``new_axis``: stack on a new leading model axis instead of concatenating
    along the existing axis 0 (rules.py:34-45)."""

    slot: str
    mode: str
    new_axis: bool = False


@dataclass(frozen=True)
class MergeRule:
    source: OpKind
    target: OpKind | None
    dim: MergeDim
    recipes: tuple[WeightRecipe, ...] = ()
    note: str = ""

    @property
    def mergeable(self) -> bool:
        return self.target is not None


def _concat(*slots: str) -> tuple[WeightRecipe, ...]:
    return tuple(WeightRecipe(s, CHANNEL_CONCAT) for s in slots)


def _stack(*slots: str, new_axis: bool) -> tuple[WeightRecipe, ...]:
    return tuple(WeightRecipe(s, BATCH_STACK, new_axis=new_axis) for s in slots)


_AGNOSTIC = {
    OpKind.RELU: "elementwise; packing-agnostic",
    OpKind.TANH: "elementwise; packing-agnostic",
    OpKind.GELU: "elementwise; packing-agnostic",
    OpKind.SOFTMAX: "reduction axis must not be the packed axis",
    OpKind.MAX_POOL2D: "spatial only; packing-agnostic",
    OpKind.MEAN_POOL2D: "spatial only; packing-agnostic",
    OpKind.ADD: "elementwise; packing-agnostic",
    OpKind.MUL: "elementwise; packing-agnostic",
}

_STRUCTURAL = (OpKind.CONCAT, OpKind.RESHAPE, OpKind.TRANSPOSE, OpKind.PACK, OpKind.UNPACK,
               OpKind.SLICE)


def _build_rules() -> dict[OpKind, MergeRule]:
    table: dict[OpKind, MergeRule] = {
        OpKind.CONV2D: MergeRule(OpKind.CONV2D, OpKind.GROUPED_CONV2D, MergeDim.CHANNEL,
                                 _concat("kernel", "bias"), "becomes a grouped conv with M groups"),
        OpKind.GROUPED_CONV2D: MergeRule(OpKind.GROUPED_CONV2D, OpKind.GROUPED_CONV2D,
                                         MergeDim.CHANNEL, _concat("kernel", "bias"),
                                         "group count scales from G to M*G"),
        OpKind.MATMUL: MergeRule(OpKind.MATMUL, OpKind.BATCH_MATMUL, MergeDim.BATCH,
                                 _stack("weight", "bias", new_axis=True),
                                 "weights stack on a new leading model axis"),
        OpKind.BATCH_MATMUL: MergeRule(OpKind.BATCH_MATMUL, OpKind.BATCH_MATMUL, MergeDim.BATCH,
                                       _stack("weight", "bias", new_axis=False),
                                       "batch count scales from b to M*b"),
        OpKind.LAYER_NORM: MergeRule(OpKind.LAYER_NORM, OpKind.GROUP_NORM, MergeDim.CHANNEL,
                                     _concat("gamma", "beta"),
                                     "becomes a group norm with M groups"),
        OpKind.GROUP_NORM: MergeRule(OpKind.GROUP_NORM, OpKind.GROUP_NORM, MergeDim.CHANNEL,
                                     _concat("gamma", "beta"), "group count scales from G to M*G"),
        OpKind.BATCH_NORM: MergeRule(OpKind.BATCH_NORM, OpKind.BATCH_NORM, MergeDim.CHANNEL,
                                     _concat("gamma", "beta", "running_mean", "running_var"),
                                     "per-channel affine; all four vectors concatenate"),
        OpKind.ATTENTION: MergeRule(OpKind.ATTENTION, OpKind.ATTENTION, MergeDim.BATCH, (),
                                    "per-instance heads; packs on the model axis"),
        OpKind.REL_ATTENTION: MergeRule(OpKind.REL_ATTENTION, OpKind.REL_ATTENTION,
                                        MergeDim.BATCH,
                                        _stack("r_w_bias", "r_r_bias", new_axis=True),
                                        "per-instance heads and biases; packs on the model axis"),
    }
    for kind, note in _AGNOSTIC.items():
        table[kind] = MergeRule(kind, kind, MergeDim.DONT_CARE, (), note)
    for kind in _STRUCTURAL:
        table[kind] = MergeRule(kind, None, MergeDim.DONT_CARE, (),
                                "not mergeable: rearranges the axes packing relies on")
    return table


RULES: dict[OpKind, MergeRule] = _build_rules()
assert set(RULES) == set(OpKind), "every op kind needs exactly one rule"


def rule_for(kind: OpKind) -> MergeRule:
    """Merge rule of a kind; structural kinds raise UnsupportedOpError."""
    rule = RULES[kind]
    if rule.target is None:
        raise UnsupportedOpError(f"{kind.value} cannot appear in a graph to be merged: {rule.note}")
    return rule


def forbidden_dims(kind: OpKind, attrs: dict, input_spec: TensorSpec) -> set[MergeDim]:
    """Packings that would pack a node's reduction axis (rules.py:129-146):
    a softmax over the channel axis cannot pack on channels, and a rank-4
    softmax over axis 0 cannot pack on batch (batch packing folds models into
    axis 0 there)."""
    if kind is not OpKind.SOFTMAX:
        return set()
    rank = input_spec.rank
    axis = attrs["axis"] % rank
    out = set()
    if axis == channel_axis(rank):
        out.add(MergeDim.CHANNEL)
    if rank == 4 and axis == 0:
        out.add(MergeDim.BATCH)
    return out


_GROUP_SCALING = {
    OpKind.CONV2D: ("groups", None),
    OpKind.GROUPED_CONV2D: ("groups", "groups"),
    OpKind.MATMUL: ("batch_count", None),
    OpKind.BATCH_MATMUL: ("batch_count", "batch_count"),
    OpKind.LAYER_NORM: ("groups", None),
    OpKind.GROUP_NORM: ("groups", "groups"),
}


def merged_attrs(kind: OpKind, attrs: dict, num_models: int) -> dict:
    """Attributes of the merged counterpart (rules.py:149-164): the group or
    batch count becomes M (fresh) or multiplies by M (already grouped)."""
    out = dict(attrs)
    if kind in _GROUP_SCALING:
        key, base = _GROUP_SCALING[kind]
        out[key] = num_models * (attrs[base] if base else 1)
    return out


def merge_weight_slot(recipe: WeightRecipe, values: list[TensorValue]) -> TensorValue:
    """Merge M same-spec tensors of one slot, model-major (rules.py:167-184)."""
    ref = values[0].spec
    for i, v in enumerate(values):
        if v.spec.dims != ref.dims or v.spec.dtype != ref.dtype:
            raise ArchitectureMismatchError(
                f"slot {recipe.slot!r}: model 0 has {ref.dims} ({ref.dtype}) but "
                f"model {i} has {v.spec.dims} ({v.spec.dtype})")
    parts = [v.data for v in values]
    merged = torch.stack(parts, 0) if recipe.new_axis else torch.cat(parts, 0)
    return TensorValue(TensorSpec(ref.dtype, tuple(merged.shape)), merged)


def merge_weights(rule: MergeRule, slot_values: list[list[TensorValue]]) -> list[TensorValue]:
    if len(slot_values) > len(rule.recipes):
        raise ArchitectureMismatchError(
            f"{rule.source.value} has at most {len(rule.recipes)} weight slots, "
            f"got {len(slot_values)}")
    return [merge_weight_slot(r, vals) for r, vals in zip(rule.recipes, slot_values)]


def rules_as_json() -> dict:
    """The rule table as a JSON document (reference `rules dump`)."""
    return {
        "schema": 1,
        "kinds_covered": len(OpKind),
        "rules": [{
            "source": k.value,
            "target": RULES[k].target.value if RULES[k].target else None,
            "mergeable": RULES[k].mergeable,
            "dim": RULES[k].dim.value,
            "weights": [{"slot": r.slot, "recipe": r.mode} for r in RULES[k].recipes],
            "note": RULES[k].note,
        } for k in OpKind],
    }
