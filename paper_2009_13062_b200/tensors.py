"""Concrete tensors and weight stores (reference engine.py:49-103).

``TensorValue.data`` is a ``torch.Tensor`` (host or CUDA) instead of a numpy
array, so bf16 is representable and device residency is explicit. numpy
arrays are accepted everywhere a tensor is and converted on construction.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .errors import ShapeError
from .ir import Layout, TensorSpec

TORCH_DTYPES = {"f32": torch.float32, "f64": torch.float64, "bf16": torch.bfloat16}
DTYPE_NAMES = {v: k for k, v in TORCH_DTYPES.items()}
NUMPY_DTYPES = {"f32": np.float32, "f64": np.float64}


def as_tensor(data) -> torch.Tensor:
    if isinstance(data, torch.Tensor):
        return data
    return torch.from_numpy(np.ascontiguousarray(data))


@dataclass(frozen=True)
class TensorValue:
    """A spec plus contiguous data of exactly ``spec.dims``."""

    spec: TensorSpec
    data: torch.Tensor

    def __post_init__(self):
        t = as_tensor(self.data)
        want = TORCH_DTYPES[self.spec.dtype]
        if t.dtype != want:
            t = t.to(want)
        if tuple(t.shape) != self.spec.dims:
            if t.numel() != self.spec.size:
                raise ShapeError(f"data has {t.numel()} elements, spec wants {self.spec.size}")
            t = t.reshape(self.spec.dims)
        if not t.is_contiguous():
            t = t.contiguous()
        object.__setattr__(self, "data", t)

    @classmethod
    def from_array(cls, arr, layout: Layout = Layout.UNLAID) -> "TensorValue":
        t = as_tensor(arr)
        name = DTYPE_NAMES.get(t.dtype)
        if name is None:
            raise ShapeError(f"unsupported dtype {t.dtype}")
        return cls(TensorSpec(name, tuple(t.shape), layout), t)

    def numpy(self) -> np.ndarray:
        t = self.data.detach()
        if t.dtype == torch.bfloat16:
            t = t.float()
        return t.cpu().numpy()

    def to(self, device) -> "TensorValue":
        return TensorValue(self.spec, self.data.to(device))

    def bit_equal(self, other: "TensorValue") -> bool:
        """Same dtype, dims and payload bits (reference engine.py:74-80)."""
        if self.spec.dtype != other.spec.dtype or self.spec.dims != other.spec.dims:
            return False
        a = self.data.detach().cpu().contiguous().view(torch.uint8)
        b = other.data.detach().cpu().contiguous().view(torch.uint8)
        return torch.equal(a, b)


@dataclass
class WeightStore:
    """Named parameter tensors of one model (or of a merged model)."""

    tensors: dict[str, TensorValue]
    model_index: int = 0

    def __getitem__(self, name: str) -> TensorValue:
        if name not in self.tensors:
            raise KeyError(f"weight {name!r} not in store")
        return self.tensors[name]

    def __contains__(self, name: str) -> bool:
        return name in self.tensors

    def names(self) -> set[str]:
        return set(self.tensors)

    def total_bytes(self) -> int:
        return sum(t.data.numel() * t.data.element_size() for t in self.tensors.values())
