"""Merged CNN families on the GPU vs the CPU oracle (per-instance forwards).

* exact mode, f32: every op restates the reference order (direct conv, BN,
  ReLU, Add, pools) -> merged ResNet slices are byte-identical to the oracle;
* fast f32 (fused conv+BN+residual+ReLU, FFMA): normwise <= 1e-4;
* fast bf16 (NHWC tensor-core implicit GEMM, folded BN): <= 2e-2, top-1 exact.
"""

import numpy as np
import pytest

from oracle import executor as OX
from paper_2009_13062_b200 import execute, merge, merge_backbone, model_inputs
from paper_2009_13062_b200 import workloads as W

pytestmark = pytest.mark.gpu


def normwise(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30)


def _run(name, m, dtype, mode, heads=True, batch=1):
    graph = W.build_graph(name, batch=batch, dtype=dtype)
    stores = [W.build_weights(name, dtype=dtype, model=j) for j in range(m)]
    inputs = [model_inputs(graph, model=j) for j in range(m)]
    if heads:
        out = graph.node_map()["pool"].output_spec
        hs = [W.fc_head(out, 10 + 3 * j, seed=j) for j in range(m)]
        merged, mstore = merge_backbone(graph, {n.id for n in graph.nodes}, stores, hs)
    else:
        hs = None
        merged, mstore = merge(graph, stores)
    outs, _ = execute(merged.graph, mstore, merged.bind_inputs(inputs), mode=mode)
    per = merged.slice_outputs(outs)
    return graph, stores, inputs, hs, per


def _oracle(graph, stores, inputs, hs, j):
    feat = OX.execute(graph, stores[j].tensors, inputs[j])[0]
    if hs is None:
        return feat
    return OX.execute(hs[j][0], hs[j][1].tensors, {"feat": feat})[0]


@pytest.mark.parametrize("name", ["resnet-mini", "resnext-mini"])
def test_exact_f32_merged_cnn_bit_identical(name):
    graph, stores, inputs, hs, per = _run(name, 2, "f32", "exact", heads=False, batch=2)
    for j in range(2):
        assert per[j][0].numpy().tobytes() == _oracle(graph, stores, inputs, None, j).tobytes()


@pytest.mark.parametrize("name", ["resnet-mini", "resnext-mini"])
def test_fast_f32_fused_cnn(name):
    graph, stores, inputs, hs, per = _run(name, 3, "f32", "fast")
    for j in range(3):
        want = _oracle(graph, stores, inputs, hs, j)
        got = per[j][0].numpy()
        assert normwise(got, want) < 1e-4
        assert (got.argmax(-1) == want.argmax(-1)).all()


@pytest.mark.parametrize("name", ["resnet-mini", "resnext-mini"])
def test_fast_bf16_tensor_core_cnn(name):
    graph, stores, inputs, hs, per = _run(name, 4, "bf16", "fast")
    for j in range(4):
        want = _oracle(graph, stores, inputs, hs, j)
        assert normwise(per[j][0].numpy(), want) < 2e-2


@pytest.mark.parametrize("name,m", [("resnet50", 2), ("resnext50_32x4d", 4)])
def test_full_size_cnn_sampled_instance(name, m):
    """BASELINE configs[0]/[2] architectures at 224x224 (N reduced for the
    oracle's CPU time; slices are independent): instance 0 and m-1."""
    graph, stores, inputs, hs, per = _run(name, m, "bf16", "fast")
    for j in (0, m - 1):
        want = _oracle(graph, stores, inputs, hs, j)
        got = per[j][0].numpy()
        assert normwise(got, want) < 2e-2
        assert int(got.argmax()) == int(want.argmax())
