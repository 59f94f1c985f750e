"""Parity at every BASELINE.json configuration, through the exact plan the
bench runs (``workloads.merged_workload`` + ``compile_plan`` defaults: heads
attached with merge_backbone, default fusion / LayerNorm folding, the same
G / T / batch that select tiles, CTA pairs, split-K and folding).

Per SURVEY §8c the oracle is the per-instance CPU forward built from the
reference kernels (merged == per-instance is the reference's own theorem,
PAPER.md:620-670), run on sampled instances 0 and N-1 (slices independent):
  * logits normwise  max|y_gpu - y_cpu| / max|y_cpu|  <= 2e-2 (bf16) / 1e-4 (fp32),
  * top-1 argmax bit-exact per sequence / image, top-1/top-2 margin reported.

Set NF_PARITY_LOG=<file> to append one JSON line per checked instance
(error, top-1 agreement, smallest oracle margin) — profiles/r02_parity.jsonl.
"""

import json
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

from oracle import executor as OX
from paper_2009_13062_b200 import execute
from paper_2009_13062_b200 import workloads as W

pytestmark = pytest.mark.gpu

TOL = {"bf16": 2e-2, "f32": 1e-4}


def normwise(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def _oracle_instance(graph, store, inputs, head):
    feat = OX.execute(graph, store.tensors, inputs)[0]
    return OX.execute(head[0], head[1].tensors, {"feat": feat})[0]


def _margins(logits):
    srt = np.sort(np.asarray(logits, np.float64), axis=-1)
    return srt[..., -1] - srt[..., -2]


def _check_config(cfg):
    model, n, batch, dtype = W.BASELINE_CONFIGS[cfg]
    graph, stores, inputs, merged, mstore, heads = W.merged_workload(model, n, batch, dtype)
    outs, trace = execute(merged.graph, mstore, merged.bind_inputs(inputs))
    per = merged.slice_outputs(outs)
    sample = (0, n - 1)
    with ThreadPoolExecutor(max_workers=len(sample)) as ex:
        wants = list(ex.map(lambda j: _oracle_instance(graph, stores[j], inputs[j], heads[j]),
                            sample))
    log = os.environ.get("NF_PARITY_LOG")
    for j, want in zip(sample, wants):
        got = per[j][0].numpy().astype(np.float64)
        want = want.reshape(got.shape)
        err = normwise(got, want)
        top_ok = bool((got.argmax(-1) == want.argmax(-1)).all())
        rec = {"config": cfg, "model": model, "instances": n, "batch": batch, "dtype": dtype,
               "instance": j, "normwise": err, "tol": TOL[dtype], "top1_exact": top_ok,
               "rows": int(np.prod(got.shape[:-1])), "classes": int(got.shape[-1]),
               "min_margin_oracle": float(_margins(want).min()),
               "max_abs_logit": float(np.abs(want).max()),
               "kernel_launches": trace.kernel_launches}
        print(json.dumps(rec))
        if log:
            with open(log, "a") as f:
                f.write(json.dumps(rec) + "\n")
        assert err <= TOL[dtype], rec
        assert top_ok, rec
    torch.cuda.empty_cache()


def test_c1_resnet50_n2_fp32():
    """configs[0]: ResNet-50, N=2, B=1, 224x224, fp32 (<= 1e-4, top-1 exact)."""
    _check_config("C1")


def test_c2_bert_base_n8_b1_with_heads():
    """configs[1]: BERT-base N=8 B=1 S=128, 12 layers + per-task heads."""
    _check_config("C2")


def test_c3_resnext50_n32():
    """configs[2]: ResNeXt-50 32x4d N=32 B=1 (super-grouped implicit GEMM)."""
    _check_config("C3")


def test_c4_xlnet_base_n32_b4():
    """configs[3]: XLNet-base 12 layers N=32 B=4 S=128 (relative attention)."""
    _check_config("C4")


def test_c5_bert_base_n32_b8():
    """configs[4] per-GPU shard: BERT-base N=32 B=8 S=128 (the bench default)."""
    _check_config("C5")
