"""Normwise error of the merged BERT-2l (+ heads) features and logits vs the
oracle, for the current NF_FOLD_LN setting (diagnostic)."""
import numpy as np
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from test_gpu_execute import _bert_setup, normwise  # noqa: E402
from oracle import executor as OX  # noqa: E402
from paper_2009_13062_b200 import execute  # noqa: E402

graph, stores, inputs, merged, mstore, heads = _bert_setup("bert-2l", 4, 1)
outs, _ = execute(merged.graph, mstore, merged.bind_inputs(inputs))
per = merged.slice_outputs(outs)
for j in range(4):
    feat = OX.execute(graph, stores[j].tensors, inputs[j])[0]
    want = OX.execute(heads[j][0], heads[j][1].tensors, {"feat": feat})[0]
    print(j, "logits", normwise(per[j][0].numpy(), want), per[j][0].numpy(), want)
graph, stores, inputs, merged, mstore, _ = _bert_setup("bert-2l", 4, 1, heads=False)
outs, _ = execute(merged.graph, mstore, merged.bind_inputs(inputs))
per = merged.slice_outputs(outs)
for j in range(4):
    want = OX.execute(graph, stores[j].tensors, inputs[j])[0]
    print(j, "features", normwise(per[j][0].numpy(), want))
