export PYTHONPATH=.
timeout 600 python -m pytest tests/test_gpu_fold.py tests/test_gpu_execute.py -q --timeout 300 2>&1 | tail -3
NF_FOLD_LN=1 python - <<'PY'
import sys; sys.path.insert(0, "tests")
import numpy as np
from test_gpu_execute import _bert_setup, normwise
from oracle import executor as OX
from paper_2009_13062_b200 import execute, engine
engine._FOLD_LN = True
for rows_cap in (False,):
    graph, stores, inputs, merged, mstore, _ = _bert_setup("bert-2l", 2, 4, heads=False)
    outs, _ = execute(merged.graph, mstore, merged.bind_inputs(inputs))
    per = merged.slice_outputs(outs)
    for j in range(2):
        want = OX.execute(graph, stores[j].tensors, inputs[j])[0]
        print("large-batch err", j, normwise(per[j][0].numpy(), want))
PY
