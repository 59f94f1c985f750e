"""Node-by-node comparison of a GPU plan against the oracle (debug aid)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from oracle import executor as OX
from paper_2009_13062_b200 import Plan, model_inputs
from paper_2009_13062_b200 import workloads as W

name = sys.argv[1] if len(sys.argv) > 1 else "resnet-mini"
dtype = sys.argv[2] if len(sys.argv) > 2 else "bf16"
g = W.build_graph(name, dtype=dtype)
st = W.build_weights(name, dtype=dtype, model=0)
inp = model_inputs(g, model=0)
plan = Plan(g, st)
plan.load_inputs(inp)
plan.launch()
torch.cuda.synchronize()
_, vals = OX.execute(g, st.tensors, inp, keep=True)
for n in g.nodes:
    v = plan.vals.get(n.id)
    if v is None or v.split is not None:
        continue
    got = v.t.float().cpu().numpy()
    want = vals[n.id]
    err = np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-30)
    flag = "  <-- BAD" if err > 3e-2 else ""
    print(f"{n.id:24s} {n.kind.value:14s} {err:.3e}{flag}")
