import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2009_13062_b200 import Plan, model_inputs
from paper_2009_13062_b200 import workloads as W
g = W.build_graph("resnet-mini", dtype="bf16")
st = W.build_weights("resnet-mini", dtype="bf16", model=0)
inp = model_inputs(g, model=0)
plan = Plan(g, st)
plan.load_inputs(inp); plan.launch(); torch.cuda.synchronize()
x = plan.vals["stem.pool"].t.float()           # (1,64,16,16) logical
wf, bias = plan._wcache[("convchain", "l1.b0.conv1")]
wg, bg = plan._wcache[("convchain", "l1.b0.conv1", "gemm")]
print("wf", wf.shape, "wg", wg.shape, bg.shape)
ref = torch.nn.functional.conv2d(x, wf.permute(0, 3, 1, 2), bias)
ref = torch.relu(ref)
got = plan.vals["l1.b0.relu1"].t.float()
print("err vs folded torch", ((got - ref).abs().max() / ref.abs().max()).item())
# unfolded oracle-like
w = st["l1.b0.conv1.w"].data.cuda().float()
gm, be, mu, va = (st[f"l1.b0.bn1.{s}"].data.cuda().float() for s in "gbmv")
y = torch.nn.functional.conv2d(x, w)
y = (y - mu.view(1,-1,1,1)) / torch.sqrt(va.view(1,-1,1,1) + 1e-5) * gm.view(1,-1,1,1) + be.view(1,-1,1,1)
y = torch.relu(y)
print("err vs unfolded", ((got - y).abs().max() / y.abs().max()).item(), "folded-vs-unfolded", ((ref - y).abs().max()/y.abs().max()).item())
xn = plan.vals["stem.pool"].t
print("pool strides", xn.shape, xn.stride(), "out strides", plan.vals["l1.b0.relu1"].t.stride())
for i,(nid, fn, _) in enumerate(plan.steps[:8]):
    print(i, nid, [c for c in fn.__code__.co_consts if isinstance(c,str)], fn.__code__.co_freevars)
scale = gm / torch.sqrt(va + 1e-5)
wman = (w * scale.view(-1,1,1,1)).permute(0,2,3,1)
print("wf vs manual fold", (wf - wman).abs().max().item(), "bias vs manual", (bias - (be - mu*scale)).abs().max().item())
print("chain", [ (k, [n.id for n in v["nodes"]]) for k,v in plan._conv_chains(__import__('paper_2009_13062_b200').topological_order(g), {}, set()).items()][:2])
print("bn attrs", [n.attrs for n in g.nodes if n.id=="l1.b0.bn1"])
