"""Experiment: the merged BERT-8 forward as L instance lanes (each a merged
forward of N/L instances) captured on L streams of one CUDA graph."""
import sys, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import bench
from paper_2009_13062_b200 import compile_plan, merge_backbone
from paper_2009_13062_b200 import workloads as W

def run(model, n, b, lanes):
    graph, stores, inputs, merged, mstore, heads = bench.build_workload(model, n, b, "bf16", 0)
    per = n // lanes
    plans = []
    for l in range(lanes):
        sl = slice(l * per, (l + 1) * per)
        mg, ms = merge_backbone(graph, {x.id for x in graph.nodes}, stores[sl], heads[sl])
        p = compile_plan(mg.graph, ms)
        p.load_inputs(mg.bind_inputs(inputs[sl]))
        plans.append(p)
    streams = [torch.cuda.Stream() for _ in plans]
    def launch():
        cur = torch.cuda.current_stream()
        for s in streams:
            s.wait_stream(cur)
        for p, s in zip(plans, streams):
            with torch.cuda.stream(s):
                p.launch()
        for s in streams:
            cur.wait_stream(s)
    launch(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        launch()
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    ms = bench._time_steps(g.replay, 5, flush, torch.cuda.current_stream())
    ms = bench._time_steps(g.replay, 30, flush, torch.cuda.current_stream())
    return ms

for model, n, b in (("bert-base", 8, 1), ("bert-base", 32, 1)):
    for lanes in (1, 2, 4):
        ms = run(model, n, b, lanes)
        print(json.dumps({"model": model, "n": n, "b": b, "lanes": lanes, "ms": round(ms, 4),
                          "inf_s": round(n * b / ms * 1e3, 1)}))
