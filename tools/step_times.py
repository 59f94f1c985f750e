"""Per-launch device time of a BASELINE config's plan: every launch of the
plan bracketed by CUDA events recorded into one CUDA graph (the bench's
instrumented replay), averaged over replays, with its algorithmic bytes/flops.

    python tools/step_times.py --config C1 [--top 20]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2009_13062_b200 import compile_plan  # noqa: E402
from paper_2009_13062_b200.workloads import BASELINE_CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--top", type=int, default=25)
    args = ap.parse_args()
    model, n, batch, dtype = BASELINE_CONFIGS[args.config]
    _, _, inputs, merged, mstore, _ = bench.build_workload(model, n, batch, dtype, 0, heads=True)
    plan = compile_plan(merged.graph, mstore)
    plan.load_inputs(merged.bind_inputs(inputs))
    lin = bench.linear_launch_bytes(merged, mstore, {nid for nid, _, _ in plan.steps})
    steps = plan.steps
    evs = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(len(steps) + 1)]
    plan.launch()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        st = torch.cuda.current_stream()
        for i, (_, fn, _) in enumerate(steps):
            evs[i].record(st)
            fn(st.cuda_stream)
        evs[-1].record(st)
    per = [0.0] * len(steps)
    for _ in range(args.reps):
        g.replay()
        torch.cuda.synchronize()
        for i in range(len(steps)):
            per[i] += evs[i].elapsed_time(evs[i + 1]) * 1e3 / args.reps
    total = sum(per)
    print(f"{args.config}: {len(steps)} launches, {total:.1f} us summed (instrumented, serialised)")
    order = sorted(range(len(steps)), key=lambda i: -per[i])[:args.top]
    for i in order:
        nid = steps[i][0]
        b, f = lin.get(nid, (0, 0))
        gbs = b / per[i] / 1e3 if per[i] else 0
        tf = f / per[i] / 1e6 if per[i] else 0
        print(f"{per[i]:8.1f} us  {100 * per[i] / total:5.1f}%  {gbs:7.0f} GB/s {tf:7.1f} TF/s  {nid[:90]}")


if __name__ == "__main__":
    main()
