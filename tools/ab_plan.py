"""A/B of plan options on a BASELINE config: graph-replay ms/step (L2
flushed between steps, CUDA events) for compile_plan variants.

    python tools/ab_plan.py --config C5 --variants fold_ln=1 fold_ln=0
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
    ap.add_argument("--config", default="C5")
    ap.add_argument("--variants", nargs="+", default=["fold_ln=1", "fold_ln=0"])
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    model, n, batch, dtype = BASELINE_CONFIGS[args.config]
    _, _, inputs, merged, mstore, _ = bench.build_workload(model, n, batch, dtype, 0, heads=True)
    bound = merged.bind_inputs(inputs)
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    outs = {}
    for v in args.variants:
        kw = {k: bool(int(x)) for k, x in (a.split("=") for a in v.split(","))}
        plan = compile_plan(merged.graph, mstore, **kw)
        plan.load_inputs(bound)
        g = plan.capture()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.steps):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            g.replay()
            e.record()
            ts.append((s, e))
        torch.cuda.synchronize()
        ms = sum(s.elapsed_time(e) for s, e in ts) / len(ts)
        outs[v] = [o.float().clone() for o in plan.outputs()]
        print(f"{args.config} {v}: {ms:.4f} ms/step, {plan.kernel_launches} launches", flush=True)
        del g, plan
        torch.cuda.empty_cache()
    ref = outs[args.variants[0]]
    for v in args.variants[1:]:
        err = max(((a - b).abs().max() / b.abs().max()).item() for a, b in zip(outs[v], ref))
        print(f"  {v} vs {args.variants[0]}: normwise {err:.3e}")


if __name__ == "__main__":
    main()
