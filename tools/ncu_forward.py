"""One merged forward of a bench workload inside a cudaProfilerStart/Stop
range, for ncu runs with `--profile-from-start off`:

    ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,\
        dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/x.csv \
        python tools/ncu_forward.py --config C5

Builds the exact plan bench.py times (same workload builder, heads, mode),
replays it a few times unprofiled (warm instruction caches, lazy module
loads), then launches one forward eagerly inside the profiled range. Also
writes the plan's per-launch algorithmic bytes/flops (bench.linear_launch_bytes)
next to the step list so the summary can pair ncu rows with them.
"""

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2009_13062_b200 import compile_plan  # noqa: E402
from paper_2009_13062_b200.workloads import BASELINE_CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5", choices=sorted(BASELINE_CONFIGS))
    ap.add_argument("--forwards", type=int, default=1)
    ap.add_argument("--meta", default=None, help="write the step list + algorithmic bytes here")
    args = ap.parse_args()
    model, n, batch, dtype = BASELINE_CONFIGS[args.config]
    _, _, inputs, merged, mstore, _ = bench.build_workload(model, n, batch, dtype, 0, heads=True)
    plan = compile_plan(merged.graph, mstore, mode="fast")
    plan.load_inputs(merged.bind_inputs(inputs))
    for _ in range(3):
        plan.launch()
    torch.cuda.synchronize()
    if args.meta:
        lin = bench.linear_launch_bytes(merged, mstore, {nid for nid, _, _ in plan.steps})
        Path(args.meta).write_text(json.dumps({
            "config": args.config, "workload": f"{model}/N{n}/B{batch}/{dtype}",
            "steps": [nid for nid, _, _ in plan.steps],
            "family": {k: list(v) for k, v in lin.items()},
            "kernel_launches": plan.kernel_launches}, indent=0))
    torch.cuda.cudart().cudaProfilerStart()
    for _ in range(args.forwards):
        plan.launch()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()


if __name__ == "__main__":
    main()
