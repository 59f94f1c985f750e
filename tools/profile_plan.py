"""Timeline of one merged forward inside a CUDA-graph replay (CUPTI via
torch.profiler): per-kernel device time, and the idle gaps between kernels.

    python tools/profile_plan.py [--model bert-base] [--instances 8] [--batch 1]
"""

import argparse
import collections
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2009_13062_b200 import compile_plan  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="bert-base")
    ap.add_argument("--instances", type=int, default=8)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--no-heads", action="store_true")
    ap.add_argument("--out", default="gpurun_out/timeline.json")
    ap.add_argument("--no-pdl", action="store_true",
                    help="serialise kernels (NF_PDL=0) so per-kernel durations are exact")
    args = ap.parse_args()
    if args.no_pdl:
        import os
        os.environ["NF_PDL"] = "0"
    _, _, inputs, merged, mstore, _ = bench.build_workload(
        args.model, args.instances, args.batch, args.dtype, 0, heads=not args.no_heads)
    plan = compile_plan(merged.graph, mstore)
    plan.load_inputs(merged.bind_inputs(inputs))
    g = plan.capture()
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    kern = sorted([(e.time_range.start, e.time_range.end, e.name) for e in evs],
                  key=lambda t: t[0])
    n = len(kern) // 3
    one = kern[n:2 * n]  # middle replay
    span = one[-1][1] - one[0][0]
    busy = sum(e - s for s, e, _ in one)
    per = collections.defaultdict(lambda: [0, 0.0])
    for s, e, name in one:
        short = name.split("(")[0][:70]
        per[short][0] += 1
        per[short][1] += e - s
    print(json.dumps({"kernels_per_forward": n, "span_us": round(span, 1),
                      "busy_us": round(busy, 1), "gap_us": round(span - busy, 1)}))
    for name, (cnt, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        print(f"{t:9.1f} us {100 * t / busy:5.1f}%  n={cnt:3d} avg={t / cnt:7.2f}  {name}")
    seq = [{"name": nm.split("(")[0][:60], "start": round(s - one[0][0], 2),
            "dur": round(e - s, 2)} for s, e, nm in one]
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(seq, indent=0))


if __name__ == "__main__":
    main()
