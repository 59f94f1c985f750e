"""Per-kernel critical-path share of a PDL timeline (gpurun_out/timeline.json
from tools/profile_plan.py): delta between consecutive kernel end times."""
import collections
import json
import sys

seq = json.load(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/timeline.json"))
prev_end = None
acc = collections.defaultdict(list)
for k in seq:
    end = k["start"] + k["dur"]
    if prev_end is not None:
        acc[k["name"][:60]].append(end - prev_end)
    prev_end = end
for name, v in sorted(acc.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v):8.1f} us  n={len(v):3d}  avg={sum(v)/len(v):6.2f}  {name}")
