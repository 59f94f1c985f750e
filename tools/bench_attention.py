"""Graph-timed microbenchmark of the merged attention kernel (BERT shapes)."""
import argparse, json
import torch
from paper_2009_13062_b200 import kernels as K

ap = argparse.ArgumentParser()
ap.add_argument("--bt", type=int, default=8)
ap.add_argument("--heads", type=int, default=12)
ap.add_argument("--seq", type=int, default=128)
ap.add_argument("--reps", type=int, default=50)
a = ap.parse_args()
qkv = (torch.rand(a.bt, a.seq, 3 * 64 * a.heads, device="cuda") - 0.5).bfloat16()
for _ in range(3):
    K.attention(qkv, heads=a.heads)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(a.reps):
        K.attention(qkv, heads=a.heads)
g.replay(); torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); g.replay(); e.record(); torch.cuda.synchronize()
print(json.dumps({"bt": a.bt, "heads": a.heads, "seq": a.seq, "us": s.elapsed_time(e) * 1e3 / a.reps}))
