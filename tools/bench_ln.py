"""Time nf_grouped_linear_ln (cluster LayerNorm epilogue) vs the plain merged
Linear at batch-1 shapes (CUDA graph of L2-flushed launches)."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2009_13062_b200 import _lib

def t_graph(fn, reps, flush):
    def cap(k):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(reps):
                flush.zero_()
                if k:
                    fn(torch.cuda.current_stream().cuda_stream)
        return g
    out = []
    for k in (True, False):
        g = cap(k); g.replay(); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); g.replay(); e.record(); torch.cuda.synchronize()
        out.append(s.elapsed_time(e))
    return (out[0] - out[1]) / reps * 1e3

flush = torch.empty(64 * 1024 * 1024, device="cuda")
for G, T, K, N in [(8, 128, 768, 768), (8, 128, 3072, 768), (32, 128, 768, 768)]:
    x = (torch.rand(G, T, K, device="cuda") - 0.5).bfloat16()
    w = ((torch.rand(G, N, K, device="cuda") - 0.5) / K ** 0.5).bfloat16()
    b = torch.zeros(G, N, device="cuda"); r = torch.zeros(G, T, N, device="cuda").bfloat16()
    gam = torch.ones(G, N, device="cuda"); bet = torch.zeros(G, N, device="cuda")
    y = torch.empty(G, T, N, device="cuda").bfloat16()
    ln = lambda st: _lib.call("nf_grouped_linear_ln", x.data_ptr(), K, T * K, w.data_ptr(), b.data_ptr(), r.data_ptr(), gam.data_ptr(), bet.data_ptr(), 1e-12, y.data_ptr(), N, T * N, G, T, K, N, st)
    pl = lambda st: _lib.call("nf_grouped_linear_ws", x.data_ptr(), K, T * K, w.data_ptr(), b.data_ptr(), r.data_ptr(), y.data_ptr(), N, T * N, G, T, K, N, _lib.NF_BF16, _lib.NF_W_NK, 0, _lib.NF_MODE_FAST, None, 0, st)
    print(json.dumps({"G": G, "T": T, "K": K, "N": N, "ln_us": round(t_graph(ln, 20, flush), 2), "plain_us": round(t_graph(pl, 20, flush), 2)}))

# direct launches (no CUDA graph), with / without residual
def t_direct(fn, reps):
    for _ in range(3):
        fn(torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(torch.cuda.current_stream().cuda_stream); e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return round(sorted(ts)[len(ts) // 2], 2)

G, T, K, N = 8, 128, 768, 768
x = (torch.rand(G, T, K, device="cuda") - 0.5).bfloat16()
w = ((torch.rand(G, N, K, device="cuda") - 0.5) / K ** 0.5).bfloat16()
b = torch.zeros(G, N, device="cuda"); r = torch.zeros(G, T, N, device="cuda").bfloat16()
gam = torch.ones(G, N, device="cuda"); bet = torch.zeros(G, N, device="cuda")
y = torch.empty(G, T, N, device="cuda").bfloat16()
for rp in (r.data_ptr(), None):
    ln = lambda st: _lib.call("nf_grouped_linear_ln", x.data_ptr(), K, T * K, w.data_ptr(), b.data_ptr(), rp, gam.data_ptr(), bet.data_ptr(), 1e-12, y.data_ptr(), N, T * N, G, T, K, N, st)
    print(json.dumps({"residual": rp is not None, "direct_us": t_direct(ln, 20), "graph_us": round(t_graph(ln, 20, flush), 2)}))
