"""Micro-benchmark of the merged-Linear kernel at BASELINE config shapes.

Times each shape with CUDA events (warm-up, then the mean of R launches, L2
flushed between launches by a 256 MB write) and prints achieved HBM GB/s
(algorithmic bytes: weights + activations in + out) and TFLOP/s.
"""

import argparse
import json

import torch

from paper_2009_13062_b200 import _lib

SHAPES = {
    # name: (G, T, K, N)
    "bert_b1_qkv": (8, 128, 768, 2304),
    "bert_b1_proj": (8, 128, 768, 768),
    "bert_b1_ff1": (8, 128, 768, 3072),
    "bert_b1_ff2": (8, 128, 3072, 768),
    "bert_b1_ff1_gelu": (8, 128, 768, 3072),
    "xlnet_b4_ff1": (32, 512, 768, 3072),
    "xlnet_b4_ff2": (32, 512, 3072, 768),
    "bert_b8_ff1": (32, 1024, 768, 3072),
    "bert_b8_ff1_gelu": (32, 1024, 768, 3072),
    "bert_b8_qkv": (32, 1024, 768, 2304),
    "bert_b8_ff2": (32, 1024, 3072, 768),
    "bert_b8_proj_res": (32, 1024, 768, 768),
    "bert_b8_ff2_res": (32, 1024, 3072, 768),
    "xlnet_b4_ff1_gelu": (32, 512, 768, 3072),
    "xlnet_b4_proj_res": (32, 512, 768, 768),
}


def run(name, G, T, K, N, reps, flush):
    dev = "cuda"
    x = (torch.rand(G, T, K, device=dev) - 0.5).bfloat16()
    w = (torch.rand(G, N, K, device=dev) - 0.5).bfloat16() * 0.05
    b = torch.zeros(G, N, device=dev)
    y = torch.empty(G, T, N, device=dev, dtype=torch.bfloat16)
    stream = torch.cuda.current_stream().cuda_stream

    def launch():
        _lib.call("nf_grouped_linear", x.data_ptr(), w.data_ptr(), b.data_ptr(), None,
                  y.data_ptr(), G, T, K, N, _lib.NF_BF16, _lib.NF_W_NK, _lib.NF_ACT_NONE,
                  _lib.NF_MODE_FAST, stream)

    for _ in range(5):
        launch()
    torch.cuda.synchronize()
    # Capture `reps` launches, each preceded by an L2 flush, in one CUDA graph
    # so host launch latency is excluded; time flush-only graph separately.
    def capture(with_kernel):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(reps):
                if flush is not None:
                    flush.zero_()
                if with_kernel:
                    launch_on(torch.cuda.current_stream().cuda_stream)
        return g

    act = _lib.NF_ACT_GELU if name.endswith("gelu") else _lib.NF_ACT_NONE
    res = torch.zeros_like(y) if name.endswith("_res") else None

    wsb = int(_lib.load().nf_linear_workspace_bytes(G, T, K, N))
    ws = torch.zeros(max(wsb, 1), dtype=torch.uint8, device=dev)

    def launch_on(st):
        _lib.call("nf_grouped_linear_ws", x.data_ptr(), K, T * K, w.data_ptr(), b.data_ptr(),
                  res.data_ptr() if res is not None else None, y.data_ptr(), N, T * N, G, T, K, N, _lib.NF_BF16, _lib.NF_W_NK, act,
                  _lib.NF_MODE_FAST, ws.data_ptr() if wsb else None, wsb, st)

    def timed(g):
        g.replay()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g.replay()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) * 1e-3

    t = (timed(capture(True)) - timed(capture(False))) / reps
    nbytes = 2 * (G * N * K + G * T * K + G * T * N)
    flops = 2 * G * T * N * K
    return {"shape": name, "G": G, "T": T, "K": K, "N": N, "us": t * 1e6,
            "GBps": nbytes / t / 1e9, "TFLOPs": flops / t / 1e12}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--only", default="")
    ap.add_argument("--shapes", default="", help="extra G,T,K,N;G,T,K,N;... to time")
    args = ap.parse_args()
    flush = None if args.no_flush else torch.empty(256 * 1024 * 1024 // 4, device="cuda")
    shapes = dict(SHAPES)
    if args.shapes:
        shapes = {f"g{s}": tuple(int(v) for v in s.split(",")) for s in args.shapes.split(";")}
    for name, shp in shapes.items():
        if args.only and name not in args.only.split(","):
            continue
        print(json.dumps(run(name, *shp, args.reps, flush)))


if __name__ == "__main__":
    main()
