"""Micro-benchmark of the merged LayerNorm (+ residual) at the C5 / C4 shape
(model-major split storage, per-instance affine): L2 flushed, CUDA events,
algorithmic bytes = x + residual read, y written."""
import argparse
import json

import torch

from paper_2009_13062_b200 import _lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=32)
    ap.add_argument("--rows", type=int, default=1024)
    ap.add_argument("--d", type=int, default=768)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--add", action="store_true",
                    help="time torch.add(x, r, out=y) instead: the same 2-read + 1-write streams")
    ap.add_argument("--copy", action="store_true", help="time y.copy_(x) (1 read + 1 write)")
    a = ap.parse_args()
    x = torch.randn(a.m, a.rows, a.d, device="cuda").bfloat16()
    r = torch.randn_like(x)
    y = torch.empty_like(x)
    g = torch.rand(a.m * a.d, device="cuda")
    b = torch.rand(a.m * a.d, device="cuda")
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    args = (x.data_ptr(), r.data_ptr(), g.data_ptr(), b.data_ptr(), y.data_ptr(), a.m, a.rows,
            a.rows * a.d, a.d, 1, a.d, a.d, 1, a.rows, 1e-12, _lib.NF_BF16, st)
    def run():
        if a.copy:
            y.copy_(x)
        elif a.add:
            torch.add(x, r, out=y)
        else:
            _lib.call("nf_group_norm", *args)

    for _ in range(3):
        run()
    ts = []
    for _ in range(a.reps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        run()
        e.record()
        ts.append((s, e))
    torch.cuda.synchronize()
    us = sum(s.elapsed_time(e) for s, e in ts) / len(ts) * 1e3
    nbytes = (2 if a.copy else 3) * x.numel() * 2
    print(json.dumps({"op": "copy" if a.copy else ("torch.add" if a.add else "nf_group_norm"), "rows": a.m * a.rows, "d": a.d, "us": round(us, 2),
                      "GBps": round(nbytes / us / 1e3, 1)}))


if __name__ == "__main__":
    main()
