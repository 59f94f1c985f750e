"""Per-CTA timeline of the last chained batch-1 Linear launch of a merged
forward (csrc/gemm_chain.cuh built with -DNF_CHAIN_TRACE):

    tools/build_var.sh ctrace -DNF_CHAIN_TRACE
    NF_LIB_PATH=varlib/lib_ctrace.so python tools/chain_trace.py --config C2
"""
import argparse
import ctypes
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2009_13062_b200 import _lib, compile_plan  # noqa: E402
from paper_2009_13062_b200.workloads import BASELINE_CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    args = ap.parse_args()
    model, n, batch, dtype = BASELINE_CONFIGS[args.config]
    _, _, inputs, merged, mstore, _ = bench.build_workload(model, n, batch, dtype, 0, heads=True)
    plan = compile_plan(merged.graph, mstore)
    plan.load_inputs(merged.bind_inputs(inputs))
    g = plan.capture()
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    buf = (ctypes.c_uint64 * (148 * 4 * 16))()
    fn = _lib.load().nf_debug_chain_trace
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
    assert fn(ctypes.addressof(buf), ctypes.sizeof(buf)) == 0
    tr = np.frombuffer(buf, dtype=np.uint64).reshape(148, 4, 16).astype(np.int64)
    t0 = tr[:, 0, 7][tr[:, 0, 7] > 0].min()
    print(f"CTA entry: min 0, max {(tr[:, 0, 7].max() - t0) / 1e3:.2f} us")
    rows = []
    for b in range(148):
        for u in range(4):
            r = tr[b, u]
            if r[0] == 0 or r[0] < t0 or (u > 0 and r[0] < tr[b, u - 1, 0]):
                continue
            rows.append((b, u, int(r[6]), *(((r[:6] - t0) / 1e3).tolist())))
    print("op  n   start(min/med/max)   dep_ok(med/max)  first_stage(med)  mma_done(med/max)  "
          "epi_start(med)  published(min/med/max)")
    for op in sorted({r[2] for r in rows}):
        a = np.array([r[3:] for r in rows if r[2] == op])
        q = lambda c, f: f(a[:, c])  # noqa: E731
        print(f"{op:2d} {len(a):3d}  {q(0, np.min):6.2f} {q(0, np.median):6.2f} {q(0, np.max):6.2f}"
              f"   {q(1, np.median):6.2f} {q(1, np.max):6.2f}   {q(2, np.median):6.2f}"
              f"        {q(3, np.median):6.2f} {q(3, np.max):6.2f}      {q(4, np.median):6.2f}"
              f"     {q(5, np.min):6.2f} {q(5, np.median):6.2f} {q(5, np.max):6.2f}")
    # per-unit durations
    a = np.array([r[3:] for r in rows])
    print(f"median unit phases (us): dep wait {np.median(a[:, 1] - a[:, 0]):.2f}, "
          f"dep->first stage {np.median(a[:, 2] - a[:, 1]):.2f}, main loop "
          f"{np.median(a[:, 3] - a[:, 2]):.2f}, acc->epi {np.median(a[:, 4] - a[:, 3]):.2f}, "
          f"epilogue {np.median(a[:, 5] - a[:, 4]):.2f}")
    for op in range(3):
        pre = np.array([(tr[b, u, [0, 12, 13, 4]] - t0) / 1e3 for b in range(148) for u in range(4)
                        if tr[b, u, 0] >= t0 and tr[b, u, 6] == op and tr[b, u, 4] > 0
                        and tr[b, u, 12] >= tr[b, u, 0]])
        if len(pre):
            d = np.diff(pre, axis=1)
            print(f"op{op} epilogue pre-accumulator (median us): start->dep ok %.2f, "
                  "dep ok->stats %.2f, stats->acc ready %.2f" % tuple(np.median(d, axis=0)))
        ep = np.array([(tr[b, u, [4, 8, 9, 10, 11, 5]] - t0) / 1e3 for b in range(148)
                       for u in range(4) if tr[b, u, 0] >= t0 and tr[b, u, 6] == op
                       and tr[b, u, 5] >= tr[b, u, 4] > 0 and tr[b, u, 5] - tr[b, u, 0] < 10 ** 6])
        if len(ep) == 0:
            continue
        d = np.diff(ep, axis=1)
        print(f"op{op} epilogue phases (median us, n={len(ep)}): residual wait %.2f, chunks %.2f, "
              "stats %.2f, store completion %.2f, publish %.2f" % tuple(np.median(d, axis=0)))
    wb = (ctypes.c_uint64 * (148 * 4 * 8 * 8))()
    fw = _lib.load().nf_debug_chain_wtrace
    fw.argtypes = [ctypes.c_void_p, ctypes.c_int]
    assert fw(ctypes.addressof(wb), ctypes.sizeof(wb)) == 0
    wt = np.frombuffer(wb, dtype=np.uint64).reshape(148, 4, 8, 8).astype(np.int64)
    for op in range(3):
        sel = [(b, u) for b in range(148) for u in range(4)
               if tr[b, u, 0] >= t0 and tr[b, u, 6] == op and wt[b, u, 0, 0] >= tr[b, u, 4] > 0]
        if not sel:
            continue
        st = np.array([(wt[b, u, :, 0] - tr[b, u, 8]) / 1e3 for b, u in sel])
        du = np.array([(wt[b, u, :, 7] - wt[b, u, :, 0]) / 1e3 for b, u in sel])
        ph = np.array([np.diff(wt[b, u, 0, :]) / 1e3 for b, u in sel])
        print(f"op{op} warp-2 chunk phases (median us): ld0 %.2f, math0 %.2f, act+store0 %.2f, "
              "ld1 %.2f, math1 %.2f, act+store1 %.2f, tail %.2f" % tuple(np.median(ph, axis=0)))
        print(f"op{op} per-warp chunk loop: start after residual (median per warp) "
              + " ".join(f"{x:.2f}" for x in np.median(st, axis=0))
              + " | duration " + " ".join(f"{x:.2f}" for x in np.median(du, axis=0)))
    for b in (0, 47, 48, 90, 147):
        print(f"CTA {b}: " + " | ".join(
            f"op{int(tr[b, u, 6])} " + " ".join(f"{(tr[b, u, s] - t0) / 1e3:.1f}" for s in range(6))
            for u in range(4) if tr[b, u, 0] >= t0 and tr[b, u, 0] > 0))


if __name__ == "__main__":
    main()
