"""GPU serving strategies of the paper's evaluation, B200 edition.

The reference benchmarks its CPU executor with three strategies
(`pkg/src/modelmerge/bench.py:102-199`: ``sequential``, ``threaded``,
``merged``, each with a tracemalloc peak-memory figure); the paper compares
NetFuse on the GPU against:

  * **sequential** — one process runs the N models one after another;
  * **concurrent** — a process per model, all running at once with no
    synchronisation across processes;
  * **hybrid** — P processes, each running N/P models sequentially
    ("(Ap, Bm)");
  * **merged** — NetFuse: the N models merged into one forward.

and reports peak GPU memory per strategy (the per-process
framework base memory is what sinks the concurrent baseline).

Every strategy here runs in its own spawned worker process(es) so all of
them pay the same per-process costs (CUDA context, allocator, module load),
and every model is served by this framework's own kernels: unmerged models
as N per-instance plans (one CUDA graph per process replaying that
process's models back to back), the merged one as a single merged plan.
A round = every process serves each of its models once (one request per
model, inputs resident on the device) and synchronises. All processes start
their timed rounds at a shared barrier; throughput = inferences completed by
all processes / (last finish - first start), host wall clock (CLOCK_MONOTONIC
is shared by the processes; device events cannot be compared across CUDA
contexts). Memory: the device's used bytes (NVML, sampled by the parent
every ~20 ms) above the idle baseline taken before any worker starts, plus
each worker's own allocator peak (weights + activations).

    python -m paper_2009_13062_b200.serving --model bert-base --num-models 32 \
        [--batch 1] [--strategies sequential,concurrent,hybrid:4,merged]
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import threading
import time
from dataclasses import asdict, dataclass, field

STRATEGIES = ("sequential", "concurrent", "hybrid", "merged")


@dataclass
class ServingReport:
    strategy: str
    model: str
    num_models: int
    batch: int
    dtype: str
    processes: int
    models_per_process: list[int]
    rounds: int
    wall_s: float = 0.0
    inferences_per_s: float = 0.0
    ms_per_round: float = 0.0
    peak_device_bytes: int | None = None      # NVML used above the idle baseline
    worker_allocated_bytes: list[int] = field(default_factory=list)  # torch peak per worker
    worker_reserved_bytes: list[int] = field(default_factory=list)
    kernel_launches_per_round: int = 0
    error: str | None = None

    def to_dict(self) -> dict:
        return asdict(self)


def partition(num_models: int, processes: int) -> list[list[int]]:
    """Model ids per process: contiguous, sizes differing by at most one
    (the hybrid baseline's "(Ap, Bm)" split)."""
    if num_models < 1:
        raise ValueError("num_models must be >= 1")
    if not 1 <= processes <= num_models:
        raise ValueError(f"processes must be in [1, {num_models}], got {processes}")
    base, extra = divmod(num_models, processes)
    out, start = [], 0
    for p in range(processes):
        n = base + (1 if p < extra else 0)
        out.append(list(range(start, start + n)))
        start += n
    return out


def resolve(strategy: str, num_models: int, processes: int | None = None) -> tuple[str, int]:
    """(strategy name, process count) for a strategy spec: ``sequential``,
    ``concurrent``, ``merged``, ``hybrid`` (needs ``processes``) or
    ``hybrid:P``."""
    name, _, arg = strategy.partition(":")
    if name not in STRATEGIES:
        raise ValueError(f"unknown strategy {strategy!r}; choose from {STRATEGIES}")
    if name == "hybrid":
        p = int(arg) if arg else processes
        if p is None:
            raise ValueError("hybrid needs a process count (hybrid:P)")
        if not 1 <= p <= num_models:
            raise ValueError(f"hybrid processes must be in [1, {num_models}], got {p}")
        return name, p
    if arg:
        raise ValueError(f"strategy {name!r} takes no argument")
    return name, (num_models if name == "concurrent" else 1)


# ----------------------------------------------------------------------------
# worker side
# ----------------------------------------------------------------------------

def _build_round(model: str, ids: list[int], batch: int, dtype: str, total: int,
                 heads: bool, merged: bool):
    """Plans for this worker's models captured into one CUDA graph; returns
    (graph, kernel launches per replay, keep-alive objects)."""
    import torch

    from . import workloads as W
    from .engine import compile_plan

    if merged:
        _, _, inputs, mg, mstore, _ = W.merged_workload(model, len(ids), batch, dtype, ids[0],
                                                        heads)
        plan = compile_plan(mg.graph, mstore, mode="fast")
        plan.load_inputs(mg.bind_inputs(inputs))
        torch.cuda.synchronize()
        return plan.capture(), plan.kernel_launches, [plan]
    plans = []
    for m in ids:
        g, st, x, head = W.instance_workload(model, m, batch, dtype, heads, total)
        p = compile_plan(g, st, mode="fast")
        p.load_inputs(x)
        hp = compile_plan(head[0], head[1], mode="fast") if head else None
        plans.append((p, hp))

    def one_round():
        for p, hp in plans:
            p.launch()
            if hp is not None:
                hp.input_views["feat"].copy_(p.outputs()[0])
                hp.launch()

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        one_round()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    cg = torch.cuda.CUDAGraph()
    with torch.cuda.graph(cg):
        one_round()
    launches = sum(p.kernel_launches + (hp.kernel_launches + 1 if hp else 0) for p, hp in plans)
    return cg, launches, plans


def _worker(rank: int, model: str, ids: list[int], batch: int, dtype: str, total: int,
            heads: bool, merged: bool, rounds: int, warmup: int, barrier, queue) -> None:
    res = {"rank": rank}
    try:
        import torch
        torch.cuda.set_device(0)
        cg, launches, keep = _build_round(model, ids, batch, dtype, total, heads, merged)
        for _ in range(warmup):
            cg.replay()
        torch.cuda.synchronize()
        res["launches"] = launches
        barrier.wait()
        t0 = time.perf_counter()
        for _ in range(rounds):
            cg.replay()
            torch.cuda.synchronize()
        t1 = time.perf_counter()
        res.update(t0=t0, t1=t1, allocated=torch.cuda.max_memory_allocated(),
                   reserved=torch.cuda.max_memory_reserved())
        barrier.wait()  # stay resident until every worker is done (memory sampling)
        del cg, keep
    except BaseException as e:  # reported to the parent, which raises
        res["error"] = f"{type(e).__name__}: {e}"
        try:
            barrier.abort()
        except Exception:
            pass
    queue.put(res)


# ----------------------------------------------------------------------------
# parent side
# ----------------------------------------------------------------------------

class _MemSampler:
    """Device used-memory (NVML) sampled from a thread: baseline at start,
    peak while running."""

    def __init__(self, index: int = 0, period_s: float = 0.02):
        self.index, self.period = index, period_s
        self.baseline = self.peak = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self._nv = pynvml
            self.baseline = self.peak = pynvml.nvmlDeviceGetMemoryInfo(self._h).used

            def poll():
                while not self._stop.is_set():
                    self.peak = max(self.peak, self._nv.nvmlDeviceGetMemoryInfo(self._h).used)
                    time.sleep(self.period)

            self._t = threading.Thread(target=poll, daemon=True)
            self._t.start()
        except Exception:
            self._t = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=1.0)

    def used_above_baseline(self) -> int | None:
        if self.baseline is None or self.peak is None:
            return None
        return int(self.peak - self.baseline)


def run_serving(model: str, strategy: str, num_models: int, *, batch: int = 1,
                dtype: str = "bf16", processes: int | None = None, rounds: int = 20,
                warmup: int = 3, heads: bool = True, timeout_s: float = 1800.0) -> ServingReport:
    """Serve ``num_models`` instances of ``model`` with ``strategy`` and
    report throughput and peak device memory (see the module docstring)."""
    name, nproc = resolve(strategy, num_models, processes)
    if rounds < 1 or warmup < 0:
        raise ValueError("rounds must be >= 1 and warmup >= 0")
    parts = partition(num_models, nproc)
    rep = ServingReport(strategy=name if name != "hybrid" else f"hybrid:{nproc}", model=model,
                        num_models=num_models, batch=batch, dtype=dtype, processes=nproc,
                        models_per_process=[len(p) for p in parts], rounds=rounds)
    ctx = mp.get_context("spawn")
    barrier = ctx.Barrier(nproc)
    queue = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, model, ids, batch, dtype, num_models, heads,
                                               name == "merged", rounds, warmup, barrier, queue),
                         daemon=True)
             for r, ids in enumerate(parts)]
    results = []
    with _MemSampler() as mem:
        for p in procs:
            p.start()
        deadline = time.monotonic() + timeout_s
        while len(results) < nproc and time.monotonic() < deadline:
            try:
                results.append(queue.get(timeout=5.0))
            except Exception:
                if not any(p.is_alive() for p in procs) and queue.empty():
                    break
        for p in procs:
            p.join(timeout=30.0)
            if p.is_alive():
                p.kill()
    errors = [r["error"] for r in results if "error" in r]
    if errors or len(results) < nproc:
        rep.error = errors[0] if errors else f"{nproc - len(results)} worker(s) never reported"
        return rep
    t0 = min(r["t0"] for r in results)
    t1 = max(r["t1"] for r in results)
    rep.wall_s = t1 - t0
    rep.inferences_per_s = num_models * batch * rounds / rep.wall_s
    rep.ms_per_round = rep.wall_s / rounds * 1e3
    rep.peak_device_bytes = mem.used_above_baseline()
    results.sort(key=lambda r: r["rank"])
    rep.worker_allocated_bytes = [int(r["allocated"]) for r in results]
    rep.worker_reserved_bytes = [int(r["reserved"]) for r in results]
    rep.kernel_launches_per_round = sum(r["launches"] for r in results)
    return rep


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__,
                                 formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--model", default="bert-base")
    ap.add_argument("--num-models", type=int, default=32)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--strategies", default="sequential,concurrent,hybrid:4,merged")
    ap.add_argument("--rounds", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--no-heads", action="store_true")
    args = ap.parse_args(argv)
    reports = []
    for s in args.strategies.split(","):
        r = run_serving(args.model, s.strip(), args.num_models, batch=args.batch,
                        dtype=args.dtype, rounds=args.rounds, warmup=args.warmup,
                        heads=not args.no_heads)
        reports.append(r)
        print(json.dumps(r.to_dict()), flush=True)
    merged = next((r for r in reports if r.strategy == "merged" and not r.error), None)
    if merged:
        print(json.dumps({"merged_speedup": {r.strategy: round(merged.inferences_per_s /
                                                              r.inferences_per_s, 3)
                                             for r in reports if not r.error and r is not merged}}))
    return 0


if __name__ == "__main__":
    os.environ.setdefault("PYTHONUNBUFFERED", "1")
    raise SystemExit(main())
