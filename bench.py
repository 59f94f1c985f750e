"""Benchmark: merged inferences/s of N same-architecture instances in one
forward (BASELINE.json metric), on B200.

Workload (default): BASELINE configs[1] — BERT-base merged N=8 instances,
batch 1, seq 128, bf16, each instance with its own random-init weights and
per-task classifier head (unmerged, merge_backbone), synthetic embeddings.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

Multi-GPU = instance sharding: every rank hosts its own
`--instances` merged instances (weak scaling), no collective on the hot path;
the step time is the max over ranks.

`value`: device-timed CUDA-graph replays of the merged forward with inputs
resident in HBM; the L2 is flushed (256 MiB write) between steps, outside the
timed events. `e2e`: the same through the public plan API with host buffers —
H2D of every instance's input from pinned memory, forward, D2H of the logits
— each step. `--impl reference` times the reference CPU algorithm (the
oracle's numpy restatement of pkg/src/modelmerge/engine.py) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "merged inferences/sec (N instances x batch); speedup vs N separate runs"
UNIT = "inferences/s"


def _peaks() -> tuple[dict, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text()), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region: NVML
    polled every ~2 ms from a thread (a 50-step batch-1 region lasts only
    tens of ms), nvidia-smi -lms 100 when NVML is unavailable."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []
        self._stop = threading.Event()
        self._t = None

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            pr = torch.cuda.get_device_properties(self.index)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def __enter__(self):
        try:
            nv, h = self._nvml_handle()
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            bits = (nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap)
            first = threading.Event()

            def poll():
                while not self._stop.is_set():
                    sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    flags = ["Active" if r & b else "Not Active" for b in bits]
                    self.lines.append(", ".join([str(sm), str(mx), hex(r)] + flags))
                    first.set()
                    time.sleep(0.002)

            self._t = threading.Thread(target=poll, daemon=True)
            self._t.start()
            first.wait(1.0)  # the first sample precedes the timed region
            return self
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        self._stop.set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        elif self._t is not None:
            self._t.join(timeout=1.0)

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for name, val in zip(names, f[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# Workload construction
# ---------------------------------------------------------------------------

def build_workload(model: str, instances: int, batch: int, dtype: str, first_instance: int,
                   heads: bool = True):
    """The merged workload (shared with tests/test_gpu_configs.py)."""
    from paper_2009_13062_b200 import workloads as W
    return W.merged_workload(model, instances, batch, dtype, first_instance, heads)


def linear_launch_bytes(merged, mstore, step_ids=None) -> dict[str, tuple[int, int]]:
    """Algorithmic (bytes, flops) per weight-streaming launch of the merged
    plan: merged Linear (weights + inputs + outputs, each touched once; SURVEY
    §8d per-kernel operands), the fused QKV+attention launch (keyed by the
    attention node when the plan fused the pair) and merged convs (weights +
    input + output activations)."""
    from paper_2009_13062_b200 import OpKind
    from paper_2009_13062_b200.ir import parse_ref

    specs = dict(merged.graph.graph_inputs)
    specs.update({n.id: n.output_spec for n in merged.graph.nodes})
    users: dict[str, list] = {}
    for n in merged.graph.nodes:
        for r in n.inputs:
            users.setdefault(parse_ref(r)[0], []).append(n)
    out = {}
    for n in merged.graph.nodes:
        if n.kind in (OpKind.BATCH_MATMUL, OpKind.MATMUL):
            w = mstore[n.weights[0]].spec
            x = specs[parse_ref(n.inputs[0])[0]]
            esz = 2 if x.dtype == "bf16" else 4
            k_in = x.dims[-1]
            rows = math.prod(x.dims[:-1])
            n_out = w.dims[-1]
            b = (math.prod(w.dims) + rows * k_in + rows * n_out) * esz
            out[n.id] = (b, 2 * rows * k_in * n_out)
            us = users.get(n.id, [])
            if (step_ids is not None and n.id not in step_ids and len(us) == 1
                    and us[0].kind is OpKind.ATTENTION and us[0].id in step_ids):
                # fused QKV+attention launch: the projection's weights and input
                # plus the context output (QKV itself never reaches HBM)
                ctx = math.prod(us[0].output_spec.dims) * esz
                out[us[0].id] = (b - rows * n_out * esz + ctx, 2 * rows * k_in * n_out)
        elif n.kind in (OpKind.CONV2D, OpKind.GROUPED_CONV2D):
            w = mstore[n.weights[0]].spec
            x = specs[parse_ref(n.inputs[0])[0]]
            esz = 2 if x.dtype == "bf16" else 4
            y = n.output_spec
            pix = y.dims[0] * y.dims[2] * y.dims[3]
            b = (math.prod(w.dims) + math.prod(x.dims) + math.prod(y.dims)) * esz
            out[n.id] = (b, 2 * pix * math.prod(w.dims))
    return out


# ---------------------------------------------------------------------------
# Our arm
# ---------------------------------------------------------------------------

def run_ours(args) -> dict | None:
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)

    from paper_2009_13062_b200 import PipelinedRunner, compile_plan

    from paper_2009_13062_b200.sharding import shard_range
    shard = shard_range(args.instances * world, world, rank)  # weak scaling: N per GPU
    graph, stores, inputs, merged, mstore, heads = build_workload(
        args.model, len(shard), args.batch, args.dtype, shard.start, heads=not args.no_heads)
    plan = compile_plan(merged.graph, mstore, mode="fast")
    bound = merged.bind_inputs(inputs)
    plan.load_inputs(bound)
    torch.cuda.synchronize()
    graph_exec = plan.capture()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    def step_timed(n: int) -> list[float]:
        evs = []
        for _ in range(n):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            graph_exec.replay()
            e.record(stream)
            evs.append((s, e))
        torch.cuda.synchronize()
        return [s.elapsed_time(e) for s, e in evs]

    step_timed(args.warmup)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        times_ms = step_timed(args.steps)
    total_ms = sum(times_ms)
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    per_step_items = args.instances * args.batch * world
    value = per_step_items / (ms_per_step / 1e3)

    # ---- e2e through the public API with host buffers --------------------
    pinned = {k: v.data.pin_memory() for k, v in bound.items()}
    h2d = sum(t.numel() * t.element_size() for t in pinned.values())

    # serving loop of the public API: each step's H2D copy (pinned host ->
    # device staging) overlaps the previous step's forward; the logits come
    # back with one D2H copy per output buffer
    runner = PipelinedRunner(plan)
    outs_host = runner.alloc_host_outputs(1)[0]
    d2h = runner.d2h_bytes(outs_host)

    def e2e_steps(n: int) -> float:
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        runner.run([pinned] * n, outs_host)
        e.record(stream)
        torch.cuda.synchronize()
        return s.elapsed_time(e)

    e2e_steps(args.warmup)
    if world > 1:
        dist.barrier()
    e2e_ms = e2e_steps(args.steps)
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = per_step_items / (e2e_ms / args.steps / 1e3)

    # ---- dominant kernel roofline (merged Linear), CUDA events per launch --
    lin = linear_launch_bytes(merged, mstore, {nid for nid, _, _ in plan.steps})
    events: list = []
    for _ in range(2):
        events = []
        plan.launch(events=events)
    torch.cuda.synchronize()
    is_cnn = "res" in args.model
    lin_ms, lin_bytes, lin_flops, lin_n, all_ms = 0.0, 0, 0, 0, 0.0
    for i, (nid, _, _) in enumerate(plan.steps):
        ms = events[i].elapsed_time(events[i + 1])
        all_ms += ms
        if nid in lin:
            lin_ms += ms
            lin_bytes += lin[nid][0]
            lin_flops += lin[nid][1]
            lin_n += 1
    peaks, peak_src = _peaks()
    achieved = lin_bytes / (lin_ms / 1e3) / 1e9
    traffic = None
    tfile = ROOT / "profiles" / "gemm_traffic.json"
    if tfile.exists():
        traffic = json.loads(tfile.read_text()).get(f"{args.model}/N{args.instances}/B{args.batch}")

    unmerged = None if args.no_unmerged else unmerged_legs(
        args, graph, stores, inputs, heads, flush, stream, value)

    if world > 1:
        dist.barrier()
    if rank != 0:
        dist.destroy_process_group()
        return None
    cpu = cpu_baseline(args, graph, stores, inputs, heads) if world == 1 and not args.no_cpu \
        else None
    # Bound of the dominant kernel family: HBM when its arithmetic intensity is
    # under the measured ridge (bf16 peak / copy bandwidth), tensor otherwise.
    ridge = peaks["bf16_tflops"] * 1e12 / (peaks["hbm_gbs"] * 1e9)
    tensor_bound = lin_bytes > 0 and lin_flops / lin_bytes > ridge
    tflops = lin_flops / (lin_ms / 1e3) / 1e12 if lin_ms else 0.0
    roofline = {
        "bound": "tensor" if tensor_bound else "hbm",
        "kernel": ("k_grouped_gemm_tc (merged Linear) + k_qkv_attention_tc" if not is_cnn else
                   "k_grouped_gemm_tc (implicit-GEMM merged conv + Linear)"),
        "achieved": round(tflops if tensor_bound else achieved, 1),
        "peak": peaks["bf16_tflops"] if tensor_bound else peaks["hbm_gbs"],
        "unit": "TFLOP/s" if tensor_bound else "GB/s",
        "frac": round((tflops / peaks["bf16_tflops"]) if tensor_bound
                      else (achieved / peaks["hbm_gbs"]), 4),
        "traffic": traffic,
        "peak_source": peak_src,
        "launches_per_step": lin_n,
        "algorithmic_bytes_per_step": lin_bytes,
        "algorithmic_flops_per_step": lin_flops,
        "hbm_gbs_achieved": round(achieved, 1),
        "tflops_achieved": round(tflops, 1),
        "share_of_step": round(lin_ms / all_ms, 4) if all_ms else None,
    }
    if world > 1:
        dist.destroy_process_group()
    return {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": args.dtype,
        "data": "synthetic (seeded U[-1,1] embeddings; fan-in-scaled random-init weights)",
        "config": {
            "workload": f"{args.model} merged N={args.instances} B={args.batch} per GPU"
                        + ("" if args.no_heads else " + per-task classifier heads"),
            "model": args.model,
            "instances_per_gpu": args.instances,
            "global_instances": args.instances * world,
            "global_batch": args.instances * args.batch * world,
            "batch": args.batch,
            "seq_len": 128 if "bert" in args.model or "xlnet" in args.model else None,
            "image": 224 if "res" in args.model else None,
            "parallelism": f"instance-shard x{world} (no collective on the hot path)",
            "l2": "flushed between timed steps (256 MiB write outside the events)",
            "timing": "CUDA events around each CUDA-graph replay; max over ranks",
        },
        "e2e": {"value": round(e2e_value, 2), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "roofline": roofline,
        "unmerged": unmerged,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "gpu_launches": plan.kernel_launches * args.steps,
    }


def _time_steps(fn, n: int, flush, stream) -> float:
    """Mean device ms of ``fn`` over ``n`` L2-flushed steps (CUDA events)."""
    import torch
    evs = []
    for _ in range(n):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        fn()
        e.record(stream)
        evs.append((s, e))
    torch.cuda.synchronize()
    return sum(s.elapsed_time(e) for s, e in evs) / n


def unmerged_legs(args, graph, stores, inputs, heads, flush, stream, merged_value) -> dict:
    """The metric's denominator: the same N instances run as N separate
    (unmerged) forwards, sequentially in one stream on this GPU (SURVEY §8d,
    PAPER.md:394-399 "sequential" baseline):
      * ours_sequential: this framework's kernels at M=1, N per-instance plans
        (backbone + head) recorded into one CUDA graph;
      * ours_concurrent: the same N plans on N streams of one graph (the
        paper's concurrent baseline);
      * torch_eager_sequential: stock PyTorch ops (cuBLAS / cuDNN / SDPA),
        eager, one instance after another;
      * torch_graph_sequential: the same PyTorch ops captured in a CUDA graph
        (no launch overhead: the strongest unmerged baseline)."""
    import torch

    from baselines.torch_eager import TorchModel
    from paper_2009_13062_b200 import compile_plan

    n_inst = len(stores)
    items = n_inst * args.batch
    steps = max(3, min(args.steps, 20))
    out: dict = {"instances": n_inst, "steps": steps}

    plans = []
    for m in range(n_inst):
        p = compile_plan(graph, stores[m], mode="fast")
        p.load_inputs(inputs[m])
        hp = compile_plan(heads[m][0], heads[m][1], mode="fast") if heads else None
        plans.append((p, hp))

    def ours_all():
        for p, hp in plans:
            p.launch()
            if hp is not None:
                hp.input_views["feat"].copy_(p.outputs()[0])
                hp.launch()

    ours_all()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ours_all()
    _time_steps(g.replay, 3, flush, stream)
    ms = _time_steps(g.replay, steps, flush, stream)
    out["ours_sequential"] = {"value": round(items / (ms / 1e3), 2), "ms_per_step": round(ms, 4),
                              "kernel_launches": sum(p.kernel_launches +
                                                     (hp.kernel_launches if hp else 0)
                                                     for p, hp in plans)}
    del g

    # the paper's "concurrent" baseline: the N separate
    # forwards on N streams of one CUDA graph, free to overlap on the GPU
    streams = [torch.cuda.Stream() for _ in plans]

    def ours_concurrent():
        cur = torch.cuda.current_stream()
        for s_ in streams:
            s_.wait_stream(cur)
        for (p, hp), s_ in zip(plans, streams):
            with torch.cuda.stream(s_):
                p.launch()
                if hp is not None:
                    hp.input_views["feat"].copy_(p.outputs()[0])
                    hp.launch()
        for s_ in streams:
            cur.wait_stream(s_)

    ours_concurrent()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ours_concurrent()
    _time_steps(g.replay, 3, flush, stream)
    ms = _time_steps(g.replay, steps, flush, stream)
    out["ours_concurrent"] = {"value": round(items / (ms / 1e3), 2), "ms_per_step": round(ms, 4),
                              "streams": len(streams)}
    del g, plans

    models = []
    for m in range(n_inst):
        tm = TorchModel(graph, stores[m])
        tm.load(inputs[m])
        hm = TorchModel(heads[m][0], heads[m][1]) if heads else None
        models.append((tm, hm))

    @torch.inference_mode()
    def torch_all():
        res = []
        for tm, hm in models:
            y = tm.forward()[0]
            if hm is not None:
                hm.inputs["feat"].copy_(y)
                y = hm.forward()[0]
            res.append(y)
        return res

    torch_all()
    _time_steps(torch_all, 3, flush, stream)
    ms = _time_steps(torch_all, steps, flush, stream)
    out["torch_eager_sequential"] = {"value": round(items / (ms / 1e3), 2),
                                     "ms_per_step": round(ms, 4)}
    s2 = torch.cuda.Stream()
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s2):
        torch_all()
    torch.cuda.current_stream().wait_stream(s2)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        torch_all()
    _time_steps(g.replay, 3, flush, stream)
    ms = _time_steps(g.replay, steps, flush, stream)
    out["torch_graph_sequential"] = {"value": round(items / (ms / 1e3), 2),
                                     "ms_per_step": round(ms, 4)}
    del g, models
    out["speedup"] = {k: round(merged_value / out[k]["value"], 3)
                      for k in ("ours_sequential", "ours_concurrent", "torch_eager_sequential",
                                "torch_graph_sequential")}
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------------
# Reference CPU path (oracle restatement of the reference numpy kernels)
# ---------------------------------------------------------------------------

def _layer_graph(model: str, batch: int, dtype: str):
    from paper_2009_13062_b200 import workloads as W
    return W.build_graph("bert-2l" if model.startswith("bert") else model, batch=batch,
                         dtype=dtype)


def reference_sample(args, instances: list[int], threads: int) -> tuple[float, str]:
    """Run the reference algorithm on a bounded sample and return the
    extrapolated whole-workload inferences/s plus a description."""
    from oracle import executor as OX
    from paper_2009_13062_b200 import model_inputs
    from paper_2009_13062_b200 import workloads as W

    sample_layers = 1
    g2 = _layer_graph(args.model, args.batch, args.dtype)
    one = W.BertConfig(layers=sample_layers)
    g1, _ = W._bert(args.batch, args.dtype, one)
    jobs = []
    for m in instances:
        st = W.build_weights("bert-2l", dtype=args.dtype, seed=0, model=m)
        x = model_inputs(g2, seed=0, model=m)
        jobs.append((st, x))

    def run(job):
        st, x = job
        return OX.execute(g1, st.tensors, x)

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(run, jobs))
    dt = time.perf_counter() - t0
    layers = W.BERT_BASE.layers
    per_instance_s = dt * layers / sample_layers / len(jobs)
    value = args.batch / per_instance_s
    desc = (f"{len(jobs)} instance(s) x {sample_layers} of {layers} encoder layers, "
            f"{threads} thread(s); extrapolated x{layers // sample_layers} layers "
            f"(slices independent, PAPER.md:620-670); heads excluded")
    return value, desc


def cpu_baseline(args, graph, stores, inputs, heads) -> dict:
    """One complete instance forward (all layers + its head) of the reference
    algorithm on one host core: no extrapolation over layers."""
    from oracle import executor as OX
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    feat = OX.execute(graph, stores[0].tensors, inputs[0])[0]
    if heads:
        OX.execute(heads[0][0], heads[0][1].tensors, {"feat": feat})
    dt = time.perf_counter() - t0
    return {"value": round(args.batch / dt, 5), "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"1 full instance forward ({args.model}, B={args.batch}, + head) of the "
                      f"numpy restatement of the reference kernels, {dt:.1f} s on 1 of "
                      f"{cores} host cores"}


def run_reference(args) -> dict | None:
    world, rank, _ = dist_env()
    if rank != 0:
        return None
    threads = min(args.instances, os.cpu_count() or 1)
    inst = list(range(min(args.instances, threads)))
    vals = []
    for _ in range(args.warmup):
        reference_sample(args, inst, threads)
    for _ in range(args.steps):
        v, desc = reference_sample(args, inst, threads)
        vals.append(v)
    value = statistics.mean(vals)
    ms_per_step = args.instances * args.batch / value * 1e3
    return {
        "impl": "reference",
        "metric": METRIC,
        "value": round(value, 4),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 2),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": args.dtype,
        "data": "synthetic (same seeds as our arm)",
        "config": {"workload": f"{args.model} N={args.instances} B={args.batch} S=128",
                   "model": args.model, "instances_per_gpu": args.instances,
                   "batch": args.batch, "seq_len": 128,
                   "parallelism": "host threads (reference `threaded` strategy, bench.py:112-121)"},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads,
                         "kind": "port", "sample": desc},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawTextHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--model", default="bert-base")
    ap.add_argument("--instances", type=int, default=8, help="merged instances per GPU")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--no-heads", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    ap.add_argument("--no-unmerged", action="store_true",
                    help="skip the N-separate-runs legs (speedup denominator)")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        res = run_reference(args)
    else:
        res = run_ours(args)
    if res is not None:
        print(json.dumps(res), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
