"""Benchmark: merged inferences/s of N same-architecture instances in one
forward (BASELINE.json metric: "merged inferences/sec (N instances x batch) at
N=32; speedup vs N separate runs"), on B200.

Workload (default, BASELINE configs[4] per GPU): BERT-base, 32 merged
instances per GPU, batch 8, seq 128, bf16, each instance with its own
random-init weights and per-task classifier head (unmerged, merge_backbone),
synthetic embeddings. `--gpus 8` under torchrun is config C5 itself (N=256
sharded 32 per GPU). `--config C1..C5` selects another BASELINE config.

    python bench.py [--config C5] [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N [--scaling weak|strong] ...

Multi-GPU = instance sharding: weak scaling (default) gives every
rank `--instances` merged instances; `--scaling strong` splits `--instances`
(e.g. 256) over the ranks. No collective on the hot path; the step time is the
max over ranks; one all_gather of the per-instance logits after the timed
region is timed and reported separately (`gather`).

`value`: device-timed CUDA-graph replays of the merged forward with inputs
resident in HBM; the L2 is flushed (256 MiB write) between steps, outside the
timed events. `e2e`: the same through the public serving API with host
buffers (PipelinedRunner: H2D of every instance's input from pinned memory,
forward, D2H of the logits) each step. `roofline`: the dominant kernel family
(merged Linear / implicit-GEMM conv launches) — its share of a forward from
per-launch CUDA events in an instrumented graph replay, times the real
replay's ms_per_step, against its algorithmic bytes / flops. `--impl reference`
times the reference CPU algorithm (the oracle's numpy restatement of
pkg/src/modelmerge/engine.py) on the host cores, on a bounded sample of the
same workload.
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
    # chained launches (engine._ChainStep, id "chain:a+b+c"): their members' sum
    for sid in step_ids or ():
        if sid.startswith("chain:"):
            mem = sid[len("chain:"):].split("+")
            if all(m in out for m in mem):
                out[sid] = (sum(out[m][0] for m in mem), sum(out[m][1] for m in mem))
    return out


# ---------------------------------------------------------------------------
# Our arm
# ---------------------------------------------------------------------------

def shard_for(args, world: int, rank: int) -> range:
    """This rank's instance ids: weak scaling = `--instances` per rank;
    strong scaling = `--instances` in total, split over the ranks."""
    from paper_2009_13062_b200.sharding import shard_range
    total = args.instances * world if args.scaling == "weak" else args.instances
    return shard_range(total, world, rank)


def family_roofline(plan, lin: dict, ms_per_step: float, peaks: dict, reps: int = 5) -> dict:
    """Dominant-kernel roofline from a live, instrumented CUDA-graph replay:
    every launch of the plan bracketed by (external) CUDA events recorded
    into the graph on the launching stream, replayed `reps` times. The
    family's SHARE of the summed per-launch times is applied to the real
    (PDL-overlapped) replay's ms_per_step, so the family time can never
    exceed the step; achieved = algorithmic bytes (flops) / that time."""
    import torch

    steps = plan.steps
    dev = plan.device
    evs = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(len(steps) + 1)]
    s = torch.cuda.Stream(device=dev)
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        plan.launch()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        st = torch.cuda.current_stream()
        for i, (_, fn, _) in enumerate(steps):
            evs[i].record(st)
            fn(st.cuda_stream)
        evs[-1].record(st)
    per = [0.0] * len(steps)
    for _ in range(reps):
        g.replay()
        torch.cuda.synchronize(dev)
        for i in range(len(steps)):
            per[i] += evs[i].elapsed_time(evs[i + 1]) / reps
    del g
    all_ms = sum(per)
    fam_ms_inst, fam_bytes, fam_flops, fam_n = 0.0, 0, 0, 0
    for i, (nid, _, _) in enumerate(steps):
        if nid in lin:
            fam_ms_inst += per[i]
            fam_bytes += lin[nid][0]
            fam_flops += lin[nid][1]
            fam_n += 1
    share = fam_ms_inst / all_ms if all_ms else 0.0
    fam_ms = share * ms_per_step
    assert fam_ms <= ms_per_step + 1e-9
    # bound: HBM when the family's arithmetic intensity is under the measured
    # ridge (sustained bf16 peak / copy bandwidth), tensor otherwise. The
    # family is timed inside a long step (back-to-back forwards under the
    # power cap), so its tensor denominator is the SUSTAINED cuBLAS figure
    # (B200_PROFILING.md: burst for a kernel timed alone, sustained for one
    # timed inside a long step); the burst fraction is reported beside it.
    sus = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    ridge = sus * 1e12 / (peaks["hbm_gbs"] * 1e9)
    tensor_bound = fam_bytes > 0 and fam_flops / fam_bytes > ridge
    gbs = fam_bytes / (fam_ms / 1e3) / 1e9 if fam_ms else 0.0
    tflops = fam_flops / (fam_ms / 1e3) / 1e12 if fam_ms else 0.0
    return {
        "bound": "tensor" if tensor_bound else "hbm",
        "achieved": round(tflops if tensor_bound else gbs, 1),
        "peak": sus if tensor_bound else peaks["hbm_gbs"],
        "peak_kind": ("bf16 sustained (kernel family timed inside a long step)" if tensor_bound
                      else "HBM copy bandwidth"),
        "unit": "TFLOP/s" if tensor_bound else "GB/s",
        "frac": round((tflops / sus) if tensor_bound else (gbs / peaks["hbm_gbs"]), 4),
        "frac_of_burst_peak": round(tflops / peaks["bf16_tflops"], 4) if tensor_bound else None,
        "launches_per_step": fam_n,
        "share_of_step": round(share, 4),
        "family_ms_per_step": round(fam_ms, 4),
        "instrumented_ms_per_step": round(all_ms, 4),
        "algorithmic_bytes_per_step": fam_bytes,
        "algorithmic_flops_per_step": fam_flops,
        "algorithmic_bytes_per_launch": fam_bytes // max(fam_n, 1),
        "hbm_gbs_achieved": round(gbs, 1),
        "tflops_achieved": round(tflops, 1),
    }


def run_ours(args) -> dict | None:
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    # one rank per GPU; --dist-backend gloo lets several ranks share a GPU
    # (a functional check of the multi-rank path on a one-GPU box)
    dev = torch.device("cuda", local % max(torch.cuda.device_count(), 1) if world > 1 else 0)
    torch.cuda.set_device(dev)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    from paper_2009_13062_b200 import PipelinedRunner, compile_plan

    shard = shard_for(args, world, rank)
    total_instances = args.instances * world if args.scaling == "weak" else args.instances
    graph, stores, inputs, merged, mstore, heads = build_workload(
        args.model, len(shard), args.batch, args.dtype, shard.start, heads=not args.no_heads)
    torch.cuda.reset_peak_memory_stats(dev)
    plan = compile_plan(merged.graph, mstore, mode="fast")
    bound = merged.bind_inputs(inputs)
    plan.load_inputs(bound)
    torch.cuda.synchronize()
    graph_exec = plan.capture()
    graph_exec.replay()
    torch.cuda.synchronize()
    plan_peak = torch.cuda.max_memory_allocated(dev)
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
    per_step_items = total_instances * args.batch
    value = per_step_items / (ms_per_step / 1e3)

    # ---- end-of-run gather of every instance's logits (not on the hot path)
    gather = None
    if world > 1:
        logits = _per_instance_logits(plan, merged)
        dist.barrier()
        ge0, ge1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ge0.record(stream)
        from paper_2009_13062_b200.sharding import gather_instance_outputs
        got = gather_instance_outputs(logits, total_instances)
        ge1.record(stream)
        torch.cuda.synchronize()
        gms = ge0.elapsed_time(ge1)
        t = torch.tensor([gms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        gather = {"collective": f"all_gather ({args.dist_backend}) of per-instance logits, "
                                "after timing",
                  "ms": round(float(t.item()), 4),
                  "bytes_per_rank": sum(x.numel() * x.element_size() for x in logits),
                  "instances_gathered": len(got) if got is not None else None}

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

    # ---- dominant kernel family roofline (live, instrumented replay) ------
    peaks, peak_src = _peaks()
    lin = linear_launch_bytes(merged, mstore, {nid for nid, _, _ in plan.steps})
    roofline = family_roofline(plan, lin, ms_per_step, peaks)
    is_cnn = "res" in args.model
    chained = any(nid.startswith("chain:") for nid, _, _ in plan.steps)
    roofline["kernel"] = (
        ("k_conv_tf32x3 (3xTF32 merged conv) + fp32 heads" if args.dtype == "f32" else
         "k_grouped_gemm_tc (implicit-GEMM merged conv + Linear)") if is_cnn
        else "k_linear_chain_tc (chained merged Linears) + k_qkv_attention_tc" if chained
        else "k_grouped_gemm_tc (merged Linear) + k_qkv_attention_tc")
    roofline["peak_source"] = peak_src
    roofline["traffic"] = _ncu_traffic(args)
    roofline["ncu_share"] = _ncu_share(args)

    unmerged = None if (args.no_unmerged or world > 1) else unmerged_legs(
        args, graph, stores, inputs, heads, flush, stream, value)

    if world > 1:
        dist.barrier()
    if rank != 0:
        dist.destroy_process_group()
        return None
    cpu = cpu_baseline(args) if world == 1 and not args.no_cpu else None
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
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": args.dtype,
        "data": "synthetic (seeded U[-1,1] embeddings / images; fan-in-scaled random-init "
                "weights)",
        "config": {
            "workload": f"{args.model} merged N={len(shard)} B={args.batch} per GPU"
                        + (f" ({total_instances} instances on {world} GPUs)" if world > 1 else "")
                        + ("" if args.no_heads else " + per-task heads"),
            "baseline_config": args.config,
            "model": args.model,
            "instances_per_gpu": len(shard),
            "global_instances": total_instances,
            "global_batch": per_step_items,
            "batch": args.batch,
            "seq_len": 128 if "bert" in args.model or "xlnet" in args.model else None,
            "image": 224 if "res" in args.model else None,
            "parallelism": f"instance-shard x{world} (no collective on the hot path)"
                           + (f", {args.dist_backend}" if world > 1 else ""),
            "l2": "flushed between timed steps (256 MiB write outside the events)",
            "timing": "CUDA events around each CUDA-graph replay; max over ranks",
        },
        "e2e": {"value": round(e2e_value, 2), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "roofline": roofline,
        "gather": gather,
        "memory": {"peak_hbm_allocated_bytes": plan_peak,
                   "merged_weights_bytes": mstore.total_bytes()},
        "unmerged": unmerged,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "gpu_launches": plan.kernel_launches * args.steps,
    }


def _per_instance_logits(plan, merged) -> list:
    """Per-instance head outputs of this rank's plan as same-shape tensors
    (the heads' widths differ per task: padded to the widest)."""
    import torch
    flat = [g[0] for g in merged.slice_outputs(list(plan.outputs()))]
    width = max(t.shape[-1] for t in flat)
    return [torch.nn.functional.pad(t, (0, width - t.shape[-1])).contiguous() for t in flat]


def _profiles_json(name: str):
    f = ROOT / "profiles" / name
    return json.loads(f.read_text()) if f.exists() else {}


def _workload_key(args) -> str:
    return f"{args.model}/N{args.instances}/B{args.batch}/{args.dtype}"


def _ncu_traffic(args):
    """DRAM bytes per dominant-family launch from the committed ncu --set full
    capture of this workload (profiles/r02_ncu_traffic.json), or None."""
    got = _profiles_json("r02_ncu_traffic.json").get(_workload_key(args)) or {}
    return got.get("dram_bytes_per_family_launch")


def _ncu_share(args):
    """The dominant family's share of a forward in the committed ncu launch
    list of this workload (serialised, cold cache: shares compare, absolute
    times do not), or None."""
    got = _profiles_json("r02_ncu_share.json").get(_workload_key(args)) or {}
    return got.get("family_share")


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

class ReferenceSampler:
    """Bounded samples of the reference CPU algorithm on this config: the
    oracle's numpy restatement of pkg/src/modelmerge/engine.py (bit-identical
    to it on every golden vector), one instance per host thread (the
    reference's `threaded` strategy, bench.py:102-121).

    One job = the work of one instance that is independent of everything
    else (sequences and layers are independent units of
    work for the clock): transformers run ONE encoder layer of ONE sequence
    (1/L of an inference, L = 12); CNNs run one full forward of the instance's
    batch plus its FC head. Throughput = inference-equivalents completed / the
    measured wall time of the sample: nothing is extrapolated beyond the
    sample's own work and the reported time is the time the sample took."""

    def __init__(self, args, instances: list[int]):
        from paper_2009_13062_b200 import model_inputs
        from paper_2009_13062_b200 import workloads as W

        self.model = args.model
        one = W.one_layer_model(args.model)
        self.layers = W.layer_count(args.model)
        self.jobs = []
        if one is not None:
            g = W.build_graph(one, batch=1, dtype=args.dtype)
            for m in instances:
                st = W.build_weights(one, dtype=args.dtype, seed=0, model=m)
                self.jobs.append((g, st.tensors, model_inputs(g, seed=0, model=m), None))
            self.items_per_job = 1.0 / self.layers
            self.unit = f"1 of {self.layers} encoder layers x 1 sequence"
        else:
            g = W.build_graph(args.model, batch=args.batch, dtype=args.dtype)
            out = g.node_map()[g.graph_outputs[0].rsplit(":", 1)[0]].output_spec
            for m in instances:
                st = W.build_weights(args.model, dtype=args.dtype, seed=0, model=m)
                self.jobs.append((g, st.tensors, model_inputs(g, seed=0, model=m),
                                  W.fc_head(out, 1000, seed=100 + m)))
            self.items_per_job = float(args.batch)
            self.unit = f"1 full forward (B={args.batch}) + FC head"

    @staticmethod
    def _run(job):
        from oracle import executor as OX
        g, tensors, x, head = job
        out = OX.execute(g, tensors, x)[0]
        if head is not None:
            OX.execute(head[0], head[1].tensors, {"feat": out})
        return out

    def step(self, threads: int, jobs: list | None = None) -> tuple[float, float]:
        """Run `jobs` (default: all) on `threads` host threads; return
        (inference-equivalents done, wall seconds)."""
        jobs = self.jobs if jobs is None else jobs
        t0 = time.perf_counter()
        if threads == 1:
            for j in jobs:
                self._run(j)
        else:
            with ThreadPoolExecutor(max_workers=threads) as ex:
                list(ex.map(self._run, jobs))
        return len(jobs) * self.items_per_job, time.perf_counter() - t0


def cpu_baseline(args, budget_s: float = 10.0) -> dict:
    """The reference CPU algorithm on ONE host core (a scalar port): jobs of
    the sampler run back to back until ~`budget_s` of work is done."""
    cores = os.cpu_count() or 1
    sampler = ReferenceSampler(args, list(range(min(args.instances, 8))))
    items, secs, n = 0.0, 0.0, 0
    while secs < budget_s and n < 64:
        i, dt = sampler.step(1, [sampler.jobs[n % len(sampler.jobs)]])
        items, secs, n = items + i, secs + dt, n + 1
    return {"value": round(items / secs, 5), "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{n} job(s) of [{sampler.unit}] of the numpy restatement of the "
                      f"reference kernels ({args.model}, same seeds), {secs:.1f} s on 1 of "
                      f"{cores} host cores; value = inference-equivalents / wall time"}


def run_reference(args) -> dict | None:
    """--impl reference: the reference CPU algorithm on this config with all
    the host threads it can use (min(N, cores) instances, one per thread),
    each step one bounded sample. Under torchrun only rank 0 runs."""
    world, rank, _ = dist_env()
    if rank != 0:
        return None
    cores = os.cpu_count() or 1
    threads = max(1, min(args.instances, cores))
    sampler = ReferenceSampler(args, list(range(threads)))
    for _ in range(args.warmup):
        sampler.step(threads)
    items, secs = 0.0, 0.0
    for _ in range(args.steps):
        i, dt = sampler.step(threads)
        items, secs = items + i, secs + dt
    value = items / secs
    ms_per_step = secs / args.steps * 1e3
    desc = (f"{threads} instance(s) x [{sampler.unit}] per step on {threads} thread(s) "
            f"({cores} host cores); {items / args.steps:.4g} inference-equivalents per step")
    return {
        "impl": "reference",
        "metric": METRIC,
        "value": round(value, 5),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 2),
        "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": args.dtype,
        "data": "synthetic (same seeds as our arm)",
        "config": {"workload": f"{args.model} N={args.instances} B={args.batch} per GPU",
                   "baseline_config": args.config, "model": args.model,
                   "instances_per_gpu": args.instances, "batch": args.batch,
                   "items_per_step": round(items / args.steps, 5),
                   "parallelism": "host threads (reference `threaded` strategy, "
                                  "bench.py:112-121)"},
        "cpu_baseline": {"value": round(value, 5), "unit": UNIT, "cores": threads,
                         "kind": "port", "sample": desc},
        "e2e": {"value": round(value, 5), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main(argv=None) -> int:
    from paper_2009_13062_b200.workloads import BASELINE_CONFIGS

    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawTextHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(BASELINE_CONFIGS), default="C5",
                    help="BASELINE.json config (C5 = BERT-base N=32/GPU B=8, the default)")
    ap.add_argument("--model", default=None)
    ap.add_argument("--instances", type=int, default=None,
                    help="merged instances per GPU (weak) / in total (strong)")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--dtype", default=None)
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="torch.distributed backend under torchrun (gloo: ranks may share a GPU)")
    ap.add_argument("--no-heads", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    ap.add_argument("--no-unmerged", action="store_true",
                    help="skip the N-separate-runs legs (speedup denominator)")
    args = ap.parse_args(argv)
    model, n, batch, dtype = BASELINE_CONFIGS[args.config]
    args.model = args.model or model
    args.instances = args.instances or n
    args.batch = args.batch or batch
    args.dtype = args.dtype or dtype
    if (args.model, args.instances, args.batch, args.dtype) != (model, n, batch, dtype):
        args.config = None  # a custom workload, not the named BASELINE config
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
