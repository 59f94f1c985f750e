"""Turn a round's raw GPU evidence (gpurun_out/final_*) into the committed
summaries under profiles/:

  * <tag>_launches_summary.txt — ncu launch list (gpu__time_duration.sum,
    --clock-control none) of `bench.py --steps 2 --warmup 3`, our kernels
    grouped by name with count / mean / share;
  * <tag>_bert8_ncu_full.json — per-kernel key metrics of the --set full
    capture (time, DRAM bytes, DRAM / tensor / SM throughput, L2 hit rate);
  * gemm_traffic.json — mean DRAM bytes per weight-streaming launch of the
    BERT-base N=8 B=1 forward (bench.py's roofline `traffic`).

    python tools/summarize_profiles.py [--tag r01]
"""
import argparse
import collections
import csv
import io
import json
import subprocess
from pathlib import Path

OURS = ("nf::", "k_grouped_gemm_tc", "k_qkv_attention", "k_group_norm", "k_attention",
        "k_rel_attention", "k_pool", "k_elementwise", "k_copy", "k_conv", "k_linear")
METRICS = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__t_sector_hit_rate.pct", "launch__grid_size", "launch__registers_per_thread")


def launches(csv_path: Path, out: Path) -> None:
    text = csv_path.read_text(errors="replace")
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per = collections.defaultdict(list)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        if not any(k in name for k in OURS):
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ns = v * {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
        per[name.split("(")[0]].append(ns)
    total = sum(sum(v) for v in per.values())
    lines = ["# ncu launch list (bench.py --steps 2 --warmup 3 --no-cpu --no-unmerged; BERT-base N=8 B=1;",
             "# cold-cache, serialised: compare SHARES, not absolutes). Our kernels only.",
             f"# total {int(total)} ns over {sum(len(v) for v in per.values())} launches", ""]
    for name, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{100 * sum(v) / total:6.2f}%  n={len(v):5d}  avg={sum(v) / len(v):10.0f}ns  {name}")
    out.write_text("\n".join(lines) + "\n")


def ncu_full(rep: Path, out: Path) -> dict:
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, body = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(head)}
    res = []
    for r in body:
        d = {"Kernel Name": r[idx["Kernel Name"]][:90]}
        for m in METRICS:
            if m in idx:
                d[m] = f"{r[idx[m]]} {units[idx[m]]}".strip()
        res.append(d)
    out.write_text(json.dumps({"ncu_set_full_bert8": res}, indent=1) + "\n")
    return {"rows": res, "idx": idx}


def _bytes(s: str) -> float:
    v, _, u = s.partition(" ")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    return float(v.replace(",", "")) * scale


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--src", default="gpurun_out")
    args = ap.parse_args()
    src, dst = Path(args.src), Path("profiles")
    dst.mkdir(exist_ok=True)
    if (src / "final_launches.csv").exists():
        launches(src / "final_launches.csv", dst / f"{args.tag}_launches_summary.txt")
    rep = src / "final_ncu_bert8.ncu-rep"
    if rep.exists():
        got = ncu_full(rep, dst / f"{args.tag}_bert8_ncu_full.json")
        stream = [r for r in got["rows"]
                  if any(k in r["Kernel Name"] for k in ("k_grouped_gemm_tc<128, true",
                                                          "k_grouped_gemm_tc<128, 1,", "qkv"))]
        if stream:
            per = [_bytes(r["dram__bytes_read.sum"]) + _bytes(r["dram__bytes_write.sum"])
                   for r in stream]
            tr = dst / "gemm_traffic.json"
            doc = json.loads(tr.read_text()) if tr.exists() else {}
            doc["bert-base/N8/B1"] = int(sum(per) / len(per))
            doc[f"per_launch_{args.tag}"] = [
                {"kernel": r["Kernel Name"], "dram_bytes": int(b),
                 "ncu_time": r["gpu__time_duration.sum"]} for r, b in zip(stream, per)]
            tr.write_text(json.dumps(doc, indent=1) + "\n")
    for f in sorted(src.glob("final_bench_*.json")):
        name = f.name.replace("final_bench_", f"{args.tag}_bench_")
        (dst / name).write_text(f.read_text())


if __name__ == "__main__":
    main()
