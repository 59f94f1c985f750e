"""Summarise a round's per-config ncu evidence (gpurun_out/<tag>_ncu_<C>.csv
from tools/ncu_forward.py, plus the plan metadata) into the committed files
bench.py reads:

  * profiles/<tag>_ncu_share.json   — per workload: the dominant family's share
    of one forward's summed kernel time (ncu, serialised, cold-ish cache) and a
    per-kernel table (count, mean time, share, DRAM bytes per launch);
  * profiles/<tag>_ncu_traffic.json — per workload: mean DRAM bytes
    (read + write) per dominant-family launch, beside the plan's algorithmic
    bytes per family launch.

    python tools/summarize_ncu.py [--tag r02] [--src gpurun_out]
"""
import argparse
import collections
import csv
import io
import json
import re
from pathlib import Path

# the dominant (weight-streaming / tensor) family, as bench.family_roofline
# defines it: merged Linear + implicit-GEMM conv launches, the fused
# QKV+attention launch, the fp32 3xTF32 conv
FAMILY = re.compile(r"k_grouped_gemm_tc|k_linear_chain_tc|k_qkv_attention_tc|k_conv_tf32|k_linear_tf32")
OURS = re.compile(r"^(nf::|k_)|nf::")
SCALE = {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
         "KB": 1e3, "MB": 1e6, "GB": 1e9}


def read_launches(path: Path) -> list[dict]:
    text = path.read_text(errors="replace")
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    by_id: dict[str, dict] = collections.OrderedDict()
    for r in rows:
        d = by_id.setdefault(r["ID"], {"name": r["Kernel Name"]})
        v = float(r["Metric Value"].replace(",", "") or 0)
        d[r["Metric Name"]] = v * SCALE.get(r.get("Metric Unit", ""), 1.0)
    return list(by_id.values())


def short(name: str) -> str:
    s = name.split("(")[0]
    s = re.sub(r"^void\s+", "", s)
    return s.replace("nf::(anonymous namespace)::", "").replace("nf::", "")[:80]


def summarise(launches: list[dict], meta: dict) -> tuple[dict, dict]:
    per = collections.defaultdict(lambda: {"n": 0, "ns": 0.0, "dram": 0.0})
    for l in launches:
        k = short(l["name"])
        per[k]["n"] += 1
        per[k]["ns"] += l.get("gpu__time_duration.sum", 0.0)
        per[k]["dram"] += l.get("dram__bytes_read.sum", 0.0) + l.get("dram__bytes_write.sum", 0.0)
    total = sum(v["ns"] for v in per.values())
    fam = [l for l in launches if FAMILY.search(l["name"])]
    fam_ns = sum(l.get("gpu__time_duration.sum", 0.0) for l in fam)
    fam_dram = [l.get("dram__bytes_read.sum", 0.0) + l.get("dram__bytes_write.sum", 0.0)
                for l in fam]
    alg = [v[0] for v in meta.get("family", {}).values()]
    share = {
        "family_share": round(fam_ns / total, 4) if total else None,
        "family_launches": len(fam),
        "launches": len(launches),
        "summed_kernel_us": round(total / 1e3, 1),
        "family_us": round(fam_ns / 1e3, 1),
        "kernels": [
            {"kernel": k, "n": v["n"], "avg_us": round(v["ns"] / v["n"] / 1e3, 2),
             "share": round(v["ns"] / total, 4),
             "dram_mb_per_launch": round(v["dram"] / v["n"] / 1e6, 2)}
            for k, v in sorted(per.items(), key=lambda kv: -kv[1]["ns"])],
        "source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                  "--clock-control none, one eager forward (tools/ncu_forward.py); serialised: "
                  "compare shares, not absolutes",
    }
    traffic = {
        "dram_bytes_per_family_launch": int(sum(fam_dram) / len(fam_dram)) if fam_dram else None,
        "algorithmic_bytes_per_family_launch": int(sum(alg) / len(alg)) if alg else None,
        "family_launches": len(fam),
    }
    if traffic["dram_bytes_per_family_launch"] and traffic["algorithmic_bytes_per_family_launch"]:
        traffic["dram_over_algorithmic"] = round(
            traffic["dram_bytes_per_family_launch"] / traffic["algorithmic_bytes_per_family_launch"], 3)
    return share, traffic


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="r02")
    ap.add_argument("--src", default="gpurun_out")
    args = ap.parse_args()
    src, dst = Path(args.src), Path("profiles")
    # configs without a new capture keep their committed summaries
    old = lambda n: json.loads((dst / n).read_text()) if (dst / n).exists() else {}  # noqa: E731
    shares, traffics = old(f"{args.tag}_ncu_share.json"), old(f"{args.tag}_ncu_traffic.json")
    for f in sorted(src.glob(f"{args.tag}_ncu_C*.csv")):
        cfg = f.stem.rsplit("_", 1)[-1]
        mf = src / f"{args.tag}_ncu_{cfg}_meta.json"
        meta = json.loads(mf.read_text()) if mf.exists() else {}
        key = meta.get("workload", cfg)
        s, t = summarise(read_launches(f), meta)
        s["config"] = t["config"] = cfg
        shares[key], traffics[key] = s, t
        print(f"{cfg} {key}: family share {s['family_share']}, {s['family_launches']} launches, "
              f"DRAM/alg {t.get('dram_over_algorithmic')}")
    (dst / f"{args.tag}_ncu_share.json").write_text(json.dumps(shares, indent=1) + "\n")
    (dst / f"{args.tag}_ncu_traffic.json").write_text(json.dumps(traffics, indent=1) + "\n")


if __name__ == "__main__":
    main()
