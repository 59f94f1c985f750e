"""Key metrics of the round's `ncu --set full` captures (tools/gpu_evidence.sh
full) per launch: duration, DRAM bytes and throughput, tensor-pipe activity,
bf16 tensor op rate, L2 hit rate, occupancy, registers.

    python tools/summarize_full.py gpurun_out/ev_full_c5.ncu-rep ... > profiles/r02_ncu_full_summary.txt
"""
import csv
import io
import subprocess
import sys

COLS = [
    ("gpu__time_duration.sum", "us", 1e-3),
    ("dram__bytes_read.sum", "MB rd", 1e-6),
    ("dram__bytes_write.sum", "MB wr", 1e-6),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "%dram", 1),
    # tensor-core operand reads from shared memory (tcgen05.mma; the legacy
    # hmma pipe counters do not see tcgen05)
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "%tc smem", 1),
    ("lts__t_sector_hit_rate.pct", "%L2 hit", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "%occ", 1),
    ("launch__registers_per_thread", "regs", 1),
    ("launch__grid_size", "grid", 1),
]


def unit_scale(u):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
            "msecond": 1e6, "ns": 1, "us": 1e3, "ms": 1e6}.get(u, 1)


def main():
    for rep in sys.argv[1:]:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        if len(rows) < 3:
            continue
        hdr, units = rows[0], rows[1]
        print(f"## {rep.split('/')[-1]}")
        print("kernel".ljust(46) + "".join(f"{name:>11s}" for _, name, _ in COLS))
        for r in rows[2:]:
            name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
            name = name.replace("nf::", "").replace("(anonymous namespace)::", "")[:45]
            vals = []
            for key, _, sc in COLS:
                key2 = next((h for h in hdr if h.endswith(key)), None)
                if key2 is None:
                    vals.append(float("nan"))
                    continue
                i = hdr.index(key2)
                try:
                    v = float(r[i].replace(",", "")) * unit_scale(units[i]) * sc
                except ValueError:
                    v = float("nan")
                vals.append(v)
            print(name.ljust(46) + "".join(f"{v:11.1f}" for v in vals))
        print()


if __name__ == "__main__":
    main()
