"""Source lines with the most warp-stall samples for one kernel launch of an
`ncu --set full --import-source on` capture (what the profile-driven epilogue
fixes of this round were read from).

    python tools/stall_lines.py gpurun_out/p3_c5.ncu-rep --kernel k_grouped_gemm \
        --skip 2 [--top 16]
"""
import argparse
import csv
import io
import subprocess


def _int(x):
    try:
        return int(x)
    except ValueError:
        return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--kernel", required=True, help="kernel name regex")
    ap.add_argument("--skip", type=int, default=0, help="matching launches to skip")
    ap.add_argument("--top", type=int, default=16)
    a = ap.parse_args()
    out = subprocess.run(
        ["ncu", "-i", a.rep, "--page", "source", "--csv", "--kernel-name", f"regex:{a.kernel}",
         "--launch-skip", str(a.skip), "--launch-count", "1", "--print-source", "sass,cuda"],
        capture_output=True, text=True, check=True).stdout
    sections, cur = [], None
    for row in csv.reader(io.StringIO(out)):
        if row and row[0] == "File Path":
            cur = {"file": row[1], "rows": []}
            sections.append(cur)
        elif row and row[0] == "Function Name" and cur is not None:
            cur["func"] = row[1]
        elif cur is not None:
            cur["rows"].append(row)
    if sections:
        print(sections[0].get("func", "")[:150])
    total = 0
    lines = []
    for s in sections:
        hdr = next((r for r in s["rows"] if r and r[0] == "Line No"), None)
        if hdr is None:
            continue
        i_s = hdr.index("Warp Stall Sampling (All Samples)")
        for r in s["rows"]:
            if r and r[0].isdigit():
                n = _int(r[i_s])
                total += n
                lines.append((n, s["file"].split("/")[-1], r[0], r[1].strip()))
    print(f"samples {total}")
    for n, f, ln, src in sorted(lines, reverse=True)[:a.top]:
        print(f"{n:6d} {100 * n / max(total, 1):5.1f}%  {f}:{ln}  {src[:90]}")


if __name__ == "__main__":
    main()
