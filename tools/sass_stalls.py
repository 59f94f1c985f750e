"""Top warp-stall instructions of an ncu --set full capture (SASS view):

    python tools/sass_stalls.py gpurun_out/x.ncu-rep [--top 25] [--context 0]

Prints each hot instruction's share of all stall samples and its leading
stall reasons (long_sb = waiting on a global/local load, barrier = named /
CTA barrier, mio = shared-memory queue, ...), optionally with neighbours.
"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=25)
    ap.add_argument("--context", type=int, default=0)
    args = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", args.rep, "--page", "source", "--csv", "--print-source",
                          "sass"], capture_output=True, text=True).stdout
    hdr, body = None, []
    for r in csv.reader(io.StringIO(raw)):
        if r and r[0] == "Address":
            hdr = r
        elif hdr and r and r[0].startswith("0x"):
            body.append(r)
    H = {h: i for i, h in enumerate(hdr)}
    col = H["Warp Stall Sampling (All Samples)"]
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(int(r[col] or 0) for r in body)
    print(f"{len(body)} instructions, {tot} stall samples")
    hot = sorted(range(len(body)), key=lambda i: -int(body[i][col] or 0))[:args.top]
    for i in sorted(hot):
        r = body[i]
        n = int(r[col] or 0)
        top = sorted(((int(r[H[h]] or 0), h[6:]) for h in reasons), reverse=True)[:3]
        why = ", ".join(f"{h} {v}" for v, h in top if v)
        for j in range(max(0, i - args.context), i):
            print(f"        {j:5d} {body[j][H['Source']].strip()[:90]}")
        print(f"{100 * n / tot:5.1f}% {i:5d} {r[H['Source']].strip()[:70]:70s} [{why}]")


if __name__ == "__main__":
    main()
