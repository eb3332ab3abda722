"""Warp-instructions and stall samples per CUDA source line (needs -lineinfo + --import-source).

    python profiles/src_lines.py <prof.ncu-rep> <kernel regex> [top]
"""
import csv
import io
import subprocess
import sys


def main(rep, kernel, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda",
                          "--kernel-name", f"regex:{kernel}", "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    res, fname, hdr = [], None, None
    for r in rows:
        if len(r) == 2 and r[0] == "File Name":
            fname = r[1].split("/")[-1]
            hdr = None
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            try:
                ei, si = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
            except ValueError:
                continue
            num = lambda x: float(x) if x not in ("", "-") else 0.0
            res.append((num(r[ei]), num(r[si]), f"{fname}:{r[0]}", r[1].strip()[:80]))
    tot_i = sum(x[0] for x in res) or 1
    tot_s = sum(x[1] for x in res) or 1
    print(f"total warp-instructions {tot_i:.0f}")
    for i, s, loc, src in sorted(res, key=lambda x: -x[0])[:int(top)]:
        print(f"{100 * i / tot_i:5.1f}% inst {100 * s / tot_s:5.1f}% stall  {loc:22s} {src}")


if __name__ == "__main__":
    main(*sys.argv[1:])
