"""Stall samples / executed warp instructions per CUDA source line (needs an --import-source
capture; ncu's cuda,sass source view).

    python profiles/source_lines.py <prof.ncu-rep> <kernel regex> [top]
"""
import csv
import io
import subprocess
import sys


def main(rep, kernel, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kernel}",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    fname, hdr, data = None, None, []
    for r in csv.reader(io.StringIO(out)):
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            hdr = r
        elif hdr and len(r) == len(hdr) and r[0]:
            data.append((fname, r))
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ei = hdr.index("Instructions Executed")
    num = lambda x: float(x) if x not in ("", "-") else 0.0
    tot = sum(num(r[si]) for _, r in data) or 1.0
    toti = sum(num(r[ei]) for _, r in data) or 1.0
    print(f"stall samples {tot:.0f}, warp instructions {toti:.0f}")
    data.sort(key=lambda fr: -num(fr[1][si]))
    for f, r in data[:int(top)]:
        print(f"{100 * num(r[si]) / tot:5.1f}% stall {100 * num(r[ei]) / toti:5.1f}% inst  {f}:{r[0]}  {r[1].strip()[:80]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
