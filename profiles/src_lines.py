"""Warp-instructions and stall samples per CUDA source line of one kernel (ncu capture taken
with -lineinfo builds and --import-source on).

    python profiles/src_lines.py <prof.ncu-rep> <kernel regex> [top]
"""
import collections
import csv
import io
import subprocess
import sys


def main(rep, kernel, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--kernel-name", f"regex:{kernel}", "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    inst, stall, text = collections.Counter(), collections.Counter(), {}
    fname, hdr, cur = "?", None, None
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        if r[0]:
            cur = (fname, int(r[0]))
            text[cur] = r[1].strip()[:70]
        if cur is None or not r[2]:
            continue
        num = lambda x: float(x) if x not in ("", "-") else 0.0
        inst[cur] += num(r[hdr.index("Instructions Executed")])
        stall[cur] += num(r[hdr.index("Warp Stall Sampling (All Samples)")])
    ti, ts = sum(inst.values()) or 1, sum(stall.values()) or 1
    print(f"total warp-instructions {ti:.0f}")
    for k, v in inst.most_common(int(top)):
        print(f"{100 * v / ti:5.1f}% inst {100 * stall[k] / ts:5.1f}% stall  {k[0]}:{k[1]:<5d} {text.get(k, '')}")


if __name__ == "__main__":
    main(*sys.argv[1:])
