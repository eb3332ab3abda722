"""Basic-block instruction counts of one kernel from an ncu --set full capture (SASS page).

    python profiles/inst_blocks.py <prof.ncu-rep> <kernel regex> [top]
Groups consecutive SASS instructions with the same execution count (a basic block) and
prints the blocks that execute the most warp-instructions, with their stall share.
"""
import csv
import io
import subprocess
import sys


def main(rep, kernel, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kernel}",
                          "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
    hdr = rows[h]
    data = [r for r in rows[h + 1:] if len(r) == len(hdr) and r[0] != "Address"]
    ei, si = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    num = lambda x: float(x) if x not in ("", "-") else 0.0
    tot = sum(num(r[ei]) for r in data)
    stot = sum(num(r[si]) for r in data) or 1.0
    blocks, cur = [], None
    for r in data:
        c = num(r[ei])
        if cur is None or c != cur[0]:
            cur = [c, 0, 0.0, r[0][-5:] + " " + r[1][:60]]
            blocks.append(cur)
        cur[1] += 1
        cur[2] += num(r[si])
    print(f"total warp-instructions {tot:.0f}")
    for c, n, st, s in sorted(blocks, key=lambda b: -b[0] * b[1])[:int(top)]:
        print(f"{100 * c * n / tot:5.1f}% inst  {100 * st / stot:5.1f}% stall  count={c:9.0f} x{n:3d}  {s}")


if __name__ == "__main__":
    main(*sys.argv[1:])
