"""Aggregate ncu SASS-page stall samples (needs a --set full --import-source capture).

    python profiles/source_hotspots.py <prof.ncu-rep> <kernel regex> [top]
Prints the hottest SASS instructions and the share per opcode.
"""
import collections
import csv
import io
import subprocess
import sys


def main(rep, kernel, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kernel}"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    data = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr) and r[0] != "Address"]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ei = hdr.index("Instructions Executed")
    num = lambda x: float(x) if x not in ("", "-") else 0.0
    tot = sum(num(r[si]) for r in data)
    ops = collections.Counter()
    inst = collections.Counter()
    for r in data:
        op = r[1].split()[0] if r[1].split() else "?"
        if op.startswith("@"):
            op = r[1].split()[1]
        op = op.split(".")[0]
        ops[op] += num(r[si])
        inst[op] += num(r[ei])
    print(f"total stall samples {tot:.0f}; by opcode (stall share / executed warp-instr):")
    for op, v in ops.most_common(18):
        print(f"  {op:10s} {100 * v / tot:5.1f}%  {inst[op]:12.0f}")
    print("hottest instructions:")
    data.sort(key=lambda r: -num(r[si]))
    for r in data[:int(top)]:
        print(f"  {100 * num(r[si]) / tot:5.1f}%  {r[0]}  {r[1][:90]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
