"""Summarise ncu artefacts for profiles/ (run here, on the CPU box).

    python profiles/summarize.py launches <launches.csv>      # per-kernel device time shares
    python profiles/summarize.py full <prof.ncu-rep> [...]    # key metrics of a --set full capture
"""
import collections
import csv
import io
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__grid_size",
        "launch__block_size", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio"]


def launches(path):
    rows = list(csv.reader(open(path)))
    h = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[h], rows[h + 1:]
    k, v = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in data:
        name = r[k].split("(")[0].replace("void ", "").replace("ss::<unnamed>::", "")
        tot[name] += float(r[v].replace(",", ""))
        cnt[name] += 1
    s = sum(tot.values())
    print(f"{'kernel':48s} {'launches':>8s} {'avg us':>9s} {'share':>7s}")
    for name, t in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{name:48s} {cnt[name]:8d} {t / cnt[name] / 1e3:9.1f} {100 * t / s:6.1f}%")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"== {name.split('(')[0]}")
        for key in KEYS:
            if key in hdr:
                i = hdr.index(key)
                print(f"  {key:75s} {r[i]:>14s} {units[i]}")


def traffic(*paths):
    """JSON {kernel: {"dram_bytes": read+write per launch (mean), "us": duration}} from full captures."""
    import json
    agg = collections.defaultdict(list)
    for path in paths:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        hdr, units = rows[0], rows[1]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        ir, iw, it = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum"), \
            hdr.index("gpu__time_duration.sum")
        ii = hdr.index("smsp__inst_executed.sum") if "smsp__inst_executed.sum" in hdr else None
        for r in rows[2:]:
            name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("unnamed>::", "")
            b = float(r[ir]) * scale[units[ir]] + float(r[iw]) * scale[units[iw]]
            us = float(r[it]) * (1e-3 if units[it] == "nsecond" else 1.0)
            wi = float(r[ii]) if ii is not None and r[ii] else 0.0
            agg[name].append((b, us, wi))
    src = ", ".join(os.path.basename(p) for p in paths)
    print(json.dumps({"source": f"ncu --set full ({src}): dram__bytes_read.sum + dram__bytes_write.sum per launch",
                      "kernels": {k: {"dram_bytes": sum(x[0] for x in v) / len(v), "us": sum(x[1] for x in v) / len(v),
                                      "warp_inst": sum(x[2] for x in v) / len(v),
                                      "captures": len(v)} for k, v in agg.items()}}, indent=1))


if __name__ == "__main__":
    {"launches": launches, "full": full, "traffic": traffic}[sys.argv[1]](*sys.argv[2:])
