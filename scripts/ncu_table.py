"""Per-kernel table of the key ncu metrics (raw CSV page) incl. stall reasons per issue.

    python scripts/ncu_table.py <raw.csv>
"""
import csv
import sys

KEYS = [("us", "gpu__time_duration.sum"), ("dramR", "dram__bytes_read.sum"), ("dramW", "dram__bytes_write.sum"),
        ("issue%", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        ("warps%", "sm__warps_active.avg.pct_of_peak_sustained_active"), ("regs", "launch__registers_per_thread"),
        ("grid", "launch__grid_size"), ("inst", "smsp__inst_executed.sum")]
STALLS = ["barrier", "long_scoreboard", "short_scoreboard", "wait", "math_pipe_throttle", "mio_throttle",
          "lg_throttle", "not_selected", "selected", "dispatch_stall", "no_instruction", "branch_resolving",
          "membar", "sleeping", "tex_throttle", "drain", "misc"]


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = rows[0]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        out = [f"{k}={r[hdr.index(m)]}" for k, m in KEYS if m in hdr]
        st = []
        for s in STALLS:
            m = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if m in hdr:
                v = float(r[hdr.index(m)] or 0)
                if v >= 0.1:
                    st.append(f"{s}={v:.2f}")
        print(name[:40], " ".join(out))
        print("   stalls/issue:", " ".join(st))
        for m in ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
                  "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"):
            if m in hdr:
                print(f"   {m} = {r[hdr.index(m)]}")


if __name__ == "__main__":
    main(sys.argv[1])
