"""Print a compact table from an ncu --page raw --csv export (one row per launch)."""
import csv
import sys

COLS = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "rdMB"), ("dram__bytes_write.sum", "wrMB"),
        ("lts__t_sector_hit_rate.pct", "L2hit"), ("sm__warps_active.avg.pct_of_peak_sustained_active", "wact"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "smthr"), ("launch__grid_size", "grid"),
        ("launch__registers_per_thread", "reg"), ("smsp__inst_executed.sum", "Minst"),
        ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "lsb"),
        ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "bar"),
        ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "ssb"),
        ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "wait"),
        ("smsp__average_warps_issue_stalled_membar_per_issue_active.ratio", "mbar"),
        ("smsp__thread_inst_executed_per_inst_executed.ratio", "thr/inst")]
r = list(csv.reader(open(sys.argv[1])))
h = r[0]
units = r[1]
print("kernel".ljust(22) + "".join(c[1].rjust(8) for c in COLS))
for row in r[2:]:
    d = dict(zip(h, row))
    u = dict(zip(h, units))
    out = []
    for m, _ in COLS:
        v = d.get(m, "")
        try:
            x = float(v.replace(",", ""))
            un = u.get(m, "")
            if m.startswith("dram__bytes"):
                x *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(un, 1)
            if m == "gpu__time_duration.sum":
                x *= {"ns": 1e-3, "us": 1, "ms": 1e3}.get(un, 1)
            if m == "smsp__inst_executed.sum":
                x /= 1e6
            out.append(f"{x:8.2f}")
        except ValueError:
            out.append(v[:8].rjust(8))
    print(d["Kernel Name"].split("(")[0].replace("gps::", "").replace("void ", "")[:22].ljust(22) + "".join(out))
