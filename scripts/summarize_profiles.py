"""Summarise ncu outputs into profiles/ (committed evidence).

  python scripts/summarize_profiles.py ROUND LAUNCH_CSV [NCU_REP ...]

Writes profiles/<round>_launches.csv (kernel, grid, block, duration_us per launch,
load-time kernels excluded), profiles/<round>_summary.md (per-kernel share of the
serialised step + the full-capture metrics of every captured launch) and
updates profiles/traffic.json (DRAM bytes per launch per kernel class).
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LOAD = ("k_rs_", "k_degrees", "k_make_keys", "k_build_rows", "k_dup_flags", "k_transpose_keys", "k_label_hist")
CLASS = [("k_explore", "explore"), ("k_ec", "ec_write"), ("k_join<0>", "join_count"), ("k_join<1>", "join_write"),
         ("k_join<2>", "join_write"), ("k_join_v", "join_write"), ("k_join_fast", "join_write"), ("k_join_bulk", "join_write"),
         ("k_join_seg", "join_len"), ("k_join_job_totals", "join_len"), ("k_collect", "collect"),
         ("k_check", "check"), ("k_post", "bitand"), ("k_scan", "scan")]
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__thread_inst_executed_per_inst_executed.ratio",
           "smsp__sass_average_branch_targets_threads_uniform.pct", "launch__registers_per_thread",
           "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1, "ms": 1e3,
         "nsecond": 1e-3, "msecond": 1e3}


def short(name):
    n = name.split("(")[0].replace("void ", "").replace("gps::", "")
    n = n.replace("(unsigned int)", "").replace("u>", ">")
    n = n.replace("(bool)0", "0").replace("(bool)1", "1").replace("<false>", "<0>").replace("<true>", "<1>")
    return n


def klass(n):
    for pre, c in CLASS:
        if n.startswith(pre):
            return c
    return n


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] != "gpu__time_duration.sum":
                continue
            v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1e-3)
            n = short(d["Kernel Name"])
            if n.startswith(LOAD):
                continue
            out.append((n, d["Grid Size"], d["Block Size"], v))
    return out


def full(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for d in data:
        e = {"kernel": short(d[hdr.index("Kernel Name")])}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                try:
                    val = float(d[i].replace(",", ""))
                except ValueError:
                    continue
                if m.startswith("dram__bytes"):
                    val *= SCALE.get(units[i], 1)
                if m == "gpu__time_duration.sum":
                    val *= SCALE.get(units[i], 1)
                e[m] = val
        res.append(e)
    return res


def main():
    rnd, lpath, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    L = launches(lpath)
    with open(os.path.join(prof, f"{rnd}_launches.csv"), "w") as fh:
        w = csv.writer(fh)
        w.writerow(["kernel", "grid", "block", "duration_us"])
        for r in L:
            w.writerow([r[0], r[1], r[2], f"{r[3]:.3f}"])
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, _, _, v in L:
        agg[n][0] += 1
        agg[n][1] += v
    tot = sum(v[1] for v in agg.values())
    md = [f"# {rnd}: ncu evidence", "",
          f"Launch list: `{os.path.basename(lpath)}` (ncu `--metrics gpu__time_duration.sum --clock-control none`,",
          "cold-cache and serialised: compare SHARES).  Graph-load kernels excluded.", "",
          "| kernel | class | launches | total µs | avg µs | share |", "|---|---|---|---|---|---|"]
    for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        md.append(f"| `{n}` | {klass(n)} | {c} | {v:.1f} | {v / c:.2f} | {v / tot:.3f} |")
    md.append(f"| total | | {sum(v[0] for v in agg.values())} | {tot:.1f} | | 1.000 |")
    traffic_path = os.path.join(prof, "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for rep in reps:
        F = full(rep)
        md += ["", f"## Full capture `{os.path.basename(rep)}` (`ncu --set full --clock-control none`)", "",
               "| kernel | µs | DRAM read MB | DRAM write MB | L2 hit % | L1 hit % | warps active % | SM thr % "
               "| DRAM % | threads/inst | uniform br % | regs | stall long-sb | stall barrier |",
               "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
        per = collections.defaultdict(list)
        for e in F:
            g = lambda k: e.get(k, float("nan"))  # noqa: E731
            md.append(f"| `{e['kernel']}` | {g('gpu__time_duration.sum'):.1f} | {g('dram__bytes_read.sum') / 1e6:.2f} | "
                      f"{g('dram__bytes_write.sum') / 1e6:.2f} | {g('lts__t_sector_hit_rate.pct'):.1f} | "
                      f"{g('l1tex__t_sector_hit_rate.pct'):.1f} | {g('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
                      f"{g('sm__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
                      f"{g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.2f} | "
                      f"{g('smsp__thread_inst_executed_per_inst_executed.ratio'):.1f} | "
                      f"{g('smsp__sass_average_branch_targets_threads_uniform.pct'):.1f} | "
                      f"{g('launch__registers_per_thread'):.0f} | "
                      f"{g('smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio'):.2f} | "
                      f"{g('smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio'):.2f} |")
            per[klass(e["kernel"])].append((e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0),
                                           e.get("lts__t_sector_hit_rate.pct", float("nan")),
                                           e.get("gpu__time_duration.sum", 0.0)))
        pre = os.environ.get("TRAFFIC_PREFIX", "")
        for c, v in per.items():
            traffic[pre + c] = sum(x[0] for x in v) / len(v)   # DRAM bytes per launch
            tw = sum(x[2] for x in v)
            if tw > 0:   # duration-weighted L2 hit rate of the class
                traffic[pre + c + ":l2_hit_pct"] = sum(x[1] * x[2] for x in v if x[1] == x[1]) / tw
    json.dump(traffic, open(traffic_path, "w"), indent=1)
    open(os.path.join(prof, f"{rnd}_summary.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md[:40]))


if __name__ == "__main__":
    main()
