"""Summarise an ncu report per CUDA source line (instructions + stall samples).

usage: python scripts/ncu_lines.py REPORT.ncu-rep OUT_PREFIX [max_launches]
Writes OUT_PREFIX_<i>.txt for each profiled launch: kernel name, duration,
DRAM bytes, and the 40 source lines with the most executed instructions.
"""
import csv, io, subprocess, sys


def ncu(*args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main():
    rep, out = sys.argv[1], sys.argv[2]
    nmax = int(sys.argv[3]) if len(sys.argv) > 3 else 64
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv", "--metrics",
                                          "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
                                          "smsp__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed"))))
    hdr = raw[0]
    rows = [dict(zip(hdr, r)) for r in raw[2:]]
    for i, r in enumerate(rows[:nmax]):
        src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                                              "--launch-skip", str(i), "--launch-count", "1"))))
        agg, text, fn, h = {}, {}, None, None
        cur = None
        for s in src:
            if len(s) >= 2 and s[0] == "File Path":
                fn = s[1].split("/")[-1]
                continue
            if s and s[0] == "Line No":
                h = s
                continue
            if h and s and len(s) >= 8:
                if s[0].strip():
                    cur = (fn, s[0])
                    text[cur] = s[1][:100]
                try:
                    ie, ws = float(s[7] or 0), float(s[4] or 0)
                except ValueError:
                    continue
                a = agg.setdefault(cur, [0.0, 0.0])
                a[0] += ie
                a[1] += ws
        ti = sum(a[0] for a in agg.values()) or 1
        tw = sum(a[1] for a in agg.values()) or 1
        with open(f"{out}_{i}.txt", "w") as fh:
            fh.write(f"kernel {r.get('Kernel Name')}\n")
            for k in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
                      "sm__throughput.avg.pct_of_peak_sustained_elapsed"):
                fh.write(f"{k} {r.get(k)}\n")
            for k, a in sorted(agg.items(), key=lambda x: -x[1][0])[:40]:
                fh.write(f"{a[0] / ti * 100:5.1f}% inst {a[1] / tw * 100:5.1f}% stall  {k[0]}:{k[1]}  {text.get(k, '')}\n")


if __name__ == "__main__":
    main()
