"""Summarise an ncu capture (raw page) and a launch list into markdown for profiles/.

usage: python tools/ncu_summary.py REPORT.ncu-rep LAUNCHES.csv OUT.md "title"
"""
import collections
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum"]


def main(rep, launches, out, title):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    lines = [f"# {title}", "", f"ncu --set full capture `{rep.split('/')[-1]}` (cold-cache, serialised replays: "
             "compare shares, not absolute times with bench.py).", ""]
    for r in rows[2:]:
        lines.append(f"## `{r[hdr.index('Kernel Name')][:90]}`")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"| {k} | {r[i]} | {units[i]} |")
        lines.append("")
    agg = collections.defaultdict(lambda: [0, 0.0])
    hdr2 = None
    for r in csv.reader(open(launches)):
        if "Kernel Name" in r:
            hdr2 = r
            continue
        if hdr2 and len(r) == len(hdr2):
            d = dict(zip(hdr2, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                name = d["Kernel Name"].split("(")[0]
                agg[name][0] += 1
                agg[name][1] += float(d["Metric Value"].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    lines += ["## Launch list (ncu --metrics gpu__time_duration.sum, whole bench run incl. setup)", "",
              "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k[:70]}` | {c} | {t / 1e6:.3f} | {t / tot * 100:.1f}% |")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:5])
