"""Summarise ncu outputs into profiles/ (launch list shares + full-capture
metrics of the top kernels).  Usage:
  python tools/ncu_summary.py launches <launches.csv> > profiles/..._launches.md
  python tools/ncu_summary.py full <report.ncu-rep> [...] > profiles/..._full.md
"""
import collections
import csv
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
    "launch__block_size", "launch__cluster_dim_x", "launch__registers_per_thread",
    "lts__t_sector_hit_rate.pct",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
]


def short(name):
    m = re.search(r"(k_[a-z_0-9]+)(<[^>]*>)?", name)
    return (m.group(1) + (m.group(2) or "")) if m else name[:60]


def launches(path):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    h = rows[0]
    iname, ival = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    other = 0.0
    for r in rows[1:]:
        ns = float(r[ival].replace(",", ""))
        if "hsvdcu" not in r[iname] and "unnamed>::k_" not in r[iname]:
            other += ns
            continue
        k = short(r[iname])
        c, t = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, t + ns)
    tot = sum(t for _, t in agg.values())
    print("| kernel | launches | total ms | share of library time |")
    print("|---|---|---|---|")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {c} | {t / 1e6:.3f} | {100 * t / tot:.1f}% |")
    print(f"\nlibrary kernels total {tot / 1e6:.1f} ms; non-library (torch input generation) "
          f"{other / 1e6:.1f} ms.  ncu per-launch times are serialised and cold-cache: compare "
          f"shares, not absolutes.")


def full(paths):
    for p in paths:
        out = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(out.splitlines()))
        h, units = rows[0], rows[1]
        for r in rows[2:]:
            print(f"### `{short(r[h.index('Kernel Name')])}` ({p.split('/')[-1]})\n")
            print("| metric | value |")
            print("|---|---|")
            for k in KEYS:
                if k in h:
                    i = h.index(k)
                    print(f"| {k} | {r[i]} {units[i]} |")
            print()


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2:])
