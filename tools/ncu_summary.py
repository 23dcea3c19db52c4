"""Summarise ncu outputs into profiles/ (launch list shares + full-capture
metrics of the top kernels).  Usage:
  python tools/ncu_summary.py launches <launches.csv> > profiles/..._launches.md
  python tools/ncu_summary.py full <report.ncu-rep> [...] > profiles/..._full.md
  python tools/ncu_summary.py traffic <launches.csv> <workload> <passes> [profiles/traffic.json]
    (DRAM bytes per launch of the DMMA GEMM family from a launch list that
    also collected dram__bytes_read/write.sum; `passes` = rank-k HSVD steps in
    the profiled command; what bench.py's roofline.traffic reads)
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


UNIT = {"ns": 1.0, "us": 1e3, "ms": 1e6, "s": 1e9, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6,
        "Gbyte": 1e9, "Tbyte": 1e12}


def launches(path):
    """Launch list of one command: per kernel the launches, the summed
    gpu__time_duration and, when the pass also collected them, the summed
    dram__bytes_read/write (-> average DRAM bytes per launch)."""
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    h = rows[0]
    iname, ival, imet, iunit, iid = (h.index("Kernel Name"), h.index("Metric Value"),
                                     h.index("Metric Name"), h.index("Metric Unit"), h.index("ID"))
    agg = collections.OrderedDict()
    other = 0.0
    seen = set()
    for r in rows[1:]:
        v = float(r[ival].replace(",", "")) * UNIT.get(r[iunit], 1.0)
        lib = "hsvdcu" in r[iname] or "unnamed>::k_" in r[iname]
        if r[imet].startswith("gpu__time_duration"):
            if not lib:
                other += v
                continue
            k = short(r[iname])
            a = agg.setdefault(k, [0, 0.0, 0.0, 0.0])
            a[1] += v
            if r[iid] not in seen:
                seen.add(r[iid])
                a[0] += 1
        elif lib and r[imet].startswith("dram__bytes"):
            a = agg.setdefault(short(r[iname]), [0, 0.0, 0.0, 0.0])
            a[2 if "read" in r[imet] else 3] += v
    tot = sum(a[1] for a in agg.values())
    traffic = any(a[2] + a[3] > 0 for a in agg.values())
    print("| kernel | launches | total ms | share of library time |"
          + (" DRAM read GB | DRAM written GB | DRAM GB/s |" if traffic else ""))
    print("|---|---|---|---|" + ("---|---|---|" if traffic else ""))
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        line = f"| `{k}` | {a[0]} | {a[1] / 1e6:.3f} | {100 * a[1] / tot:.1f}% |"
        if traffic:
            line += f" {a[2] / 1e9:.2f} | {a[3] / 1e9:.2f} | {(a[2] + a[3]) / max(a[1], 1.0):.0f} |"
        print(line)
    print(f"\nlibrary kernels total {tot / 1e6:.1f} ms; non-library (torch input generation, "
          f"peak probes) {other / 1e6:.1f} ms.  ncu per-launch times are serialised and "
          f"cold-cache: compare shares, not absolutes.")


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


def traffic(path, workload, passes, out):
    import json
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    h = rows[0]
    iname, ival, imet, iunit, iid = (h.index("Kernel Name"), h.index("Metric Value"),
                                     h.index("Metric Name"), h.index("Metric Unit"), h.index("ID"))
    ids, byts = set(), 0.0
    for r in rows[1:]:
        k = short(r[iname])
        if not (k.startswith("k_gemm<") or k == "k_gemm" or k == "k_gemm_sk"):
            continue
        ids.add(r[iid])
        if r[imet].startswith("dram__bytes"):
            byts += float(r[ival].replace(",", "")) * UNIT.get(r[iunit], 1.0)
    try:
        data = json.load(open(out))
    except Exception:
        data = {}
    data[workload] = {
        "k_gemm": byts / max(1, len(ids)),
        "_source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over {passes} rank-k "
                   f"HSVD steps of bench.py ({len(ids)} launches of k_gemm + k_gemm_sk, "
                   f"{byts / 1e9:.1f} GB read + written); {path.split('/')[-1]}",
        "launches_per_step": len(ids) / passes,
    }
    with open(out, "w") as f:
        json.dump(data, f, indent=1)
    print(json.dumps(data[workload]))


if __name__ == "__main__":
    if sys.argv[1] == "traffic":
        traffic(sys.argv[2], sys.argv[3], int(sys.argv[4]),
                sys.argv[5] if len(sys.argv) > 5 else "profiles/traffic.json")
    elif sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2:])
