"""Summarise ncu outputs for profiles/.

    python tools/ncu_summary.py report <file.ncu-rep>     # key metrics per profiled kernel
    python tools/ncu_summary.py launches <launches.csv>   # per-kernel share of device time
    python tools/ncu_summary.py traffic <file.ncu-rep> <workload>   # -> profiles/traffic.json
"""
import csv
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("lts__t_bytes.sum", "L2 bytes"),
]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        print(f"== {r[col['Kernel Name']]}")
        for key, label in METRICS:
            if key in col:
                print(f"   {label:18s} {r[col[key]]:>14s} {units[col[key]]}")


def launches(path):
    tot = defaultdict(float)
    cnt = defaultdict(int)
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    rd = csv.DictReader(lines)
    unit = None
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        unit = r.get("Metric Unit")
        v = float(r["Metric Value"].replace(",", ""))
        tot[r["Kernel Name"]] += v
        cnt[r["Kernel Name"]] += 1
    allt = sum(tot.values())
    print(f"{'kernel':60s} {'launches':>8s} {'total':>12s} {'avg':>12s} {'share':>7s}  ({unit})")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{k[:60]:60s} {cnt[k]:8d} {tot[k]:12.1f} {tot[k] / cnt[k]:12.1f} {100 * tot[k] / allt:6.1f}%")


def traffic(*args):
    """dram__bytes_read.sum + dram__bytes_write.sum per profiled kernel (first launch of each):
    traffic <report.ncu-rep> [<report2.ncu-rep> ...] <workload>"""
    import json
    import os

    *paths, workload = args
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    kern = {}
    for path in paths:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(out.splitlines()))
        hdr, units = rows[0], rows[1]
        col = {h: i for i, h in enumerate(hdr)}
        for r in rows[2:]:
            name = r[col["Kernel Name"]]
            if name in kern:
                continue
            tot = 0.0
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                tot += float(r[col[m]].replace(",", "")) * scale.get(units[col[m]], 1)
            kern[name] = tot
    dst = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
    try:  # one entry per workload; other workloads' captures are kept
        with open(dst) as fh:
            allw = json.load(fh).get("workloads", {})
    except Exception:
        allw = {}
    allw[workload] = {"source": [os.path.basename(p) for p in paths], "kernels": kern}
    with open(dst, "w") as fh:
        json.dump({"workloads": allw}, fh, indent=1)
    print(json.dumps(allw[workload], indent=1))


if __name__ == "__main__":
    fn = {"report": report, "launches": launches, "traffic": traffic}[sys.argv[1]]
    fn(*sys.argv[2:])
