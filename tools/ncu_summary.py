"""Summarise ncu outputs for profiles/: per-kernel share of a launch list (csv from
`ncu --metrics gpu__time_duration.sum --csv`) and key metrics of a `--set full` report."""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def launch_list(path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v = v * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
        per[name][0] += 1
        per[name][1] += v
    tot = sum(v[1] for v in per.values())
    out = [f"{'kernel':60s} {'launches':>8s} {'total_us':>12s} {'share':>7s}"]
    for k, (n, t) in sorted(per.items(), key=lambda x: -x[1][1]):
        out.append(f"{k[:60]:60s} {n:8d} {t:12.1f} {t / tot * 100:6.2f}%")
    out.append(f"{'TOTAL':60s} {sum(v[0] for v in per.values()):8d} {tot:12.1f}")
    return "\n".join(out)


KEYS = ["Duration", "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy",
        "Registers Per Thread", "Executed Instructions", "L1/TEX Hit Rate", "L2 Hit Rate",
        "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Eligible Warps Per Scheduler", "Avg. Active Threads Per Warp", "Grid Size", "Block Size",
        "Dynamic Shared Memory Per Block", "dram__bytes_read.sum", "dram__bytes_write.sum"]


def full_report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    lines = [f"report: {path}"]
    for r in csv.DictReader(io.StringIO(out)):
        if r.get("Metric Name") in KEYS:
            lines.append(f"  {r['Kernel Name'][:50]:50s} {r['Metric Name']:40s} {r['Metric Value']} {r['Metric Unit']}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) > 2:
        hdr = rows[0]
        for want in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                     "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                     "smsp__thread_inst_executed_per_inst_executed.ratio", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                     "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active"):
            if want in hdr:
                k = hdr.index(want)
                for r in rows[2:]:
                    lines.append(f"  raw {want:60s} {rows[1][k]:>8s} {r[k]}")
    return "\n".join(lines)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(launch_list(p) if p.endswith(".csv") else full_report(p))
        print()
