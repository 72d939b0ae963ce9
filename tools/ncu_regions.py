"""Summarise an ncu --set full report of k_interact: headline metrics, stall reasons and
per-SASS-region instruction counts (regions split at backward branches = loops).
Usage: python tools/ncu_regions.py report.ncu-rep"""
import csv
import io
import subprocess
import sys
from collections import Counter


def run(args):
    return subprocess.run(["ncu", "-i", sys.argv[1]] + args, capture_output=True, text=True).stdout


def details():
    rows = list(csv.reader(io.StringIO(run(["--page", "details", "--csv"]))))
    hdr = rows[0]
    want = ["Duration", "Executed Ipc Active", "Issue Slots Busy", "Executed Instructions",
            "Registers Per Thread", "Achieved Active Warps Per SM", "L1/TEX Hit Rate", "L2 Hit Rate",
            "DRAM Throughput", "Compute (SM) Throughput", "Warp Cycles Per Issued Instruction"]
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") in want:
            print(f"{d['Metric Name']:40s} {d['Metric Value']:>16s} {d['Metric Unit']}")


def sass():
    text = run(["--page", "source", "--csv", "--print-source", "sass"])
    rows = list(csv.reader(io.StringIO(text)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    data = rows[2:]
    tot = sum(int(r[ix["Instructions Executed"]] or 0) for r in data)
    samp = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
    print(f"total warp instructions {tot / 1e9:.3f} G, stall samples {samp}")
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    for c in cols:
        v = sum(int(r[ix[c]] or 0) for r in data)
        if v > 0.01 * samp:
            print(f"  {c:28s} {100 * v / samp:5.1f}%")
    # loops: backward branches; report the hottest instruction-count regions
    base = int(data[0][0], 16)
    addr = [int(r[0], 16) - base for r in data]
    ex = [int(r[ix["Instructions Executed"]] or 0) for r in data]
    sm = [int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data]
    loops = []
    for k, r in enumerate(data):
        src = r[1]
        if "BRA" in src and ex[k] > 0:
            try:
                tgt = int(src.split("BRA")[1].split()[-1].strip(" ;"), 16) - base
            except ValueError:
                continue
            if tgt < addr[k]:
                loops.append((tgt, addr[k]))
    seen = set()
    for lo, hi in sorted(loops, key=lambda x: x[1] - x[0]):
        idx = [k for k in range(len(data)) if lo <= addr[k] <= hi]
        e = sum(ex[k] for k in idx)
        s = sum(sm[k] for k in idx)
        if e < 0.02 * tot or (lo, hi) in seen:
            continue
        seen.add((lo, hi))
        iters = ex[idx[-1]]
        ops = Counter()
        for k in idx:
            if ex[k] >= 0.9 * iters:
                op = data[k][1].split()
                op = op[1] if op[0].startswith("@") else op[0]
                ops[op.split(".")[0]] += 1
        print(f"loop [{lo:#x},{hi:#x}] inst {e / 1e9:.3f}G ({100 * e / tot:.1f}%) samples {100 * s / samp:.1f}% "
              f"iters {iters / 1e6:.2f}M hot-body {sum(ops.values())} instr")
        print("   ", ", ".join(f"{k}:{v}" for k, v in ops.most_common(14)))


if __name__ == "__main__":
    details()
    sass()
