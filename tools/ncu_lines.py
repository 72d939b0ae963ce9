"""Stall samples and executed warp instructions per CUDA source line of an ncu --set full
report (compiled with -lineinfo): python tools/ncu_lines.py REPORT [TOP]."""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40
text = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                      capture_output=True, text=True).stdout
samp, inst, src = defaultdict(int), defaultdict(int), {}
fname, hdr, cur = "?", None, None
for row in csv.reader(io.StringIO(text)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = {h: i for i, h in enumerate(row)}
        continue
    if hdr is None or len(row) < 5:
        continue
    if row[0]:  # a source line row
        cur = (fname, int(row[0]))
        src[cur] = row[1].strip()
    if cur is None:
        continue
    try:
        s = int(row[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        n = int(row[hdr["Instructions Executed"]] or 0)
    except (ValueError, IndexError):
        continue
    samp[cur] += s
    inst[cur] += n
ts, ti = sum(samp.values()) or 1, sum(inst.values()) or 1
print(f"samples {ts}, warp instructions {ti / 1e9:.3f} G")
for k in sorted(samp, key=lambda k: -samp[k])[:top]:
    print(f"{100 * samp[k] / ts:5.1f}% samp {100 * inst[k] / ti:5.1f}% inst  {k[0]}:{k[1]:<5d} {src.get(k, '')[:90]}")
