"""Stall samples and executed instructions of an ncu report's SASS, summed per
bucket of consecutive lines:  python tools/ncu_regions.py rep.ncu-rep [bucket]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
B = int(sys.argv[2]) if len(sys.argv) > 2 else 100
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
lines = txt.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
tot_s = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
for b0 in range(0, len(rows), B):
    chunk = rows[b0:b0 + B]
    s = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in chunk)
    ex = sum(int(r["Instructions Executed"] or 0) for r in chunk)
    if s * 200 < tot_s:
        continue
    first = next((r["Source"].strip() for r in chunk if int(r["Instructions Executed"] or 0)), "")
    print(f"{b0:5d}-{b0 + len(chunk) - 1:5d} {100 * s / tot_s:5.1f}% ex={ex:>11d}  {first[:60]}")
