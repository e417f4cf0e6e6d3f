"""Summarise an ncu report's SASS source page: hottest instructions by stall
samples and by executed instructions.   python tools/ncu_hot.py rep.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
lines = txt.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
tot_s = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
tot_i = sum(int(r["Instructions Executed"] or 0) for r in rows)
print(f"{len(rows)} SASS lines, {tot_s} stall samples, {tot_i} warp instructions executed")
idx = {r["Address"]: i for i, r in enumerate(rows)}
hot = sorted(rows, key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))[:N]
for r in sorted(hot, key=lambda r: idx[r["Address"]]):
    s = int(r["Warp Stall Sampling (All Samples)"] or 0)
    print(f"{idx[r['Address']]:5d} {100*s/tot_s:5.1f}% ex={int(r['Instructions Executed'] or 0):>10d}  {r['Source'].strip()[:90]}")
