"""Aggregates warp-stall samples of an ncu source page (cuda,sass) by CUDA line.
usage: ncu -i REP --page source --csv --print-source=cuda,sass > x.csv; python scripts/ncu_lines.py x.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
agg = defaultdict(int)
src = {}
f = None
line = None
iS = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        iS = r.index("Warp Stall Sampling (All Samples)")
        continue
    if iS is None or len(r) <= iS:
        continue
    if r[0]:
        line = (f, int(r[0]))
        src[line] = r[1]
        if r[iS].isdigit():
            agg[line] += 0
    elif r[iS].isdigit() and line:
        agg[line] += int(r[iS])
tot = sum(agg.values())
print("total", tot)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{100*v/tot:5.1f}% {k[0]}:{k[1]}  {src[k][:90]}")
