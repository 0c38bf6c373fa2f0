import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
agg = defaultdict(int); src = {}; f = None; line = None; iE = None
for r in rows:
    if not r: continue
    if r[0] == "File Path": f = r[1].split("/")[-1]; continue
    if r[0] == "Line No": iE = r.index("Instructions Executed"); continue
    if iE is None or len(r) <= iE: continue
    if r[0]:
        line = (f, int(r[0])); src[line] = r[1]
    elif r[iE].isdigit() and line:
        agg[line] += int(r[iE])
tot = sum(agg.values()); print("total", tot)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{100*v/tot:5.1f}% {k[0]}:{k[1]}  {src[k][:90]}")
