"""Splits a kernel's SASS (ncu source page CSV, --print-source=cuda,sass) at its BAR.SYNC instructions and prints,
per segment, executed instructions, stall samples and the top stall reasons.  python scripts/ncu_phases.py FILE.csv"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
sass = {}
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0] == "" and r[2].startswith("0x"):
        a = int(r[2], 16)
        if a not in sass:
            sass[a] = r
iS = hdr.index("# Samples"); iE = hdr.index("Instructions Executed")
stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
seg = []; cur = {"n": 0, "inst": 0, "samp": 0, "st": {}, "first": None, "fp64": 0, "lds": 0}
def flush():
    global cur
    seg.append(cur); cur = {"n": 0, "inst": 0, "samp": 0, "st": {}, "first": None, "fp64": 0, "lds": 0}
for a in sorted(sass):
    r = sass[a]; txt = r[3].strip()
    if cur["first"] is None: cur["first"] = hex(a & 0xffff)
    cur["n"] += 1
    e = int(r[iE]) if r[iE].isdigit() else 0
    cur["inst"] += e; cur["samp"] += int(r[iS]) if r[iS].isdigit() else 0
    op = txt.split()[0] if not txt.startswith("@") else txt.split()[1]
    if op.startswith(("DFMA", "DMUL", "DADD", "DSETP")): cur["fp64"] += e
    if op.startswith(("LDS", "STS", "ATOMS")): cur["lds"] += e
    for i, h in stall_cols:
        if r[i].isdigit() and int(r[i]): cur["st"][h] = cur["st"].get(h, 0) + int(r[i])
    if "BAR.SYNC" in txt: flush()
flush()
tot = sum(s["samp"] for s in seg)
print("%4s %6s %8s %10s %9s %9s %7s  top stalls" % ("seg", "start", "static", "warp-inst", "fp64", "smem", "samp%"))
for k, s in enumerate(seg):
    top = sorted(s["st"].items(), key=lambda kv: -kv[1])[:4]
    print("%4d %6s %8d %10d %9d %9d %6.1f%%  %s" % (k, s["first"], s["n"], s["inst"], s["fp64"], s["lds"], 100.0 * s["samp"] / max(tot, 1),
          ", ".join("%s %.0f%%" % (h[6:], 100.0 * v / max(s["samp"], 1)) for h, v in top)))
