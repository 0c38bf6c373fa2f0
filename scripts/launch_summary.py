"""Summarises an ncu --csv launch list: per kernel count, mean/total time, mean DRAM bytes.
python scripts/launch_summary.py FILE.csv"""
import csv, sys, collections, re
rows = []
with open(sys.argv[1]) as f:
    lines = [l for l in f if not l.startswith("==")]
rd = csv.DictReader(lines)
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rd:
    name = re.sub(r"\(.*", "", r["Kernel Name"])
    grid = r.get("Grid Size", "")
    v = float(r["Metric Value"].replace(",", ""))
    u = r["Metric Unit"]
    m = r["Metric Name"]
    if m == "gpu__time_duration.sum":
        v = v / 1e3 if u in ("ns", "nsecond") else (v * 1e3 if u in ("ms", "msecond") else v)  # -> us
    elif m.startswith("dram__bytes"):
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        v = v * mult
    agg[name][m].append(v)
    agg[name]["grid"].append(grid)
tot = sum(sum(a["gpu__time_duration.sum"]) for a in agg.values())
print("%-60s %6s %10s %10s %6s %10s %10s" % ("kernel", "n", "mean us", "total us", "share", "rd MB", "wr MB"))
for name, a in sorted(agg.items(), key=lambda kv: -sum(kv[1]["gpu__time_duration.sum"])):
    t = a["gpu__time_duration.sum"]
    rdb = a.get("dram__bytes_read.sum", [0]); wrb = a.get("dram__bytes_write.sum", [0])
    print("%-60s %6d %10.1f %10.1f %5.1f%% %10.2f %10.2f  grid %s" % (name[:60], len(t), sum(t) / len(t), sum(t), 100 * sum(t) / tot,
          sum(rdb) / len(rdb) / 1e6, sum(wrb) / len(wrb) / 1e6, a["grid"][len(a["grid"])//2]))
print("total us", tot)
