"""Prints the key counters of an .ncu-rep (raw page): python scripts/ncu_keys.py REPORT [regex]"""
import csv, subprocess, sys, re
rep = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
for vals in rows[2:]:
    print("==", vals[hdr.index("Kernel Name")][:90])
    for i, h in enumerate(hdr):
        if pat:
            if pat.search(h): print("%-90s %s %s" % (h, vals[i], units[i]))
            continue
        keep = (h in ("gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
                      "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
                      "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
                      "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
                      "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__cycles_elapsed.avg", "smsp__thread_inst_executed_per_inst_executed.ratio")
                or (h.startswith("sm__inst_executed_pipe_") and h.endswith("pct_of_peak_sustained_active"))
                or (h.startswith("sm__pipe_") and h.endswith("pct_of_peak_sustained_active")))
        if keep: print("%-90s %s %s" % (h, vals[i], units[i]))
        if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
            try:
                v = float(vals[i])
                if v > 0.1: print("  stall %-55s %.2f" % (h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], v))
            except ValueError:
                pass
