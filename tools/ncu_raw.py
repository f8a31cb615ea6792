"""Print the key raw counters of every kernel in an ncu report (stall reasons included).
usage: python tools/ncu_raw.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum"]
idx = [h.index(w) if w in h else None for w in want]
stall = [i for i, c in enumerate(h) if c.startswith("smsp__average_warps_issue_stalled_") and c.endswith("_per_issue_active.ratio")]
for r in rows[2:]:
    print("----")
    for w, i in zip(want, idx):
        if i is not None:
            print("  ", w, r[i])
    st = sorted([(float(r[i]) if r[i] else 0, h[i].replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")) for i in stall], reverse=True)[:6]
    print("   stalls", [(round(a, 2), b) for a, b in st])
