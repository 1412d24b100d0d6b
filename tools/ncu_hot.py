"""Hot SASS lines of one kernel from an ncu report: python tools/ncu_hot.py report.ncu-rep [min_share]."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
for k in ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
          "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
          "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "lts__t_bytes.sum", "smsp__inst_executed.sum"]:
    if k in h:
        print(f"{k:70s} {v[h.index(k)]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
iS, iE, iW = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
tw = sum(int(r[iW]) for r in data if r[iW].isdigit()) or 1
te = sum(int(r[iE]) for r in data if r[iE].isdigit()) or 1
print("total inst", te, "samples", tw)
for r in data:
    w = int(r[iW]) if r[iW].isdigit() else 0
    e = int(r[iE]) if r[iE].isdigit() else 0
    if w >= thr * tw:
        print(f"{100 * w / tw:5.1f}% {e:10d} {r[iS].strip()[:90]}")
