"""Aggregate warp-stall reasons per source region for one kernel of an ncu report.
usage: ncu_stalls.py report.ncu-rep kernel_regex file.cu:start-end:name [...]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
regions = []
for a in sys.argv[3:]:
    f, rng, name = a.split(":")
    lo, hi = rng.split("-")
    regions.append((f, int(lo), int(hi), name))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
cur_file, hdr = None, None
agg = {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        cur_file = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    line = int(r[0])
    d = dict(zip(hdr, r))
    name = "other"
    for f, lo, hi, nm in regions:
        if cur_file == f and lo <= line <= hi:
            name = nm
    a = agg.setdefault(name, {})
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k or k in ("Warp Stall Sampling (All Samples)", "Instructions Executed"):
            try:
                a[k] = a.get(k, 0) + float(v)
            except ValueError:
                pass
tot = sum(a.get("Warp Stall Sampling (All Samples)", 0) for a in agg.values()) or 1
for name, a in sorted(agg.items(), key=lambda kv: -kv[1].get("Warp Stall Sampling (All Samples)", 0)):
    s = a.get("Warp Stall Sampling (All Samples)", 0)
    top = sorted(((k[6:], v) for k, v in a.items() if k.startswith("stall_")), key=lambda kv: -kv[1])[:5]
    print(f"{name:14s} {100*s/tot:5.1f}%  inst {a.get('Instructions Executed',0)/1e6:7.1f}M  " +
          "  ".join(f"{k}={100*v/max(s,1):.0f}%" for k, v in top))
