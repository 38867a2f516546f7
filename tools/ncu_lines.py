"""Top source lines by warp-stall samples for one kernel of an ncu report."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", kern], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = {}
cur = None
for r in rows:
    if len(r) < 8 or r[0] in ("Line No", "File Path", "Function Name"):
        continue
    try:
        samp = float(r[4] or 0)
        ins = float(r[7] or 0)
    except ValueError:
        continue
    if r[0].strip():
        cur = (int(r[0]), r[1].strip()[:100])
        agg.setdefault(cur, [0.0, 0.0])
        agg[cur][0] += samp
        agg[cur][1] += ins
tot = sum(v[0] for v in agg.values()) or 1
toti = sum(v[1] for v in agg.values()) or 1
print(f"{kern}: samples {tot:.0f}, warp-instructions {toti:.0f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0] / tot * 100:5.1f}% stall {v[1] / toti * 100:5.1f}% inst  L{k[0]}: {k[1]}")
