"""Top source lines by warp-stall samples from an ncu report (cuda,sass
source view): python tools/ncu_lines.py REPORT.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg, src, fname = {}, {}, ""
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5 or not r[0]:
        continue
    key = (fname, int(r[0]))
    try:
        v = float(r[4])
    except ValueError:
        v = 0.0
    agg[key] = agg.get(key, 0) + v
    src[key] = r[1]
tot = sum(agg.values()) or 1
for key, v in sorted(agg.items(), key=lambda kv: -kv[1])[:n]:
    print(f"{100 * v / tot:5.1f}%  {key[0]}:{key[1]:<5} {src[key].strip()[:100]}")
