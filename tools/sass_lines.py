"""Per-source-line warp-stall samples of one kernel from an ncu report.

ncu's CUDA source page needs the report's own source correlation; this joins
the SASS page (per-instruction samples, in address order) with `nvdisasm -g`
line info of the same cubin instead (instruction i of the function <-> row i).

    python tools/sass_lines.py gpurun_out/prof.ncu-rep kernels_8b 'Li1EEEE' [--top 40]
"""
import argparse
import collections
import csv
import io
import os
import re
import subprocess
import tempfile

ap = argparse.ArgumentParser()
ap.add_argument("report")
ap.add_argument("cubin", help="cubin stem inside libffb200.so, e.g. kernels_8b")
ap.add_argument("func", help="substring of the mangled kernel name, e.g. Li1EEEE")
ap.add_argument("--lib", default=os.path.join(os.path.dirname(os.path.dirname(
    os.path.abspath(__file__))), "paper_2505_22758_b200", "libffb200.so"))
ap.add_argument("--top", type=int, default=40)
ap.add_argument("--lines", default="", help="lo-hi: only report lines in this range")
a = ap.parse_args()

tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", a.lib], cwd=tmp, check=True,
               stdout=subprocess.DEVNULL)
cub = [f for f in os.listdir(tmp) if f.startswith(a.cubin) and f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True,
                     text=True, check=True).stdout
# instruction -> innermost source line of the selected function
lines, cur, inside = [], None, False
for ln in dis.splitlines():
    if ln.startswith("//--------------------- .text."):
        inside = a.func in ln and "decode_step_kernel" in ln
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m and "inlined at" not in ln:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln):
        lines.append(cur)

out = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
data = rows[hdr_i + 1:]
col = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
print(f"{len(data)} SASS rows in report, {len(lines)} instructions in {cub}:{a.func}")
per = collections.defaultdict(lambda: collections.Counter())
tot = collections.Counter()
for i, r in enumerate(data):
    if i >= len(lines) or lines[i] is None:
        continue
    key = lines[i]
    s = int(r[col["Warp Stall Sampling (All Samples)"]] or 0)
    per[key]["samples"] += s
    per[key]["inst"] += int(r[col["Instructions Executed"]] or 0)
    for h in stall_cols:
        v = int(float(r[col[h]] or 0))
        per[key][h] += v
        tot[h] += v
    tot["samples"] += s
lo, hi = (int(x) for x in a.lines.split("-")) if a.lines else (0, 1 << 30)
items = [(k, v) for k, v in per.items() if lo <= k[1] <= hi]
items.sort(key=lambda kv: -kv[1]["samples"])
T = max(1, tot["samples"])
print(f"total samples {T}")
for (f, n), v in items[:a.top]:
    top = ", ".join(f"{h[6:]} {v[h]}" for h in sorted(stall_cols, key=lambda h: -v[h])[:3] if v[h])
    print(f"{f}:{n:5d} {100 * v['samples'] / T:5.1f}%  inst {v['inst']:9d}  {top}")
