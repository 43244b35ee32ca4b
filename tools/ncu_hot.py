"""Top stall-sampled source lines of an ncu report (needs -lineinfo):
    python tools/ncu_hot.py gpurun_out/front_c2_r01.ncu-rep [n] [--sass]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
sass = "--sass" in sys.argv
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
per_line = defaultdict(float)
per_sass = []
src_of = {}
cur = None
si = None
fname = ""
for r in rows:
    if r and r[0] == "File Name":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        si = r.index("Warp Stall Sampling (All Samples)")
        continue
    if si is None or len(r) <= si:
        continue
    if r[0] not in ("", "-") and r[0].isdigit():
        cur = (fname, int(r[0]))
        src_of[cur] = r[1].strip()[:100]
    try:
        v = float(r[si])
    except ValueError:
        continue
    if cur is not None:
        per_line[cur] += v
    per_sass.append((v, r[2], r[3].strip()[:80], cur))
tot = sum(per_line.values())
print(f"total samples {tot:.0f}")
if sass:
    for v, addr, ins, cur in sorted(per_sass, key=lambda x: -x[0])[:top_n]:
        print(f"{v:7.0f} {100*v/max(tot,1):5.1f}%  {ins:60s} {cur}")
else:
    for key, v in sorted(per_line.items(), key=lambda x: -x[1])[:top_n]:
        print(f"{v:7.0f} {100*v/max(tot,1):5.1f}%  {key[0]}:{key[1]}  {src_of.get(key,'')}")
