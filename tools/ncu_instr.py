"""Per-source-line executed warp instructions from an ncu report (cuda,sass view)."""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
per = defaultdict(float)
txt = {}
cur = None
hdr = None
f = ""
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        continue
    if hdr is None or len(r) <= ie:
        continue
    if r[0]:
        cur = (f, r[0])
        txt[cur] = r[1][:90]
    try:
        per[cur] += float(r[ie] or 0)
    except ValueError:
        pass
tot = sum(per.values())
print(f"total warp instructions {tot:.3e}")
for k, v in sorted(per.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100*v/tot:5.1f}% {v:10.3e} {k[0]}:{k[1]:>4} {txt.get(k,'')}")
