"""Per-SASS-instruction executed counts and stall samples from an ncu report
(development tool): python tools/ncu_sass.py <rep> [min_exec_fraction]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ia, ie, isamp = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[ie] or 0) for r in rows[2:] if len(r) > ie)
stot = sum(int(r[isamp] or 0) for r in rows[2:] if len(r) > ie)
print(f"total instr {tot:.4g} samples {stot}")
for r in rows[2:]:
    if len(r) <= ie:
        continue
    n = int(r[ie] or 0)
    s = int(r[isamp] or 0)
    if n >= thr * tot or s >= thr * stot:
        print(f"{r[0][-5:]} {n/1e6:9.2f}M {100*s/max(stot,1):5.1f}%  {r[ia].strip()}")
