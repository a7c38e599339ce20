"""Aggregate an ncu source page (--print-source cuda,sass --csv) per CUDA source
line: stall samples and top stall reasons.  Usage: python tools/ncu_lines.py rep.ncu-rep [N]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
per_line = defaultdict(float)
src_text = {}
reasons = defaultdict(lambda: defaultdict(float))
cur_file = ""
hdr = None
cur_line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5:
        continue
    if r[0]:
        cur_line = (cur_file, r[0])
        src_text[cur_line] = r[1][:100]
    try:
        s = float(r[4] or 0)
    except ValueError:
        continue
    per_line[cur_line] += s
    for i, name in enumerate(hdr):
        if name.startswith("stall_") or name.startswith("Warp Stall Sampling (All Samples):"):
            try:
                reasons[cur_line][name] += float(r[i] or 0)
            except ValueError:
                pass
tot = sum(per_line.values()) or 1
for key, s in sorted(per_line.items(), key=lambda kv: -kv[1])[:top]:
    rs = sorted(reasons[key].items(), key=lambda kv: -kv[1])[:3]
    rtxt = " ".join(f"{n.split(':')[-1].strip()[:18]}={v/tot*100:.1f}" for n, v in rs if v > 0)
    print(f"{100*s/tot:5.1f}% {key[0]}:{key[1]:>4} {src_text.get(key, '')[:70]:70s} {rtxt}")
