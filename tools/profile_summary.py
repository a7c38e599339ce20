"""Summarise ncu captures into profiles/ (committed evidence).

python tools/profile_summary.py <tag> <rep.ncu-rep> [<launches.csv>]
writes profiles/<tag>.md (key metrics, top stall lines, top instruction lines) and
merges dram bytes per launch into profiles/traffic.json under the mode key
parsed from the kernel's template arguments (bf_kernel<METRIC, FAST, ...>)."""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, rep = sys.argv[1], sys.argv[2]
launches = sys.argv[3] if len(sys.argv) > 3 else None


def run(*a):
    return subprocess.run(list(a), capture_output=True, text=True).stdout


raw = list(csv.reader(run("ncu", "-i", rep, "--page", "raw", "--csv").splitlines()))
h, u, v = raw[0], raw[1], raw[2]
R = {n: (v[i], u[i]) for i, n in enumerate(h)}
kname = R.get("Kernel Name", ("?", ""))[0]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
        "launch__block_size", "launch__occupancy_limit_shared_mem", "sm__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]
lines = [f"# ncu capture `{tag}`", "", f"kernel: `{kname}`", "", "| metric | value | unit |", "|---|---|---|"]
for w in want:
    if w in R:
        lines.append(f"| {w} | {R[w][0]} | {R[w][1]} |")


def to_bytes(val, unit):
    x = float(val.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


rd = to_bytes(*R["dram__bytes_read.sum"])
wr = to_bytes(*R["dram__bytes_write.sum"])
lines += ["", f"DRAM traffic per launch: read {rd/1e9:.3f} GB + write {wr/1e9:.3f} GB", ""]
lines += ["## Warp-stall samples by source line (top 25)", "", "```"]
lines += run(sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, "25").splitlines()
lines += ["```", "", "## Executed warp instructions by source line (top 25)", "", "```"]
lines += run(sys.executable, os.path.join(ROOT, "tools", "ncu_instr.py"), rep, "25").splitlines()
lines += ["```"]
if launches:
    agg = {}
    rows = [r for r in csv.reader(open(launches)) if len(r) > 5]
    hh = rows[0]
    for r in rows[1:]:
        d = dict(zip(hh, r))
        key = d["Kernel Name"].split("(")[0]
        agg.setdefault(key, {}).setdefault(d["Metric Name"], []).append(
            float(d["Metric Value"].replace(",", "")))
    lines += ["", "## Launch list (ncu --metrics gpu__time_duration.sum, cold-cache, serialised)", "",
              "| kernel | launches | mean duration (us) | mean dram read (MB) |", "|---|---|---|---|"]
    for kk, m in agg.items():
        t = m.get("gpu__time_duration.sum", [0])
        dr = m.get("dram__bytes_read.sum", [0])
        lines.append(f"| `{kk[:70]}` | {len(t)} | {sum(t)/len(t)/1e3:.1f} | {sum(dr)/len(dr)/1e6:.1f} |")
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
with open(os.path.join(ROOT, "profiles", f"{tag}.md"), "w") as f:
    f.write("\n".join(lines) + "\n")
# traffic.json
mode = os.environ.get("TRAFFIC_KEY")  # e.g. c4_fast; default: parsed for the C2 captures
if mode is None and "bf_kernel<" in kname:
    fast = kname.split("bf_kernel<")[1].split(",")[1].strip()
    mode = "fast" if fast in ("1", "true") else "det"
if mode:
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    t = json.load(open(tp)) if os.path.exists(tp) else {}
    t[mode] = {"kernel": kname, "dram_bytes_read": rd, "dram_bytes_write": wr, "capture": tag}
    json.dump(t, open(tp, "w"), indent=1)
print("\n".join(lines[:30]))
