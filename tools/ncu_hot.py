"""Hottest SASS lines (warp-stall samples) of the first launch of a kernel in an ncu report.
    python tools/ncu_hot.py <rep> <kernel regex> [n]"""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern, "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
si, ie = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
num = lambda v: float(v) if v.replace('.', '', 1).isdigit() else 0.0
data = []
for r in rows[2:]:
    if len(r) != len(h):
        break          # next launch
    data.append(r)
tot = sum(num(r[si]) for r in data)
print(f"samples {tot:.0f}, instructions {sum(num(r[ie]) for r in data):.0f}, sass lines {len(data)}")
for r in sorted(data, key=lambda r: -num(r[si]))[:n]:
    print(f"{r[0][-5:]} {num(r[si]):6.0f} {100 * num(r[si]) / max(tot, 1):5.1f}% ex={r[ie]:>7}  {r[1].strip()[:90]}")
