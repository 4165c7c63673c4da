"""Top SASS instructions (by executed count and by stall samples) of one kernel
in an .ncu-rep, grouped into basic-block-ish windows."""
import csv
import subprocess
import sys

path, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
ia, isrc, isamp, iexe = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
data = []
for r in rows[2:]:
    if len(r) < len(h):
        continue
    data.append((r[ia], r[isrc].strip(), int(r[isamp] or 0), int(r[iexe] or 0)))
tot_e = sum(d[3] for d in data)
tot_s = sum(d[2] for d in data)
print(f"instructions executed (warp-level) {tot_e:,}  samples {tot_s:,}  sass lines {len(data)}")
# opcode histogram weighted by executed count
from collections import Counter
c = Counter()
for d in data:
    op = d[1].split()[0] if d[1] else "?"
    if op.startswith("@"):
        op = d[1].split()[1]
    c[op.split(".")[0]] += d[3]
print("opcode mix:", ", ".join(f"{k}={100*v/tot_e:.1f}%" for k, v in c.most_common(25)))
print("--- hottest by stall samples")
for d in sorted(data, key=lambda x: -x[2])[:top]:
    print(f"{d[2]:7d} {d[3]:12,} {d[0][-5:]}  {d[1][:90]}")
print("--- execution-count profile along the code (runs of lines with equal count)")
runs = []
for d in data:
    if runs and runs[-1][1] == d[3]:
        runs[-1][2] += 1
        runs[-1][3].append(d[1].split()[0] if d[1] else "?")
    else:
        runs.append([d[0][-5:], d[3], 1, [d[1].split()[0] if d[1] else "?"]])
big = sorted(runs, key=lambda r: -r[1] * r[2])[:top]
for r in sorted(big, key=lambda r: r[0]):
    print(f"{r[0]} count={r[1]:>12,} n={r[2]:4d} share={100*r[1]*r[2]/tot_e:5.1f}%  {' '.join(r[3][:12])}")
