"""Per-CUDA-source-line stall samples / executed warp instructions of one kernel
from an .ncu-rep (needs -lineinfo): python scripts/ncu_lines.py rep kernel [top]."""
import csv
import subprocess
import sys

path, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
f = "?"
rows = []
hdr = None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue
    try:
        rows.append((f, int(r[0]), r[1].strip(), int(r[4] or 0), int(r[7] or 0)))
    except ValueError:
        pass
ts = sum(x[3] for x in rows) or 1
te = sum(x[4] for x in rows) or 1
print(f"samples {ts:,}  warp-instr {te:,}")
by_file = {}
for x in rows:
    a = by_file.setdefault(x[0], [0, 0])
    a[0] += x[3]
    a[1] += x[4]
for k, v in sorted(by_file.items(), key=lambda kv: -kv[1][0]):
    print(f"  {k:24s} samples {100*v[0]/ts:5.1f}%  instr {100*v[1]/te:5.1f}%")
print("--- top lines by samples (file:line samples% instr%)")
for x in sorted(rows, key=lambda x: -x[3])[:top]:
    print(f"{x[0]}:{x[1]:<5d} {100*x[3]/ts:5.1f}% {100*x[4]/te:5.1f}%  {x[2][:100]}")
