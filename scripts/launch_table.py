"""Print an ncu --csv per-launch metric log as one row per launch."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
h = rows[i]
data = {}
for r in rows[i + 1:]:
    d = dict(zip(h, r))
    key = (int(d["ID"]), d["Kernel Name"].split("(")[0][-40:], d["Grid Size"])
    data.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
tot = 0.0
for k, v in sorted(data.items()):
    t = v.get("gpu__time_duration.sum", 0) / 1e3
    tot += t
    rw = (v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)) / 1e6
    print(f"{k[0]:3d} {k[1]:40s} {k[2]:14s} {t:9.1f} us  dram {rw:8.1f} MB  {rw / max(t, 1e-9):6.2f} TB/s"
          f"  inst {v.get('smsp__inst_executed.sum', 0) / 1e6:8.1f} M")
print(f"total {tot:.1f} us")
agg = {}
for k, v in data.items():
    a = agg.setdefault(k[1], [0, 0.0, 0.0])
    a[0] += 1
    a[1] += v.get("gpu__time_duration.sum", 0) / 1e3
    a[2] += (v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)) / 1e6
print("by kernel:")
for name, (n, t, mb) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {name:40s} n={n:4d} {t:10.1f} us  {100 * t / max(tot, 1e-9):5.1f}%  dram {mb:9.1f} MB  {mb / max(t, 1e-9):6.2f} TB/s")
