"""Per-kernel summary of an ncu launch list (--csv --log-file, metrics
gpu__time_duration.sum [+ dram__bytes_read.sum, dram__bytes_write.sum]):

    python scripts/launch_summary.py launches.csv [n]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
hdr = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hdr]
ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
data, names = defaultdict(dict), {}
for r in rows[hdr + 1:]:
    if len(r) > vi:
        data[r[0]][r[mi]] = (float(r[vi].replace(",", "")), r[ui])
        names[r[0]] = r[ki].split("(")[0][:60]
T = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}
Bs = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
agg = defaultdict(lambda: [0, 0.0, 0.0])
for i, d in data.items():
    t, tu = d.get("gpu__time_duration.sum", (0.0, "us"))
    b = sum(v * Bs.get(u, 1) for k, (v, u) in d.items() if k.startswith("dram__bytes"))
    a = agg[names[i]]
    a[0] += 1
    a[1] += t * T.get(tu, 1)
    a[2] += b
tot = sum(v[1] for v in agg.values()) or 1
print(f"{'n':>5s} {'avg us':>9s} {'share':>6s} {'MB/launch':>10s} {'GB/s':>7s}  kernel")
for k, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1])[:n]:
    print(f"{c:5d} {t / c:9.2f} {t / tot * 100:5.1f}% {b / c / 1e6:10.2f} {b / t / 1e3 if t else 0:7.0f}  {k}")
