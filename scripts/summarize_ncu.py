"""Summarise an ncu --csv launch list: per-kernel count, total/avg time, DRAM bytes."""
import csv, sys, collections, re

def load(path):
    rows = [r for r in csv.reader(open(path)) if r]
    # find header
    for i, r in enumerate(rows):
        if "Kernel Name" in r and "Metric Name" in r:
            hdr = r; body = rows[i+1:]; break
    ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    launches = collections.OrderedDict()
    for r in body:
        key = r[ii]
        d = launches.setdefault(key, {"name": r[ki]})
        v = r[vi].replace(",", "")
        try: d[r[mi]] = float(v)
        except ValueError: pass
    return list(launches.values())

def short(n):
    n = re.sub(r"\(.*", "", n)
    return n[:70]

if __name__ == "__main__":
    L = load(sys.argv[1])
    agg = collections.OrderedDict()
    for d in L:
        k = short(d["name"])
        a = agg.setdefault(k, [0, 0.0, 0.0])
        a[0] += 1; a[1] += d.get("gpu__time_duration.sum", 0); a[2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':72s} {'n':>4s} {'avg_us':>9s} {'share':>6s} {'MB/launch':>10s} {'GB/s':>8s}")
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:72s} {n:4d} {t/n/1e3:9.1f} {t/tot*100:5.1f}% {b/n/1e6:10.2f} {b/t if t else 0:8.0f}")
