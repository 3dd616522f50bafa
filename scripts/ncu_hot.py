"""Top stall-sampled SASS lines of one kernel in an ncu report:
    python scripts/ncu_hot.py report.ncu-rep kernel_regex [n]"""
import csv, io, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 16
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-units", "base",
                      "-k", f"regex:{kern}", "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
body = [r for r in rows[hdr + 1:] if len(r) > 3 and r[2].isdigit()]
tot = sum(int(r[2]) for r in body) or 1
print(f"total samples {tot}")
for r in sorted(body, key=lambda r: -int(r[2]))[:n]:
    print(f"{int(r[2]) / tot * 100:5.1f}%  {r[1].strip()[:100]}")
