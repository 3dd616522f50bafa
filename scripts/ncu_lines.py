"""Warp-stall samples of one kernel in an ncu report, summed per CUDA source
line (needs -lineinfo and --import-source on):

    python scripts/ncu_lines.py report.ncu-rep kernel_regex [n]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}", "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, acc = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit():
        try:
            s = int(r[4])
        except ValueError:
            continue
        if s:
            acc.append((s, fname, int(r[0]), r[1].strip()))
tot = sum(a[0] for a in acc) or 1
print(f"total samples {tot}")
for s, f, ln, src in sorted(acc, reverse=True)[:n]:
    print(f"{s / tot * 100:5.1f}%  {f}:{ln:<5d} {src[:90]}")
