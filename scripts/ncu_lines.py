"""Warp-stall samples of one kernel in an ncu report, summed per CUDA source
line (needs -lineinfo and --import-source on), with each line's top stall
reasons:

    python scripts/ncu_lines.py report.ncu-rep kernel_regex [n] [launch_skip]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}", "--launch-skip", skip, "-c", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, line, acc = None, None, None, {}
reasons = defaultdict(lambda: defaultdict(int))
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if not hdr:
        continue
    if r[0].isdigit():  # a source line: aggregated samples in column 4
        line = (fname, int(r[0]), r[1].strip())
        try:
            s = int(r[4])
        except ValueError:
            s = 0
        if s:
            acc[line] = s
    elif line and len(r) == len(hdr) and r[2].startswith("0x"):  # its SASS rows
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    reasons[line][h[6:]] += int(r[i])
                except ValueError:
                    pass
tot = sum(acc.values()) or 1
print(f"total samples {tot}")
for line, s in sorted(acc.items(), key=lambda kv: -kv[1])[:n]:
    f, ln, src = line
    top = sorted(reasons[line].items(), key=lambda kv: -kv[1])[:3]
    why = " ".join(f"{k}:{v}" for k, v in top if v)
    print(f"{s / tot * 100:5.1f}%  {f}:{ln:<5d} {src[:70]:70s} [{why}]")
