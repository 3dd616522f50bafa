"""Executed warp instructions of one kernel in an ncu report, summed per CUDA
source line (needs -lineinfo and --import-source on), with the SASS opcode mix
of each line:

    python scripts/ncu_inst_lines.py report.ncu-rep kernel_regex [n] [launch_skip]
"""
import csv
import io
import subprocess
import sys
from collections import Counter, defaultdict

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}", "--launch-skip", skip, "-c", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, line = None, None, None
inst = Counter()
ops = defaultdict(Counter)
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        continue
    if not hdr:
        continue
    if r[0].isdigit():
        line = (fname, int(r[0]), r[1].strip())
    elif line and len(r) == len(hdr) and r[2].startswith("0x"):
        try:
            v = int(r[ie])
        except ValueError:
            v = 0
        if v:
            inst[line] += v
            op = r[3].split()[0] if r[3].split() else "?"
            if op.startswith("@"):
                op = r[3].split()[1]
            ops[line][op.split(".")[0]] += v
tot = sum(inst.values()) or 1
print(f"total warp instructions {tot}")
for line, v in inst.most_common(n):
    f, ln, src = line
    mix = " ".join(f"{k}:{c * 100 // v}%" for k, c in ops[line].most_common(4))
    print(f"{v / tot * 100:5.1f}%  {f}:{ln:<5d} {src[:60]:60s} [{mix}]")
