"""Summarise an `ncu --set full` report: one row per kernel launch with time,
DRAM bytes, tensor-pipe activity, SM / memory throughput and issue activity.

    python scripts/summarize_full.py report.ncu-rep [--traffic profiles/traffic.json]

With --traffic, also (re)writes the per-launch DRAM traffic table that
bench.py reports as roofline.traffic (keys = bench.py kernel keys).
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread",
]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

# bench.py roofline keys -> kernel-name prefixes whose launches make up one unit
GROUPS = {
    "ssd_scan": ("ssd_tc_cumsum", "ssd_tc_chunkscan", "ssd_tc_out"),
    "ssd_tc_chunkscan": ("ssd_tc_cumsum", "ssd_tc_chunkscan"),  # bench phase scan_states
    "ssd_tc_out": ("ssd_tc_out",),                                # bench phase scan_out
    "tc_gemm_kernel<256,2>": ("void tc_gemm_kernel<256, 2",),
    "tc_gemm_kernel<256,4>": ("void tc_gemm_kernel<256, 4",),
    "conv_silu_tma": ("conv_silu_tma",),
}


def rows(report):
    out = subprocess.run(
        ["ncu", "-i", report, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
        check=True, capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units, body = r[0], r[1], r[2:]
    res = []
    for row in body:
        d = {"kernel": row[hdr.index("Kernel Name")].split("(")[0]}
        for m in METRICS:
            if m not in hdr:
                continue
            i = hdr.index(m)
            try:
                v = float(row[i].replace(",", ""))
            except ValueError:
                continue
            if m.startswith("dram__bytes"):
                v *= UNIT.get(units[i], 1)
            if m == "gpu__time_duration.sum":  # normalise to microseconds
                v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
                      "second": 1e6, "s": 1e6}.get(units[i], 1.0)
            d[m] = v
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--traffic", help="traffic json to update (bench.py roofline.traffic)")
    ap.add_argument("--model", default="2.7b", help="key of the traffic table to (re)write")
    a = ap.parse_args()
    rs = rows(a.report)
    print(f"{'kernel':44s} {'us':>8s} {'DRAM MB':>8s} {'GB/s':>7s} {'SM%':>5s} "
          f"{'mem%':>5s} {'issue%':>6s} {'tensor%':>7s} {'regs':>4s}")
    for d in rs:
        t = d.get("gpu__time_duration.sum", 0.0)
        b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        print(f"{d['kernel'][:44]:44s} {t:8.1f} {b / 1e6:8.1f} {b / (t * 1e3) if t else 0:7.0f} "
              f"{d.get(METRICS[3], 0):5.1f} {d.get(METRICS[4], 0):5.1f} "
              f"{d.get(METRICS[5], 0):6.1f} {d.get(METRICS[6], 0):7.1f} {d.get(METRICS[7], 0):4.0f}")
    if a.traffic:
        try:
            with open(a.traffic) as f:
                full = json.load(f)
        except (OSError, ValueError):
            full = {}
        table = dict(full.get(a.model, {}))
        for key, names in GROUPS.items():
            tot, seen = 0.0, False
            for n in names:
                hit = [d for d in rs if d["kernel"].startswith(n)]
                if hit:
                    seen = True
                    tot += hit[0].get("dram__bytes_read.sum", 0.0) + hit[0].get("dram__bytes_write.sum", 0.0)
            if seen:
                table[key] = tot
        full[a.model] = table
        with open(a.traffic, "w") as f:
            json.dump(full, f, indent=1)
        print("wrote", a.traffic, a.model, table)


if __name__ == "__main__":
    main()
