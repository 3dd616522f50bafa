"""Per-head clock timeline of ssd_tc_out's CTA 0 (MMA warp + first math warp).

    python scripts/trace_ssd_out.py

Columns are clock64 offsets (cycles) from the MMA warp's first loop entry.
MMA warp: loop start, yfree ok, prev ok, mrdy[0..3] ok, last MMA issued.
Math warp: iteration start, build_m(i+1) done, bar_y(i) ok, epilogue done.
"""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_09555_b200 as m  # noqa: E402
from paper_2603_09555_b200 import _abi  # noqa: E402


def main():
    cfg = m.named_config("370m", compute="bf16", n_layers=1)
    params = m.synthetic_init(cfg, seed=0)
    tok = torch.randint(0, cfg.vocab_size, (4, 8192), device="cuda")
    m.prefill(params, tok, cfg, logits="last")
    buf = torch.zeros(8192, dtype=torch.int64, device="cuda")
    _abi.lib().ssd200_debug_trace(buf.data_ptr())
    m.prefill(params, tok, cfg, logits="last")
    torch.cuda.synchronize()
    _abi.lib().ssd200_debug_trace(None)
    t = buf.cpu().numpy().astype(np.float64)
    mma = t[:512].reshape(64, 8)
    mat = t[1024:1024 + 512].reshape(64, 8)
    n = int((mma[:, 0] > 0).sum())
    t0 = mma[0, 0]

    def rel(v):
        return f"{v - t0:7.0f}" if v > 0 else "      -"

    print("head | mma: start  yfree   prev  kb0    kb1    kb2    kb3    issued | "
          "math: start  built  y_ok   epi_done")
    for i in range(n):
        a, b = mma[i], mat[i]
        print(f"{i:3d}  | " + " ".join(rel(a[k]) for k in (0, 1, 2, 3, 4, 5, 6, 7))
              + " | " + " ".join(rel(b[k]) for k in range(4)))
    warp_detail(t)
    d = t[6144:6144 + 256].reshape(16, 16)
    w = t[2048:2048 + 16 * 16 * 8].reshape(16, 16, 8)
    print("warp 0 build(h) steps from iteration start: commit fetch diag chunk0..6")
    for h in range(1, 16):
        t0 = w[0, h - 1, 0]
        print(f"{h:3d} " + " ".join(f"{v - t0:6.0f}" for v in d[h, :10]))




def warp_detail(t):
    """Per math warp and head i: [build(i+1) math | st wait | y wait | epilogue] cycles."""
    d = t[2048:2048 + 16 * 16 * 8].reshape(16, 16, 8)
    print("warp  head: build-math/st-wait/ywait/epi")
    for w in range(16):
        row = []
        for i in range(16):
            a = d[w, i]
            if a[0] <= 0:
                continue
            if a[4] > 0:
                row.append(f"{a[4]-a[0]:5.0f}/{a[5]-a[4]:4.0f}/{a[2]-a[1]:5.0f}/{a[3]-a[2]:5.0f}")
            else:
                row.append(f"{a[1]-a[0]:5.0f}/   -/{a[2]-a[1]:5.0f}/{a[3]-a[2]:5.0f}")
        if row:
            print(f"w{w:2d} " + " ".join(row[:7]))


if __name__ == "__main__":
    main()
