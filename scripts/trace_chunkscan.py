"""Per-chunk clock timeline of ssd_tc_chunkscan's CTA 0.

    python scripts/trace_chunkscan.py
Columns (cycles from the producer's first stamp): producer stage free | MMA: X scaled,
accumulator free | math: stage landed, scale done, S ready, state updated.
"""
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
    t = buf.cpu().numpy().astype(np.float64)[4096:4096 + 64 * 8].reshape(64, 8)
    t0 = t[0, 0]
    print("chunk | prod_free | mma_xsd mma_tfree | land scaled sready updated")
    for c in range(32):
        r = t[c]
        print(f"{c:3d} " + " ".join(f"{v - t0:8.0f}" if v > 0 else "       -" for v in r[:7]))


if __name__ == "__main__":
    main()
