"""Phase timeline of the fused decode step (CTA 0 %globaltimer stamps).

    python scripts/trace_decode.py --model 1.3b --batch 1
"""

from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_09555_b200 as m  # noqa: E402
from paper_2603_09555_b200 import _abi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="1.3b")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--prefetch", type=int, default=1)
    args = ap.parse_args()
    kw = {"n_layers": args.layers} if args.layers else {}
    cfg = m.named_config(args.model, compute="bf16", **kw)
    params = m.synthetic_init(cfg, seed=0)
    _abi.lib().ssd200_set_option(3, args.prefetch)
    prompt = torch.randint(0, cfg.vocab_size, (args.batch, 16), device="cuda")
    _, cache = m.prefill(params, prompt, cfg, logits=None)
    dec = m.GreedyDecoder(params, cfg, cache, 20, use_graph=False)
    for _ in range(3):
        dec.step()
    buf = torch.zeros(8192, dtype=torch.int64, device="cuda")
    _abi.lib().ssd200_debug_trace(buf.data_ptr())
    torch.cuda.synchronize()
    dec.step()
    torch.cuda.synchronize()
    _abi.lib().ssd200_debug_trace(None)
    t = buf.cpu().numpy().astype(np.float64)
    L = cfg.n_layers
    t0 = t[0]
    names = ["stage_x", "P1_gemv", "P1_bar", "P2", "P2_bar", "P3_stage", "P3_gemv", "P3_bar"]
    durs = np.zeros(8)
    for l in range(L):
        row = t[l * 8:(l + 1) * 8]
        nxt = t[(l + 1) * 8] if l + 1 < L else t[4000]
        seg = np.diff(np.concatenate([row, [nxt]]))
        durs += seg
        if l < 3 or l == L - 1:
            print(f"layer {l:2d} start {(row[0]-t0)/1e3:8.1f} us  " +
                  " ".join(f"{n}={d/1e3:6.2f}" for n, d in zip(names, seg)))
    print("mean per layer (us):", " ".join(f"{n}={d/L/1e3:.2f}" for n, d in zip(names, durs)))
    print(f"layers total {(t[4000]-t0)/1e3:.1f} us, head {(t[4001]-t[4000])/1e3:.1f} us")
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    p1e = t[5000:5000 + nsm]
    p1x = t[5200:5200 + nsm]
    if p1e.min() > 0:
        print(f"layer-1 P1 end over CTAs: min {(p1e.min()-t0)/1e3:.1f} median {(np.median(p1e)-t0)/1e3:.1f} "
              f"max {(p1e.max()-t0)/1e3:.1f} us (slowest CTA {int(p1e.argmax())}); barrier exit "
              f"min {(p1x.min()-t0)/1e3:.1f} max {(p1x.max()-t0)/1e3:.1f} us")
        order = np.argsort(p1e)[-8:]
        print("slowest CTAs:", [(int(i), round((p1e[i]-t0)/1e3, 1)) for i in order])
    prod = t[4096:4096 + 2 * L + 1]
    print("producer done W_in/W_out per layer (us from t0):",
          " ".join(f"{(p-t0)/1e3:.0f}" for p in prod[:8]), "... E at", f"{(prod[-1]-t0)/1e3:.0f}")



    arr = t[5400:5400 + nsm]
    rel = t[5600:5600 + nsm]
    if arr.min() > 0:
        print(f"layer-1 P1 barrier: CTA arrival min {(arr.min()-t0)/1e3:.1f} max {(arr.max()-t0)/1e3:.1f} us; "
              f"release seen min {(rel.min()-t0)/1e3:.1f} max {(rel.max()-t0)/1e3:.1f} us; "
              f"thread-0 P1 end -> CTA arrival: max {(arr - p1e).max()/1e3:.2f} us")


    ps = t[6000:6000 + 40]
    cs = t[6600:6600 + 40]
    print("pf_ahead", int(t[7000]), "pf_bytes", int(t[7001]), "cp_bytes", int(t[7002]))
    print("stage k: producer slot acquired / consumer warp0 data ready (us from t0)")
    for k in range(0, 24):
        print(f"  {k:2d} {(ps[k]-t0)/1e3:8.2f} {(cs[k]-t0)/1e3:8.2f}")

if __name__ == "__main__":
    main()
