"""Decode step time under library options (tuning sweeps).

    python scripts/decode_opts.py --batch 64 --set "" --set "dec_pdl=0" --set "dec_split_in=1,dec_split_out=1"

(fields of ssd200_tuning_t, passed per call through _abi.tuning)
"""

from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2603_09555_b200 as m  # noqa: E402
from paper_2603_09555_b200 import _abi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="1.3b")
    ap.add_argument("--batch", type=int, action="append", default=[])
    ap.add_argument("--steps", type=int, default=32)
    ap.add_argument("--set", action="append", default=[])
    args = ap.parse_args()
    cfg = m.named_config(args.model, compute="bf16")
    params = m.synthetic_init(cfg, seed=0)
    for B in args.batch or [64]:
        prompt = torch.randint(0, cfg.vocab_size, (B, 16), device="cuda")
        _, cache = m.prefill(params, prompt, cfg, logits=None)
        for spec in args.set or [""]:
            opts = {}
            for kv in filter(None, spec.split(",")):
                k, v = kv.split("=")
                opts[k] = int(v)
            with _abi.tuning(**opts):  # the graph captures the tuned launches
                dec = m.GreedyDecoder(params, cfg, cache, args.steps + 8)
                for _ in range(3):
                    dec.step()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(args.steps):
                dec.step()
            e.record()
            torch.cuda.synchronize()
            ms = s.elapsed_time(e) / args.steps
            gbs = m.decode_step_bytes(cfg, B) / ms / 1e6
            print(f"B={B:4d} opts[{spec or 'default':>12s}] {ms:8.3f} ms/step  {gbs:7.0f} GB/s",
                  flush=True)
            del dec


if __name__ == "__main__":
    main()
