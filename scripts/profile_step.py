"""Small, ncu-friendly driver: a few prefill or decode steps of one model
config with a reduced layer count (same per-layer shapes as the bench).

    python scripts/profile_step.py prefill --model 370m --layers 2 --batch 4 --seqlen 8192
    python scripts/profile_step.py decode  --model 1.3b --layers 2 --batch 1
"""

from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2603_09555_b200 as m  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=("prefill", "decode"))
    ap.add_argument("--model", default="370m")
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--seqlen", type=int, default=8192)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--opt", action="append", default=[], help="ssd200_tuning_t field=value")
    args = ap.parse_args()
    from paper_2603_09555_b200 import _abi

    opts = dict(kv.split("=") for kv in args.opt)
    with _abi.tuning(**opts):
        run(args)


def run(args):
    cfg = m.named_config(args.model, compute="bf16", n_layers=args.layers)
    params = m.synthetic_init(cfg, seed=0)
    if args.what == "prefill":
        tok = torch.randint(0, cfg.vocab_size, (args.batch, args.seqlen), device="cuda")
        for _ in range(args.iters):
            m.prefill(params, tok, cfg, logits="last")
    else:
        prompt = torch.randint(0, cfg.vocab_size, (args.batch, 16), device="cuda")
        _, cache = m.prefill(params, prompt, cfg, logits=None)
        dec = m.GreedyDecoder(params, cfg, cache, args.iters + 4, use_graph=False)
        for _ in range(args.iters):
            dec.step()
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
