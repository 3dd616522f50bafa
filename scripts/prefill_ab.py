"""A/B of prefill implementation choices in ONE process, interleaved so both
arms see the same power / clock state:

    python scripts/prefill_ab.py --model 2.7b --batch 32 --seqlen 8192 \
        --arm "" --arm "gemm_group_m=1" [--rounds 3] [--steps 3]

Prints ms per step and tok/s per arm and round (fields of ssd200_tuning_t)."""

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
    ap.add_argument("--model", default="2.7b")
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--seqlen", type=int, default=8192)
    ap.add_argument("--layers", type=int, default=0, help="0 = the model's")
    ap.add_argument("--arm", action="append", default=[])
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    kw = {"n_layers": args.layers} if args.layers else {}
    cfg = m.named_config(args.model, compute="bf16", **kw)
    params = m.synthetic_init(cfg, seed=0)
    tok = torch.randint(0, cfg.vocab_size, (args.batch, args.seqlen), device="cuda")
    arms = args.arm or [""]
    for rnd in range(args.rounds):
        for spec in arms:
            opts = dict(kv.split("=") for kv in filter(None, spec.split(",")))
            with _abi.tuning(**opts):
                m.prefill(params, tok, cfg, logits="last")  # warm
                torch.cuda.synchronize()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                for _ in range(args.steps):
                    m.prefill(params, tok, cfg, logits="last")
                e.record()
                torch.cuda.synchronize()
            ms = s.elapsed_time(e) / args.steps
            print(f"round {rnd} arm[{spec or 'default':>24s}] {ms:9.2f} ms/step "
                  f"{args.batch * args.seqlen / ms * 1e3:12.0f} tok/s", flush=True)


if __name__ == "__main__":
    main()
