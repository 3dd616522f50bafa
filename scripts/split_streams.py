"""Experiment: a wide decode batch as two half-batch chains on two CUDA
streams in one graph, so one half's HBM-bound state stream can overlap the
other half's tensor-core GEMMs (rows are independent).  Prints ms per token
step for the single chain and the split chains, and checks the tokens agree.

    python scripts/split_streams.py --batch 256 --parts 2
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
from paper_2603_09555_b200.cache import Mamba2Cache  # noqa: E402
from paper_2603_09555_b200.decode import _step_into  # noqa: E402
from paper_2603_09555_b200.model import _Runner  # noqa: E402


def timed(fn, n):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="1.3b")
    ap.add_argument("--batch", type=int, action="append", default=[])
    ap.add_argument("--parts", type=int, action="append", default=[])
    ap.add_argument("--steps", type=int, default=32)
    args = ap.parse_args()
    cfg = m.named_config(args.model, compute="bf16")
    params = m.synthetic_init(cfg, seed=0)
    for B in args.batch or [256]:
        prompt = torch.randint(0, cfg.vocab_size, (B, 16), device="cuda")
        _, cache0 = m.prefill(params, prompt, cfg, logits=None)
        for parts in args.parts or [1, 2]:
            cache = cache0.copy()
            rows = B // parts
            chains = []
            for j in range(parts):
                sl = slice(j * rows, (j + 1) * rows)
                c = Mamba2Cache(cache.ssm_all[:, sl], cache.conv_all[:, sl])
                tok = torch.zeros((rows,), dtype=torch.int64, device="cuda")
                lg = torch.empty((rows, cfg.vocab_size), dtype=torch.float32, device="cuda")
                chains.append((_Runner(params, cfg), c, tok, lg))
            streams = [torch.cuda.Stream() for _ in range(parts)]

            def body():
                cur = torch.cuda.current_stream()
                for (r, c, tok, lg), s in zip(chains, streams):
                    s.wait_stream(cur)
                    with torch.cuda.stream(s):
                        r.stream = _abi.stream_handle(s)
                        _step_into(r, cfg, tok, c, c, logits=lg, argmax=tok)
                for s in streams:
                    cur.wait_stream(s)

            body()  # warm-up (workspaces, attributes)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                body()
            ms = timed(g.replay, args.steps)
            toks = torch.cat([ch[2] for ch in chains])
            gbs = m.decode_step_bytes(cfg, B) / ms / 1e6
            print(f"B={B:4d} parts={parts} {ms:8.3f} ms/step {gbs:7.0f} GB/s "
                  f"tok-checksum={int(toks.sum())}", flush=True)
            del g, chains, cache


if __name__ == "__main__":
    main()
