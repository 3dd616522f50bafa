"""Run the same bf16 prefill (370M width, 1 layer, B=4, T=2048) many times and
count runs whose hidden state differs bitwise from the first (a race detector)."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
import paper_2603_09555_b200 as m  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
cfg = m.named_config("370m", compute="bf16", vocab_size=512, n_layers=1)
params = m.from_reference(m.random_init_host(cfg, 91), cfg)
toks = torch.as_tensor(np.random.default_rng(92).integers(0, cfg.vocab_size, size=(4, 2048))).cuda()
_, _, base = m.prefill(params, toks, cfg, logits="last", return_hidden=True)
base = base.clone()
bad = 0
worst = 0.0
for _ in range(n):
    _, _, h = m.prefill(params, toks, cfg, logits="last", return_hidden=True)
    if not torch.equal(h, base):
        bad += 1
        worst = max(worst, (h - base).abs().max().item())
print(f"mismatching runs: {bad} / {n}  worst |d| {worst:.3e}")
