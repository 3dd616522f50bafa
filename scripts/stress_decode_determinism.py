"""Decode determinism stress: graph-replayed generate vs eager, bitwise, at the
state stream's tile hand-out modes (counter chunks at B = 160 / 256, register state
at B = 1).  python scripts/stress_decode_determinism.py"""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2603_09555_b200 as m
for model, B, steps in (("370m", 256, 24), ("1.3b", 1, 64), ("370m", 1, 64), ("370m", 160, 24)):
    cfg = m.named_config(model, compute="bf16", vocab_size=512, n_layers=2)
    params = m.from_reference(m.random_init_host(cfg, 5), cfg)
    toks = np.random.default_rng(6).integers(0, cfg.vocab_size, size=(B, 9))
    ref = m.generate(params, toks, steps, cfg=cfg, use_graph=False, keep_logits=True)
    bad = 0
    for rep in range(3):
        g = m.generate(params, toks, steps, cfg=cfg, use_graph=True, keep_logits=True)
        bad += int(not (torch.equal(g.tokens, ref.tokens) and torch.equal(g.per_step_logits, ref.per_step_logits)))
        m.decode.clear_graph_cache()
    print(model, B, steps, "mismatching graph runs:", bad, flush=True)
