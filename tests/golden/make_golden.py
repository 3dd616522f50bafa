"""Generate golden vectors from the REAL reference engine (run in the build
container, where /root/reference exists; the GPU box only reads the .npz).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Fixtures written next to this script:
  ssd_cases.npz     ssd_forward (ssd.py:209) + sequential_ssm (oracle.py:42)
                    outputs on seeded instances, incl. padding / T=1 / G=H /
                    initial-state / L=1 edge cases, f64 and f32.
  small_model.npz   prefill / decode_step / generate (model.py:177,
                    decode.py:77,147) on the reference test config
                    (tests/conftest.py:42-57), f32 and f64, several seeds.
  c1_130m.npz       config 1: 130M random_init(seed 0) f32, prompt 512 tokens
                    (seed 0), generate(gen_len=65) tokens + logits.
  weights_digest.npz per-tensor float64 sums of random_init weights, pinning
                    the Philox draw order of our re-implementation.
  ref_bundle/       manifest.json + data.bin written by the reference's
                    save_bundle (bundle.py:134-168) for random_init(small
                    config with d_model 16, 1 layer, seed 9): pins the bundle
                    format byte for byte.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import ssd_engine as se  # noqa: E402  (the reference itself)
from ssd_engine import ModelConfig, SsdInputs  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def small_config(**overrides) -> ModelConfig:
    kw = dict(
        vocab_size=64, d_model=32, n_layers=2, d_state=8, head_dim=8, expand=2,
        n_groups=1, conv_kernel=4, chunk_size=16, norm_eps=1e-12,
    )
    kw.update(overrides)
    return ModelConfig(**kw)


def make_instance(rng, batch, seq, heads, pdim, ndim, groups):
    """Same distributions as the reference fixture (tests/conftest.py:7-24)."""
    return dict(
        X=rng.standard_normal((batch, seq, heads, pdim)),
        dt=rng.uniform(0.0, 1.2, size=(batch, seq, heads)),
        a=-rng.uniform(0.3, 4.0, size=heads),
        B=rng.standard_normal((batch, seq, groups, ndim)),
        C=rng.standard_normal((batch, seq, groups, ndim)),
    )


SSD_SHAPES = [
    # (batch, seq, heads, pdim, ndim, groups, chunk, with_init)
    (1, 16, 2, 4, 4, 1, 4, False),
    (2, 37, 3, 5, 6, 3, 8, False),      # pad, G == H
    (1, 1, 2, 8, 8, 1, 256, False),     # T = 1 padded to one 256 chunk
    (2, 300, 4, 8, 8, 1, 128, True),    # pad + initial state
    (1, 64, 2, 4, 3, 2, 1, False),      # L = 1
    (1, 512, 2, 16, 16, 1, 256, False), # two full chunks at L = 256
    (1, 257, 2, 64, 128, 1, 256, True), # production head dims, ragged tail
    (1, 70, 4, 8, 8, 2, 64, True),
]


def gen_ssd_cases():
    rng = np.random.default_rng(20261018)
    out = {"n": len(SSD_SHAPES)}
    for i, (b, t, h, p, n, g, L, with_init) in enumerate(SSD_SHAPES):
        inst = make_instance(rng, b, t, h, p, n, g)
        init = rng.standard_normal((b, h, p, n)) if with_init else None
        for k, v in inst.items():
            out[f"{i}.{k}"] = v
        out[f"{i}.L"] = L
        out[f"{i}.has_init"] = int(with_init)
        if with_init:
            out[f"{i}.init"] = init
        for tag, dt in (("f64", np.float64), ("f32", np.float32)):
            si = SsdInputs(
                X=inst["X"].astype(dt), dt=inst["dt"].astype(dt), a=inst["a"].astype(dt),
                Bmat=inst["B"].astype(dt), Cmat=inst["C"].astype(dt),
            )
            res = se.ssd_forward(si, L, initial_state=None if init is None else init.astype(dt))
            out[f"{i}.Y_{tag}"] = res.Y
            out[f"{i}.final_{tag}"] = res.final_state
        Ys, hs = se.sequential_ssm(inst["X"], inst["dt"], inst["a"], inst["B"], inst["C"],
                                   initial_state=init)
        out[f"{i}.Y_seq"] = Ys
        out[f"{i}.final_seq"] = hs
    np.savez_compressed(os.path.join(HERE, "ssd_cases.npz"), **out)


SMALL_MODELS = [
    # (name, overrides, seed)
    ("base", {}, 2),
    ("k2", dict(d_model=8, n_layers=1, head_dim=4, d_state=4, conv_kernel=2, chunk_size=4), 3),
    ("wide", dict(d_model=64, n_layers=4), 1),
    ("grp", dict(d_model=32, n_groups=2, head_dim=8), 7),
]


def gen_small_model():
    out = {"names": np.array([m[0] for m in SMALL_MODELS])}
    for name, ov, seed in SMALL_MODELS:
        for comp in ("f32", "f64"):
            cfg = small_config(**ov).with_policy(compute=comp)
            params = se.random_init(cfg, seed)
            rng = np.random.default_rng(100 + seed)
            toks = rng.integers(0, cfg.vocab_size, size=(2, 21))
            logits, cache = se.prefill(params, toks, cfg)
            key = f"{name}.{comp}"
            out[f"{key}.tokens"] = toks
            out[f"{key}.logits"] = logits
            out[f"{key}.ssm"] = np.stack(cache.ssm)
            out[f"{key}.conv"] = np.stack(cache.conv)
            nxt = rng.integers(0, cfg.vocab_size, size=(2,))
            step_logits, cache2 = se.decode_step(params, cache, nxt, cfg)
            out[f"{key}.next"] = nxt
            out[f"{key}.step_logits"] = step_logits
            out[f"{key}.step_ssm"] = np.stack(cache2.ssm)
            out[f"{key}.step_conv"] = np.stack(cache2.conv)
            prompt = rng.integers(0, cfg.vocab_size, size=(1, 16))
            res = se.generate(params, prompt, 64, mode="cached", cfg=cfg)
            out[f"{key}.prompt"] = prompt
            out[f"{key}.gen"] = res.tokens
        # bf16e ablation (decay_exp rounding) in f32
        cfg = small_config(**ov).with_policy(decay_exp="bf16e")
        params = se.random_init(cfg, seed)
        toks = np.random.default_rng(200 + seed).integers(0, cfg.vocab_size, size=(1, 19))
        out[f"{name}.bf16e.tokens"] = toks
        out[f"{name}.bf16e.logits"] = se.prefill(params, toks, cfg)[0]
    np.savez_compressed(os.path.join(HERE, "small_model.npz"), **out)


C1_TAP_ROWS = [0, 1, 127, 255, 256, 383, 510, 511]


def c1_config() -> ModelConfig:
    return ModelConfig(vocab_size=50288, d_model=768, n_layers=24)


def gen_c1():
    cfg = c1_config()
    t0 = time.perf_counter()
    params = se.random_init(cfg, 0)
    prompt = np.random.default_rng(0).integers(0, cfg.vocab_size, size=(1, 512))
    res = se.generate(params, prompt, 65, mode="cached", cfg=cfg, keep_logits=True)
    lg = res.per_step_logits[0]  # (65, V)
    srt = np.sort(lg, axis=-1)
    out = dict(
        prompt=prompt,
        tokens=res.tokens,
        logits_first=lg[0].astype(np.float32),   # last prefill position
        logits_last=lg[-1].astype(np.float32),   # after 64 decode steps
        top2_gap=(srt[:, -1] - srt[:, -2]).astype(np.float32),
    )
    # one block's hidden output on the prompt (layer 0), rows 0..3 and tail
    hidden0 = params.embedding[prompt]
    h1, s1, c1 = se.block_forward(params.layers[0], hidden0, cfg)
    out["layer0_hidden_rows"] = h1[0, [0, 1, 255, 256, 510, 511]].astype(np.float32)
    out["layer0_state_head0"] = s1[0, 0].astype(np.float32)
    out["layer0_conv_tail"] = c1[0].astype(np.float32)
    # the residual stream after every layer (model.py:198-203 re-run block by
    # block): sampled rows (chunk edges included) + full-tensor norm and sum
    h = hidden0
    rows, norms, sums = [], [], []
    for lyr in params.layers:
        h, _, _ = se.block_forward(lyr, h, cfg)
        rows.append(h[0, C1_TAP_ROWS].astype(np.float32))
        norms.append(float(np.linalg.norm(h)))
        sums.append(float(h.sum(dtype=np.float64)))
    out["tap_rows"] = np.stack(rows)
    out["tap_norm"] = np.asarray(norms)
    out["tap_sum"] = np.asarray(sums)
    # bf16 mode: the reference on the SAME bf16-rounded weights,
    # f32 compute: greedy tokens + the first step's logits
    pb = se.random_init(cfg, 0)
    rne = lambda a: se.numerics.bf16_round(a).astype(a.dtype)  # noqa: E731
    for lyr in pb.layers:
        lyr.W_in, lyr.W_out = rne(lyr.W_in), rne(lyr.W_out)
    pb.embedding = rne(pb.embedding)
    rb = se.generate(pb, prompt, 65, mode="cached", cfg=cfg, keep_logits=True)
    out["bf16w_tokens"] = rb.tokens
    out["bf16w_logits_first"] = rb.per_step_logits[0, 0].astype(np.float32)
    np.savez_compressed(os.path.join(HERE, "c1_130m.npz"), **out)
    print(f"c1 golden in {time.perf_counter() - t0:.1f}s tokens={res.tokens[0, :8]}...")


def gen_digest():
    out = {}
    for name, cfg, seed in (
        ("small", small_config(), 2),
        ("c1", c1_config(), 0),
    ):
        p = se.random_init(cfg, seed)
        out[f"{name}.embedding"] = np.float64(p.embedding.astype(np.float64).sum())
        out[f"{name}.embedding_first"] = p.embedding[:2, :8]
        for i in (0, cfg.n_layers - 1):
            l = p.layers[i]
            for f in ("W_in", "conv_w", "dt_bias", "A_log", "D", "W_out"):
                out[f"{name}.{i}.{f}"] = np.float64(getattr(l, f).astype(np.float64).sum())
        out[f"{name}.n_params"] = se.n_params(cfg)
    np.savez_compressed(os.path.join(HERE, "weights_digest.npz"), **out)


def gen_bundle():
    cfg = small_config(d_model=16, n_layers=1, vocab_size=32)
    se.save_bundle(se.random_init(cfg, 9), cfg, os.path.join(HERE, "ref_bundle"))


if __name__ == "__main__":
    which = sys.argv[1:] or ["ssd", "small", "digest", "c1", "bundle"]
    if "ssd" in which:
        gen_ssd_cases()
    if "small" in which:
        gen_small_model()
    if "digest" in which:
        gen_digest()
    if "c1" in which:
        gen_c1()
    if "bundle" in which:
        gen_bundle()
    print("golden fixtures written to", HERE)
