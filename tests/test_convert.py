"""HF checkpoint converter, the reference converter's
test cases (pkg/converter/test/convert.test.ts:20-160) on synthetic HF-layout
checkpoints: every canonical tensor exactly once and in order, (out, in) ->
(in, out) transposes, the conv squeeze, bf16 storage cast to f32, unmapped
tensors reported, deterministic bytes, named errors, config translation."""

from __future__ import annotations

import json

import numpy as np
import pytest
import torch
from safetensors.torch import save_file

from paper_2603_09555_b200 import bundle, convert
from paper_2603_09555_b200.config import ModelConfig

CFG = ModelConfig(vocab_size=64, d_model=32, n_layers=2, d_state=8, head_dim=8, chunk_size=16,
                  norm_eps=1e-5)


def _hf_checkpoint(path, dtype=torch.float32, drop=None, extra=True, limit=(0.0, float("inf"))):
    g = torch.Generator().manual_seed(0)
    c = CFG

    def r(*shape):
        return torch.randn(*shape, generator=g).to(dtype)

    t = {"backbone.embeddings.weight": r(c.vocab_size, c.d_model),
         "backbone.norm_f.weight": r(c.d_model)}
    for i in range(c.n_layers):
        p = f"backbone.layers.{i}."
        t[p + "mixer.in_proj.weight"] = r(c.d_in_proj, c.d_model)   # torch Linear (out, in)
        t[p + "mixer.conv1d.weight"] = r(c.conv_dim, 1, c.conv_kernel)
        t[p + "mixer.conv1d.bias"] = r(c.conv_dim)
        t[p + "mixer.dt_bias"] = r(c.n_heads)
        t[p + "mixer.A_log"] = r(c.n_heads)
        t[p + "mixer.D"] = r(c.n_heads)
        t[p + "mixer.norm.weight"] = r(c.d_inner)
        t[p + "mixer.out_proj.weight"] = r(c.d_model, c.d_inner)
        if extra:
            t[p + "norm.weight"] = r(c.d_model)  # residual pre-norm: no engine slot
    if extra:
        t["lm_head.weight"] = t["backbone.embeddings.weight"].clone()
        t["mystery.tensor"] = r(3)
    if drop:
        t.pop(drop)
    path.mkdir(parents=True, exist_ok=True)
    save_file(t, str(path / "model.safetensors"))
    hf = {"vocab_size": c.vocab_size, "hidden_size": c.d_model, "num_hidden_layers": c.n_layers,
          "state_size": c.d_state, "head_dim": c.head_dim, "expand": c.expand,
          "n_groups": c.n_groups, "conv_kernel": c.conv_kernel, "chunk_size": c.chunk_size,
          "layer_norm_epsilon": c.norm_eps,
          "time_step_limit": [limit[0], "Infinity" if limit[1] == float("inf") else limit[1]]}
    (path / "config.json").write_text(json.dumps(hf))
    return {k: v.float().numpy() for k, v in t.items()}


def test_convert_layout_and_report(tmp_path):
    src = _hf_checkpoint(tmp_path / "hf")
    cfg, converted, unmapped = convert.convert(str(tmp_path / "hf"), str(tmp_path / "out"))
    assert cfg == CFG
    assert sorted(converted) == sorted(bundle.tensor_names(CFG))
    man = json.loads((tmp_path / "out" / "manifest.json").read_text())
    assert [e["name"] for e in man["tensors"]] == bundle.tensor_names(CFG)
    assert man["config"]["dt_limits"] == [0.0, None]
    params, _ = bundle.load_bundle_host(tmp_path / "out")
    for i, lp in enumerate(params.layers):
        p = f"backbone.layers.{i}.mixer."
        assert np.array_equal(lp.W_in, src[p + "in_proj.weight"].T)
        assert np.array_equal(lp.W_out, src[p + "out_proj.weight"].T)
        assert np.array_equal(lp.conv_w, src[p + "conv1d.weight"][:, 0, :])
        assert np.array_equal(lp.norm_w, src[p + "norm.weight"])
    assert np.array_equal(params.embedding, src["backbone.embeddings.weight"])
    assert "mystery.tensor" in unmapped
    assert "lm_head.weight (expected, no engine slot)" in unmapped
    assert "backbone.layers.0.norm.weight (expected, no engine slot)" in unmapped


def test_bf16_storage_is_cast_and_deterministic(tmp_path):
    src = _hf_checkpoint(tmp_path / "hf", dtype=torch.bfloat16, extra=False)
    convert.convert(str(tmp_path / "hf"), str(tmp_path / "a"))
    convert.convert(str(tmp_path / "hf"), str(tmp_path / "b"))
    for f in ("manifest.json", "data.bin"):
        assert (tmp_path / "a" / f).read_bytes() == (tmp_path / "b" / f).read_bytes()
    params, _ = bundle.load_bundle_host(tmp_path / "a")
    assert np.array_equal(params.final_norm_w, src["backbone.norm_f.weight"])


def test_missing_tensor_and_config_errors(tmp_path):
    _hf_checkpoint(tmp_path / "hf", drop="backbone.layers.1.mixer.D")
    with pytest.raises(bundle.MissingTensorError, match="layers.1.D"):
        convert.convert(str(tmp_path / "hf"), str(tmp_path / "out"))
    with pytest.raises(bundle.BundleError, match="does not exist"):
        convert.convert(str(tmp_path / "nope"), str(tmp_path / "out"))
    with pytest.raises(ValueError, match="hidden_size"):
        convert.translate_config({"vocab_size": 4})


def test_finite_time_step_limit(tmp_path):
    _hf_checkpoint(tmp_path / "hf", limit=(0.001, 0.1))
    cfg, _, _ = convert.convert(str(tmp_path / "hf"), str(tmp_path / "out"))
    assert cfg.dt_limits == (0.001, 0.1)


def test_keep_pre_norm_round_trip_and_oracle(tmp_path):
    """--keep-pre-norm: backbone.layers.N.norm.weight lands in the bundle as
    layers.N.pre_norm.weight (instead of being reported unmapped), the bundle
    reader returns it as pre_norm_w, and the oracle block with the pre-norm is
    residual + mixer(rmsnorm(hidden) * w) — the real state-spaces/mamba2 block."""
    import warnings

    import oracle as orc

    src = _hf_checkpoint(tmp_path / "hf")
    cfg, converted, unmapped = convert.convert(str(tmp_path / "hf"), str(tmp_path / "b"),
                                               keep_pre_norm=True)
    assert not any("layers.0.norm.weight" in u for u in unmapped)
    assert "layers.1.pre_norm.weight" in converted
    with warnings.catch_warnings():
        warnings.simplefilter("error")  # the pre-norm tensors are not "unknown"
        host, cfg2 = bundle.load_bundle_host(tmp_path / "b")
    for i in range(cfg.n_layers):
        assert np.array_equal(host.layers[i].pre_norm_w, src[f"backbone.layers.{i}.norm.weight"])
    # without the flag the reference behaviour is unchanged
    _, _, unmapped0 = convert.convert(str(tmp_path / "hf"), str(tmp_path / "b0"))
    assert any("backbone.layers.0.norm.weight" in u for u in unmapped0)
    host0, _ = bundle.load_bundle_host(tmp_path / "b0")
    assert host0.layers[0].pre_norm_w is None
    # oracle block with the pre-norm = manual composition
    rng = np.random.default_rng(3)
    hid = rng.standard_normal((2, 20, cfg.d_model)).astype(np.float32)
    lyr = host.layers[0]
    out, _, _ = orc.block(lyr, hid, cfg)
    from types import SimpleNamespace

    plain = SimpleNamespace(**{k: v for k, v in vars(lyr).items() if k != "pre_norm_w"})
    normed = orc.rms_norm(hid, lyr.pre_norm_w, cfg.norm_eps)
    mix, _, _ = orc.block(plain, normed, cfg)
    assert np.allclose(out, hid + (mix - normed), atol=1e-5, rtol=1e-5)
