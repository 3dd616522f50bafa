"""HuggingFace Mamba-2 checkpoint -> bundle converter.

A Python restatement of the reference's TypeScript converter
(pkg/converter/src/convert.ts, mapping.ts, safetensors.ts; node is not in this
image) producing the same bundle: the tensor mapping of pkg/converter/
mapping.json (HF ``backbone.*`` names -> canonical names, torch Linear
(out, in) transposed to the engine's row-vector (in, out), depthwise conv
(C, 1, k) squeezed to (C, k)), HF config.json fields translated the same way
(``time_step_limit`` infinity -> null), every tensor cast to float32 from F32 /
BF16 / F16 / F64 storage, deterministic output.  Source tensors without an
engine slot are reported, never silently dropped: the per-block residual
pre-norm (the reference block has none, mapping.json "known_unmapped") and the
tied ``lm_head``.  ``keep_pre_norm=True`` (``--keep-pre-norm``) instead carries
the pre-norm weights into the bundle as ``layers.N.pre_norm.weight``, which
this package's block applies (``LayerParams.pre_norm_w``), so real
state-spaces/mamba2 checkpoints compute what they were trained to.

    python -m paper_2603_09555_b200.convert --source <hf dir> --out <bundle dir>
"""

from __future__ import annotations

import json
import math
import os
from types import SimpleNamespace

import numpy as np

from .bundle import BundleError, MissingTensorError, TensorShapeError, save_bundle, tensor_shape
from .config import ModelConfig

# mapping.json "config_fields": HF config.json key -> engine field
CONFIG_FIELDS = {
    "vocab_size": "vocab_size",
    "hidden_size": "d_model",
    "num_hidden_layers": "n_layers",
    "state_size": "d_state",
    "head_dim": "head_dim",
    "expand": "expand",
    "n_groups": "n_groups",
    "conv_kernel": "conv_kernel",
    "chunk_size": "chunk_size",
    "layer_norm_epsilon": "norm_eps",
    "time_step_limit": "dt_limits",
}

# mapping.json "tensors": (source pattern, canonical target, transform)
TENSOR_RULES = (
    ("backbone.embeddings.weight", "embedding", "none"),
    ("backbone.layers.{i}.mixer.in_proj.weight", "layers.{i}.in_proj.weight", "transpose2d"),
    ("backbone.layers.{i}.mixer.conv1d.weight", "layers.{i}.conv1d.weight", "squeeze_mid"),
    ("backbone.layers.{i}.mixer.conv1d.bias", "layers.{i}.conv1d.bias", "none"),
    ("backbone.layers.{i}.mixer.dt_bias", "layers.{i}.dt_bias", "none"),
    ("backbone.layers.{i}.mixer.A_log", "layers.{i}.A_log", "none"),
    ("backbone.layers.{i}.mixer.D", "layers.{i}.D", "none"),
    ("backbone.layers.{i}.mixer.norm.weight", "layers.{i}.norm.weight", "none"),
    ("backbone.layers.{i}.mixer.out_proj.weight", "layers.{i}.out_proj.weight", "transpose2d"),
    ("backbone.norm_f.weight", "final_norm.weight", "none"),
)
KNOWN_UNMAPPED = ("backbone.layers.{i}.norm.weight", "lm_head.weight")

_LEAF_ATTR = {"in_proj.weight": "W_in", "conv1d.weight": "conv_w", "conv1d.bias": "conv_b",
              "dt_bias": "dt_bias", "A_log": "A_log", "D": "D", "norm.weight": "norm_w",
              "out_proj.weight": "W_out"}


def _limit(value, fallback):
    """mapping.ts normalizeLimit: None -> fallback; non-finite -> None (null)."""
    if value is None:
        return fallback
    if isinstance(value, (int, float)):
        return float(value) if math.isfinite(value) else None
    if isinstance(value, str):
        try:
            v = float(value)
        except ValueError:
            raise ValueError(f"cannot interpret dt limit {value!r}") from None
        return v if math.isfinite(v) else None
    raise ValueError(f"cannot interpret dt limit {value!r}")


def translate_config(raw: dict) -> ModelConfig:
    """mapping.ts translateConfig: every mapped field is required."""
    cfg = {}
    for src, dst in CONFIG_FIELDS.items():
        if src not in raw:
            raise ValueError(f"config.json is missing required field '{src}'")
        cfg[dst] = raw[src]
    limits = cfg["dt_limits"] or [None, None]
    lo, hi = _limit(limits[0] if len(limits) > 0 else None, 0.0), _limit(
        limits[1] if len(limits) > 1 else None, None)
    cfg["dt_limits"] = (float(lo), float("inf") if hi is None else float(hi))
    return ModelConfig(**cfg)


def _expand(pattern: str, n_layers: int):
    return [pattern.replace("{i}", str(i)) for i in range(n_layers)] if "{i}" in pattern else [pattern]


def apply_transform(arr: np.ndarray, transform: str) -> np.ndarray:
    """mapping.ts applyTransform."""
    if transform == "none":
        return arr
    if transform == "squeeze_mid":
        if arr.ndim != 3 or arr.shape[1] != 1:
            raise ValueError(f"squeeze_mid expects (C, 1, k), got {list(arr.shape)}")
        return arr[:, 0, :]
    if transform == "transpose2d":
        if arr.ndim != 2:
            raise ValueError(f"transpose2d expects a matrix, got {list(arr.shape)}")
        return np.ascontiguousarray(arr.T)
    raise ValueError(f"unknown transform {transform}")


def _read_checkpoint(source: str):
    """convert.ts loadCheckpoint + safetensors.ts: config.json and every
    *.safetensors file (sorted), tensors decoded to float32."""
    if not os.path.isdir(source):
        raise BundleError(f"source {source} does not exist (remote repo ids are not fetched; "
                          f"pass a local checkout)")
    cfg_path = os.path.join(source, "config.json")
    if not os.path.exists(cfg_path):
        raise BundleError(f"missing config.json under {source}")
    with open(cfg_path, encoding="utf-8") as f:
        raw_cfg = json.load(f)
    files = sorted(f for f in os.listdir(source) if f.endswith(".safetensors"))
    if not files:
        raise BundleError(f"no .safetensors files under {source}")
    from safetensors import safe_open

    tensors = {}
    for fn in files:
        with safe_open(os.path.join(source, fn), framework="pt") as f:
            for name in f.keys():
                # torch decodes F32 / BF16 / F16 / F64; bf16 -> f32 is exact
                tensors[name] = f.get_tensor(name).float().numpy()
    return raw_cfg, tensors


PRE_NORM_RULE = ("backbone.layers.{i}.norm.weight", "layers.{i}.pre_norm.weight", "none")


def convert(source: str, out: str, keep_pre_norm: bool = False):
    """convert.ts convert: HF checkpoint dir -> bundle dir.  Returns
    (cfg, converted canonical names, unmapped source names)."""
    raw_cfg, tensors = _read_checkpoint(source)
    cfg = translate_config(raw_cfg)
    rules = {}
    for src, dst, tr in TENSOR_RULES + ((PRE_NORM_RULE,) if keep_pre_norm else ()):
        for s_name, d_name in zip(_expand(src, cfg.n_layers), _expand(dst, cfg.n_layers)):
            rules[s_name] = (d_name, tr)
    known = {n for p in KNOWN_UNMAPPED for n in _expand(p, cfg.n_layers)} - set(rules)
    produced, unmapped = {}, []
    for name in sorted(tensors):
        if name not in rules:
            unmapped.append(f"{name} (expected, no engine slot)" if name in known else name)
            continue
        target, tr = rules[name]
        if target in produced:
            raise BundleError(f"duplicate production of canonical tensor {target}")
        arr = apply_transform(np.asarray(tensors[name], dtype=np.float32), tr)
        want = (cfg.d_model,) if target.endswith("pre_norm.weight") else tensor_shape(target, cfg)
        if tuple(arr.shape) != tuple(want):
            raise TensorShapeError(f"{target}: shape {list(arr.shape)} != expected {list(want)}")
        produced[target] = arr
    for _, dst, _ in TENSOR_RULES + ((PRE_NORM_RULE,) if keep_pre_norm else ()):
        for d_name in _expand(dst, cfg.n_layers):
            if d_name not in produced:
                raise MissingTensorError(f"missing canonical tensor {d_name}")
    layers = []
    for i in range(cfg.n_layers):
        layers.append(SimpleNamespace(**{attr: produced[f"layers.{i}.{leaf}"]
                                         for leaf, attr in _LEAF_ATTR.items()},
                                      pre_norm_w=produced.get(f"layers.{i}.pre_norm.weight")))
    params = SimpleNamespace(embedding=produced["embedding"], layers=layers,
                             final_norm_w=produced["final_norm.weight"])
    save_bundle(params, cfg, out)
    return cfg, list(produced), unmapped


def main(argv=None) -> int:
    import argparse

    ap = argparse.ArgumentParser(description="HF Mamba-2 checkpoint -> bundle")
    ap.add_argument("--source", required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--keep-pre-norm", action="store_true",
                    help="carry backbone.layers.N.norm into the bundle (applied by this engine)")
    args = ap.parse_args(argv)
    cfg, converted, unmapped = convert(args.source, args.out, keep_pre_norm=args.keep_pre_norm)
    print(f"converted {len(converted)} tensors ({cfg.n_layers} layers, d_model={cfg.d_model}) "
          f"-> {args.out}")
    for name in unmapped:
        print(f"  unmapped: {name}")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
