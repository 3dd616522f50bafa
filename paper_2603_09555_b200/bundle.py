"""Two-file tensor bundle (manifest.json + data.bin) straight onto the GPU —
SURVEY.md §8(f) row 1; mirrors ``ssd_engine.bundle`` (bundle.py:1-243).

The format is the reference's bit-exact contract with its checkpoint
converter: UTF-8 JSON manifest {format_version, config, tensors: [name, dtype,
shape, offset, length]} and a raw little-endian float32 payload, every section
64-byte aligned, tensors in canonical order (bundle.py:44-59).

* ``save_bundle`` writes the same bytes as the reference for the same
  reference-layout weights (tested byte-for-byte against a bundle the
  reference wrote).
* ``load_bundle_host`` validates exactly like the reference (same checks in
  the same order, same exception classes and messages) and returns zero-copy
  views of a memory-mapped payload in the reference layout.
* ``load_bundle`` validates the same way, then streams each tensor from the
  mapped file to the device in f32 and does the device-layout conversion
  there (K-major transposes, bf16 rounding, norm_w folded into W_out for the
  bf16 path) — bitwise the layout ``from_reference`` builds on the host, but
  without materialising a host copy of a 2.7B model.
"""

from __future__ import annotations

import json
import mmap
import warnings
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import torch

from .config import ElemPolicy, ModelConfig
from .params import LayerParams, ModelParams, decay_coefficient

FORMAT_VERSION = 1
ALIGNMENT = 64


class BundleError(Exception):
    """Base class for bundle load/save failures (bundle.py:24-25)."""


class FormatVersionError(BundleError):
    pass


class MissingTensorError(BundleError):
    pass


class TensorShapeError(BundleError):
    pass


class PayloadError(BundleError):
    pass


def tensor_names(cfg: ModelConfig) -> list[str]:
    """Canonical parameter names in payload order (bundle.py:44-59)."""
    names = ["embedding"]
    for i in range(cfg.n_layers):
        names += [
            f"layers.{i}.in_proj.weight",
            f"layers.{i}.conv1d.weight",
            f"layers.{i}.conv1d.bias",
            f"layers.{i}.dt_bias",
            f"layers.{i}.A_log",
            f"layers.{i}.D",
            f"layers.{i}.norm.weight",
            f"layers.{i}.out_proj.weight",
        ]
    names.append("final_norm.weight")
    return names


_LEAF = {
    "in_proj.weight": lambda c: (c.d_model, c.d_in_proj),
    "conv1d.weight": lambda c: (c.conv_dim, c.conv_kernel),
    "conv1d.bias": lambda c: (c.conv_dim,),
    "dt_bias": lambda c: (c.n_heads,),
    "A_log": lambda c: (c.n_heads,),
    "D": lambda c: (c.n_heads,),
    "norm.weight": lambda c: (c.d_inner,),
    "out_proj.weight": lambda c: (c.d_inner, c.d_model),
}
_ATTR = {  # canonical leaf -> LayerParams attribute
    "in_proj.weight": "W_in",
    "conv1d.weight": "conv_w",
    "conv1d.bias": "conv_b",
    "dt_bias": "dt_bias",
    "A_log": "A_log",
    "D": "D",
    "norm.weight": "norm_w",
    "out_proj.weight": "W_out",
}


def tensor_shape(name: str, cfg: ModelConfig) -> tuple[int, ...]:
    """Expected shape of a canonical tensor (bundle.py:62-80)."""
    if name == "embedding":
        return (cfg.vocab_size, cfg.d_model)
    if name == "final_norm.weight":
        return (cfg.d_model,)
    _, _, leaf = name.split(".", 2)
    if leaf not in _LEAF:
        raise KeyError(f"unknown canonical tensor name {name!r}")
    return _LEAF[leaf](cfg)


def _config_dict(cfg: ModelConfig) -> dict:
    """bundle.py:97-112 (null encodes an unbounded dt limit)."""
    return {
        "vocab_size": cfg.vocab_size,
        "d_model": cfg.d_model,
        "n_layers": cfg.n_layers,
        "d_state": cfg.d_state,
        "head_dim": cfg.head_dim,
        "expand": cfg.expand,
        "n_groups": cfg.n_groups,
        "conv_kernel": cfg.conv_kernel,
        "chunk_size": cfg.chunk_size,
        "norm_eps": cfg.norm_eps,
        "dt_limits": [None if not np.isfinite(v) else v for v in cfg.dt_limits],
    }


def _config_from_dict(raw: dict, policy: ElemPolicy | None = None) -> ModelConfig:
    """bundle.py:115-131; the element policy is the caller's (not in the file)."""
    limits = [float("inf") if v is None else float(v) for v in raw.get("dt_limits", [0.0, None])]
    return ModelConfig(
        vocab_size=raw["vocab_size"],
        d_model=raw["d_model"],
        n_layers=raw["n_layers"],
        d_state=raw["d_state"],
        head_dim=raw["head_dim"],
        expand=raw["expand"],
        n_groups=raw["n_groups"],
        conv_kernel=raw["conv_kernel"],
        chunk_size=raw["chunk_size"],
        norm_eps=raw["norm_eps"],
        dt_limits=(float(limits[0]), float(limits[1])),
        policy=policy if policy is not None else ElemPolicy(),
    )


PRE_NORM = "layers.{i}.pre_norm.weight"  # optional residual pre-norm (not in the reference format)


def pre_norm_names(cfg: ModelConfig) -> list[str]:
    """The optional per-layer residual pre-norm tensors (d_model,) that a bundle
    converted from a real state-spaces/mamba2 checkpoint may carry
    (``convert(..., keep_pre_norm=True)``).  The reference's reader ignores
    them with a warning (bundle.py:186-225 tolerates unknown tensors); this
    one loads them into ``LayerParams.pre_norm_w`` when every layer has one."""
    return [PRE_NORM.format(i=i) for i in range(cfg.n_layers)]


def _host_tensors(params, cfg: ModelConfig) -> dict:
    def arr(x):
        if isinstance(x, torch.Tensor):
            x = x.detach().cpu().numpy()
        return x

    out = {"embedding": arr(params.embedding), "final_norm.weight": arr(params.final_norm_w)}
    for i, layer in enumerate(params.layers):
        for leaf, attr in _ATTR.items():
            out[f"layers.{i}.{leaf}"] = arr(getattr(layer, attr))
        if getattr(layer, "pre_norm_w", None) is not None:
            out[PRE_NORM.format(i=i)] = arr(layer.pre_norm_w)
    return out


def save_bundle(params, cfg: ModelConfig, path) -> None:
    """Write manifest.json and data.bin (bundle.py:134-168) from
    reference-layout weights (e.g. ``random_init_host``); byte-identical to
    the reference's writer."""
    path = Path(path)
    try:
        path.mkdir(parents=True, exist_ok=True)
        tensors = _host_tensors(params, cfg)
        entries, payload = [], bytearray()
        extra = [n for n in pre_norm_names(cfg) if n in tensors]
        for name in tensor_names(cfg) + extra:
            shape = (cfg.d_model,) if name in extra else tensor_shape(name, cfg)
            a = np.ascontiguousarray(tensors[name], dtype="<f4")
            if a.shape != shape:
                raise TensorShapeError(f"{name}: shape {a.shape} != expected {shape}")
            if len(payload) % ALIGNMENT:
                payload.extend(b"\x00" * (ALIGNMENT - len(payload) % ALIGNMENT))
            entries.append({"name": name, "dtype": "f32", "shape": list(a.shape),
                            "offset": len(payload), "length": a.nbytes})
            payload.extend(a.tobytes())
        manifest = {"format_version": FORMAT_VERSION, "config": _config_dict(cfg),
                    "tensors": entries}
        (path / "manifest.json").write_text(json.dumps(manifest, indent=2) + "\n",
                                            encoding="utf-8")
        (path / "data.bin").write_bytes(bytes(payload))
    except OSError as exc:
        raise BundleError(f"cannot write bundle at {path}: {exc}") from exc


def _open(path: Path):
    """Read the manifest and map the payload (bundle.py:171-184)."""
    manifest_path, payload_path = path / "manifest.json", path / "data.bin"
    try:
        manifest = json.loads(manifest_path.read_text(encoding="utf-8"))
        with open(payload_path, "rb") as f:
            size = f.seek(0, 2)
            payload = (mmap.mmap(f.fileno(), 0, access=mmap.ACCESS_READ) if size
                       else b"")
    except OSError as exc:
        raise BundleError(f"cannot read bundle at {path}: {exc}") from exc
    except json.JSONDecodeError as exc:
        raise BundleError(f"malformed manifest at {manifest_path}: {exc}") from exc
    return manifest, payload


def _validate(manifest, payload_len: int, policy: ElemPolicy | None):
    """bundle.py:186-225: the reference's checks, in its order, with its
    exception classes.  Returns (cfg, [(name, shape, offset, nelems)])."""
    version = manifest.get("format_version")
    if version != FORMAT_VERSION:
        raise FormatVersionError(f"format_version {version} != supported {FORMAT_VERSION}")
    cfg = _config_from_dict(manifest["config"], policy)
    entries = {e["name"]: e for e in manifest["tensors"]}
    if len(entries) != len(manifest["tensors"]):
        raise BundleError("duplicate tensor names in manifest")
    expected = tensor_names(cfg)
    pre = pre_norm_names(cfg)
    has_pre = all(n in entries for n in pre)
    for extra in sorted(set(entries) - set(expected) - (set(pre) if has_pre else set())):
        warnings.warn(f"ignoring unknown tensor {extra!r} in bundle", stacklevel=3)
    prev_end, table = 0, []
    for name in expected:
        entry = entries.get(name)
        if entry is None:
            raise MissingTensorError(f"bundle is missing tensor {name!r}")
        shape = tuple(entry["shape"])
        if shape != tensor_shape(name, cfg):
            raise TensorShapeError(
                f"{name}: manifest shape {shape} != expected {tensor_shape(name, cfg)}")
        if entry["dtype"] != "f32":
            raise BundleError(f"{name}: unsupported dtype {entry['dtype']!r}")
        offset, length = entry["offset"], entry["length"]
        nelems = int(np.prod(shape)) if shape else 1
        if length != 4 * nelems:
            raise PayloadError(f"{name}: length {length} != 4*prod(shape) = {4 * nelems}")
        if offset % ALIGNMENT or offset < prev_end:
            raise PayloadError(f"{name}: offset {offset} misaligned or overlapping")
        if offset + length > payload_len:
            raise PayloadError(
                f"{name}: payload truncated (need {offset + length} bytes, have {payload_len})")
        prev_end = offset + length
        table.append((name, shape, offset, nelems))
    for name in pre if has_pre else []:  # optional residual pre-norm, after the canonical set
        entry = entries[name]
        shape = tuple(entry["shape"])
        if shape != (cfg.d_model,) or entry["dtype"] != "f32" or entry["length"] != 4 * cfg.d_model:
            raise TensorShapeError(f"{name}: expected f32 ({cfg.d_model},), got {entry}")
        if entry["offset"] % ALIGNMENT or entry["offset"] + entry["length"] > payload_len:
            raise PayloadError(f"{name}: offset {entry['offset']} misaligned or truncated")
        table.append((name, shape, entry["offset"], cfg.d_model))
    return cfg, table


def _assemble(tensors: dict, cfg: ModelConfig) -> SimpleNamespace:
    layers = [SimpleNamespace(**{attr: tensors[f"layers.{i}.{leaf}"]
                                 for leaf, attr in _ATTR.items()},
                              pre_norm_w=tensors.get(PRE_NORM.format(i=i)))
              for i in range(cfg.n_layers)]
    return SimpleNamespace(embedding=tensors["embedding"], layers=layers,
                           final_norm_w=tensors["final_norm.weight"])


def load_bundle_host(path, policy: ElemPolicy | None = None):
    """``load_bundle`` of the reference (bundle.py:171-243): validated
    reference-layout float32 arrays (read-only views of the mapped payload)
    and the config."""
    manifest, payload = _open(Path(path))
    cfg, table = _validate(manifest, len(payload), policy)
    tensors = {name: np.frombuffer(payload, dtype="<f4", count=n, offset=off).reshape(shape)
               for name, shape, off, n in table}
    return _assemble(tensors, cfg), cfg


def load_bundle(path, device="cuda", compute: str = "f32"):
    """Validate like the reference, then load the bundle straight into the
    device layout of ``compute`` ("f32" | "f64" | "bf16"): each tensor goes
    from the mapped file to the device as f32 and is transposed / rounded /
    folded there.  Returns (device ModelParams, cfg with that policy)."""
    manifest, payload = _open(Path(path))
    cfg, table = _validate(manifest, len(payload), ElemPolicy(compute=compute))
    dev = torch.device(device)
    wd = torch.float64 if compute == "f64" else torch.float32
    host = {name: np.frombuffer(payload, dtype="<f4", count=n, offset=off).reshape(shape)
            for name, shape, off, n in table}

    def up(name):  # mapped f32 -> device f32 (no host-side copy of the tensor)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")  # read-only buffer: torch only reads it
            return torch.from_numpy(host[name]).to(dev)

    def small(name):
        return up(name).to(wd)

    def big(name, transpose=False, row_scale=None):
        t = up(name)
        if compute != "bf16":
            return t.to(wd)
        if row_scale is not None:  # norm_w folded into W_out's rows (numerics.py:149-158)
            t = row_scale[:, None] * t
        if transpose:
            t = t.t()
        return t.to(torch.bfloat16).contiguous()

    layers = []
    for i in range(cfg.n_layers):
        p = f"layers.{i}."
        norm_w = up(p + "norm.weight")
        layers.append(LayerParams(
            W_in=big(p + "in_proj.weight", transpose=True),
            conv_w=small(p + "conv1d.weight"),
            conv_b=small(p + "conv1d.bias"),
            dt_bias=small(p + "dt_bias"),
            A_log=small(p + "A_log"),
            D=small(p + "D"),
            norm_w=norm_w.to(wd),
            W_out=big(p + "out_proj.weight", transpose=True,
                      row_scale=norm_w if compute == "bf16" else None),
            a=torch.as_tensor(decay_coefficient(host[p + "A_log"], cfg), dtype=wd).to(dev),
            pre_norm_w=small(PRE_NORM.format(i=i)) if PRE_NORM.format(i=i) in host else None,
        ))
    params = ModelParams(embedding=big("embedding"), layers=layers,
                         final_norm_w=small("final_norm.weight"), mode=compute)
    return params, cfg
