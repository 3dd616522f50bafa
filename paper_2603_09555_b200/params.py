"""Weights on the device — mirrors of ``LayerParams`` / ``ModelParams``
(model.py:73-91) plus the host-side initialiser ``random_init``
(bundle.py:246-289) and the numpy -> device adapter ``from_reference``.

Device layout per compute mode (include/ssd200.h):
  f32 / f64  every tensor in the compute dtype, reference shapes
             (W_in (d_model, d_in_proj), W_out (d_inner, d_model)).
  bf16       W_in^T (d_in_proj, d_model) and W_out^T (d_model, d_inner) bf16,
             K-major for the tcgen05 GEMMs; embedding (V, d_model) bf16 (also
             the tied head's B operand); conv taps, biases, dt_bias, D and the
             norm weights stay f32.
The per-head decay a = -exp(A_log) is evaluated once on the host with numpy,
exactly as decay_coefficient (ssd.py:99-112) does, so the bf16e ablation
rounds identically.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from types import SimpleNamespace

import numpy as np
import torch

from .config import ModelConfig


@dataclass
class LayerParams:
    W_in: torch.Tensor
    conv_w: torch.Tensor
    conv_b: torch.Tensor
    dt_bias: torch.Tensor
    A_log: torch.Tensor
    D: torch.Tensor
    norm_w: torch.Tensor
    W_out: torch.Tensor
    a: torch.Tensor = field(default=None)  # -exp(A_log), compute dtype (f32 in bf16 mode)
    # optional residual pre-norm weight (d_model), compute dtype (f32 in bf16 mode):
    # real state-spaces/mamba2 checkpoints' backbone.layers.N.norm, which the
    # reference block drops (converter/mapping.json:75-78); None = the reference block
    pre_norm_w: torch.Tensor = field(default=None)


@dataclass
class ModelParams:
    embedding: torch.Tensor
    layers: list
    final_norm_w: torch.Tensor
    mode: str = "f32"

    @property
    def device(self) -> torch.device:
        return self.embedding.device


def _bf16_round_np(x: np.ndarray) -> np.ndarray:
    """numerics.py:76-93 (round-to-nearest-even), used for the bf16e ablation."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    lsb = (u >> np.uint32(16)) & np.uint32(1)
    return ((u + np.uint32(0x7FFF) + lsb) & np.uint32(0xFFFF0000)).view(np.float32)


def decay_coefficient(A_log, cfg: ModelConfig) -> np.ndarray:
    """ssd.py:99-112 on the host: a = -exp(A_log) in the working dtype."""
    A_log = np.asarray(A_log)
    if not np.all(np.isfinite(A_log)):
        raise ValueError("A_log must be finite")
    wd = np.float64 if cfg.policy.compute == "f64" else np.float32
    e = np.exp(A_log.astype(wd, copy=False))
    if cfg.policy.bf16_decay:
        e = _bf16_round_np(e.astype(np.float32)).astype(wd)
    return -e


def _np(x) -> np.ndarray:
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    return np.asarray(x)


def from_reference(params, cfg: ModelConfig, device="cuda") -> ModelParams:
    """Upload reference-layout (numpy) weights into the device layout of
    ``cfg.policy.compute``.  Accepts the reference's ModelParams or any object
    with the same attribute names."""
    mode = cfg.policy.compute
    dev = torch.device(device)
    wd = torch.float64 if mode == "f64" else torch.float32

    def small(x):  # f32 / f64 side tensors
        return torch.as_tensor(np.ascontiguousarray(_np(x)), dtype=wd).to(dev)

    def big(x, transpose=False):
        arr = _np(x)
        if mode == "bf16":
            t = torch.as_tensor(np.ascontiguousarray(arr.astype(np.float32)))
            if transpose:
                t = t.t()
            return t.to(torch.bfloat16).contiguous().to(dev)
        return torch.as_tensor(np.ascontiguousarray(arr), dtype=wd).to(dev)

    layers = []
    for lp in params.layers:
        W_out = _np(lp.W_out)
        if mode == "bf16":
            # the gated norm's weight is folded into W_out's rows (the norm's
            # row scale is applied after the out_proj GEMM; numerics.py:149-158)
            W_out = _np(lp.norm_w).astype(np.float32)[:, None] * W_out.astype(np.float32)
        layers.append(
            LayerParams(
                W_in=big(lp.W_in, transpose=True),
                conv_w=small(lp.conv_w),
                conv_b=small(lp.conv_b),
                dt_bias=small(lp.dt_bias),
                A_log=small(lp.A_log),
                D=small(lp.D),
                norm_w=small(lp.norm_w),
                W_out=big(W_out, transpose=True),
                a=small(decay_coefficient(_np(lp.A_log), cfg)),
                pre_norm_w=(small(lp.pre_norm_w)
                            if getattr(lp, "pre_norm_w", None) is not None else None),
            )
        )
    return ModelParams(
        embedding=big(params.embedding),
        layers=layers,
        final_norm_w=small(params.final_norm_w),
        mode=mode,
    )


def random_init_host(cfg: ModelConfig, seed: int):
    """bundle.py:246-289 — the reference's deterministic initialisation
    (numpy Philox keyed by seed, tensors drawn in canonical order), returned
    as host float32 arrays in the reference layout."""
    rng = np.random.Generator(np.random.Philox(seed))

    def normal(shape, std=0.02):
        return rng.normal(0.0, std, size=shape).astype(np.float32)

    embedding = normal((cfg.vocab_size, cfg.d_model))
    bound = 1.0 / np.sqrt(cfg.conv_kernel)
    layers = []
    for _ in range(cfg.n_layers):
        w_in = normal((cfg.d_model, cfg.d_in_proj))
        conv_w = rng.uniform(-bound, bound, size=(cfg.conv_dim, cfg.conv_kernel)).astype(np.float32)
        dt = rng.uniform(1e-3, 1e-1, size=cfg.n_heads)
        a_log = np.log(rng.uniform(1.0, 16.0, size=cfg.n_heads)).astype(np.float32)
        d = rng.normal(0.0, 1.0, size=cfg.n_heads).astype(np.float32)
        layers.append(
            SimpleNamespace(
                W_in=w_in,
                conv_w=conv_w,
                conv_b=np.zeros(cfg.conv_dim, dtype=np.float32),
                dt_bias=np.log(np.expm1(dt)).astype(np.float32),
                A_log=a_log,
                D=d,
                norm_w=np.ones(cfg.d_inner, dtype=np.float32),
                W_out=normal((cfg.d_inner, cfg.d_model)),
            )
        )
    return SimpleNamespace(
        embedding=embedding, layers=layers, final_norm_w=np.ones(cfg.d_model, dtype=np.float32)
    )


def random_init(cfg: ModelConfig, seed: int, device="cuda") -> ModelParams:
    """Reference-identical weights (bundle.py:246-289), uploaded to ``device``."""
    return from_reference(random_init_host(cfg, seed), cfg, device)


def synthetic_init(cfg: ModelConfig, seed: int = 0, device="cuda") -> ModelParams:
    """Throughput-only init drawn on the device with the reference's
    distributions (normal(0, .02) projections, U[-1/sqrt(k), 1/sqrt(k)] conv,
    a in [-16, -1], dt in [1e-3, 1e-1], D ~ N(0,1)).  Not Philox-identical:
    used by bench.py for the 370M-2.7B configs where a host numpy init would
    take minutes.  Parity tests always use ``random_init``."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    dev = torch.device(device)
    mode = cfg.policy.compute
    wd = torch.float64 if mode == "f64" else torch.float32
    big_dt = torch.bfloat16 if mode == "bf16" else wd

    def normal(shape, std=0.02):
        return (torch.randn(shape, generator=g, device=dev, dtype=torch.float32) * std).to(big_dt)

    def uniform(shape, lo, hi):
        return torch.rand(shape, generator=g, device=dev, dtype=torch.float64) * (hi - lo) + lo

    layers = []
    bound = 1.0 / np.sqrt(cfg.conv_kernel)
    for _ in range(cfg.n_layers):
        dt = uniform((cfg.n_heads,), 1e-3, 1e-1)
        a_log = torch.log(uniform((cfg.n_heads,), 1.0, 16.0)).to(torch.float32)
        w_in = normal((cfg.d_in_proj, cfg.d_model) if mode == "bf16" else (cfg.d_model, cfg.d_in_proj))
        w_out = normal((cfg.d_model, cfg.d_inner) if mode == "bf16" else (cfg.d_inner, cfg.d_model))
        layers.append(
            LayerParams(
                W_in=w_in.contiguous(),
                conv_w=uniform((cfg.conv_dim, cfg.conv_kernel), -bound, bound).to(wd),
                conv_b=torch.zeros(cfg.conv_dim, device=dev, dtype=wd),
                dt_bias=torch.log(torch.expm1(dt)).to(wd),
                A_log=a_log.to(wd),
                D=torch.randn(cfg.n_heads, generator=g, device=dev, dtype=torch.float32).to(wd),
                norm_w=torch.ones(cfg.d_inner, device=dev, dtype=wd),
                W_out=w_out.contiguous(),
                a=torch.as_tensor(decay_coefficient(a_log.cpu().numpy(), cfg), dtype=wd).to(dev),
            )
        )
    return ModelParams(
        embedding=normal((cfg.vocab_size, cfg.d_model)).contiguous(),
        layers=layers,
        final_norm_w=torch.ones(cfg.d_model, device=dev, dtype=wd),
        mode=mode,
    )
