"""Model configuration and element policy — mirrors of the reference
``ModelConfig`` (model.py:20-70) and ``ElemPolicy`` (numerics.py:20-53).

Same fields, same derived widths, same validation messages.  One addition:
``ElemPolicy.compute`` also accepts ``"bf16"`` — bf16 weights and GEMM
operands with fp32 accumulation, fp32 decays/cumsums/exps, an fp32 residual
stream and an fp32 SSM state (the B200 tensor-core mode; the reference itself
only has f32/f64, numerics.py:17,37-38).
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

_COMPUTE = {"f32": np.float32, "f64": np.float64, "bf16": np.float32}


@dataclass(frozen=True)
class ElemPolicy:
    """numerics.py:20-53.  compute in {"f32", "f64", "bf16"}; decay_exp in
    {"f32", "bf16e"} (the bf16-rounded exp(A_log) ablation)."""

    compute: str = "f32"
    decay_exp: str = "f32"

    def __post_init__(self):
        if self.compute not in _COMPUTE:
            raise ValueError(f"compute must be 'f32', 'f64' or 'bf16', got {self.compute!r}")
        if self.decay_exp not in ("f32", "bf16e"):
            raise ValueError(f"decay_exp must be 'f32' or 'bf16e', got {self.decay_exp!r}")

    @property
    def dtype(self) -> np.dtype:
        """Host dtype of activations/caches handed back to callers."""
        return np.dtype(_COMPUTE[self.compute])

    @property
    def residual_dtype(self) -> np.dtype:
        # never below float32 (numerics.py:46-49)
        return self.dtype

    @property
    def bf16_decay(self) -> bool:
        return self.decay_exp == "bf16e"

    @property
    def tensor_core(self) -> bool:
        return self.compute == "bf16"


@dataclass(frozen=True)
class ModelConfig:
    """model.py:20-70 — same defaults (N=128, P=64, expand 2, G=1, k=4, L=256)."""

    vocab_size: int
    d_model: int
    n_layers: int
    d_state: int = 128
    head_dim: int = 64
    expand: int = 2
    n_groups: int = 1
    conv_kernel: int = 4
    chunk_size: int = 256
    norm_eps: float = 1e-5
    dt_limits: tuple = (0.0, float("inf"))
    mask_strategy: str = "static"
    policy: ElemPolicy = field(default_factory=ElemPolicy)

    def __post_init__(self):
        if self.d_inner % self.head_dim != 0:
            raise ValueError(
                f"expand*d_model = {self.d_inner} not divisible by head_dim {self.head_dim}"
            )
        if self.n_heads % self.n_groups != 0:
            raise ValueError(f"n_heads {self.n_heads} not divisible by n_groups {self.n_groups}")
        if self.conv_kernel < 1 or self.chunk_size < 1:
            raise ValueError("conv_kernel and chunk_size must be >= 1")
        if self.mask_strategy not in ("static", "rowwise"):
            raise ValueError(f"unknown mask strategy {self.mask_strategy!r}")

    @property
    def d_inner(self) -> int:
        return self.expand * self.d_model

    @property
    def n_heads(self) -> int:
        return self.d_inner // self.head_dim

    @property
    def conv_dim(self) -> int:
        return self.d_inner + 2 * self.n_groups * self.d_state

    @property
    def d_in_proj(self) -> int:
        # [z | xBC | dt_raw]   (model.py:60-63)
        return 2 * self.d_inner + 2 * self.n_groups * self.d_state + self.n_heads

    @property
    def dtype(self) -> np.dtype:
        return self.policy.dtype

    def with_policy(self, **kwargs) -> "ModelConfig":
        return replace(self, policy=replace(self.policy, **kwargs))


# Named model configs.  Only 130M is pinned by the reference
# (test_model.py:160-172); the rest follow the upstream mamba2 sizes
# (n_params cross-checks them).
MODEL_SIZES = {
    "130m": dict(d_model=768, n_layers=24),
    "370m": dict(d_model=1024, n_layers=48),
    "780m": dict(d_model=1536, n_layers=48),
    "1.3b": dict(d_model=2048, n_layers=48),
    "2.7b": dict(d_model=2560, n_layers=64),
}


def named_config(name: str, compute: str = "bf16", vocab_size: int = 50288, **kw) -> ModelConfig:
    base = dict(MODEL_SIZES[name.lower()])
    base.update(kw)
    return ModelConfig(vocab_size=vocab_size, policy=ElemPolicy(compute=compute), **base)
