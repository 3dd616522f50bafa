"""Device-resident O(1) decode cache — mirror of ``Mamba2Cache``
(decode.py:21-37) and ``GenerationResult`` (decode.py:40-46).

One contiguous allocation per kind:
  ssm  (n_layers, B, H, P, N)        compute dtype (f32 in bf16 mode)
  conv (n_layers, B, conv_dim, k-1)  newest column last
``.ssm[i]`` / ``.conv[i]`` are per-layer views, so list semantics are kept,
and the base pointers stay fixed across steps (one CUDA graph replays them).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .config import ModelConfig


def state_dtype(cfg: ModelConfig) -> torch.dtype:
    return torch.float64 if cfg.policy.compute == "f64" else torch.float32


class Mamba2Cache:
    def __init__(self, ssm: torch.Tensor, conv: torch.Tensor):
        self.ssm_all = ssm
        self.conv_all = conv

    @classmethod
    def empty(cls, cfg: ModelConfig, batch: int, device="cuda", zero=True):
        mk = torch.zeros if zero else torch.empty
        dt = state_dtype(cfg)
        ssm = mk((cfg.n_layers, batch, cfg.n_heads, cfg.head_dim, cfg.d_state), dtype=dt, device=device)
        conv = mk((cfg.n_layers, batch, cfg.conv_dim, cfg.conv_kernel - 1), dtype=dt, device=device)
        return cls(ssm, conv)

    @property
    def ssm(self) -> list:
        return list(self.ssm_all.unbind(0))

    @property
    def conv(self) -> list:
        return list(self.conv_all.unbind(0))

    @property
    def batch(self) -> int:
        return self.ssm_all.shape[1]

    def copy(self) -> "Mamba2Cache":
        return Mamba2Cache(self.ssm_all.clone(), self.conv_all.clone())

    def to_bytes(self) -> bytes:
        """All ssm buffers then all conv buffers (decode.py:31-33)."""
        return self.ssm_all.cpu().numpy().tobytes() + self.conv_all.cpu().numpy().tobytes()

    @property
    def nbytes(self) -> int:
        return self.ssm_all.numel() * self.ssm_all.element_size() + (
            self.conv_all.numel() * self.conv_all.element_size()
        )


@dataclass
class GenerationResult:
    """tokens (B, G) int64; per_step_logits optional (B, G, vocab)."""

    tokens: torch.Tensor
    steps: int
    per_step_logits: torch.Tensor | None = None
