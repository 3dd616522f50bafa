"""Multi-GPU partitioning of the hot path.

Two ways the path shards across the GPUs of one box:

* **batch** — rows are independent in prefill and decode (model.py:124-206,
  decode.py:77-144), so rank r owns rows ``batch_slice(B, r, world)`` and no
  collective touches the data path.  The kernels are batch-invariant, so a
  sharded run equals the single-GPU run row for row; ``gather_rows``
  reassembles per-rank results (tokens, logits) when a caller wants them on
  one rank.
* **SSD head groups** — heads are independent in the scan (ssd.py:139-198).
  ``shard_layer_by_heads`` cuts one layer's weights so rank r owns heads
  ``head_slice(H, r, world)``: its z / x / dt columns of W_in, its x conv
  channels, its D / dt_bias / A_log / norm_w entries and its W_out rows; the
  B / C columns and their conv channels (G = 1, shared by every head) are
  replicated.  A layer then needs exactly one all-reduce (sum) after out_proj
  over ``[partial (rows, d_model) | sum u^2 (rows)]``; the rsqrt row scale of
  the gated RMSNorm commutes with the out_proj GEMM once ``norm_w`` is folded
  into W_out, so every rank finishes ``hidden += partial * rsqrt(ssq / d_inner
  + eps)`` identically.

Only partitioning and collectives live here; the arithmetic is the CUDA path.
"""

from __future__ import annotations

from types import SimpleNamespace

import numpy as np
import torch

from .config import ModelConfig


def _split(n: int, rank: int, world: int) -> tuple[int, int]:
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def batch_slice(batch: int, rank: int, world: int) -> slice:
    """Contiguous near-equal row range of `rank` (the first batch % world
    ranks take one extra row)."""
    lo, hi = _split(batch, rank, world)
    return slice(lo, hi)


def head_slice(n_heads: int, rank: int, world: int) -> slice:
    """Contiguous head range of `rank` for head-group sharding."""
    if n_heads < world:
        raise ValueError(f"cannot shard {n_heads} heads over {world} ranks")
    lo, hi = _split(n_heads, rank, world)
    return slice(lo, hi)


def gather_rows(local: torch.Tensor, batch: int, group=None) -> torch.Tensor:
    """All-gather per-rank row slices (dim 0, sizes from batch_slice) into the
    full (batch, ...) tensor on every rank.  Works with gloo (CPU tensors) and
    NCCL (CUDA tensors)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rows = max(batch_slice(batch, r, world).stop - batch_slice(batch, r, world).start
               for r in range(world))
    pad = torch.zeros((rows,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    out = []
    for r in range(world):
        s = batch_slice(batch, r, world)
        out.append(parts[r][: s.stop - s.start])
    return torch.cat(out, dim=0)


def local_dims(cfg: ModelConfig, heads: slice) -> SimpleNamespace:
    """Widths of one rank's head-sharded layer."""
    h = heads.stop - heads.start
    d_inner = h * cfg.head_dim
    gn = cfg.n_groups * cfg.d_state
    return SimpleNamespace(n_heads=h, d_inner=d_inner, conv_dim=d_inner + 2 * gn,
                           d_in_proj=2 * d_inner + 2 * gn + h, d_inner_full=cfg.d_inner)


def shard_layer_by_heads(layer, cfg: ModelConfig, rank: int, world: int) -> SimpleNamespace:
    """Cut one layer (reference layout, numpy or CPU tensors: W_in
    (d_model, d_in_proj) with columns [z | x | B | C | dt_raw], model.py:107-121;
    conv_w (conv_dim, k) over [x | B | C]; W_out (d_inner, d_model)) down to
    the heads of `rank`.  Returns the local arrays plus `heads` and `dims`."""
    heads = head_slice(cfg.n_heads, rank, world)
    P, di, gn = cfg.head_dim, cfg.d_inner, cfg.n_groups * cfg.d_state
    ch = slice(heads.start * P, heads.stop * P)  # this rank's d_inner channels
    W_in = np.asarray(layer.W_in)
    z = W_in[:, ch]
    x = W_in[:, di + ch.start: di + ch.stop]
    bc = W_in[:, 2 * di: 2 * di + 2 * gn]
    dt = W_in[:, 2 * di + 2 * gn + heads.start: 2 * di + 2 * gn + heads.stop]
    conv_w, conv_b = np.asarray(layer.conv_w), np.asarray(layer.conv_b)
    cw = np.concatenate([conv_w[ch], conv_w[di: di + 2 * gn]], axis=0)
    cb = np.concatenate([conv_b[ch], conv_b[di: di + 2 * gn]], axis=0)
    return SimpleNamespace(
        W_in=np.ascontiguousarray(np.concatenate([z, x, bc, dt], axis=1)),
        conv_w=np.ascontiguousarray(cw),
        conv_b=np.ascontiguousarray(cb),
        dt_bias=np.asarray(layer.dt_bias)[heads].copy(),
        A_log=np.asarray(layer.A_log)[heads].copy(),
        D=np.asarray(layer.D)[heads].copy(),
        norm_w=np.asarray(layer.norm_w)[ch].copy(),
        W_out=np.ascontiguousarray(np.asarray(layer.W_out)[ch]),
        heads=heads,
        dims=local_dims(cfg, heads),
    )
