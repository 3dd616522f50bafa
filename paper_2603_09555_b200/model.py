"""Prefill over the C-ABI — mirrors ``block_forward`` / ``prefill``
(model.py:124-206).  Python only validates, allocates and sequences per-layer
calls onto one CUDA stream; every FLOP runs in libssd200.so.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _abi
from .cache import Mamba2Cache, state_dtype
from .config import ModelConfig
from .params import LayerParams, ModelParams


class PolicyAudit:
    """model.py:94-104 — records (site, dtype) events."""

    def __init__(self):
        self.events = []

    def record(self, site, dtype):
        self.events.append((site, str(dtype)))

    def sites(self, name):
        return [d for s, d in self.events if s == name]


def dims_struct(cfg: ModelConfig) -> _abi.Dims:
    """ssd200_dims_t for cfg; carries the implementation choices in scope
    (``_abi.tuning(...)``), or NULL for the library defaults."""
    lo, hi = cfg.dt_limits
    if not (0 <= lo < hi):
        raise ValueError(f"need 0 <= dt_min < dt_max, got {cfg.dt_limits}")
    tune = _abi.current_tuning()
    d = _abi.Dims(
        dtype=_abi.DTYPE_CODE[cfg.policy.compute],
        d_model=cfg.d_model,
        d_inner=cfg.d_inner,
        n_heads=cfg.n_heads,
        head_dim=cfg.head_dim,
        d_state=cfg.d_state,
        n_groups=cfg.n_groups,
        conv_kernel=cfg.conv_kernel,
        chunk_size=cfg.chunk_size,
        norm_eps=float(cfg.norm_eps),
        dt_min=float(lo),
        dt_max=float(hi),
        tuning=ctypes.pointer(tune) if tune is not None else None,
    )
    d._keep = tune  # the struct points at it
    return d


def layer_struct(lp: LayerParams) -> _abi.Layer:
    return _abi.Layer(
        W_in=lp.W_in.data_ptr(),
        conv_w=lp.conv_w.data_ptr(),
        conv_b=lp.conv_b.data_ptr(),
        dt_bias=lp.dt_bias.data_ptr(),
        a=lp.a.data_ptr(),
        D=lp.D.data_ptr(),
        norm_w=lp.norm_w.data_ptr(),
        W_out=lp.W_out.data_ptr(),
        pre_norm_w=lp.pre_norm_w.data_ptr() if lp.pre_norm_w is not None else None,
    )


def _audit(audit, cfg):
    if audit is not None:
        audit.record("decay_exp", "bf16e" if cfg.policy.bf16_decay else cfg.dtype)
        audit.record("residual_add", cfg.policy.residual_dtype)


def check_tokens(tokens, cfg: ModelConfig, ndim: int, device) -> torch.Tensor:
    """model.py:191-195 / decode.py:88-92 validation, then upload as int64.

    Host ids (numpy, lists, CPU tensors) are range-checked here and raise
    ValueError like the reference.  Ids already on the device are not read
    back (no host sync on the hot path): the embedding kernel checks them and
    an id outside [0, vocab) yields a NaN row instead of an out-of-bounds read."""
    if isinstance(tokens, torch.Tensor):
        t = tokens
    else:
        t = torch.as_tensor(np.asarray(tokens))
    if t.dim() != ndim:
        shape = tuple(t.shape)
        if ndim == 2:
            raise ValueError(f"tokens must be (B, T), got shape {shape}")
        raise ValueError(f"token must be (B,), got shape {shape}")
    if t.numel() == 0:
        raise ValueError("empty token array")
    if t.dtype.is_floating_point or t.dtype == torch.bool:
        raise ValueError(f"token ids must be integers, got {t.dtype}")
    if not t.is_cuda:
        lo, hi = int(t.min()), int(t.max())
        if lo < 0 or hi >= cfg.vocab_size:
            raise ValueError("token id out of range")
        if t.dtype != torch.int64:
            t = t.to(torch.int64)
        return t.contiguous().to(device=device, non_blocking=t.is_pinned())
    return t.to(device=device, dtype=torch.int64).contiguous()


class _Runner:
    """Per-call context: dims, stream, one workspace reused across layers."""

    def __init__(self, params: ModelParams, cfg: ModelConfig):
        if params.mode != cfg.policy.compute:
            raise ValueError(
                f"params were uploaded for compute={params.mode!r}, cfg asks {cfg.policy.compute!r}"
            )
        self.cfg = cfg
        self.params = params
        self.dev = torch.device(params.device)
        self.dims = dims_struct(cfg)
        self.lib = _abi.lib()
        # the caller's current stream ON THE PARAMS' DEVICE; every ABI call runs
        # under a device guard so the library's per-device state matches
        self.stream = _abi.stream_handle(torch.cuda.current_stream(self.dev))
        self.sdt = state_dtype(cfg)
        self._ws = None
        self._layers = [layer_struct(lp) for lp in params.layers]
        self._layer_arr = (_abi.Layer * len(self._layers))(*self._layers)

    def workspace(self, nbytes: int) -> torch.Tensor:
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.dev)
        return self._ws

    def embed(self, tok: torch.Tensor):
        if tok.dtype != torch.int64 or not tok.is_contiguous():  # the C-ABI reads dense int64
            tok = tok.to(torch.int64).contiguous()
        rows = tok.numel()
        cfg = self.cfg
        hidden = torch.empty((rows, cfg.d_model), dtype=self.sdt, device=self.dev)
        lp = (
            torch.empty((rows, cfg.d_model), dtype=torch.bfloat16, device=self.dev)
            if cfg.policy.compute == "bf16"
            else None
        )
        self._call("ssd200_embed", self.lib.ssd200_embed, self.dims, tok.data_ptr(), rows,
                   cfg.vocab_size, self.params.embedding.data_ptr(), hidden.data_ptr(),
                   _abi.ptr(lp), self.stream)
        return hidden, lp

    def _call(self, what, fn, *args):
        with torch.cuda.device(self.dev):
            _abi.check(fn(*args), what)

    def prefill_layer(self, i, hidden, hidden_lp, ssm_out, conv_out, B, T):
        ws = self.workspace(self.lib.ssd200_prefill_layer_workspace(self.dims, B, T))
        self._call("ssd200_prefill_layer", self.lib.ssd200_prefill_layer, self.dims,
                   self._layers[i], hidden.data_ptr(), _abi.ptr(hidden_lp), ssm_out.data_ptr(),
                   _abi.ptr(conv_out) if conv_out.numel() else None, B, T, ws.data_ptr(),
                   ws.numel(), self.stream)

    def decode_layer(self, i, hidden, hidden_lp, ssm_in, ssm_out, conv_in, conv_out, B):
        ws = self.workspace(self.lib.ssd200_decode_layer_workspace(self.dims, B))
        has_conv = conv_in.numel() > 0
        self._call("ssd200_decode_layer", self.lib.ssd200_decode_layer, self.dims,
                   self._layers[i], hidden.data_ptr(), _abi.ptr(hidden_lp), ssm_in.data_ptr(),
                   ssm_out.data_ptr(), conv_in.data_ptr() if has_conv else None,
                   conv_out.data_ptr() if has_conv else None, B, ws.data_ptr(), ws.numel(),
                   self.stream)

    def decode_layers(self, hidden, hidden_lp, ssm_in, ssm_out, conv_in, conv_out, B):
        """Every layer of one decode step (ssd200_decode_layers: chained layers)."""
        ws = self.workspace(self.lib.ssd200_decode_layers_workspace(self.dims, B))
        has_conv = conv_in.numel() > 0
        self._call("ssd200_decode_layers", self.lib.ssd200_decode_layers, self.dims,
                   self._layer_arr, len(self._layers), hidden.data_ptr(), _abi.ptr(hidden_lp),
                   ssm_in.data_ptr(), ssm_out.data_ptr(),
                   conv_in.data_ptr() if has_conv else None,
                   conv_out.data_ptr() if has_conv else None, B, ws.data_ptr(), ws.numel(),
                   self.stream)

    def head(self, hidden, row_stride, rows, logits=None, argmax=None, base_offset=0):
        cfg = self.cfg
        ws = self.workspace(self.lib.ssd200_head_workspace(self.dims, cfg.vocab_size, rows))
        hptr = hidden.data_ptr() + base_offset * hidden.element_size()
        self._call("ssd200_head", self.lib.ssd200_head, self.dims, cfg.vocab_size, hptr,
                   row_stride, self.params.final_norm_w.data_ptr(),
                   self.params.embedding.data_ptr(), _abi.ptr(logits), _abi.ptr(argmax), rows,
                   ws.data_ptr(), ws.numel(), self.stream)


def _as_hidden(hidden, cfg, dev):
    h = hidden if isinstance(hidden, torch.Tensor) else torch.as_tensor(np.asarray(hidden))
    return h.to(device=dev, dtype=state_dtype(cfg)).contiguous()


def block_forward(layer: LayerParams, hidden, cfg: ModelConfig, audit: PolicyAudit | None = None):
    """model.py:124-174 — one residual block over (B, T, d_model).

    Returns (hidden_out, final ssm state (B,H,P,N), conv tail (B,conv_dim,k-1)).
    The input is not mutated."""
    dev = layer.W_in.device
    h = _as_hidden(hidden, cfg, dev).clone()
    if h.dim() != 3 or h.shape[-1] != cfg.d_model:
        raise ValueError(f"hidden must be (B, T, {cfg.d_model}), got {tuple(h.shape)}")
    B, T, _ = h.shape
    # the layer's own upload mode (its W_in dtype), so a layer/cfg mismatch raises in
    # _Runner instead of running kernels on the wrong layout; only the layer is used
    mode = {torch.bfloat16: "bf16", torch.float32: "f32", torch.float64: "f64"}[layer.W_in.dtype]
    params = ModelParams(embedding=layer.W_in, layers=[layer], final_norm_w=layer.norm_w, mode=mode)
    r = _Runner(params, cfg)
    lp = h.to(torch.bfloat16) if cfg.policy.compute == "bf16" else None
    sdt = state_dtype(cfg)
    ssm = torch.empty((B, cfg.n_heads, cfg.head_dim, cfg.d_state), dtype=sdt, device=dev)
    conv = torch.empty((B, cfg.conv_dim, cfg.conv_kernel - 1), dtype=sdt, device=dev)
    r.prefill_layer(0, h.view(B * T, -1), lp, ssm, conv, B, T)
    _audit(audit, cfg)
    return h, ssm, conv


def prefill(params: ModelParams, tokens, cfg: ModelConfig, audit: PolicyAudit | None = None,
            logits: str = "all", return_hidden: bool = False, argmax_out=None):
    """model.py:177-206 — embed, every block, final RMSNorm, tied head.

    logits="all" returns (B, T, vocab) like the reference; "last" returns only
    the last position (B, vocab) (what generate needs); None skips the head.
    ``argmax_out`` (B,) int64 receives the greedy token of the last position
    (ties -> lowest id) from the head kernel.  Returns (logits, Mamba2Cache)."""
    dev = params.device
    tok = check_tokens(tokens, cfg, 2, dev)
    B, T = tok.shape
    r = _Runner(params, cfg)
    hidden, lp = r.embed(tok.view(-1))
    cache = Mamba2Cache.empty(cfg, B, device=dev, zero=False)
    for i in range(cfg.n_layers):
        r.prefill_layer(i, hidden, lp, cache.ssm_all[i], cache.conv_all[i], B, T)
        _audit(audit, cfg)
    out = None
    if logits == "all":
        out = torch.empty((B, T, cfg.vocab_size), dtype=state_dtype(cfg), device=dev)
        r.head(hidden, cfg.d_model, B * T, logits=out)
    elif logits == "last":
        out = torch.empty((B, cfg.vocab_size), dtype=state_dtype(cfg), device=dev)
        r.head(hidden, T * cfg.d_model, B, logits=out, argmax=argmax_out,
               base_offset=(T - 1) * cfg.d_model)
    elif logits is not None:
        raise ValueError(f"logits must be 'all', 'last' or None, got {logits!r}")
    if argmax_out is not None and logits != "last":
        r.head(hidden, T * cfg.d_model, B, argmax=argmax_out, base_offset=(T - 1) * cfg.d_model)
    if return_hidden:
        return out, cache, hidden.view(B, T, cfg.d_model)
    return out, cache
