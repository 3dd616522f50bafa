"""Cached decode over the C-ABI — mirrors ``cache_init``, ``decode_step`` and
``generate`` (decode.py:49-194).

``decode_step`` is functional like the reference (a new cache is returned;
the input cache is not mutated).  ``generate`` updates one cache in place and
replays the whole per-token step (embed -> every layer -> norm -> head ->
argmax -> token feedback) as ONE CUDA graph, G-1 times, with no host
synchronisation until the tokens are read back.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _abi
from .cache import GenerationResult, Mamba2Cache, state_dtype
from .config import ModelConfig
from .model import PolicyAudit, _audit, _Runner, check_tokens, layer_table, prefill
from .params import ModelParams


def cache_init(cfg: ModelConfig, batch: int, device="cuda") -> Mamba2Cache:
    """decode.py:49-62 — all-zero cache."""
    if batch < 1:
        raise ValueError("batch must be >= 1")
    return Mamba2Cache.empty(cfg, batch, device=device, zero=True)


def _fused_step(r: _Runner, cfg, tok, cache: Mamba2Cache, logits, argmax, bar) -> bool:
    """The whole step as one persistent kernel (ssd200_decode_step), cache
    updated in place.  Returns False when the configuration is outside the
    fused kernel's coverage (the caller then runs the per-layer sequence)."""
    if cfg.policy.compute != "bf16" or tok.shape[0] > 8:
        return False
    B = tok.shape[0]
    hidden = torch.empty((B, cfg.d_model), dtype=torch.float32, device=r.dev)
    lp = torch.empty((B, cfg.d_model), dtype=torch.bfloat16, device=r.dev)
    need = r.lib.ssd200_decode_step_workspace(r.dims, B)
    ws = r.workspace(need)
    rc = r.lib.ssd200_decode_step(
        r.dims, layer_table(r.params).data_ptr(), cfg.n_layers, cfg.vocab_size,
        r.params.embedding.data_ptr(), r.params.final_norm_w.data_ptr(), tok.data_ptr(),
        hidden.data_ptr(), lp.data_ptr(), cache.ssm_all.data_ptr(),
        cache.conv_all.data_ptr() if cache.conv_all.numel() else None,
        _abi.ptr(logits), _abi.ptr(argmax), bar.data_ptr(), B, ws.data_ptr(), ws.numel(),
        r.stream,
    )
    if rc == _abi.EUNSUPPORTED:
        return False
    _abi.check(rc, "ssd200_decode_step")
    return True


def _step_into(r: _Runner, cfg, tok, cache_in: Mamba2Cache, cache_out: Mamba2Cache,
               logits=None, argmax=None):
    B = tok.shape[0]
    hidden, lp = r.embed(tok)
    for i in range(cfg.n_layers):
        r.decode_layer(
            i, hidden, lp, cache_in.ssm_all[i], cache_out.ssm_all[i],
            cache_in.conv_all[i], cache_out.conv_all[i], B,
        )
    r.head(hidden, cfg.d_model, B, logits=logits, argmax=argmax)


def decode_step(params: ModelParams, cache: Mamba2Cache, token, cfg: ModelConfig,
                audit: PolicyAudit | None = None):
    """decode.py:77-144 — (B,) ids -> ((B, vocab) logits, new cache)."""
    dev = params.device
    tok = check_tokens(token, cfg, 1, dev)
    if cache.batch != tok.shape[0]:
        raise ValueError(f"cache batch {cache.batch} != token batch {tok.shape[0]}")
    r = _Runner(params, cfg)
    new = Mamba2Cache.empty(cfg, tok.shape[0], device=dev, zero=False)
    logits = torch.empty((tok.shape[0], cfg.vocab_size), dtype=state_dtype(cfg), device=dev)
    _step_into(r, cfg, tok, cache, new, logits=logits)
    for _ in range(cfg.n_layers):
        _audit(audit, cfg)
    return logits, new


class GreedyDecoder:
    """In-place greedy decoding loop captured as one CUDA graph per step.

    The graph reads the current token from ``self.tok`` and writes the next
    greedy token back into it, updates the cache in place, and records the
    token (and optionally the logits) at the device-side step counter."""

    def __init__(self, params: ModelParams, cfg: ModelConfig, cache: Mamba2Cache, gen_len: int,
                 keep_logits: bool = False, use_graph: bool = True, fused: bool = True):
        self.cfg = cfg
        self.dev = params.device
        B = cache.batch
        self.B = B
        self.cache = cache
        self.runner = _Runner(params, cfg)
        self.tok = torch.zeros((B,), dtype=torch.int64, device=self.dev)
        self.tokens = torch.zeros((B, gen_len), dtype=torch.int64, device=self.dev)
        self.logits = torch.empty((B, cfg.vocab_size), dtype=state_dtype(cfg), device=self.dev)
        self.kept = (
            torch.empty((B, gen_len, cfg.vocab_size), dtype=state_dtype(cfg), device=self.dev)
            if keep_logits
            else None
        )
        self.step_idx = torch.zeros((1,), dtype=torch.int64, device=self.dev)
        self.bar = torch.zeros((2,), dtype=torch.int32, device=self.dev)  # grid-barrier state
        self.graph = None
        self.use_graph = use_graph
        self.fused = fused

    def _body(self):
        cfg = self.cfg
        done = self.fused and _fused_step(self.runner, cfg, self.tok, self.cache, self.logits,
                                          self.tok, self.bar)
        if not done:
            _step_into(self.runner, cfg, self.tok, self.cache, self.cache, logits=self.logits,
                       argmax=self.tok)
        # bookkeeping: tokens[:, step] = tok; step += 1
        self.tokens.index_copy_(1, self.step_idx, self.tok.view(-1, 1))
        if self.kept is not None:
            self.kept.index_copy_(1, self.step_idx, self.logits.unsqueeze(1))
        self.step_idx.add_(1)

    def capture(self):
        # warm up once on a side stream (workspace allocation, attributes)
        saved = (self.cache.copy(), self.tok.clone(), self.tokens.clone(), self.step_idx.clone())
        s = torch.cuda.Stream(device=self.dev)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.runner.stream = _abi.stream_handle(s)
            self._body()
        torch.cuda.current_stream().wait_stream(s)
        # restore the state the warm-up step consumed
        self.cache.ssm_all.copy_(saved[0].ssm_all)
        self.cache.conv_all.copy_(saved[0].conv_all)
        self.tok.copy_(saved[1])
        self.tokens.copy_(saved[2])
        self.step_idx.copy_(saved[3])
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.runner.stream = _abi.stream_handle()
            self._body()
        self.graph = g
        self.runner.stream = _abi.stream_handle()

    def step(self):
        if self.use_graph:
            if self.graph is None:
                self.capture()
            self.graph.replay()
        else:
            self.runner.stream = _abi.stream_handle()
            self._body()


# captured decode graphs kept across generate() calls (a capture costs ~100x a token step);
# keyed by the parameters' identity, config, batch and length; only modest caches are kept
_GRAPH_CACHE: dict = {}
_GRAPH_CACHE_MAX = 2
_GRAPH_CACHE_MAX_BYTES = 8 << 30  # per entry: the decoder keeps its own copy of the cache


def clear_graph_cache() -> None:
    """Drop the decode graphs (and their cache buffers) kept by generate()."""
    _GRAPH_CACHE.clear()


def _decoder_for(params: ModelParams, cfg: ModelConfig, cache: Mamba2Cache, gen_len: int,
                 keep_logits: bool, use_graph: bool) -> "GreedyDecoder":
    nbytes = cache.ssm_all.numel() * cache.ssm_all.element_size() + \
        cache.conv_all.numel() * cache.conv_all.element_size()
    if not use_graph or nbytes > _GRAPH_CACHE_MAX_BYTES:
        return GreedyDecoder(params, cfg, cache, gen_len, keep_logits=keep_logits,
                             use_graph=use_graph)
    key = (id(params), cfg, cache.batch, gen_len, keep_logits, str(params.device))
    hit = _GRAPH_CACHE.get(key)
    if hit is not None and hit[0] is params:
        dec = hit[1]
        dec.cache.ssm_all.copy_(cache.ssm_all)  # the graph's buffers take this prefill's state
        dec.cache.conv_all.copy_(cache.conv_all)
        dec.tokens.zero_()
        return dec
    dec = GreedyDecoder(params, cfg, cache.copy(), gen_len, keep_logits=keep_logits,
                        use_graph=True)
    if len(_GRAPH_CACHE) >= _GRAPH_CACHE_MAX:
        _GRAPH_CACHE.pop(next(iter(_GRAPH_CACHE)))
    _GRAPH_CACHE[key] = (params, dec)
    return dec


def generate(params: ModelParams, prompt, gen_len: int, mode: str = "cached",
             cfg: ModelConfig | None = None, keep_logits: bool = False,
             use_graph: bool = True) -> GenerationResult:
    """decode.py:147-194 — greedy generation of gen_len tokens after (B, P)
    prompt.  cached: one prefill then gen_len-1 in-place steps (graph
    replays); non_cached: re-prefill the whole prefix per token (the
    quadratic baseline).  Ties resolve to the lowest id."""
    if cfg is None:
        raise ValueError("cfg is required")
    if gen_len < 1:
        raise ValueError("gen_len must be >= 1")
    if mode not in ("cached", "non_cached"):
        raise ValueError(f"unknown mode {mode!r}")
    dev = params.device
    ptok = check_tokens(prompt, cfg, 2, dev)
    B = ptok.shape[0]

    if mode == "non_cached":
        tokens = torch.zeros((B, gen_len), dtype=torch.int64, device=dev)
        kept = (
            torch.empty((B, gen_len, cfg.vocab_size), dtype=state_dtype(cfg), device=dev)
            if keep_logits
            else None
        )
        seq = ptok
        pick = torch.empty((B,), dtype=torch.int64, device=dev)
        for g in range(gen_len):
            last, _ = prefill(params, seq, cfg, logits="last", argmax_out=pick)
            if kept is not None:
                kept[:, g] = last
            tokens[:, g] = pick
            seq = torch.cat([ptok, tokens[:, : g + 1]], dim=1)
        return GenerationResult(tokens=tokens, steps=gen_len, per_step_logits=kept)

    pick = torch.empty((B,), dtype=torch.int64, device=dev)
    last, cache = prefill(params, ptok, cfg, logits="last", argmax_out=pick)
    dec = _decoder_for(params, cfg, cache, gen_len, keep_logits, use_graph)
    dec.tok.copy_(pick)
    dec.tokens[:, 0] = pick
    if dec.kept is not None:
        dec.kept[:, 0] = last
    dec.step_idx.fill_(1)
    for _ in range(gen_len - 1):
        dec.step()
    # the decoder may be reused by the next call: hand back copies
    return GenerationResult(tokens=dec.tokens.clone(), steps=gen_len,
                            per_step_logits=None if dec.kept is None else dec.kept.clone())
