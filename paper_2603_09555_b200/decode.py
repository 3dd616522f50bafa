"""Cached decode over the C-ABI — mirrors ``cache_init``, ``decode_step`` and
``generate`` (decode.py:49-194).

``decode_step`` is functional like the reference (a new cache is returned;
the input cache is not mutated).  ``generate`` updates one cache in place and
replays the whole per-token step (embed -> every layer -> norm -> head ->
argmax -> token feedback) as ONE CUDA graph, G-1 times, with no host
synchronisation until the tokens are read back.
"""

from __future__ import annotations

import weakref

import numpy as np
import torch

from . import _abi
from .cache import GenerationResult, Mamba2Cache, state_dtype
from .config import ModelConfig
from .model import PolicyAudit, _audit, _Runner, check_tokens, prefill
from .params import ModelParams


def cache_init(cfg: ModelConfig, batch: int, device="cuda") -> Mamba2Cache:
    """decode.py:49-62 — all-zero cache."""
    if batch < 1:
        raise ValueError("batch must be >= 1")
    return Mamba2Cache.empty(cfg, batch, device=device, zero=True)


def _step_into(r: _Runner, cfg, tok, cache_in: Mamba2Cache, cache_out: Mamba2Cache,
               logits=None, argmax=None, chained: bool = True):
    B = tok.shape[0]
    hidden, lp = r.embed(tok)
    if chained:  # all layers in one ABI call
        r.decode_layers(hidden, lp, cache_in.ssm_all, cache_out.ssm_all, cache_in.conv_all,
                        cache_out.conv_all, B)
    else:
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
                 keep_logits: bool = False, use_graph: bool = True):
        self.cfg = cfg
        self.dev = torch.device(params.device)
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
        self.graph = None
        self.use_graph = use_graph

    def nbytes(self) -> int:
        """Device bytes this decoder keeps alive (cache + token / logits buffers)."""
        n = self.cache.nbytes + self.tokens.numel() * 8 + self.logits.numel() * self.logits.element_size()
        if self.kept is not None:
            n += self.kept.numel() * self.kept.element_size()
        return n

    def _body(self):
        cfg = self.cfg
        _step_into(self.runner, cfg, self.tok, self.cache, self.cache, logits=self.logits,
                   argmax=self.tok)
        # bookkeeping: tokens[:, step] = tok; step += 1
        self.tokens.index_copy_(1, self.step_idx, self.tok.view(-1, 1))
        if self.kept is not None:
            self.kept.index_copy_(1, self.step_idx, self.logits.unsqueeze(1))
        self.step_idx.add_(1)

    def capture(self):
        with torch.cuda.device(self.dev):
            # warm up once on a side stream (workspace allocation, attributes)
            saved = (self.cache.copy(), self.tok.clone(), self.tokens.clone(), self.step_idx.clone())
            s = torch.cuda.Stream(device=self.dev)
            s.wait_stream(torch.cuda.current_stream(self.dev))
            with torch.cuda.stream(s):
                self.runner.stream = _abi.stream_handle(s)
                self._body()
            torch.cuda.current_stream(self.dev).wait_stream(s)
            # restore the state the warm-up step consumed
            self.cache.ssm_all.copy_(saved[0].ssm_all)
            self.cache.conv_all.copy_(saved[0].conv_all)
            self.tok.copy_(saved[1])
            self.tokens.copy_(saved[2])
            self.step_idx.copy_(saved[3])
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.runner.stream = _abi.stream_handle(torch.cuda.current_stream(self.dev))
                self._body()
            self.graph = g
            self.runner.stream = _abi.stream_handle(torch.cuda.current_stream(self.dev))

    def step(self):
        if self.use_graph:
            if self.graph is None:
                self.capture()
            self.graph.replay()
        else:
            self.runner.stream = _abi.stream_handle(torch.cuda.current_stream(self.dev))
            self._body()


# Captured decode graphs kept across generate() calls (a capture costs ~100x a
# token step).  Keyed by the parameters' identity, config, batch and length;
# the parameters are held weakly (an entry dies with its params).  Only
# modest decoders are kept: each holds its own cache copy and token buffers
# (counted against _GRAPH_CACHE_MAX_BYTES per entry and _GRAPH_CACHE_TOTAL_BYTES
# overall); keep_logits runs are never cached (their (B, G, V) buffer is the
# caller's result).  clear_graph_cache() drops everything.
_GRAPH_CACHE: dict = {}
_GRAPH_CACHE_MAX = 2
_GRAPH_CACHE_MAX_BYTES = 8 << 30
_GRAPH_CACHE_TOTAL_BYTES = 12 << 30


def clear_graph_cache() -> None:
    """Drop the decode graphs (and their cache buffers) kept by generate()."""
    _GRAPH_CACHE.clear()


def _decoder_for(params: ModelParams, cfg: ModelConfig, cache: Mamba2Cache, gen_len: int,
                 keep_logits: bool, use_graph: bool) -> "GreedyDecoder":
    B = cache.batch
    need = cache.nbytes + B * gen_len * 8 + B * cfg.vocab_size * 4
    if not use_graph or keep_logits or need > _GRAPH_CACHE_MAX_BYTES:
        return GreedyDecoder(params, cfg, cache, gen_len, keep_logits=keep_logits,
                             use_graph=use_graph)
    key = (id(params), cfg, B, gen_len, str(params.device))
    hit = _GRAPH_CACHE.get(key)
    if hit is not None and hit[0]() is params:
        dec = hit[1]
        dec.cache.ssm_all.copy_(cache.ssm_all)  # the graph's buffers take this prefill's state
        dec.cache.conv_all.copy_(cache.conv_all)
        dec.tokens.zero_()
        return dec
    for k in [k for k, (ref, _) in _GRAPH_CACHE.items() if ref() is None]:
        del _GRAPH_CACHE[k]  # entries whose params are gone
    dec = GreedyDecoder(params, cfg, cache.copy(), gen_len, use_graph=True)
    while _GRAPH_CACHE and (len(_GRAPH_CACHE) >= _GRAPH_CACHE_MAX or
                            sum(d.nbytes() for _, d in _GRAPH_CACHE.values()) + dec.nbytes()
                            > _GRAPH_CACHE_TOTAL_BYTES):
        _GRAPH_CACHE.pop(next(iter(_GRAPH_CACHE)))
    _GRAPH_CACHE[key] = (weakref.ref(params), dec)
    return dec


def generate(params: ModelParams, prompt, gen_len: int, mode: str = "cached",
             cfg: ModelConfig | None = None, keep_logits: bool = False,
             use_graph: bool = True) -> GenerationResult:
    """decode.py:147-194 — greedy generation of gen_len tokens after (B, P)
    prompt.  cached: one prefill then gen_len-1 in-place steps (graph
    replays); non_cached: re-prefill the whole prefix per token (the
    quadratic baseline).  Ties resolve to the lowest id.

    The captured decode graph is kept for the next call with the same params,
    config, batch and gen_len (not for keep_logits runs; see _GRAPH_CACHE);
    ``decode.clear_graph_cache()`` releases it."""
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
