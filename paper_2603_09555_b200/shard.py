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


# ------------------------------------------------------------------ head-group-sharded prefill


def upload_shard(host, cfg: ModelConfig, rank: int, world: int, device="cuda"):
    """bf16 device weights of this rank's head group (reference-layout host
    weights in, e.g. ``random_init_host``).  The embedding and final norm are
    replicated; every layer holds ``shard_layer_by_heads`` re-laid out like
    ``params.from_reference`` (K-major bf16, norm_w folded into W_out)."""
    from .params import LayerParams, ModelParams, decay_coefficient

    if cfg.policy.compute != "bf16":
        raise ValueError("head-group sharding runs the bf16 tensor-core path")
    dev = torch.device(device)

    def f32(x):
        return torch.as_tensor(np.ascontiguousarray(np.asarray(x, dtype=np.float32))).to(dev)

    def bf16_t(x):  # (K, N) host -> (N, K) bf16 device (K-major for the GEMMs)
        t = torch.as_tensor(np.ascontiguousarray(np.asarray(x, dtype=np.float32)))
        return t.t().to(torch.bfloat16).contiguous().to(dev)

    layers, heads, dims = [], None, None
    for lp in host.layers:
        sh = shard_layer_by_heads(lp, cfg, rank, world)
        heads, dims = sh.heads, sh.dims
        w_out = sh.norm_w.astype(np.float32)[:, None] * sh.W_out.astype(np.float32)
        layers.append(LayerParams(
            W_in=bf16_t(sh.W_in), conv_w=f32(sh.conv_w), conv_b=f32(sh.conv_b),
            dt_bias=f32(sh.dt_bias), A_log=f32(sh.A_log), D=f32(sh.D), norm_w=f32(sh.norm_w),
            W_out=bf16_t(w_out), a=f32(decay_coefficient(sh.A_log, cfg)),
        ))
    emb = torch.as_tensor(np.asarray(host.embedding, dtype=np.float32)).to(torch.bfloat16).to(dev)
    params = ModelParams(embedding=emb, layers=layers, final_norm_w=f32(host.final_norm_w),
                         mode="bf16")
    params.heads, params.local = heads, dims
    return params


def synthetic_shard(cfg: ModelConfig, rank: int, world: int, seed: int = 0, device="cuda"):
    """Throughput-only device weights of one head shard (the distributions of
    ``params.synthetic_init``), for benchmarking head-group sharding at sizes
    where a host init would take minutes."""
    from .params import LayerParams, ModelParams, decay_coefficient

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    dev = torch.device(device)
    heads = head_slice(cfg.n_heads, rank, world)
    loc = local_dims(cfg, heads)

    def normal(shape, std=0.02):
        return (torch.randn(shape, generator=g, device=dev) * std).to(torch.bfloat16).contiguous()

    def uniform(shape, lo, hi):
        return torch.rand(shape, generator=g, device=dev, dtype=torch.float64) * (hi - lo) + lo

    bound = 1.0 / np.sqrt(cfg.conv_kernel)
    layers = []
    for _ in range(cfg.n_layers):
        dt = uniform((loc.n_heads,), 1e-3, 1e-1)
        a_log = torch.log(uniform((loc.n_heads,), 1.0, 16.0)).to(torch.float32)
        layers.append(LayerParams(
            W_in=normal((loc.d_in_proj, cfg.d_model)),
            conv_w=uniform((loc.conv_dim, cfg.conv_kernel), -bound, bound).float(),
            conv_b=torch.zeros(loc.conv_dim, device=dev),
            dt_bias=torch.log(torch.expm1(dt)).float(),
            A_log=a_log,
            D=torch.randn(loc.n_heads, generator=g, device=dev),
            norm_w=torch.ones(loc.d_inner, device=dev),
            W_out=normal((cfg.d_model, loc.d_inner)),
            a=torch.as_tensor(decay_coefficient(a_log.cpu().numpy(), cfg),
                              dtype=torch.float32).to(dev),
        ))
    params = ModelParams(embedding=normal((cfg.vocab_size, cfg.d_model)), layers=layers,
                         final_norm_w=torch.ones(cfg.d_model, device=dev), mode="bf16")
    params.heads, params.local = heads, loc
    return params


def _local_dims_struct(cfg: ModelConfig, local):
    from .model import dims_struct

    d = dims_struct(cfg)
    d.d_inner = local.d_inner
    d.n_heads = local.n_heads
    return d


class HeadShardedPrefill:
    """One rank's side of a head-group-sharded ``prefill`` (model.py:177-206),
    driven layer by layer: ``partial(i)`` runs this rank's heads of layer i
    (in_proj / conv / SSD / gate / partial out_proj) into ``self.buf`` =
    ``[partial (rows, d_model) | sum u^2]``; the caller sums ``buf`` over the
    ranks (one all-reduce) and calls ``finish()``; ``logits()`` runs the
    replicated final norm + tied head on the last position."""

    def __init__(self, shard_params, tokens, cfg: ModelConfig):
        from .model import _Runner, check_tokens, layer_struct

        self.cfg, self.params = cfg, shard_params
        self.r = r = _Runner(shard_params, cfg)
        tok = check_tokens(tokens, cfg, 2, r.dev)
        self.B, self.T = tok.shape
        self.rows = self.B * self.T
        local = shard_params.local
        self.dims_l = _local_dims_struct(cfg, local)
        self.layers = [layer_struct(lp) for lp in shard_params.layers]
        self.hidden, self.lp = r.embed(tok.reshape(-1))
        self.ld = (cfg.d_model + 4) // 4 * 4  # 16-byte rows: [partial | sum u^2 | pad]
        self.buf = torch.empty((self.rows, self.ld), dtype=torch.float32, device=r.dev)
        self.ssm = torch.empty((cfg.n_layers, self.B, local.n_heads, cfg.head_dim, cfg.d_state),
                               dtype=torch.float32, device=r.dev)
        self.conv = torch.empty((cfg.n_layers, self.B, local.conv_dim, cfg.conv_kernel - 1),
                                dtype=torch.float32, device=r.dev)
        self.ws = r.workspace(r.lib.ssd200_prefill_layer_workspace(self.dims_l, self.B, self.T))

    def restart(self, tokens) -> None:
        """Embed a new (B, T) token batch of the same shape into the existing
        buffers (no allocation: a benchmark loop reuses one object)."""
        from . import _abi
        from .model import check_tokens

        r, cfg = self.r, self.cfg
        tok = check_tokens(tokens, cfg, 2, r.dev)
        if tuple(tok.shape) != (self.B, self.T):
            raise ValueError(f"restart needs tokens of shape {(self.B, self.T)}, got {tuple(tok.shape)}")
        r._call("ssd200_embed", r.lib.ssd200_embed, r.dims, tok.data_ptr(), self.rows,
                cfg.vocab_size, self.params.embedding.data_ptr(), self.hidden.data_ptr(),
                _abi.ptr(self.lp), r.stream)

    def partial(self, i: int) -> torch.Tensor:
        from . import _abi

        r = self.r
        _abi.check(
            r.lib.ssd200_prefill_layer_partial(
                self.dims_l, self.layers[i], self.lp.data_ptr(), self.buf.data_ptr(), self.ld,
                self.ssm[i].data_ptr(), self.conv[i].data_ptr() if self.conv.numel() else None,
                self.B, self.T, self.ws.data_ptr(), self.ws.numel(), r.stream,
            ),
            "ssd200_prefill_layer_partial",
        )
        return self.buf

    def finish(self):
        from . import _abi

        cfg, r = self.cfg, self.r
        _abi.check(
            r.lib.ssd200_resid_norm_finish(
                cfg.d_model, cfg.d_inner, float(cfg.norm_eps), self.hidden.data_ptr(),
                self.lp.data_ptr(), self.buf.data_ptr(), self.ld, self.rows, r.stream,
            ),
            "ssd200_resid_norm_finish",
        )

    def logits(self, argmax: torch.Tensor | None = None) -> torch.Tensor:
        cfg = self.cfg
        out = torch.empty((self.B, cfg.vocab_size), dtype=torch.float32, device=self.r.dev)
        self.r.head(self.hidden, self.T * cfg.d_model, self.B, logits=out, argmax=argmax,
                    base_offset=(self.T - 1) * cfg.d_model)
        return out


def prefill_head_sharded(shard_params, tokens, cfg: ModelConfig, group=None):
    """Head-group-sharded ``prefill`` for this rank: every rank holds
    ``upload_shard(...)`` of its heads and the same tokens; per layer ONE
    all-reduce (sum) of ``[partial | sum u^2]`` over ``group`` (NCCL on the
    GPU path) after the head-sharded out_proj.  Returns the last-position
    logits (B, V) (replicated) and this rank's final SSM states
    (n_layers, B, H_local, P, N)."""
    import torch.distributed as dist

    run = HeadShardedPrefill(shard_params, tokens, cfg)
    for i in range(cfg.n_layers):
        buf = run.partial(i)
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
        run.finish()
    return run.logits(), run.ssm


# ------------------------------------------------------------------ head-group-sharded decode


class HeadShardedDecoder:
    """One rank's side of head-group-sharded greedy decoding (decode.py:77-194):
    the rank keeps its heads' slice of the cache (SSM states (n_layers, B,
    H_local, P, N), conv windows over its x channels + the replicated B / C
    channels) and, per token, per layer, runs ``ssd200_decode_layer_partial``
    into ``buf`` = ``[partial (B, d_model) | sum u^2]``; the caller sums ``buf``
    over the ranks (one all-reduce per layer, as in prefill) and calls
    ``finish()``; the final norm + tied head + argmax are replicated.

    Build it from a finished ``HeadShardedPrefill`` (its states become the
    cache) or from explicit cache tensors."""

    def __init__(self, shard_params, cfg: ModelConfig, ssm: torch.Tensor, conv: torch.Tensor):
        from .model import _Runner, layer_struct

        self.cfg, self.params = cfg, shard_params
        self.r = r = _Runner(shard_params, cfg)
        local = shard_params.local
        self.dims_l = _local_dims_struct(cfg, local)
        self.layers = [layer_struct(lp) for lp in shard_params.layers]
        self.ssm, self.conv = ssm, conv  # updated in place
        self.B = ssm.shape[1]
        self.ld = (cfg.d_model + 4) // 4 * 4
        self.buf = torch.empty((self.B, self.ld), dtype=torch.float32, device=r.dev)
        self.ws = r.workspace(r.lib.ssd200_decode_layer_workspace(self.dims_l, self.B))
        self.hidden = self.lp = None
        # fixed buffers for the graph-captured step (HeadShardedGraphDecoder)
        self.tok = torch.zeros((self.B,), dtype=torch.int64, device=r.dev)
        self.logits = torch.empty((self.B, cfg.vocab_size), dtype=torch.float32, device=r.dev)
        self._hid = torch.empty((self.B, cfg.d_model), dtype=torch.float32, device=r.dev)
        self._lp = torch.empty((self.B, cfg.d_model), dtype=torch.bfloat16, device=r.dev)

    @classmethod
    def from_prefill(cls, run: "HeadShardedPrefill"):
        return cls(run.params, run.cfg, run.ssm, run.conv)

    def begin(self, tok: torch.Tensor):
        """Embed this step's tokens (B,) — replicated on every rank."""
        self.hidden, self.lp = self.r.embed(tok.reshape(-1))

    def begin_fixed(self):
        """Embed ``self.tok`` into the decoder's fixed hidden buffers (graph step)."""
        cfg, r = self.cfg, self.r
        r._call("ssd200_embed", r.lib.ssd200_embed, r.dims, self.tok.data_ptr(), self.B,
                cfg.vocab_size, self.params.embedding.data_ptr(), self._hid.data_ptr(),
                self._lp.data_ptr(), r.stream)
        self.hidden, self.lp = self._hid, self._lp

    def head_fixed(self):
        """Final norm + tied head into ``self.logits``, greedy pick into ``self.tok``."""
        self.r.head(self.hidden, self.cfg.d_model, self.B, logits=self.logits, argmax=self.tok)

    def partial(self, i: int) -> torch.Tensor:
        from . import _abi

        r = self.r
        _abi.check(
            r.lib.ssd200_decode_layer_partial(
                self.dims_l, self.layers[i], self.lp.data_ptr(), self.buf.data_ptr(), self.ld,
                self.ssm[i].data_ptr(), self.ssm[i].data_ptr(), self.conv[i].data_ptr(),
                self.conv[i].data_ptr(), self.B, self.ws.data_ptr(), self.ws.numel(), r.stream,
            ),
            "ssd200_decode_layer_partial",
        )
        return self.buf

    def finish(self):
        from . import _abi

        cfg, r = self.cfg, self.r
        _abi.check(
            r.lib.ssd200_resid_norm_finish(
                cfg.d_model, cfg.d_inner, float(cfg.norm_eps), self.hidden.data_ptr(),
                self.lp.data_ptr(), self.buf.data_ptr(), self.ld, self.B, r.stream,
            ),
            "ssd200_resid_norm_finish",
        )

    def logits_and_pick(self):
        """Replicated final RMSNorm + tied head + greedy pick (ties -> lowest id)."""
        cfg = self.cfg
        out = torch.empty((self.B, cfg.vocab_size), dtype=torch.float32, device=self.r.dev)
        pick = torch.empty((self.B,), dtype=torch.int64, device=self.r.dev)
        self.r.head(self.hidden, cfg.d_model, self.B, logits=out, argmax=pick)
        return out, pick


def sum_reduce(bufs) -> None:
    """The all-reduce of simulated ranks living in one process: every buffer
    becomes the sum over the ranks, added in rank order (a fixed order, so the
    result is deterministic)."""
    total = bufs[0].clone()
    for b in bufs[1:]:
        total.add_(b)
    for b in bufs:
        b.copy_(total)


def nccl_reduce(group=None):
    """The all-reduce of one rank per process: NCCL (sum) on the caller's
    stream, capturable in a CUDA graph."""
    import torch.distributed as dist

    def reduce(bufs):
        for b in bufs:
            dist.all_reduce(b, op=dist.ReduceOp.SUM, group=group)

    return reduce


class HeadShardedGraphDecoder:
    """Head-group-sharded greedy decoding with the WHOLE token step captured as
    one CUDA graph: embed -> per layer [every local rank's
    ``ssd200_decode_layer_partial`` -> reduce of ``[partial | sum u^2]`` ->
    ``ssd200_resid_norm_finish``] -> final norm + tied head + argmax -> token
    feedback, replayed once per token with no return to Python in between
    (the collective stays inside the captured step).

    ``ranks``: the HeadShardedDecoder(s) this process drives — one per GPU in
    a real run (``reduce = nccl_reduce(group)``; NCCL kernels are captured
    into the graph) or several on one device to simulate ranks (``reduce =
    sum_reduce``).  ``reduce=None`` is the single-rank case (no collective)."""

    def __init__(self, ranks, gen_len: int, reduce=None, use_graph: bool = True):
        self.ranks = list(ranks)
        self.reduce = reduce
        d0 = self.ranks[0]
        self.cfg, self.B, self.dev = d0.cfg, d0.B, d0.r.dev
        self.tokens = torch.zeros((self.B, gen_len), dtype=torch.int64, device=self.dev)
        self.step_idx = torch.zeros((1,), dtype=torch.int64, device=self.dev)
        self.use_graph = use_graph
        self.graph = None

    def set_token(self, tok: torch.Tensor) -> None:
        for d in self.ranks:
            d.tok.copy_(tok)

    def _set_stream(self, stream):
        for d in self.ranks:
            d.r.stream = stream

    def _body(self):
        for d in self.ranks:
            d.begin_fixed()
        for i in range(self.cfg.n_layers):
            for d in self.ranks:
                d.partial(i)
            if self.reduce is not None:
                self.reduce([d.buf for d in self.ranks])
            for d in self.ranks:
                d.finish()
        for d in self.ranks:
            d.head_fixed()
        self.tokens.index_copy_(1, self.step_idx, self.ranks[0].tok.view(-1, 1))
        self.step_idx.add_(1)

    def capture(self):
        from . import _abi

        with torch.cuda.device(self.dev):
            saved = ([(d.ssm.clone(), d.conv.clone(), d.tok.clone()) for d in self.ranks],
                     self.tokens.clone(), self.step_idx.clone())
            side = torch.cuda.Stream(device=self.dev)
            side.wait_stream(torch.cuda.current_stream(self.dev))
            with torch.cuda.stream(side):  # warm-up: workspaces, attributes, NCCL setup
                self._set_stream(_abi.stream_handle(side))
                self._body()
            torch.cuda.current_stream(self.dev).wait_stream(side)
            for d, (ssm, conv, tok) in zip(self.ranks, saved[0]):
                d.ssm.copy_(ssm)
                d.conv.copy_(conv)
                d.tok.copy_(tok)
            self.tokens.copy_(saved[1])
            self.step_idx.copy_(saved[2])
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._set_stream(_abi.stream_handle(torch.cuda.current_stream(self.dev)))
                self._body()
            self.graph = g
            self._set_stream(_abi.stream_handle(torch.cuda.current_stream(self.dev)))

    def step(self):
        from . import _abi

        if not self.use_graph:
            self._set_stream(_abi.stream_handle(torch.cuda.current_stream(self.dev)))
            self._body()
            return
        if self.graph is None:
            self.capture()
        self.graph.replay()


def generate_head_sharded(shard_params, prompt, gen_len: int, cfg: ModelConfig, group=None,
                          use_graph: bool = True):
    """Head-group-sharded cached ``generate`` (decode.py:147-194) for this rank:
    a head-sharded prefill of the prompt (one all-reduce per layer), then
    gen_len - 1 token steps replayed as ONE captured CUDA graph each
    (HeadShardedGraphDecoder: the per-layer NCCL all-reduce is inside the
    graph).  Returns the (B, gen_len) greedy tokens (replicated on every rank)."""
    import torch.distributed as dist

    if gen_len < 1:
        raise ValueError("gen_len must be >= 1")
    run = HeadShardedPrefill(shard_params, prompt, cfg)
    multi = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1
    for i in range(cfg.n_layers):
        buf = run.partial(i)
        if multi:
            dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
        run.finish()
    tok = torch.empty((run.B,), dtype=torch.int64, device=run.r.dev)
    run.logits(argmax=tok)  # greedy pick, ties -> lowest id (decode.py:72-74)
    dec = HeadShardedGraphDecoder([HeadShardedDecoder.from_prefill(run)], gen_len,
                                  reduce=nccl_reduce(group) if multi else None,
                                  use_graph=use_graph)
    dec.set_token(tok)
    dec.tokens[:, 0] = tok
    dec.step_idx.fill_(1)
    for _ in range(gen_len - 1):
        dec.step()
    return dec.tokens.clone()
