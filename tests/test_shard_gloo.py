"""Multi-process (gloo, world size 2, CPU) tests of the sharding host logic
(SURVEY.md §8(e)).  The arithmetic on each rank is the oracle here — the
point is the partitioning and the collectives, which are the same code the
GPU path runs under NCCL."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as orc
from paper_2603_09555_b200 import shard
from paper_2603_09555_b200.params import random_init_host
from conftest import small_config


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(fn, world=2, *args):
    port = _free_port()
    mp.spawn(_entry, args=(world, port, fn, args), nprocs=world, join=True)


def _entry(rank, world, port, fn, args):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world, *args)
    finally:
        dist.destroy_process_group()


# ------------------------------------------------------------------ pure host logic


@pytest.mark.parametrize("batch", [1, 2, 3, 5, 8, 13])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_batch_slice_partition(batch, world):
    seen = []  # ranks beyond the batch get empty slices; still a partition
    for r in range(world):
        s = shard.batch_slice(batch, r, world)
        seen.extend(range(s.start, s.stop))
        assert s.stop - s.start in (batch // world, batch // world + 1)
    assert seen == list(range(batch))


def test_head_slice_partition():
    for H, world in [(24, 2), (32, 8), (80, 8), (5, 2)]:
        heads = []
        for r in range(world):
            s = shard.head_slice(H, r, world)
            heads.extend(range(s.start, s.stop))
        assert heads == list(range(H))
    with pytest.raises(ValueError):
        shard.head_slice(2, 0, 4)
    with pytest.raises(ValueError):
        shard.batch_slice(4, 2, 2)


def test_shard_layer_shapes():
    cfg = small_config(d_model=32, head_dim=8)  # d_inner 64, H 8
    host = random_init_host(cfg, 0)
    lay = shard.shard_layer_by_heads(host.layers[0], cfg, 1, 2)
    d = lay.dims
    assert d.n_heads == 4 and d.d_inner == 32
    assert lay.W_in.shape == (cfg.d_model, d.d_in_proj)
    assert lay.conv_w.shape == (d.conv_dim, cfg.conv_kernel)
    assert lay.W_out.shape == (d.d_inner, cfg.d_model)
    # the B / C columns are replicated verbatim
    gn = cfg.n_groups * cfg.d_state
    full = np.asarray(host.layers[0].W_in)
    np.testing.assert_array_equal(lay.W_in[:, 2 * d.d_inner: 2 * d.d_inner + 2 * gn],
                                  full[:, 2 * cfg.d_inner: 2 * cfg.d_inner + 2 * gn])


# ------------------------------------------------------------------ gloo world size 2


def _gather_worker(rank, world, batch):
    full = torch.arange(batch * 3, dtype=torch.float64).reshape(batch, 3)
    s = shard.batch_slice(batch, rank, world)
    got = shard.gather_rows(full[s].clone(), batch)
    assert torch.equal(got, full), (rank, got)


@pytest.mark.parametrize("batch", [2, 5])
def test_gather_rows_gloo(batch):
    _run(_gather_worker, 2, batch)


def _batch_prefill_worker(rank, world):
    cfg = small_config(n_layers=2).with_policy(compute="f64")
    host = random_init_host(cfg, 3)
    ids = np.random.default_rng(0).integers(0, cfg.vocab_size, size=(5, 24))
    s = shard.batch_slice(ids.shape[0], rank, world)
    logits, _, _ = orc.prefill(host, ids[s], cfg)
    got = shard.gather_rows(torch.from_numpy(np.ascontiguousarray(logits)), ids.shape[0])
    ref, _, _ = orc.prefill(host, ids, cfg)
    # rows are independent: the sharded result equals the unsharded one bitwise
    np.testing.assert_array_equal(got.numpy(), ref)


def test_batch_sharded_prefill_gloo():
    _run(_batch_prefill_worker, 2)


def _head_sharded_block(lay, hidden, cfg):
    """One rank's part of a head-sharded block: returns (partial, sum u^2)."""
    d = lay.dims
    P, N, G = cfg.head_dim, cfg.d_state, cfg.n_groups
    nb, nt, _ = hidden.shape
    proj = hidden @ lay.W_in
    z = proj[..., : d.d_inner]
    xbc = proj[..., d.d_inner: d.d_inner + d.conv_dim]
    dt_raw = proj[..., d.d_inner + d.conv_dim:]
    act = orc.causal_conv_silu(xbc, lay.conv_w, lay.conv_b)
    x = act[..., : d.d_inner]
    Bm = act[..., d.d_inner: d.d_inner + G * N].reshape(nb, nt, G, N)
    Cm = act[..., d.d_inner + G * N:].reshape(nb, nt, G, N)
    dt = orc.step_sizes(dt_raw, lay.dt_bias, cfg.dt_limits, hidden.dtype)
    a = orc.decay_scalar(lay.A_log, hidden.dtype)
    Xh = x.reshape(nb, nt, d.n_heads, P)
    Y, _ = orc.chunked_scan(Xh, dt, a, Bm, Cm, cfg.chunk_size)
    y = (Y + lay.D[None, None, :, None] * Xh).reshape(nb, nt, d.d_inner)
    u = y * orc.silu(z)
    ssq = np.sum(u * u, axis=-1)
    partial = u @ (lay.norm_w[:, None] * lay.W_out)  # norm_w folded into W_out
    return partial, ssq


def _head_block_worker(rank, world):
    cfg = small_config(d_model=32, head_dim=8, chunk_size=8).with_policy(compute="f64")
    host = random_init_host(cfg, 5)
    layer = host.layers[0]
    rng = np.random.default_rng(1)
    layer.norm_w = (1.0 + 0.3 * rng.standard_normal(cfg.d_inner))  # non-unit norm weights
    hidden = rng.standard_normal((2, 20, cfg.d_model))
    lay = shard.shard_layer_by_heads(layer, cfg, rank, world)
    partial, ssq = _head_sharded_block(lay, hidden, cfg)
    # the single all-reduce of the layer: [partial | sum u^2]
    buf = torch.from_numpy(np.concatenate([partial, ssq[..., None]], axis=-1).copy())
    dist.all_reduce(buf, op=dist.ReduceOp.SUM)
    buf = buf.numpy()
    total, ssq_all = buf[..., :-1], buf[..., -1]
    out = hidden + total / np.sqrt(ssq_all / cfg.d_inner + cfg.norm_eps)[..., None]
    ref, _, _ = orc.block(layer, hidden, cfg)
    err = np.max(np.abs(out - ref)) / np.max(np.abs(ref))
    assert err < 1e-12, err


def test_head_sharded_block_gloo():
    _run(_head_block_worker, 2)


def _head_sharded_decode_layer(lay, hidden, ssm, conv, cfg):
    """One rank's part of a head-sharded decode layer (decode.py:99-140 on its
    heads): returns (partial, sum u^2, new ssm slice, new conv slice)."""
    d = lay.dims
    P, N, G = cfg.head_dim, cfg.d_state, cfg.n_groups
    nb = hidden.shape[0]
    proj = hidden @ lay.W_in
    z = proj[:, : d.d_inner]
    col = proj[:, d.d_inner: d.d_inner + d.conv_dim]
    dt_raw = proj[:, d.d_inner + d.conv_dim:]
    window = np.concatenate([conv, col[:, :, None]], axis=2)  # roll_and_insert, decode.py:65-69
    act = orc.silu(np.einsum("bck,ck->bc", window, lay.conv_w) + lay.conv_b)
    x = act[:, : d.d_inner].reshape(nb, d.n_heads, P)
    rep = d.n_heads // G
    Bh = np.repeat(act[:, d.d_inner: d.d_inner + G * N].reshape(nb, G, N), rep, 1)
    Ch = np.repeat(act[:, d.d_inner + G * N:].reshape(nb, G, N), rep, 1)
    dt = orc.step_sizes(dt_raw[:, None, :], lay.dt_bias, cfg.dt_limits, hidden.dtype)[:, 0, :]
    a = orc.decay_scalar(lay.A_log, hidden.dtype)
    h = np.exp(a * dt)[:, :, None, None] * ssm + dt[:, :, None, None] * x[..., None] * Bh[:, :, None]
    y = np.einsum("bhn,bhpn->bhp", Ch, h) + lay.D[None, :, None] * x
    u = y.reshape(nb, d.d_inner) * orc.silu(z)
    return u @ (lay.norm_w[:, None] * lay.W_out), np.sum(u * u, axis=-1), h, window[:, :, 1:]


def _head_decode_worker(rank, world):
    """Head-sharded decode step: each rank updates only its heads'
    cache slice and contributes [partial | sum u^2] to ONE all-reduce per layer;
    the logits equal the unsharded oracle decode_step."""
    cfg = small_config(d_model=32, head_dim=8, chunk_size=8).with_policy(compute="f64")
    host = random_init_host(cfg, 6)
    rng = np.random.default_rng(2)
    for layer in host.layers:
        layer.norm_w = 1.0 + 0.3 * rng.standard_normal(cfg.d_inner)
    B, P = 3, cfg.head_dim
    tok = rng.integers(0, cfg.vocab_size, size=B)
    conv_dim = cfg.d_inner + 2 * cfg.n_groups * cfg.d_state
    ssm = [rng.standard_normal((B, cfg.n_heads, P, cfg.d_state)) for _ in host.layers]
    conv = [rng.standard_normal((B, conv_dim, cfg.conv_kernel - 1)) for _ in host.layers]
    hidden = np.asarray(host.embedding, dtype=np.float64)[tok]
    for i, layer in enumerate(host.layers):
        lay = shard.shard_layer_by_heads(layer, cfg, rank, world)
        hs = lay.heads
        ch = slice(hs.start * P, hs.stop * P)
        conv_l = np.concatenate([conv[i][:, ch], conv[i][:, cfg.d_inner:]], axis=1)
        partial, ssq, h_new, c_new = _head_sharded_decode_layer(lay, hidden, ssm[i][:, hs],
                                                                conv_l, cfg)
        buf = torch.from_numpy(np.concatenate([partial, ssq[:, None]], axis=-1).copy())
        dist.all_reduce(buf, op=dist.ReduceOp.SUM)
        buf = buf.numpy()
        hidden = hidden + buf[:, :-1] / np.sqrt(buf[:, -1] / cfg.d_inner + cfg.norm_eps)[:, None]
        _, ref_ssm, ref_conv = orc.decode_step(host, ssm, conv, tok, cfg)
        assert np.max(np.abs(h_new - ref_ssm[i][:, hs])) < 1e-12 or i > 0
        if i == 0:
            assert np.max(np.abs(c_new[:, : ch.stop - ch.start] - ref_conv[0][:, ch])) == 0
    emb = np.asarray(host.embedding, dtype=np.float64)
    logits = orc.rms_norm(hidden, host.final_norm_w, cfg.norm_eps) @ emb.T
    ref, _, _ = orc.decode_step(host, ssm, conv, tok, cfg)
    err = np.max(np.abs(logits - ref)) / np.max(np.abs(ref))
    assert err < 1e-12, err


def test_head_sharded_decode_gloo():
    _run(_head_decode_worker, 2)
