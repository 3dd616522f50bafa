"""Parity of the CUDA path against the reference (golden vectors) and the CPU
oracle.  GPU only; every call goes through libssd200.so."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle as orc
from conftest import (BF16_BOUND, BF16_STATE_BOUND, SMALL_MODELS, golden, make_instance, report,
                      small_config)

pytestmark = pytest.mark.gpu

F64_GATE = 1e-10
F32_RTOL, F32_ATOL = 1e-5, 2e-4  # test_acceptance.py:34-38
CACHED_FULL_F32 = 1.3e-4


def _np(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


# ----------------------------------------------------------- chunked scan


@pytest.mark.parametrize("i", range(8))
def test_chunk_scan_vs_golden(i):
    import paper_2603_09555_b200 as m

    z = golden("ssd_cases.npz")
    g = lambda k: z[f"{i}.{k}"]  # noqa: E731
    init = g("init") if int(g("has_init")) else None
    L = int(g("L"))
    for dt_, tag in ((np.float64, "f64"), (np.float32, "f32")):
        inp = m.SsdInputs(X=g("X").astype(dt_), dt=g("dt").astype(dt_), a=g("a").astype(dt_),
                          Bmat=g("B").astype(dt_), Cmat=g("C").astype(dt_))
        out = m.ssd_forward(inp, L, initial_state=None if init is None else init.astype(dt_))
        Y, fin = _np(out.Y), _np(out.final_state)
        ys, hs = z[f"{i}.Y_seq"], z[f"{i}.final_seq"]
        if tag == "f64":
            assert np.abs(Y - ys).max() <= F64_GATE
            assert np.abs(fin - hs).max() <= F64_GATE * max(1.0, np.abs(hs).max())
        else:
            assert np.all(np.abs(Y - ys) <= F32_ATOL + F32_RTOL * np.abs(ys))
            assert np.all(np.abs(fin - hs) <= F32_ATOL + F32_RTOL * np.abs(hs))


def test_chunk_scan_acceptance_pool():
    """Criterion 1 (test_acceptance.py:70-94) on a 60-instance slice of the
    same distribution, chunk sizes from {1,4,16,64,256}."""
    import paper_2603_09555_b200 as m

    rng = np.random.default_rng(2024)
    pick = np.random.default_rng(77)
    for _ in range(60):
        heads = int(rng.integers(1, 5))
        groups = heads if rng.integers(2) else 1
        inst = make_instance(rng, batch=int(rng.integers(1, 3)), seq=int(rng.integers(1, 513)),
                             heads=heads, pdim=int(rng.integers(1, 9)),
                             ndim=int(rng.integers(1, 9)), groups=groups)
        L = int(pick.choice((1, 4, 16, 64, 256)))
        ys, hs = orc.sequential_scan(inst["X"], inst["dt"], inst["a"], inst["B"], inst["C"])
        out = m.ssd_forward(m.SsdInputs(inst["X"], inst["dt"], inst["a"], inst["B"], inst["C"]), L)
        assert np.abs(_np(out.Y) - ys).max() <= F64_GATE
        assert np.abs(_np(out.final_state) - hs).max() <= F64_GATE
        f = {k: v.astype(np.float32) for k, v in inst.items()}
        out32 = m.ssd_forward(m.SsdInputs(f["X"], f["dt"], f["a"], f["B"], f["C"]), L)
        assert np.all(np.abs(_np(out32.Y) - ys) <= F32_ATOL + F32_RTOL * np.abs(ys))


def test_chunk_invariance_and_masks():
    """Criterion 2 / 6: results independent of L, masks bitwise identical."""
    import paper_2603_09555_b200 as m

    rng = np.random.default_rng(5)
    inst = make_instance(rng, batch=2, seq=300, heads=3, pdim=8, ndim=8)
    si = m.SsdInputs(inst["X"], inst["dt"], inst["a"], inst["B"], inst["C"])
    base = m.ssd_forward(si, 1)
    for L in (4, 16, 64, 256):
        o = m.ssd_forward(si, L)
        assert (o.Y - base.Y).abs().max().item() <= F64_GATE
    s = m.ssd_forward(si, 16, mask_strategy="static")
    r = m.ssd_forward(si, 16, mask_strategy="rowwise")
    assert torch.equal(s.Y, r.Y) and torch.equal(s.final_state, r.final_state)


def test_chunk_scan_validation():
    import paper_2603_09555_b200 as m

    rng = np.random.default_rng(3)
    inst = make_instance(rng)
    with pytest.raises(ValueError):
        m.ssd_forward(m.SsdInputs(inst["X"], -inst["dt"], inst["a"], inst["B"], inst["C"]), 4)
    with pytest.raises(ValueError):
        m.ssd_forward(m.SsdInputs(inst["X"], inst["dt"], -inst["a"], inst["B"], inst["C"]), 4)
    with pytest.raises(ValueError):
        m.ssd_forward(m.SsdInputs(inst["X"], inst["dt"], inst["a"], inst["B"], inst["C"]), 0)


# ----------------------------------------------------------- small models


@pytest.mark.parametrize("name,ov,seed", SMALL_MODELS)
@pytest.mark.parametrize("comp", ["f32", "f64"])
def test_small_model_vs_golden(name, ov, seed, comp):
    import paper_2603_09555_b200 as m

    z = golden("small_model.npz")
    cfg = small_config(**ov).with_policy(compute=comp)
    params = m.random_init(cfg, seed)
    key = f"{name}.{comp}"
    tol = 1e-10 if comp == "f64" else 2e-5
    logits, cache = m.prefill(params, z[f"{key}.tokens"], cfg)
    ref = z[f"{key}.logits"]
    assert np.abs(_np(logits) - ref).max() <= tol * max(1.0, np.abs(ref).max())
    assert np.abs(_np(cache.ssm_all) - z[f"{key}.ssm"]).max() <= tol * max(1.0, np.abs(z[f"{key}.ssm"]).max())
    assert np.abs(_np(cache.conv_all) - z[f"{key}.conv"]).max() <= tol
    before = cache.to_bytes()
    sl, c2 = m.decode_step(params, cache, z[f"{key}.next"], cfg)
    assert cache.to_bytes() == before  # input cache not mutated (test_decode.py:107-113)
    ref = z[f"{key}.step_logits"]
    assert np.abs(_np(sl) - ref).max() <= tol * max(1.0, np.abs(ref).max())
    assert np.abs(_np(c2.ssm_all) - z[f"{key}.step_ssm"]).max() <= tol * max(1.0, np.abs(z[f"{key}.step_ssm"]).max())
    assert np.abs(_np(c2.conv_all) - z[f"{key}.step_conv"]).max() <= tol
    for use_graph in (True, False):
        res = m.generate(params, z[f"{key}.prompt"], 64, cfg=cfg, use_graph=use_graph)
        assert np.array_equal(_np(res.tokens), z[f"{key}.gen"])


@pytest.mark.parametrize("comp", ["f32", "f64"])
def test_cached_vs_full(comp):
    """Criterion 3 (test_acceptance.py:117-140) on the device."""
    import paper_2603_09555_b200 as m

    gate = CACHED_FULL_F32 if comp == "f32" else 1e-9
    cfg = small_config(d_model=64, n_layers=4, chunk_size=16).with_policy(compute=comp)
    params = m.random_init(cfg, 1)
    rng = np.random.default_rng(101)
    for prompt_len in (1, 16, 33):
        for gen in (1, 8, 64):
            toks = rng.integers(0, cfg.vocab_size, size=(1, prompt_len + gen))
            full, _ = m.prefill(params, toks, cfg)
            logits, cache = m.prefill(params, toks[:, :prompt_len], cfg)
            for g in range(gen):
                logits, cache = m.decode_step(params, cache, toks[:, prompt_len + g], cfg)
            assert (logits - full[:, -1]).abs().max().item() <= gate


def test_non_cached_matches_cached():
    import paper_2603_09555_b200 as m

    cfg = small_config(d_model=16, head_dim=4, d_state=4, chunk_size=8)
    params = m.random_init(cfg, 300)
    prompt = np.random.default_rng(400).integers(0, cfg.vocab_size, size=(1, 16))
    a = m.generate(params, prompt, 32, mode="cached", cfg=cfg)
    b = m.generate(params, prompt, 32, mode="non_cached", cfg=cfg)
    assert torch.equal(a.tokens, b.tokens)


def test_batch_invariance_bitwise():
    """Rows are independent: a batch-sharded run equals the full run bitwise
    (analogue of test_model.py:131-140; the basis of the batch sharding)."""
    import paper_2603_09555_b200 as m

    cfg = small_config(d_model=64, n_layers=2)
    params = m.random_init(cfg, 9)
    toks = np.random.default_rng(8).integers(0, cfg.vocab_size, size=(4, 37))
    full, cache = m.prefill(params, toks, cfg)
    for lo, hi in ((0, 2), (2, 4), (1, 3)):
        part, pc = m.prefill(params, toks[lo:hi], cfg)
        assert torch.equal(part, full[lo:hi])
        assert torch.equal(pc.ssm_all, cache.ssm_all[:, lo:hi])


# ----------------------------------------------------------- config 1 (130M f32)


def test_c1_130m_tokens_identical():
    """Config 1: 130M random_init(0) f32, prompt 512, generate(65): greedy
    tokens identical to the reference over all 64 decode steps; logits within
    the Table-5 gates (oracle.py:118)."""
    import paper_2603_09555_b200 as m

    z = golden("c1_130m.npz")
    cfg = m.ModelConfig(vocab_size=50288, d_model=768, n_layers=24)
    params = m.random_init(cfg, 0)
    res = m.generate(params, z["prompt"], 65, cfg=cfg, keep_logits=True)
    assert np.array_equal(_np(res.tokens), z["tokens"])
    lg = _np(res.per_step_logits[0])
    for got, ref in ((lg[0], z["logits_first"]), (lg[-1], z["logits_last"])):
        assert np.all(np.abs(got - ref) <= F32_ATOL + F32_RTOL * np.abs(ref))
    # hidden states after layer 0 within fp32 rounding (rel 1e-4, north_star)
    hidden0 = params.embedding[torch.as_tensor(z["prompt"]).cuda()]
    h1, s1, c1 = m.block_forward(params.layers[0], hidden0, cfg)
    rows = _np(h1[0, [0, 1, 255, 256, 510, 511]])
    ref = z["layer0_hidden_rows"]
    assert np.linalg.norm(rows - ref) / np.linalg.norm(ref) <= 1e-4
    assert np.all(np.abs(rows - ref) <= 1e-4 * np.abs(ref) + 1e-4 * np.abs(ref).max())
    st = _np(s1[0, 0])
    assert np.linalg.norm(st - z["layer0_state_head0"]) / np.linalg.norm(z["layer0_state_head0"]) <= 1e-4
    # the tail holds pre-activation in_proj outputs: fp32 GEMM rounding only
    ct, rt = _np(c1[0]), z["layer0_conv_tail"]
    assert np.linalg.norm(ct - rt) / np.linalg.norm(rt) <= 1e-5


# ----------------------------------------------------------- bf16 tensor-core mode


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (300, 500, 1024), (7, 3352, 768), (1000, 1024, 2048), (256, 50288, 256)])
def test_tc_gemm_matches_torch(M, N, K):
    from paper_2603_09555_b200 import _abi

    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda", generator=g).to(torch.bfloat16)
    C = torch.empty(M, N, device="cuda", dtype=torch.float32)
    _abi.check(_abi.lib().ssd200_gemm_bf16(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K,
                                           _abi.stream_handle()), "gemm")
    ref = A.float() @ B.float().t()
    err = (C - ref).abs().max().item()
    assert err <= 1e-3 * max(1.0, ref.abs().max().item()), err




def _bf16_cfg(**kw):
    from paper_2603_09555_b200 import ElemPolicy, ModelConfig

    base = dict(vocab_size=1000, d_model=256, n_layers=2, norm_eps=1e-5)
    base.update(kw)
    return ModelConfig(policy=ElemPolicy(compute="bf16"), **base)


@pytest.mark.parametrize("variant", [2, 1])
def test_bf16_prefill_vs_oracle(variant):
    """bf16 prefill (tensor-core GEMMs + SSD) vs the f32 oracle on the same
    bf16-rounded weights; both scan variants (2: parallel states + pass,
    1: the fused per-(b, h) chunk walk), which must also agree bitwise."""
    import paper_2603_09555_b200 as m
    from paper_2603_09555_b200 import _abi

    cfg = _bf16_cfg()
    host = m.random_init_host(cfg, 4)
    params = m.from_reference(host, cfg)
    toks = np.random.default_rng(5).integers(0, cfg.vocab_size, size=(2, 300))
    with _abi.tuning(scan_variant=variant):
        logits, cache = m.prefill(params, toks, cfg)
    with _abi.tuning(scan_variant=3 - variant):
        other, _ = m.prefill(params, toks, cfg)
    assert torch.equal(logits, other)  # same chunk-state arithmetic in both variants
    ref_logits, ref_ssm, _ = orc.prefill(orc.round_weights_bf16(host), toks, cfg.with_policy(compute="f32"))
    got = _np(logits)
    rel = np.linalg.norm(got - ref_logits) / np.linalg.norm(ref_logits)
    report(f"bf16_prefill[variant={variant}]", logits=float(rel))
    assert rel <= BF16_BOUND, rel
    rs = np.stack(ref_ssm)
    rel_s = np.linalg.norm(_np(cache.ssm_all) - rs) / np.linalg.norm(rs)
    assert rel_s <= BF16_STATE_BOUND, rel_s


def test_bf16_generate_graph_is_deterministic():
    """The CUDA-graph generate loop (PDL launches, in-place cache) gives the
    same tokens as the eager step loop, and decode logits stay within the
    bf16 bound of the f32 oracle on bf16-rounded weights."""
    import paper_2603_09555_b200 as m

    cfg = _bf16_cfg()
    host = m.random_init_host(cfg, 11)
    params = m.from_reference(host, cfg)
    prompt = np.random.default_rng(12).integers(0, cfg.vocab_size, size=(2, 40))
    a = m.generate(params, prompt, 24, cfg=cfg, use_graph=True, keep_logits=True)
    b = m.generate(params, prompt, 24, cfg=cfg, use_graph=False, keep_logits=True)
    assert torch.equal(a.tokens, b.tokens)
    assert torch.equal(a.per_step_logits, b.per_step_logits)
    toks = _np(a.tokens)
    seq = np.concatenate([prompt, toks[:, :-1]], axis=1)
    ref = orc.prefill(orc.round_weights_bf16(host), seq, cfg.with_policy(compute="f32"))[0]
    got = _np(a.per_step_logits)
    for g in (1, 10, 23):
        r = ref[:, prompt.shape[1] + g - 1]
        rel = np.linalg.norm(got[:, g] - r) / np.linalg.norm(r)
        report(f"bf16_generate_graph[g={g}]", logits=float(rel))
        assert rel <= BF16_BOUND, (g, rel)


@pytest.mark.parametrize("B,T", [(1, 1), (2, 2), (3, 5), (2, 63), (2, 125), (1, 253), (2, 600)])
def test_bf16_conv_edges(B, T):
    """The TMA-tiled conv1d + SiLU (64-row tiles with a 3-row halo): sequence
    starts inside tiles, T < k-1 zero-padded tails, ragged tiles — checked
    against the oracle on bf16-rounded weights."""
    import paper_2603_09555_b200 as m

    cfg = _bf16_cfg(n_layers=1)
    host = m.random_init_host(cfg, 31)
    params = m.from_reference(host, cfg)
    toks = np.random.default_rng(32 + T).integers(0, cfg.vocab_size, size=(B, T))
    logits, cache = m.prefill(params, toks, cfg)
    ref_logits, ref_ssm, ref_conv = orc.prefill(orc.round_weights_bf16(host), toks,
                                                cfg.with_policy(compute="f32"))
    got = _np(logits)
    rel = np.linalg.norm(got - ref_logits) / np.linalg.norm(ref_logits)
    report(f"bf16_conv_edges[B={B},T={T}]", logits=float(rel))
    assert rel <= BF16_BOUND, rel
    rc = np.stack(ref_conv)
    gc = _np(cache.conv_all)
    assert np.linalg.norm(gc - rc) / max(np.linalg.norm(rc), 1e-30) <= BF16_BOUND
    if T < 3:
        assert np.all(gc[..., : 3 - T] == 0)


def test_bf16_decode_vs_oracle():
    import paper_2603_09555_b200 as m

    cfg = _bf16_cfg()
    host = m.random_init_host(cfg, 6)
    params = m.from_reference(host, cfg)
    rng = np.random.default_rng(7)
    for B in (1, 3, 20):
        toks = rng.integers(0, cfg.vocab_size, size=(B, 40))
        _, cache = m.prefill(params, toks[:, :39], cfg, logits=None)
        sl, _ = m.decode_step(params, cache, toks[:, 39], cfg)
        ref_full = orc.prefill(orc.round_weights_bf16(host), toks, cfg.with_policy(compute="f32"))[0][:, -1]
        rel = np.linalg.norm(_np(sl) - ref_full) / np.linalg.norm(ref_full)
        report(f"bf16_decode[B={B}]", logits=float(rel))
        assert rel <= BF16_BOUND, (B, rel)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_bf16_head_sharded_prefill_matches_unsharded(world):
    """Head-group sharding: each simulated rank computes its
    heads and a partial out_proj; the partials + sums of u^2 are summed (the
    all-reduce) and finished.  Equals the unsharded bf16 prefill up to the
    summation order, and each rank's final states are its heads' slice."""
    import paper_2603_09555_b200 as m
    from paper_2603_09555_b200 import shard

    d_model = 256 * world  # 8 heads of 64 per rank
    cfg = m.ModelConfig(vocab_size=1024, d_model=d_model, n_layers=2, norm_eps=1e-5).with_policy(
        compute="bf16")
    host = m.random_init_host(cfg, 21)
    rng = np.random.default_rng(4)
    for lp in host.layers:  # non-unit norm weights exercise the norm_w folding
        lp.norm_w = (1.0 + 0.2 * rng.standard_normal(cfg.d_inner)).astype(np.float32)
    tok = rng.integers(0, cfg.vocab_size, size=(2, 300))
    full = m.from_reference(host, cfg)
    ref, cache = m.prefill(full, tok, cfg, logits="last")
    runs = [shard.HeadShardedPrefill(shard.upload_shard(host, cfg, r, world), tok, cfg)
            for r in range(world)]
    for i in range(cfg.n_layers):
        total = sum(run.partial(i).clone() for run in runs)  # the all-reduce
        for run in runs:
            run.buf.copy_(total)
            run.finish()
    got = runs[0].logits()
    for run in runs[1:]:
        assert torch.equal(run.logits(), got)  # replicated after the reduce
    rel = (torch.linalg.norm(got - ref) / torch.linalg.norm(ref)).item()
    assert rel <= BF16_BOUND, rel
    for r, run in enumerate(runs):
        hs = shard.head_slice(cfg.n_heads, r, world)
        for i in range(cfg.n_layers):
            a, b = run.ssm[i], cache.ssm_all[i][:, hs].float()
            assert (torch.linalg.norm(a - b) / torch.linalg.norm(b)).item() <= BF16_STATE_BOUND


@pytest.mark.parametrize("world", [2, 4])
def test_bf16_head_sharded_decode_matches_unsharded(world):
    """Head-group-sharded decode: simulated ranks run their heads
    of every layer (ssd200_decode_layer_partial), the [partial | sum u^2]
    buffers are summed (the all-reduce) and finished on every rank.  Fed the
    unsharded run's tokens, each step's logits match the unsharded bf16
    decode within the bf16 bound, and the greedy picks agree."""
    import paper_2603_09555_b200 as m
    from paper_2603_09555_b200 import shard

    d_model = 256 * world  # 8 heads of 64 per rank (the sharded prefill needs multiples of 8)
    cfg = m.ModelConfig(vocab_size=1024, d_model=d_model, n_layers=2, norm_eps=1e-5).with_policy(
        compute="bf16")
    host = m.random_init_host(cfg, 23)
    rng = np.random.default_rng(5)
    for lp in host.layers:
        lp.norm_w = (1.0 + 0.2 * rng.standard_normal(cfg.d_inner)).astype(np.float32)
    prompt = rng.integers(0, cfg.vocab_size, size=(3, 40))
    G = 6
    ref = m.generate(m.from_reference(host, cfg), prompt, G, cfg=cfg, keep_logits=True)
    runs = [shard.HeadShardedPrefill(shard.upload_shard(host, cfg, r, world), prompt, cfg)
            for r in range(world)]
    for i in range(cfg.n_layers):
        total = sum(run.partial(i).clone() for run in runs)
        for run in runs:
            run.buf.copy_(total)
            run.finish()
    decs = [shard.HeadShardedDecoder.from_prefill(run) for run in runs]
    for g in range(1, G):
        tok = ref.tokens[:, g - 1]
        for dec in decs:
            dec.begin(tok)
        for i in range(cfg.n_layers):
            total = sum(dec.partial(i).clone() for dec in decs)  # the all-reduce
            for dec in decs:
                dec.buf.copy_(total)
                dec.finish()
        outs = [dec.logits_and_pick() for dec in decs]
        for lg, pk in outs[1:]:
            assert torch.equal(lg, outs[0][0]) and torch.equal(pk, outs[0][1])  # replicated
        got, pick = outs[0]
        want = ref.per_step_logits[:, g]
        rel = (torch.linalg.norm(got - want) / torch.linalg.norm(want)).item()
        assert rel <= BF16_BOUND, (g, rel)
        assert torch.equal(pick, ref.tokens[:, g]), g


@pytest.mark.parametrize("B", [9, 16])
def test_bf16_wide_batch_decode_state_vs_oracle(B):
    """Wide-batch decode (B > 8: tensor-core in_proj, fused SSM update + gate +
    sum u^2, out_proj with the norm in its epilogue): one step's logits and the
    updated SSM / conv cache against the oracle on bf16-rounded weights, and
    the in-place graph loop against the functional step."""
    import paper_2603_09555_b200 as m

    cfg = _bf16_cfg()
    host = m.random_init_host(cfg, 41)
    params = m.from_reference(host, cfg)
    toks = np.random.default_rng(42).integers(0, cfg.vocab_size, size=(B, 30))
    _, cache = m.prefill(params, toks[:, :29], cfg, logits=None)
    before = cache.ssm_all.clone()
    sl, new = m.decode_step(params, cache, toks[:, 29], cfg)
    assert torch.equal(cache.ssm_all, before)  # the input cache is not mutated
    rl, rs, rc = orc.prefill(orc.round_weights_bf16(host), toks, cfg.with_policy(compute="f32"))
    rel = np.linalg.norm(_np(sl) - rl[:, -1]) / np.linalg.norm(rl[:, -1])
    assert rel <= BF16_BOUND, rel
    rs = np.stack(rs)
    assert np.linalg.norm(_np(new.ssm_all) - rs) / np.linalg.norm(rs) <= BF16_STATE_BOUND
    rc = np.stack(rc)
    assert np.linalg.norm(_np(new.conv_all) - rc) / np.linalg.norm(rc) <= BF16_BOUND
    a = m.generate(params, toks[:, :29], 6, cfg=cfg, use_graph=True, keep_logits=True)
    b = m.generate(params, toks[:, :29], 6, cfg=cfg, use_graph=False, keep_logits=True)
    assert torch.equal(a.tokens, b.tokens)
    assert torch.equal(a.per_step_logits, b.per_step_logits)


def test_bf16_decode_batch_invariance_bitwise():
    """bf16 decode rows do not depend on the batch they run in, within one decode
    GEMM class (here both batches are on the ~96 KB ring; at these widths the
    split-K factors coincide for every B): the basis of batch sharding for
    decode."""
    import paper_2603_09555_b200 as m

    cfg = _bf16_cfg()
    params = m.from_reference(m.random_init_host(cfg, 51), cfg)
    toks = np.random.default_rng(52).integers(0, cfg.vocab_size, size=(6, 24))
    full = m.generate(params, toks, 5, cfg=cfg, keep_logits=True)
    part = m.generate(params, toks[2:4], 5, cfg=cfg, keep_logits=True)
    assert torch.equal(full.tokens[2:4], part.tokens)
    assert torch.equal(full.per_step_logits[2:4, 1:], part.per_step_logits[:, 1:])


@pytest.mark.parametrize("B,T", [(1, 2048), (2, 1024)])
def test_bf16_prefill_production_width_vs_oracle(B, T):
    """One production-width layer (d_model 1024, the 370M block) at sizes where
    the GEMMs run 256-wide tiles over many waves and the scan walks 4-8
    chunks; the tied head on the last position.  Against the f32 oracle on the
    same bf16-rounded weights, within the stated bf16 bound."""
    import paper_2603_09555_b200 as m

    cfg = _bf16_cfg(vocab_size=2048, d_model=1024, n_layers=1)
    host = m.random_init_host(cfg, 61)
    params = m.from_reference(host, cfg)
    toks = np.random.default_rng(62).integers(0, cfg.vocab_size, size=(B, T))
    logits, cache = m.prefill(params, toks, cfg, logits="last")
    ref_logits, ref_ssm, _ = orc.prefill(orc.round_weights_bf16(host), toks,
                                         cfg.with_policy(compute="f32"))
    ref = ref_logits[:, -1]
    rel = np.linalg.norm(_np(logits) - ref) / np.linalg.norm(ref)
    assert rel <= BF16_BOUND, rel
    rs = np.stack(ref_ssm)
    rel_s = np.linalg.norm(_np(cache.ssm_all) - rs) / np.linalg.norm(rs)
    assert rel_s <= BF16_STATE_BOUND, rel_s


def test_verify_suites_pass():
    """The reference's verify suites (verify.py:22) ported to the GPU path."""
    from paper_2603_09555_b200 import verify

    results = verify.run_verify()
    assert [r.suite for r in results] == list(verify.SUITES)
    bad = [r.to_dict() for r in results if not r.passed]
    assert not bad, bad


@pytest.mark.parametrize("B,T", [(4, 4096)])
def test_bf16_prefill_cta_pair_gemms_match(B, T):
    """CTA-pair (cta_group::2) GEMMs for in_proj / out_proj (tuning gemm_pair) against
    the single-CTA GEMMs on a production-width layer at a size where both
    take 256 x 256 pair tiles; the single-CTA path is the one pinned to the
    oracle above."""
    import paper_2603_09555_b200 as m
    from paper_2603_09555_b200 import _abi

    cfg = _bf16_cfg(vocab_size=2048, d_model=1024, n_layers=2)
    params = m.from_reference(m.random_init_host(cfg, 71), cfg)
    toks = np.random.default_rng(72).integers(0, cfg.vocab_size, size=(B, T))
    outs = []
    for pair in (0, 1):
        with _abi.tuning(gemm_pair=pair):
            lg, cache = m.prefill(params, toks, cfg, logits="last")
        outs.append((lg, cache.ssm_all.clone()))
    (la, sa), (lb, sb) = outs
    assert ((la - lb).norm() / la.norm()).item() <= 1e-3
    assert ((sa - sb).norm() / sa.norm()).item() <= 1e-3


def test_bf16_prefill_gemm_cache_hints_are_bitwise_neutral():
    """The GEMM epilogues' evict-first accesses (tuning gemm_stream: 0 off, 2
    always) change only where lines live in L2, never the arithmetic: logits,
    states and the residual stream bitwise equal."""
    import paper_2603_09555_b200 as m
    from paper_2603_09555_b200 import _abi

    cfg = _bf16_cfg(vocab_size=2048, d_model=1024, n_layers=2)
    params = m.from_reference(m.random_init_host(cfg, 75), cfg)
    toks = np.random.default_rng(76).integers(0, cfg.vocab_size, size=(2, 1024))
    outs = []
    for hint in (0, 2):
        with _abi.tuning(gemm_stream=hint):
            lg, cache, hid = m.prefill(params, toks, cfg, logits="last", return_hidden=True)
        outs.append((lg, cache.ssm_all.clone(), hid.clone()))
    (la, sa, ha), (lb, sb, hb) = outs
    assert torch.equal(la, lb) and torch.equal(sa, sb) and torch.equal(ha, hb)


def test_generate_graph_cache_reuse_is_exact():
    """generate() keeps captured decode graphs across calls (decode._GRAPH_CACHE):
    a second call with another prompt through the cached graph must equal an
    uncached (eager) run, and the first call's results must not be overwritten."""
    import paper_2603_09555_b200 as m

    cfg = _bf16_cfg()
    params = m.from_reference(m.random_init_host(cfg, 81), cfg)
    rng = np.random.default_rng(82)
    p1 = rng.integers(0, cfg.vocab_size, size=(2, 20))
    p2 = rng.integers(0, cfg.vocab_size, size=(2, 20))
    a = m.generate(params, p1, 9, cfg=cfg, keep_logits=True)
    b = m.generate(params, p2, 9, cfg=cfg, keep_logits=True)  # cache hit
    ea = m.generate(params, p1, 9, cfg=cfg, keep_logits=True, use_graph=False)
    eb = m.generate(params, p2, 9, cfg=cfg, keep_logits=True, use_graph=False)
    assert torch.equal(a.tokens, ea.tokens) and torch.equal(a.per_step_logits, ea.per_step_logits)
    assert torch.equal(b.tokens, eb.tokens) and torch.equal(b.per_step_logits, eb.per_step_logits)


def test_bf16_decode_batch_invariance_across_gemm_classes():
    """At production widths (1.3B: d_model 2048) the in_proj split-K differs
    between the ~100 KB-ring class (B <= 32: split 4) and the 192 KB-ring class
    (split 2), so the f32 partial sums are added in a different order.  Forcing
    one ring (tuning dec_small_ring) makes the split a function of the widths only: rows are
    then bitwise batch-invariant across B = 2 and B = 64.  Without forcing, rows
    agree to f32 rounding of the partial sums."""
    import paper_2603_09555_b200 as m
    from paper_2603_09555_b200 import _abi

    cfg = m.named_config("1.3b", compute="bf16", vocab_size=512, n_layers=1)
    params = m.from_reference(m.random_init_host(cfg, 61), cfg)
    toks = np.random.default_rng(62).integers(0, cfg.vocab_size, size=(64, 12))
    with _abi.tuning(dec_small_ring=1):
        full = m.generate(params, toks, 4, cfg=cfg, keep_logits=True, use_graph=False)
        part = m.generate(params, toks[5:7], 4, cfg=cfg, keep_logits=True, use_graph=False)
    assert torch.equal(full.tokens[5:7], part.tokens)
    assert torch.equal(full.per_step_logits[5:7, 1:], part.per_step_logits[:, 1:])
    auto = m.generate(params, toks, 4, cfg=cfg, keep_logits=True, use_graph=False)
    a, b = auto.per_step_logits[5:7, 1:], part.per_step_logits[:, 1:]
    rel = float((a - b).norm() / b.norm())
    assert rel < 1e-2, rel


@pytest.mark.parametrize("B", [64, 200, 264])
def test_bf16_decode_production_width_wide_batches_vs_oracle(B):
    """One decode step at 370M widths (d_model 1024, 32 heads of 64 x 128) on the
    192 KB-ring swapped GEMMs (B = 64: 64-row tiles; B = 200: 256-row tiles) and
    on the tc_gemm path past 256 rows (B = 264): logits and the updated SSM /
    conv cache against the oracle on bf16-rounded weights."""
    import paper_2603_09555_b200 as m

    cfg = m.named_config("370m", compute="bf16", vocab_size=512, n_layers=1)
    host = m.random_init_host(cfg, 71)
    params = m.from_reference(host, cfg)
    toks = np.random.default_rng(72).integers(0, cfg.vocab_size, size=(B, 10))
    _, cache = m.prefill(params, toks[:, :9], cfg, logits=None)
    sl, new = m.decode_step(params, cache, toks[:, 9], cfg)
    rl, rs, rc = orc.prefill(orc.round_weights_bf16(host), toks, cfg.with_policy(compute="f32"))
    rel = np.linalg.norm(_np(sl) - rl[:, -1]) / np.linalg.norm(rl[:, -1])
    assert rel <= BF16_BOUND, rel
    rs = np.stack(rs)
    assert np.linalg.norm(_np(new.ssm_all) - rs) / np.linalg.norm(rs) <= BF16_STATE_BOUND
    rc = np.stack(rc)
    assert np.linalg.norm(_np(new.conv_all) - rc) / np.linalg.norm(rc) <= BF16_BOUND


def _sharded_setup(world, seed=33, B=3, P=40):
    import paper_2603_09555_b200 as m
    from paper_2603_09555_b200 import shard

    d_model = 256 * world  # 8 heads of 64 per rank
    cfg = m.ModelConfig(vocab_size=1024, d_model=d_model, n_layers=2, norm_eps=1e-5).with_policy(
        compute="bf16")
    host = m.random_init_host(cfg, seed)
    rng = np.random.default_rng(seed + 1)
    for lp in host.layers:  # non-unit norm weights exercise the norm_w folding
        lp.norm_w = (1.0 + 0.2 * rng.standard_normal(cfg.d_inner)).astype(np.float32)
    prompt = rng.integers(0, cfg.vocab_size, size=(B, P))
    shards = [shard.upload_shard(host, cfg, r, world) for r in range(world)]
    return m, shard, cfg, host, prompt, shards


def _sharded_decoders(shard, cfg, prompt, shards):
    runs = [shard.HeadShardedPrefill(p, prompt, cfg) for p in shards]
    for i in range(cfg.n_layers):
        shard.sum_reduce([run.partial(i) for run in runs])
        for run in runs:
            run.finish()
    tok = torch.empty((runs[0].B,), dtype=torch.int64, device="cuda")
    runs[0].logits(argmax=tok)
    return [shard.HeadShardedDecoder.from_prefill(run) for run in runs], tok


def test_bf16_head_sharded_decode_graph_matches_eager():
    """The head-sharded token step captured as ONE CUDA graph — two simulated
    ranks' layers, the per-layer reduce of [partial | sum u^2] (a fixed-order
    sum kernel standing in for the all-reduce), finish, head and argmax — gives
    the same tokens and logits, bitwise, as the same step run eagerly; and the
    tokens match the unsharded bf16 generate."""
    m, shard, cfg, host, prompt, shards = _sharded_setup(2)
    G = 8
    outs = []
    for use_graph in (True, False):
        decs, tok = _sharded_decoders(shard, cfg, prompt, shards)
        gd = shard.HeadShardedGraphDecoder(decs, G, reduce=shard.sum_reduce, use_graph=use_graph)
        gd.set_token(tok)
        gd.tokens[:, 0] = tok
        gd.step_idx.fill_(1)
        logits = []
        for _ in range(G - 1):
            gd.step()
            logits.append(gd.ranks[0].logits.clone())
        outs.append((gd.tokens.clone(), torch.stack(logits), [d.ssm.clone() for d in gd.ranks]))
    (ta, la, sa), (tb, lb, sb) = outs
    assert torch.equal(ta, tb)
    assert torch.equal(la, lb)
    for a, b in zip(sa, sb):
        assert torch.equal(a, b)
    ref = m.generate(m.from_reference(host, cfg), prompt, G, cfg=cfg, keep_logits=True)
    assert torch.equal(ta, ref.tokens)
    rel = ((la[-1] - ref.per_step_logits[:, -1]).norm() / ref.per_step_logits[:, -1].norm()).item()
    report("head_sharded_graph[world=2]", logits=rel)
    assert rel <= BF16_BOUND, rel


def test_bf16_head_sharded_generate_over_nccl_world1():
    """The product's generate_head_sharded with a real NCCL process group (one
    rank on this GPU): the prefill all-reduces and the NCCL all-reduce captured
    inside the decode graph run, and the greedy tokens equal the unsharded
    bf16 generate."""
    import socket

    import torch.distributed as dist

    m, shard, cfg, host, prompt, shards = _sharded_setup(1, seed=35)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        group = dist.new_group([0])
        run = shard.HeadShardedPrefill(shards[0], prompt, cfg)
        for i in range(cfg.n_layers):
            buf = run.partial(i)
            dist.all_reduce(buf, group=group)
            run.finish()
        tok = torch.empty((run.B,), dtype=torch.int64, device="cuda")
        run.logits(argmax=tok)
        gd = shard.HeadShardedGraphDecoder([shard.HeadShardedDecoder.from_prefill(run)], 6,
                                           reduce=shard.nccl_reduce(group))
        gd.set_token(tok)
        gd.tokens[:, 0] = tok
        gd.step_idx.fill_(1)
        for _ in range(5):
            gd.step()
        got = gd.tokens.clone()
        via_api = shard.generate_head_sharded(shards[0], prompt, 6, cfg, group=group)
        lg, ssm = shard.prefill_head_sharded(shards[0], prompt, cfg, group=group)
        # restart(): the same object re-run on new tokens equals a fresh one
        run2 = shard.HeadShardedPrefill(shards[0], prompt, cfg)
        run2.restart(prompt[::-1].copy())
        fresh = shard.HeadShardedPrefill(shards[0], prompt[::-1].copy(), cfg)
        assert torch.equal(run2.hidden, fresh.hidden) and torch.equal(run2.lp, fresh.lp)
    finally:
        dist.destroy_process_group()
    full = m.from_reference(host, cfg)
    ref = m.generate(full, prompt, 6, cfg=cfg)
    assert torch.equal(got, ref.tokens)
    assert torch.equal(via_api, ref.tokens)
    want, cache = m.prefill(full, prompt, cfg, logits="last")
    assert ((lg - want).norm() / want.norm()).item() <= BF16_BOUND
    assert ((ssm - cache.ssm_all).norm() / cache.ssm_all.norm()).item() <= BF16_STATE_BOUND


@pytest.mark.parametrize("B", [1, 9, 64])
def test_bf16_chained_decode_layers_bitwise(B):
    """ssd200_decode_layers (every layer of a token step in one ABI call, the
    (n_layers, ...) caches addressed by the library) against one
    ssd200_decode_layer call per layer: logits, greedy tokens and both caches
    agree bitwise over 4 steps."""
    import paper_2603_09555_b200 as m
    from paper_2603_09555_b200.decode import _step_into
    from paper_2603_09555_b200.model import _Runner

    cfg = m.named_config("1.3b", compute="bf16", vocab_size=512, n_layers=3)
    params = m.from_reference(m.random_init_host(cfg, 71), cfg)
    prompt = np.random.default_rng(72 + B).integers(0, cfg.vocab_size, size=(B, 12))
    _, c0 = m.prefill(params, prompt, cfg, logits=None)
    runs = []
    for chained in (True, False):
        c = c0.copy()
        r = _Runner(params, cfg)
        tok = torch.as_tensor(prompt[:, -1], device="cuda")
        lgs = []
        for _ in range(4):
            lg = torch.empty((B, cfg.vocab_size), dtype=torch.float32, device="cuda")
            _step_into(r, cfg, tok, c, c, logits=lg, argmax=tok, chained=chained)
            lgs.append(lg)
        runs.append((torch.stack(lgs), tok.clone(), c))
    (la, ta, ca), (lb, tb, cb) = runs
    assert torch.equal(la, lb)
    assert torch.equal(ta, tb)
    assert torch.equal(ca.ssm_all, cb.ssm_all)
    assert torch.equal(ca.conv_all, cb.conv_all)


@pytest.mark.parametrize("comp", ["f32", "bf16"])
def test_pre_norm_block_vs_oracle(comp):
    """The optional residual pre-norm (ssd200_layer_t.pre_norm_w; real
    state-spaces/mamba2 checkpoints' backbone.layers.N.norm, which the reference
    block drops): prefill, a cached decode step and greedy tokens against the
    oracle with the same pre-norm — f32 at the reference gates, bf16 on
    bf16-rounded weights within the stated bound."""
    import paper_2603_09555_b200 as m

    if comp == "f32":
        cfg = small_config(d_model=64, n_layers=2)
    else:
        cfg = _bf16_cfg(d_model=512)
    host = m.random_init_host(cfg, 51)
    rng = np.random.default_rng(52)
    for lp in host.layers:
        lp.pre_norm_w = (1.0 + 0.3 * rng.standard_normal(cfg.d_model)).astype(np.float32)
    params = m.from_reference(host, cfg)
    assert params.layers[0].pre_norm_w is not None
    toks = rng.integers(0, cfg.vocab_size, size=(2, 300))
    ref_host = orc.round_weights_bf16(host) if comp == "bf16" else host
    rcfg = cfg.with_policy(compute="f32")
    rl, rs, rc = orc.prefill(ref_host, toks, rcfg)
    logits, cache = m.prefill(params, toks[:, :299], cfg)
    sl, _ = m.decode_step(params, cache, toks[:, 299], cfg)
    got_p, got_d = _np(logits), _np(sl)
    if comp == "f32":
        for got, ref in ((got_p, rl[:, :299]), (got_d, rl[:, 299])):
            assert np.abs(got - ref).max() <= 2e-5 * max(1.0, np.abs(ref).max())
        gen = m.generate(params, toks[:1, :40], 12, cfg=cfg)
        assert np.array_equal(_np(gen.tokens), orc.generate(host, toks[:1, :40], 12, cfg))
    else:
        r1 = np.linalg.norm(got_p[:, -1] - rl[:, 298]) / np.linalg.norm(rl[:, 298])
        r2 = np.linalg.norm(got_d - rl[:, 299]) / np.linalg.norm(rl[:, 299])
        report("pre_norm_bf16", prefill=float(r1), decode=float(r2))
        assert r1 <= BF16_BOUND and r2 <= BF16_BOUND, (r1, r2)
    # and without the pre-norm the outputs differ (the weights are non-unit)
    for lp in params.layers:
        lp.pre_norm_w = None
    plain, _ = m.prefill(params, toks[:, :299], cfg)
    assert (plain - logits).abs().max().item() > 1e-3


@pytest.mark.parametrize("B", [3, 160])
def test_bf16_decode_groups_and_tile_handout(B):
    """The decode state stream with n_groups = 2 (B / C shared by 4 of the 8 heads,
    so a tile sequence crosses (row, group) boundaries inside a CTA) against the
    oracle, at a small batch (static tile ranges) and at B = 160 (1280 tiles:
    chunks handed out by the atomic counter).  Which CTA updates a tile must not
    change its arithmetic: the dynamic hand-out is bitwise equal to static ranges
    (tuning stream_chunk = -1) and to other chunk sizes."""
    import paper_2603_09555_b200 as m
    from paper_2603_09555_b200 import _abi

    cfg = _bf16_cfg(n_groups=2, n_layers=1, vocab_size=512)
    host = m.random_init_host(cfg, 81)
    params = m.from_reference(host, cfg)
    toks = np.random.default_rng(82).integers(0, cfg.vocab_size, size=(B, 12))
    _, cache = m.prefill(params, toks[:, :11], cfg, logits=None)
    sl, new = m.decode_step(params, cache, toks[:, 11], cfg)
    rl, rs, rc = orc.prefill(orc.round_weights_bf16(host), toks, cfg.with_policy(compute="f32"))
    rel = np.linalg.norm(_np(sl) - rl[:, -1]) / np.linalg.norm(rl[:, -1])
    report("bf16_decode_groups_logits", rel=float(rel), B=B)
    assert rel <= BF16_BOUND, rel
    rs = np.stack(rs)
    assert np.linalg.norm(_np(new.ssm_all) - rs) / np.linalg.norm(rs) <= BF16_STATE_BOUND
    rc = np.stack(rc)
    assert np.linalg.norm(_np(new.conv_all) - rc) / np.linalg.norm(rc) <= BF16_BOUND
    for chunk in (-1, 1, 3):
        with _abi.tuning(stream_chunk=chunk):
            sl2, new2 = m.decode_step(params, cache, toks[:, 11], cfg)
        assert torch.equal(sl2, sl), chunk
        assert torch.equal(new2.ssm_all, new.ssm_all), chunk
        assert torch.equal(new2.conv_all, new.conv_all), chunk


def test_bf16_decode_counter_handout_graph_replays():
    """The chunk counter of the state stream is zeroed by every layer's in_proj, so
    replaying the captured token step (the counter is reused by every layer and
    every step) gives the eager result bitwise, token for token."""
    import paper_2603_09555_b200 as m

    cfg = _bf16_cfg(n_layers=2, vocab_size=512)
    params = m.from_reference(m.random_init_host(cfg, 91), cfg)
    toks = np.random.default_rng(92).integers(0, cfg.vocab_size, size=(160, 10))
    a = m.generate(params, toks, 6, cfg=cfg, use_graph=True, keep_logits=True)
    b = m.generate(params, toks, 6, cfg=cfg, use_graph=False, keep_logits=True)
    assert torch.equal(a.tokens, b.tokens)
    assert torch.equal(a.per_step_logits, b.per_step_logits)
