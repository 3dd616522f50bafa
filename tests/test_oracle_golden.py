"""Pin the CPU oracle to the real reference: every oracle function is checked
against golden vectors produced by ``tests/golden/make_golden.py`` (which
imports the reference engine itself).  CPU only."""

from __future__ import annotations

import os
import types

import numpy as np
import pytest

import oracle as orc
from conftest import GOLDEN, SMALL_MODELS, golden, small_config


def _ssd_case(z, i):
    g = lambda k: z[f"{i}.{k}"]  # noqa: E731
    init = g("init") if int(g("has_init")) else None
    return g("X"), g("dt"), g("a"), g("B"), g("C"), int(g("L")), init


@pytest.mark.parametrize("i", range(8))
def test_chunked_scan_matches_reference(i):
    z = golden("ssd_cases.npz")
    X, dt, a, B, C, L, init = _ssd_case(z, i)
    for tag, dtp, tol in (("f64", np.float64, 1e-12), ("f32", np.float32, 2e-5)):
        Y, fin = orc.chunked_scan(
            X.astype(dtp), dt.astype(dtp), a.astype(dtp), B.astype(dtp), C.astype(dtp), L,
            None if init is None else init.astype(dtp),
        )
        ref_Y, ref_f = z[f"{i}.Y_{tag}"], z[f"{i}.final_{tag}"]
        scale = max(1.0, float(np.abs(ref_Y).max()))
        assert np.abs(Y - ref_Y).max() <= tol * scale
        assert np.abs(fin - ref_f).max() <= tol * max(1.0, float(np.abs(ref_f).max()))


@pytest.mark.parametrize("i", range(8))
def test_sequential_scan_matches_reference(i):
    z = golden("ssd_cases.npz")
    X, dt, a, B, C, L, init = _ssd_case(z, i)
    Y, h = orc.sequential_scan(X, dt, a, B, C, init=init)
    assert np.abs(Y - z[f"{i}.Y_seq"]).max() <= 1e-12
    assert np.abs(h - z[f"{i}.final_seq"]).max() <= 1e-12
    # and the chunked f64 result agrees with the sequential one (criterion 1 gate)
    assert np.abs(z[f"{i}.Y_f64"] - Y).max() <= 1e-10


def test_dense_scan_identity():
    rng = np.random.default_rng(11)
    for seq in (1, 2, 7, 16, 33):
        X = rng.standard_normal((2, seq, 2, 4))
        dt = rng.uniform(0, 1.2, (2, seq, 2))
        a = -rng.uniform(0.3, 4.0, 2)
        B = rng.standard_normal((2, seq, 1, 5))
        C = rng.standard_normal((2, seq, 1, 5))
        D = rng.standard_normal(2)
        ys, _ = orc.sequential_scan(X, dt, a, B, C, D)
        yd = orc.dense_scan(X, dt, a, B, C, D)
        assert np.abs(ys - yd).max() <= 1e-12


@pytest.mark.parametrize("name,ov,seed", SMALL_MODELS)
@pytest.mark.parametrize("comp", ["f32", "f64"])
def test_model_matches_reference(name, ov, seed, comp):
    z = golden("small_model.npz")
    cfg = small_config(**ov).with_policy(compute=comp)
    params = orc.reference_weights(cfg, seed)
    key = f"{name}.{comp}"
    tol = 1e-12 if comp == "f64" else 2e-5
    logits, ssm, conv = orc.prefill(params, z[f"{key}.tokens"], cfg)
    assert np.abs(logits - z[f"{key}.logits"]).max() <= tol * max(1, np.abs(logits).max())
    assert np.abs(np.stack(ssm) - z[f"{key}.ssm"]).max() <= tol * max(1, np.abs(z[f"{key}.ssm"]).max())
    assert np.array_equal(np.stack(conv), z[f"{key}.conv"])
    sl, s2, c2 = orc.decode_step(params, ssm, conv, z[f"{key}.next"], cfg)
    assert np.abs(sl - z[f"{key}.step_logits"]).max() <= tol * max(1, np.abs(sl).max())
    assert np.abs(np.stack(s2) - z[f"{key}.step_ssm"]).max() <= tol * max(1, np.abs(z[f"{key}.step_ssm"]).max())
    toks = orc.generate(params, z[f"{key}.prompt"], 64, cfg)
    assert np.array_equal(toks, z[f"{key}.gen"])


@pytest.mark.parametrize("name,ov,seed", SMALL_MODELS)
def test_bf16e_ablation_matches_reference(name, ov, seed):
    z = golden("small_model.npz")
    cfg = small_config(**ov).with_policy(decay_exp="bf16e")
    params = orc.reference_weights(cfg, seed)
    logits = orc.prefill(params, z[f"{name}.bf16e.tokens"], cfg)[0]
    assert np.abs(logits - z[f"{name}.bf16e.logits"]).max() <= 2e-5 * max(1, np.abs(logits).max())


def test_weights_digest():
    z = golden("weights_digest.npz")
    from paper_2603_09555_b200 import ModelConfig

    for name, cfg, seed in (
        ("small", small_config(), 2),
        ("c1", ModelConfig(vocab_size=50288, d_model=768, n_layers=24), 0),
    ):
        p = orc.reference_weights(cfg, seed)
        assert np.array_equal(p.embedding[:2, :8], z[f"{name}.embedding_first"])
        assert float(p.embedding.astype(np.float64).sum()) == float(z[f"{name}.embedding"])
        for i in (0, cfg.n_layers - 1):
            for f in ("W_in", "conv_w", "dt_bias", "A_log", "D", "W_out"):
                got = float(getattr(p.layers[i], f).astype(np.float64).sum())
                assert got == float(z[f"{name}.{i}.{f}"]), (name, i, f)


def test_primitives_known_answers():
    """Known-answer values pinned by the reference tests (test_numerics.py)."""
    assert orc.softplus(np.array(0.0)) == pytest.approx(np.log(2.0), rel=0, abs=1e-15)
    assert orc.softplus(np.array(-1.5)) == pytest.approx(0.2014132779827524, abs=1e-15)
    assert orc.softplus(np.array(30.0)) == 30.0
    assert orc.silu(np.array(-1.0)) == pytest.approx(-0.2689414213699951, abs=1e-15)
    one = np.array([1.0 + 2.0**-8], dtype=np.float32)
    assert orc.bf16_round(one)[0] == 1.0
    above = np.array([1.0 + 2.0**-8 + 2.0**-20], dtype=np.float32)
    assert orc.bf16_round(above)[0] == np.float32(1.0078125)


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "c1_130m.npz")), reason="no c1 golden")
def test_c1_golden_fixture_sane():
    z = golden("c1_130m.npz")
    assert z["tokens"].shape == (1, 65)
    assert int(np.argmax(z["logits_first"])) == int(z["tokens"][0, 0])
    assert int(np.argmax(z["logits_last"])) == int(z["tokens"][0, -1])


def test_verify_sequential_recurrence_matches_reference_golden():
    """verify.py's oracle suite compares the device scan with a host f64 time
    loop; that loop reproduces the reference's own sequential_ssm outputs
    (ssd_cases.npz, written by the real reference) to f64 rounding."""
    from paper_2603_09555_b200.ssd import SsdInputs
    from paper_2603_09555_b200.verify import sequential_recurrence

    z = golden("ssd_cases.npz")
    n = sum(1 for k in z.files if k.endswith(".Y_seq"))
    for i in range(n):
        g = lambda k: z[f"{i}.{k}"]  # noqa: E731
        if int(g("has_init")):
            continue  # the verify suite runs from a zero state
        y = sequential_recurrence(SsdInputs(X=g("X"), dt=g("dt"), a=g("a"), Bmat=g("B"),
                                            Cmat=g("C")))
        assert np.abs(y - g("Y_seq")).max() <= 1e-12 * max(1.0, np.abs(g("Y_seq")).max())
