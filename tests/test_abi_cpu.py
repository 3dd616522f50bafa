"""CPU-side checks of the boundary: the C-ABI library loads without a GPU and
exports every symbol include/ssd200.h declares; host-side validation and the
config mirror behave like the reference.  No compute calls."""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, small_config


def _declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "ssd200.h")).read()
    return sorted(set(re.findall(r"\b(ssd200_[a-z0-9_]+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol():
    from paper_2603_09555_b200 import _abi

    lib = ctypes.CDLL(_abi.LIB_PATH)
    declared = _declared_symbols()
    assert len(declared) >= 10
    for name in declared:
        assert hasattr(lib, name), name
    bound = {n for n, _, _ in _abi.SIGNATURES}
    assert bound == set(declared)


def test_abi_version_and_error_path_without_gpu():
    from paper_2603_09555_b200 import _abi

    lib = _abi.lib()
    assert lib.ssd200_abi_version() == 4
    # argument validation happens before any CUDA call
    rc = lib.ssd200_chunk_scan(0, None, None, None, None, None, None, None, None, None,
                               1, 1, 1, 1, 1, 1, 1, None, 0, None)
    assert rc == _abi.EINVAL
    assert "null pointer" in _abi.last_error()
    with pytest.raises(ValueError):
        _abi.check(rc, "probe")


def test_tuning_is_per_call_not_global():
    """Implementation choices travel inside ssd200_dims_t (no library option
    state): a scoped override changes only the calls made with it."""
    from paper_2603_09555_b200 import _abi, named_config
    from paper_2603_09555_b200.model import dims_struct

    lib = _abi.lib()
    t = _abi.default_tuning()
    assert t.size == ctypes.sizeof(_abi.Tuning)
    assert (t.gemm_pair, t.prefill_pdl, t.dec_small_ring, t.stream_cw, t.gemm_stream) == \
        (1, 1, -1, 8, 1)
    cfg = named_config("1.3b")
    base = lib.ssd200_decode_layer_workspace(dims_struct(cfg), 8)
    with _abi.tuning(dec_split_in=1, dec_split_out=1):
        d1 = dims_struct(cfg)
        assert d1.tuning and d1.tuning.contents.dec_split_in == 1
        small = lib.ssd200_decode_layer_workspace(d1, 8)
        # the defaults are unchanged for a call made without the override
        assert lib.ssd200_decode_layer_workspace(dims_struct(cfg).__class__(
            **{f: getattr(d1, f) for f, _ in d1._fields_ if f != "tuning"}), 8) == base
    assert small < base  # split-K 1 needs fewer partial buffers
    assert not dims_struct(cfg).tuning  # scope ended: NULL = library defaults
    assert lib.ssd200_decode_layer_workspace(dims_struct(cfg), 8) == base
    with pytest.raises(ValueError):
        with _abi.tuning(no_such_field=1):
            pass
    # a tuning struct from another header version is refused, not silently ignored
    bad = _abi.default_tuning()
    bad.size = ctypes.sizeof(_abi.Tuning) - 4
    d2 = dims_struct(cfg)
    d2.tuning = ctypes.pointer(bad)
    assert lib.ssd200_decode_layer_workspace(d2, 8) == 0
    assert "tuning.size" in _abi.last_error()


def test_workspace_queries_are_pure_host():
    from paper_2603_09555_b200 import _abi, named_config
    from paper_2603_09555_b200.model import dims_struct

    lib = _abi.lib()
    cfg = named_config("370m")
    d = dims_struct(cfg)
    ws = lib.ssd200_prefill_layer_workspace(d, 2, 4096)
    rows = 2 * 4096
    assert ws >= rows * (cfg.d_inner + cfg.conv_dim) * 2
    assert lib.ssd200_decode_layer_workspace(d, 8) > 0
    assert lib.ssd200_head_workspace(d, cfg.vocab_size, 4) >= 4 * cfg.vocab_size * 4
    assert lib.ssd200_chunk_scan_workspace(0, 1, 512, 24, 64, 128, 256) == (
        2 * 24 * 64 * 128 * 4 + 256
    )


def test_config_mirror_matches_reference_dims():
    """test_model.py:160-172 known-answer widths for 130M."""
    from paper_2603_09555_b200 import ModelConfig, n_params

    cfg = ModelConfig(vocab_size=50288, d_model=768, n_layers=24)
    assert (cfg.d_inner, cfg.n_heads, cfg.conv_dim, cfg.d_in_proj) == (1536, 24, 1792, 3352)
    assert n_params(cfg) == 128_971_200
    with pytest.raises(ValueError):
        ModelConfig(vocab_size=10, d_model=30, n_layers=1)  # d_inner 60 % 64
    with pytest.raises(ValueError):
        small_config().with_policy(compute="f16")


def test_random_init_matches_reference_digest():
    from conftest import golden
    from paper_2603_09555_b200 import random_init_host

    z = golden("weights_digest.npz")
    cfg = small_config()
    p = random_init_host(cfg, 2)
    assert np.array_equal(p.embedding[:2, :8], z["small.embedding_first"])
    for i in (0, cfg.n_layers - 1):
        assert float(p.layers[i].W_in.astype(np.float64).sum()) == float(z[f"small.{i}.W_in"])
        assert float(p.layers[i].A_log.astype(np.float64).sum()) == float(z[f"small.{i}.A_log"])


def test_decay_coefficient_bf16e():
    from paper_2603_09555_b200 import decay_coefficient

    cfg = small_config()
    a_log = np.log(np.array([1.5, 3.7, 15.9], dtype=np.float32))
    a = decay_coefficient(a_log, cfg)
    assert np.all(a < 0)
    ab = decay_coefficient(a_log, cfg.with_policy(decay_exp="bf16e"))
    assert np.all((ab.view(np.uint32) & 0xFFFF) == 0)  # bf16-representable
    with pytest.raises(ValueError):
        decay_coefficient(np.array([np.inf], dtype=np.float32), cfg)


def test_cost_model_matches_reference_formula():
    """Our flops_prefill is the reference cost.py formula (pinned numbers
    from SURVEY §8d: 0.343 GF/token at 130M, 6.160 GF/token at 2.7B)."""
    from paper_2603_09555_b200 import flops_prefill, named_config

    f130 = flops_prefill(named_config("130m"), 8192) / 8192
    f27 = flops_prefill(named_config("2.7b"), 8192) / 8192
    assert abs(f130 / 1e9 - 0.343) < 0.002
    assert abs(f27 / 1e9 - 6.160) < 0.002
