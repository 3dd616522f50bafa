"""Bundle I/O: the reference's manifest.json + data.bin
format, pinned byte for byte by a bundle the reference itself wrote
(tests/golden/ref_bundle, make_golden.py), and the reference's validation
cases (its tests/test_bundle.py:80-146).  CPU tests check the format and the
errors; the GPU test loads straight into the device layout and checks it is
bitwise the layout ``from_reference`` builds."""

from __future__ import annotations

import json
import os
import shutil

import numpy as np
import pytest
import torch

from paper_2603_09555_b200 import bundle
from paper_2603_09555_b200.config import ModelConfig
from paper_2603_09555_b200.params import random_init_host

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "golden", "ref_bundle")


def _ref_cfg():
    # the config make_golden.py wrote ref_bundle with
    return ModelConfig(vocab_size=32, d_model=16, n_layers=1, d_state=8, head_dim=8, expand=2,
                       n_groups=1, conv_kernel=4, chunk_size=16, norm_eps=1e-12)


def _same(a, b):
    return np.array_equal(np.asarray(a, dtype=np.float32), np.asarray(b, dtype=np.float32))


def test_reference_bundle_loads_bitwise():
    params, cfg = bundle.load_bundle_host(REF)
    assert cfg.d_model == 16 and cfg.n_layers == 1 and cfg.dt_limits == (0.0, float("inf"))
    want = random_init_host(_ref_cfg(), 9)  # the reference's random_init(cfg, 9)
    assert _same(params.embedding, want.embedding)
    assert _same(params.final_norm_w, want.final_norm_w)
    for got, exp in zip(params.layers, want.layers):
        for f in ("W_in", "conv_w", "conv_b", "dt_bias", "A_log", "D", "norm_w", "W_out"):
            assert _same(getattr(got, f), getattr(exp, f)), f


def test_save_is_byte_identical_to_reference(tmp_path):
    bundle.save_bundle(random_init_host(_ref_cfg(), 9), _ref_cfg(), tmp_path)
    for f in ("manifest.json", "data.bin"):
        with open(os.path.join(REF, f), "rb") as a, open(tmp_path / f, "rb") as b:
            assert a.read() == b.read(), f


def test_round_trip_and_layout(tmp_path):
    cfg = ModelConfig(vocab_size=64, d_model=32, n_layers=2, d_state=8, head_dim=8)
    host = random_init_host(cfg, 3)
    bundle.save_bundle(host, cfg, tmp_path)
    man = json.loads((tmp_path / "manifest.json").read_text())
    names = [e["name"] for e in man["tensors"]]
    assert names == bundle.tensor_names(cfg) and len(names) == 2 + 8 * cfg.n_layers
    prev = 0
    for e in man["tensors"]:
        assert e["offset"] % bundle.ALIGNMENT == 0 and e["offset"] >= prev
        assert e["length"] == 4 * int(np.prod(e["shape"]))
        prev = e["offset"] + e["length"]
    got, cfg2 = bundle.load_bundle_host(tmp_path)
    assert cfg2 == cfg
    assert _same(got.layers[1].W_out, host.layers[1].W_out)


def _corrupt(tmp_path, edit):
    shutil.copytree(REF, tmp_path / "b")
    p = tmp_path / "b" / "manifest.json"
    man = json.loads(p.read_text())
    edit(man)
    p.write_text(json.dumps(man))
    return tmp_path / "b"


def test_version_mismatch(tmp_path):
    b = _corrupt(tmp_path, lambda m: m.__setitem__("format_version", 2))
    with pytest.raises(bundle.FormatVersionError):
        bundle.load_bundle_host(b)


def test_missing_tensor(tmp_path):
    b = _corrupt(tmp_path, lambda m: m["tensors"].pop(3))
    with pytest.raises(bundle.MissingTensorError, match="layers.0.conv1d.bias"):
        bundle.load_bundle_host(b)


def test_shape_mismatch(tmp_path):
    def edit(m):
        m["tensors"][1]["shape"] = [1, 2]
    with pytest.raises(bundle.TensorShapeError, match="in_proj"):
        bundle.load_bundle_host(_corrupt(tmp_path, edit))


def test_corrupt_offset_names_the_tensor(tmp_path):
    def edit(m):
        m["tensors"][2]["offset"] += 4
    with pytest.raises(bundle.PayloadError, match="conv1d.weight"):
        bundle.load_bundle_host(_corrupt(tmp_path, edit))


def test_truncated_payload(tmp_path):
    shutil.copytree(REF, tmp_path / "b")
    data = (tmp_path / "b" / "data.bin").read_bytes()
    (tmp_path / "b" / "data.bin").write_bytes(data[:-64])
    with pytest.raises(bundle.PayloadError, match="truncated"):
        bundle.load_bundle_host(tmp_path / "b")


def test_duplicate_and_unknown_tensors(tmp_path):
    b = _corrupt(tmp_path, lambda m: m["tensors"].append(dict(m["tensors"][0])))
    with pytest.raises(bundle.BundleError, match="duplicate"):
        bundle.load_bundle_host(b)

    def extra(m):
        e = dict(m["tensors"][-1])
        e["name"] = "extra.weight"
        m["tensors"].append(e)
    with pytest.warns(UserWarning, match="extra.weight"):
        bundle.load_bundle_host(_corrupt(tmp_path / "x", extra))


def test_missing_directory_is_named_error(tmp_path):
    with pytest.raises(bundle.BundleError, match="cannot read bundle"):
        bundle.load_bundle_host(tmp_path / "nope")


@pytest.mark.gpu
@pytest.mark.parametrize("compute", ["f32", "bf16"])
def test_device_load_matches_from_reference(tmp_path, compute):
    """load_bundle converts on the device; the result is bitwise the layout
    from_reference builds on the host, so prefill logits are identical."""
    import paper_2603_09555_b200 as m

    cfg = ModelConfig(vocab_size=512, d_model=128, n_layers=2).with_policy(compute=compute)
    host = random_init_host(cfg, 13)
    rng = np.random.default_rng(0)
    for lp in host.layers:  # non-unit norm weights exercise the bf16 fold
        lp.norm_w = (1.0 + 0.1 * rng.standard_normal(cfg.d_inner)).astype(np.float32)
    bundle.save_bundle(host, cfg, tmp_path)
    dev, cfg2 = bundle.load_bundle(tmp_path, compute=compute)
    ref = m.from_reference(host, cfg)
    assert torch.equal(dev.embedding, ref.embedding)
    for a, b in zip(dev.layers, ref.layers):
        for f in ("W_in", "conv_w", "conv_b", "dt_bias", "A_log", "D", "norm_w", "W_out", "a"):
            assert torch.equal(getattr(a, f), getattr(b, f)), f
    toks = rng.integers(0, cfg.vocab_size, size=(2, 40))
    la, _ = m.prefill(dev, toks, cfg2, logits="last")
    lb, _ = m.prefill(ref, toks, cfg, logits="last")
    assert torch.equal(la, lb)
