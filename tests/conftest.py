"""Shared fixtures.  Markers: ``gpu`` = needs a B200 (run via gpurun)."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

# Stated bf16 bounds (relative Frobenius error against the f32 oracle / the
# reference on the SAME bf16-rounded weights), frozen at ~3x the worst value
# measured on B200 (DESIGN.md §4 lists the per-config measurements):
#   logits and the residual stream of 1-2 layer models: worst 2.6e-3
BF16_BOUND = 8e-3
#   f32 SSM states (chunk states summed from bf16 X*dt*decay operands): worst 4.1e-3
BF16_STATE_BOUND = 1.25e-2
#   logits of a full-depth model (C1: 24 bf16 layers compound): worst 2.3e-2
BF16_MODEL_BOUND = 7e-2


def report(name, **vals):
    """Append a measured error to $SSD200_PARITY_LOG (JSON lines), if set."""
    path = os.environ.get("SSD200_PARITY_LOG")
    if path:
        import json

        with open(path, "a") as f:
            f.write(json.dumps({"test": name, **vals}) + "\n")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: test needs a CUDA (B200) device")


def has_cuda() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if has_cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def golden(name: str):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def small_config(**overrides):
    """The reference's tiny test config (tests/conftest.py:42-57)."""
    from paper_2603_09555_b200 import ModelConfig

    kw = dict(
        vocab_size=64, d_model=32, n_layers=2, d_state=8, head_dim=8, expand=2,
        n_groups=1, conv_kernel=4, chunk_size=16, norm_eps=1e-12,
    )
    kw.update(overrides)
    return ModelConfig(**kw)


# (name, overrides, seed) — must match tests/golden/make_golden.py SMALL_MODELS
SMALL_MODELS = [
    ("base", {}, 2),
    ("k2", dict(d_model=8, n_layers=1, head_dim=4, d_state=4, conv_kernel=2, chunk_size=4), 3),
    ("wide", dict(d_model=64, n_layers=4), 1),
    ("grp", dict(d_model=32, n_groups=2, head_dim=8), 7),
]


def make_instance(rng, batch=1, seq=16, heads=2, pdim=4, ndim=4, groups=1, dtype=np.float64):
    """Random contract-respecting SSD inputs (reference tests/conftest.py:7-24)."""
    return dict(
        X=rng.standard_normal((batch, seq, heads, pdim)).astype(dtype),
        dt=rng.uniform(0.0, 1.2, size=(batch, seq, heads)).astype(dtype),
        a=-rng.uniform(0.3, 4.0, size=heads).astype(dtype),
        B=rng.standard_normal((batch, seq, groups, ndim)).astype(dtype),
        C=rng.standard_normal((batch, seq, groups, ndim)).astype(dtype),
    )


@pytest.fixture
def rng():
    return np.random.default_rng(1234)
