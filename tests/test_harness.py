"""Cost model + benchmark harness: the reference's byte
model and CostReport CSV schema (cost.py:138-258), pinned by values the
reference computed (PYTHONPATH=/root/reference/pkg/src: ssd_engine.cost
bytes_model / peak_activation_bytes on the same configs); the GPU harness runs
the reference's bench API on the device."""

from __future__ import annotations

import pytest

from paper_2603_09555_b200 import cost
from paper_2603_09555_b200.config import ModelConfig


def test_byte_model_matches_reference():
    c1 = ModelConfig(vocab_size=50288, d_model=768, n_layers=24)
    assert cost.bytes_model(c1, "prefill", 512) == 3948636416
    assert cost.bytes_model(c1, "decode_step") == 595432576
    assert cost.peak_activation_bytes(c1, 512) == 1716375808
    c2 = ModelConfig(vocab_size=64, d_model=32, n_layers=2, d_state=8, head_dim=8, chunk_size=16)
    assert cost.bytes_model(c2, "prefill", 37, 3) == 2171456
    assert cost.bytes_model(c2, "decode_step", batch=2) == 128704
    assert cost.peak_activation_bytes(c2, 37, 2) == 701312
    with pytest.raises(ValueError):
        cost.bytes_model(c2, "train")


def test_cost_report_csv_round_trip():
    r = cost.CostReport(model="m", phase="decode", seq_len=64, mode="cached", tokens_per_s=1.5,
                        flops=10, nbytes=20, mfu=0.1, hbu=0.2, cache_bytes=30, peak_bytes=40,
                        n_gpus=8, batch=4, algo_bytes=50, algo_hbu=0.3)
    ref_row = r.to_csv_row()
    assert len(ref_row.split(",")) == len(cost.CostReport.CSV_HEADER.split(","))
    back = cost.CostReport.from_csv_row(ref_row)
    assert back.tokens_per_s == 1.5 and back.n_gpus == 1  # reference schema: B200 columns default
    full = cost.CostReport.from_csv_row(r.to_csv_row(b200=True))
    assert full == r
    with pytest.raises(ValueError):
        cost.CostReport.from_csv_row("a,b")


def test_parse_device():
    assert cost.parse_device("a100").peak_tflops == 312.0
    assert cost.parse_device("x:1:2").peak_gbps == 2.0
    assert cost.parse_device("b200").peak_gbps > 1000
    with pytest.raises(ValueError):
        cost.parse_device("nope")


@pytest.mark.gpu
def test_harness_runs_on_device(tmp_path):
    import paper_2603_09555_b200 as m
    from paper_2603_09555_b200 import harness

    cfg = ModelConfig(vocab_size=512, d_model=128, n_layers=2).with_policy(compute="bf16")
    params = m.from_reference(m.random_init_host(cfg, 1), cfg)
    proto = harness.BenchProtocol(warmup_runs=1, timed_runs=2)
    rows = harness.bench_prefill(params, cfg, [256, 512], protocol=proto, batch=2)
    rows += harness.bench_decode(params, cfg, [8], protocol=proto, batch=2)
    rows += harness.bench_decode(params, cfg, [4], mode="non_cached", protocol=proto)
    for r in rows:
        assert not r.oom and r.report.tokens_per_s > 0 and r.wall_mean > 0
    assert rows[2].report.algo_bytes == 8 * cost.decode_step_bytes(cfg, 2)
    harness.write_csv(rows, tmp_path / "r.csv")
    lines = (tmp_path / "r.csv").read_text().splitlines()
    assert lines[0] == cost.CostReport.CSV_HEADER_B200 and len(lines) == 5


def test_prefill_phase_bytes():
    """Algorithmic bytes of the HBM-bound prefill phases (bench.py's per-phase
    rooflines): conv reads + writes xBC once; the scan reads x, z, B, C, dt and
    writes u and the final state."""
    from paper_2603_09555_b200 import cost, named_config

    cfg = named_config("2.7b")
    rows = 32 * 8192
    b = cost.bytes_prefill_layer(cfg, 8192, 32)
    assert b["conv"] == 2 * rows * cfg.conv_dim * 2
    want = (rows * (2 * cfg.d_inner + 2 * cfg.d_state) * 2 + rows * cfg.n_heads * 4
            + rows * cfg.d_inner * 2 + 32 * cfg.n_heads * cfg.head_dim * cfg.d_state * 4)
    assert b["scan"] == want
    assert cost.bytes_prefill_layer(cfg, 8192, 1)["conv"] * 32 == b["conv"]
    # the two scan kernels' own operands: every algorithmic operand once, plus the
    # split's intermediates (x read by both kernels, the bf16 chunk states, cs / dt^T)
    k = cost.bytes_scan_kernels(cfg, 8192, 32)
    prev = 32 * 32 * cfg.n_heads * cfg.head_dim * cfg.d_state * 2
    assert k["scan_states"] + k["scan_out"] > b["scan"] + 2 * prev
    assert 4.5e9 < k["scan_states"] < 4.7e9 and 9.7e9 < k["scan_out"] < 9.9e9  # ncu: 4.58 / 10.04 GB
