"""bench.py's host logic (no GPU): the driver contract's defaults, the
self-launch of N ranks for ``--gpus N``, and the split of C4's global batch."""

from __future__ import annotations

import importlib
import os
import sys

import pytest

from conftest import ROOT


def _bench(monkeypatch, argv):
    monkeypatch.setattr(sys, "argv", ["bench.py"] + argv)
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    return importlib.import_module("bench")


def test_defaults_are_the_c4_headline(monkeypatch):
    bench = _bench(monkeypatch, [])
    a = bench.parse()
    assert (a.model, a.batch, a.seqlen, a.gpus, a.workload) == ("2.7b", 32, 8192, 1, "prefill")
    assert a.warmup >= 3


def test_gpus_flag_self_launches_torchrun(monkeypatch):
    bench = _bench(monkeypatch, ["--gpus", "4", "--steps", "2"])
    seen = {}

    def fake_call(cmd, env):
        seen["cmd"], seen["env"] = cmd, env
        return 0

    monkeypatch.setattr(bench.subprocess, "call", fake_call)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    assert bench.self_launch(bench.parse()) == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-3:] == ["--gpus", "4", "--steps", "2"][-3:]
    assert os.path.basename(cmd[cmd.index("--nnodes=1") + 4]) == "bench.py"
    assert seen["env"]["NCCL_DEBUG"] == "INFO"
    assert seen["env"]["NCCL_DEBUG_FILE"] == "/dev/stderr"  # stdout stays one JSON line


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_global_batch_split(world):
    from paper_2603_09555_b200 import shard

    rows = [shard.batch_slice(32, r, world) for r in range(world)]
    assert rows[0].start == 0 and rows[-1].stop == 32
    assert all(a.stop == b.start for a, b in zip(rows, rows[1:]))
    assert {s.stop - s.start for s in rows} == {32 // world}
