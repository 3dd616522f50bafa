"""Benchmark of the Mamba-2 SSD hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload prefill|decode|serve] [--model 2.7b] [--batch 32] [--seqlen 8192]
                    [--shard batch|heads] [--tune field=value ...]

Headline (BASELINE.json configs[3], the north-star's C4): Mamba-2 2.7B bf16
chunked-SSD prefill of a GLOBAL batch of 32 sequences x 8192 tokens, one step
= one full prefill (embed, 64 blocks, final norm, tied head on the last
position) over token ids already resident in HBM.  The global batch is split
over the ranks (strong scaling: batch-sharded rows, no collective on the data
path; ``--shard heads`` instead splits every layer's SSD head groups with one
NCCL all-reduce after out_proj).  ``value`` = global tokens / max-over-ranks
step time.  ``e2e`` = the same metric through the public API ``prefill`` with
the token ids copied from pinned host memory and the last-position logits
copied back, inside the timed region.

``--gpus N`` with no torchrun environment re-launches itself through
``torch.distributed.run`` with N ranks on 127.0.0.1 (NCCL_DEBUG=INFO to
stderr, so the rank count is on record).

The JSON line also carries: ``roofline`` for the dominant kernel (timed live
with CUDA events around every launch of that phase), per-phase time shares,
``cpu_baseline`` (the numpy oracle port of the reference timed on this host,
bounded sample, rank 0 at N=1), and at N=1 two extra points: ``c2`` (370M
prefill, B=4, T=8192, BASELINE configs[1]) and ``decode`` (1.3B cached decode
sweep, configs[2]: tok/s and HBM GB/s of CUDA-graph steps), plus ``clocks``
sampled by nvidia-smi during the timed region and ``gpu_launches``.

``--impl reference`` times the reference algorithm's CPU implementation (the
oracle port; /root/reference is not on the GPU box) on this host's cores.
"""

from __future__ import annotations

import os

# host threads for the CPU legs must be fixed before numpy loads BLAS
_NCPU = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, str(_NCPU))

import argparse  # noqa: E402
import ctypes  # noqa: E402
import json  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import threading  # noqa: E402
import time  # noqa: E402

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# prefill layer phases as the library marks them (abi.cu PH_*): scan_states = chunk
# cumsum + chunk walk, scan_out = the output kernel (intra + cross-chunk outputs, D
# skip, gate; the gated norm's row scale is in the out_proj epilogue)
PHASES = ("in_proj", "conv", "scan_states", "scan_out", "out_proj")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--workload", default="prefill", choices=("prefill", "decode", "serve"))
    ap.add_argument("--model", default="2.7b")
    ap.add_argument("--batch", type=int, default=32, help="GLOBAL prefill batch (split over ranks)")
    ap.add_argument("--seqlen", type=int, default=8192)
    ap.add_argument("--c2-model", default="370m")
    ap.add_argument("--c2-batch", type=int, default=4)
    ap.add_argument("--c2-seqlen", type=int, default=8192)
    ap.add_argument("--no-c2", action="store_true")
    ap.add_argument("--decode-model", default="1.3b")
    ap.add_argument("--serve-model", default="780m")
    ap.add_argument("--serve-batch", type=int, default=64, help="GLOBAL batch (split over ranks)")
    ap.add_argument("--serve-prompt", type=int, default=4096)
    ap.add_argument("--serve-gen", type=int, default=512)
    ap.add_argument("--decode-batch", type=int, default=1)
    ap.add_argument("--decode-sweep", default="1,8,64,256",
                    help="decode batch sizes reported under decode.sweep ('' = none)")
    ap.add_argument("--decode-steps", type=int, default=64)
    ap.add_argument("--no-decode", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seqlen", type=int, default=2048,
                    help="sequence length of the bounded CPU sample (extrapolated linearly in T)")
    ap.add_argument("--shard", default="batch", choices=("batch", "heads"),
                    help="N>1: batch rows per rank (default) or SSD head groups of the whole "
                         "batch with an all-reduce after out_proj")
    ap.add_argument("--tune", action="append", default=[],
                    help="implementation choice field=value (ssd200_tuning_t), repeatable")
    return ap.parse_args()


def self_launch(args):
    """--gpus N outside torchrun: re-exec this script under torch.distributed.run
    with N local ranks (rendezvous on 127.0.0.1) and return its exit status."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # keep stdout to the one JSON line
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


# ---------------------------------------------------------------- distributed


def dist_setup(n):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def barrier(world):
    import torch

    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    torch.cuda.synchronize()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


# ---------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = (
        "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
        "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
        "clocks_event_reasons.sw_power_cap"
    )

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True,
            )
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- peaks


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return {"hbm_gbs": m["hbm_gbs"], "bf16_tflops": m["bf16_tflops"],
                "bf16_tflops_sustained": m.get("bf16_tflops_sustained", m["bf16_tflops"]),
                "source": "measured (MEASURED_PEAKS.json)"}
    except (OSError, KeyError, ValueError):
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "source": "fallback (B200_PROFILING.md)"}


def traffic_from_profiles(model, kernel_key, batch):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    --set full capture (profiles/traffic.json, keyed by model; captured at
    C4's per-GPU batch of 32 rows x 8192), or None for another shape."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            table = json.load(f).get(model.lower(), {})
    except (OSError, ValueError):
        return None
    return table.get(kernel_key) if batch == 32 else None


# ---------------------------------------------------------------- CPU legs


def cpu_prefill_sample(model, T=2048, layers=1):
    """Reference algorithm (numpy oracle port) on a bounded sample: `layers`
    blocks of `model` at (B=1, T) + the tied head on the last position.
    Returns (tok/s extrapolated linearly in n_layers, seconds, description)."""
    import oracle as orc
    from paper_2603_09555_b200 import named_config, random_init_host

    cfg = named_config(model, compute="f32", n_layers=layers)
    full = named_config(model, compute="f32")
    host = random_init_host(cfg, 0)
    toks = np.random.default_rng(0).integers(0, cfg.vocab_size, size=(1, T))
    hidden = host.embedding[toks]
    orc.block(host.layers[0], hidden[:, :256], cfg)  # warm
    t0 = time.perf_counter()
    h = hidden
    for lyr in host.layers:
        h, _, _ = orc.block(lyr, h, cfg)
    t_layers = (time.perf_counter() - t0) / layers
    t1 = time.perf_counter()
    normed = orc.rms_norm(h[:, -1], host.final_norm_w, cfg.norm_eps)
    _ = normed @ host.embedding.T
    t_head = time.perf_counter() - t1
    per_seq = full.n_layers * t_layers + t_head
    desc = (f"numpy oracle port of ssd_engine.block_forward: {layers} block(s) of {model} "
            f"f32 at B=1,T={T} ({t_layers:.2f} s/block) + last-row head, extrapolated x{full.n_layers} layers")
    return T / per_seq, t_layers * layers + t_head, desc


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    K, W = args.steps, args.warmup
    T = min(args.cpu_seqlen, args.seqlen)
    vals = []
    for i in range(W + K):
        v, _, desc = cpu_prefill_sample(args.model, T=T, layers=1)
        if i >= W:
            vals.append(v)
    val = float(np.mean(vals))
    line = {
        "impl": "reference",
        "metric": f"prefill_tokens_per_s[{args.model}]",
        "value": val,
        "unit": "tok/s",
        "n_gpus": args.gpus,
        "steps": K,
        "warmup": W,
        "higher_is_better": True,
        "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": f"Mamba-2 {args.model} prefill (reference CPU path, numpy oracle port)",
                   "global_batch": args.batch, "seq_len": args.seqlen, "sample_seq_len": T},
        "cpu_baseline": {"value": val, "unit": "tok/s", "cores": _NCPU, "kind": "port",
                         "sample": desc},
        "e2e": {"value": val, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "vs_baseline": None,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU legs


def make_events(n):
    import torch

    evs = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    for e in evs:
        e.record()
    torch.cuda.synchronize()
    return evs


def run_prefill(args, rank, world, local):
    import torch

    import paper_2603_09555_b200 as m
    from paper_2603_09555_b200 import _abi, model as mmod, shard

    cfg = m.named_config(args.model, compute="bf16")
    params = m.synthetic_init(cfg, seed=1234, device=f"cuda:{local}")
    rows = shard.batch_slice(args.batch, rank, world)  # this rank's rows of the global batch
    B, T = rows.stop - rows.start, args.seqlen
    g = torch.Generator(device="cpu").manual_seed(0)
    host_all = torch.randint(0, cfg.vocab_size, (args.batch, T), generator=g, dtype=torch.int64)
    host_tok = host_all[rows].contiguous().pin_memory()
    dev_tok = host_tok.cuda()
    lib = _abi.lib()

    # per-phase CUDA events around every layer's phases (5 phases x 2)
    L = cfg.n_layers
    K, W = args.steps, args.warmup
    ev = make_events(K * L * 10)
    ev_arr = (ctypes.c_void_p * (K * L * 10))(*[e.cuda_event for e in ev])

    class Hook:
        step = -1

    orig = mmod._Runner.prefill_layer

    def timed_layer(self, i, *a, **kw):
        if Hook.step >= 0:
            base = ctypes.addressof(ev_arr) + (Hook.step * L + i) * 10 * ctypes.sizeof(ctypes.c_void_p)
            lib.ssd200_set_phase_events(ctypes.c_void_p(base), 5)
        try:
            return orig(self, i, *a, **kw)
        finally:
            lib.ssd200_set_phase_events(None, 0)

    mmod._Runner.prefill_layer = timed_layer

    def step():
        return m.prefill(params, dev_tok, cfg, logits="last")

    for _ in range(W):
        step()
    barrier(world)
    torch.cuda.synchronize()
    n0 = lib.ssd200_launch_count()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        start.record()
        for k in range(K):
            step()
        stop.record()
        torch.cuda.synchronize()
    launches = lib.ssd200_launch_count() - n0
    ms = start.elapsed_time(stop) / K
    ms_max = max_over_ranks(ms, world)
    tokens_total = args.batch * T
    value = tokens_total / (ms_max / 1e3)

    # e2e through the public API: pinned host ids -> device, logits -> host
    host_out = torch.empty((B, cfg.vocab_size), dtype=torch.float32).pin_memory()
    barrier(world)
    s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s2.record()
    for k in range(K):
        tok = host_tok.to(f"cuda:{local}", non_blocking=True)
        lg, _ = m.prefill(params, tok, cfg, logits="last")
        host_out.copy_(lg, non_blocking=True)
    e2.record()
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(s2.elapsed_time(e2) / K, world)

    # phase shares: the same K steps again with CUDA events around every
    # layer phase (kept out of the headline timed region above)
    for k in range(K):
        Hook.step = k
        step()
    Hook.step = -1
    torch.cuda.synchronize()
    mmod._Runner.prefill_layer = orig

    # phase totals (ms per step, summed over layers)
    phase_ms = np.zeros(5)
    for k in range(K):
        for i in range(L):
            for p in range(5):
                b = ev[(k * L + i) * 10 + 2 * p]
                e = ev[(k * L + i) * 10 + 2 * p + 1]
                phase_ms[p] += b.elapsed_time(e)
    phase_ms /= K

    # the reference FLOP formula (cost.py:79-98) with the head on the last row
    flops_step = m.flops_prefill(cfg, T, B, head_rows=1)
    pk = peaks()
    # dominant kernel: the phase with the largest share
    dom = int(np.argmax(phase_ms))
    per_layer = m.cost.flops_prefill_layer(cfg, T)
    scan_flops = B * (per_layer["ssd_intra"] + per_layer["ssd_states"] + per_layer["ssd_inter"]
                      + per_layer["ssd_cross"])
    phase_flops = {
        0: B * per_layer["in_proj"],
        1: B * per_layer["conv"],
        2: B * (per_layer["ssd_states"] + per_layer["ssd_inter"]),
        3: B * (per_layer["ssd_intra"] + per_layer["ssd_cross"]),
        4: B * per_layer["out_proj"],
    }
    launch_ms = phase_ms[dom] / L
    achieved = phase_flops[dom] / (launch_ms / 1e3) / 1e12 if phase_flops[dom] else None
    peak = pk["bf16_tflops_sustained"]
    kernel_key = {0: "tc_gemm_kernel<256,2>", 1: "conv_silu_tma", 2: "ssd_tc_chunkscan",
                  3: "ssd_tc_out", 4: "tc_gemm_kernel<256,4>"}[dom]
    kernel_name = {0: "tc_gemm_kernel<256, INPROJ, CTA pair>", 1: "conv_silu_tma",
                   2: "ssd_tc_cumsum + ssd_tc_chunkscan", 3: "ssd_tc_out",
                   4: "tc_gemm_kernel<256, RESID_NORM, CTA pair>"}[dom]
    roof = {
        "kernel": f"{PHASES[dom]} ({kernel_name})",
        "bound": "tensor",
        "achieved": achieved,
        "peak": peak,
        "unit": "TFLOP/s",
        "frac": (achieved / peak) if achieved else None,
        "traffic": traffic_from_profiles(args.model, kernel_key, B),
        "traffic_source": "profiles/traffic.json (ncu --set full, one launch at B=32, T=8192)",
        "algorithmic_flops_per_launch": phase_flops[dom],
        "avg_launch_ms": launch_ms,
        "peak_source": pk["source"] + ", sustained (kernel timed inside a long step)",
    }
    # every phase against its own roofline: the GEMMs against the tensor peak; conv and
    # the two scan kernels against HBM by their operand bytes (cost.bytes_prefill_layer,
    # cost.bytes_scan_kernels); the whole scan (both kernels) by its algorithmic bytes
    # and the reference FLOP formula (what round 1 reported)
    pb = dict(m.cost.bytes_prefill_layer(cfg, T, B))
    pb.update(m.cost.bytes_scan_kernels(cfg, T, B))
    per_phase = {}

    def hbm_entry(t_launch, nbytes):
        gb = nbytes / t_launch / 1e9
        return {"ms_per_launch": t_launch * 1e3, "bound": "hbm", "achieved": gb, "unit": "GB/s",
                "frac": gb / pk["hbm_gbs"], "bytes_per_launch": nbytes}

    for p_, name in enumerate(PHASES):
        t_launch = phase_ms[p_] / L / 1e3
        if t_launch <= 0:
            continue
        if name in ("in_proj", "out_proj"):
            tf = phase_flops[p_] / t_launch / 1e12
            per_phase[name] = {"ms_per_launch": t_launch * 1e3, "bound": "tensor",
                               "achieved": tf, "unit": "TFLOP/s", "frac": tf / peak}
        else:
            per_phase[name] = hbm_entry(t_launch, pb[name])
    t_scan = (phase_ms[2] + phase_ms[3]) / L / 1e3
    if t_scan > 0:
        e = hbm_entry(t_scan, pb["scan"])
        e.update(formula_tflops=scan_flops / t_scan / 1e12,
                 formula_frac_of_tensor=scan_flops / t_scan / 1e12 / peak,
                 note="both scan kernels; algorithmic bytes (x, z, B, C, dt in; u, state out)")
        per_phase["scan"] = e
    roof["phases"] = per_phase
    step_tflops = flops_step / (ms / 1e3) / 1e12  # this rank's work / its own time
    del params, dev_tok
    return {
        "value": value,
        "ms": ms_max,
        "e2e_ms": e2e_ms,
        "e2e_value": tokens_total / (e2e_ms / 1e3),
        "d2h_global": args.batch * cfg.vocab_size * 4,
        "launches": launches,
        "roofline": roof,
        "phases_ms": {PHASES[p]: float(phase_ms[p]) for p in range(5)},
        "step_tflops_per_gpu": step_tflops,
        "step_mfu": step_tflops / pk["bf16_tflops"],
        "clocks": clk.summary(),
        "flops_step": flops_step,
        "batch_per_gpu": B,
    }


def run_prefill_point(model, B, T, K, W, local):
    """One extra prefill point (no phase pass, no e2e): tok/s and TFLOP/s."""
    import torch

    import paper_2603_09555_b200 as m

    cfg = m.named_config(model, compute="bf16")
    params = m.synthetic_init(cfg, seed=99, device=f"cuda:{local}")
    tok = torch.randint(0, cfg.vocab_size, (B, T), device=f"cuda:{local}")
    for _ in range(W):
        m.prefill(params, tok, cfg, logits="last")
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(K):
        m.prefill(params, tok, cfg, logits="last")
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / K
    tf = m.flops_prefill(cfg, T, B, head_rows=1) / (ms / 1e3) / 1e12
    pk = peaks()
    del params, tok
    torch.cuda.empty_cache()
    return {"workload": f"Mamba-2 {model} bf16 prefill (BASELINE configs[1] point)", "batch": B,
            "seq_len": T, "value": B * T / (ms / 1e3), "unit": "tok/s", "ms_per_step": ms,
            "tflops": tf, "mfu": tf / pk["bf16_tflops"], "steps": K, "warmup": W}


def run_prefill_heads(args, rank, world, local):
    """Head-group-sharded prefill: every rank runs the same
    batch on its heads; one NCCL all-reduce of [partial | sum u^2] per layer.
    Strong scaling: value = the batch's tokens / max-over-ranks step time."""
    import torch
    import torch.distributed as dist

    import paper_2603_09555_b200 as m
    from paper_2603_09555_b200 import _abi, shard

    cfg = m.named_config(args.model, compute="bf16")
    params = shard.synthetic_shard(cfg, rank, world, seed=1234, device=f"cuda:{local}")
    B, T = args.batch, args.seqlen
    g = torch.Generator(device="cpu").manual_seed(0)
    host_tok = torch.randint(0, cfg.vocab_size, (B, T), generator=g, dtype=torch.int64).pin_memory()
    dev_tok = host_tok.cuda()
    lib = _abi.lib()

    run = shard.HeadShardedPrefill(params, dev_tok, cfg)  # buffers allocated once

    def step(tok):
        run.restart(tok)
        for i in range(cfg.n_layers):
            buf = run.partial(i)
            if world > 1:
                dist.all_reduce(buf, op=dist.ReduceOp.SUM)
            run.finish()
        return run.logits()

    for _ in range(args.warmup):
        step(dev_tok)
    barrier(world)
    n0 = lib.ssd200_launch_count()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        s0.record()
        for _ in range(args.steps):
            step(dev_tok)
        s1.record()
        torch.cuda.synchronize()
    launches = lib.ssd200_launch_count() - n0
    ms = max_over_ranks(s0.elapsed_time(s1) / args.steps, world)
    host_out = torch.empty((B, cfg.vocab_size), dtype=torch.float32).pin_memory()
    barrier(world)
    s0.record()
    for _ in range(args.steps):
        lg = step(host_tok.to(f"cuda:{local}", non_blocking=True))
        host_out.copy_(lg, non_blocking=True)
    s1.record()
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(s0.elapsed_time(s1) / args.steps, world)
    flops = m.flops_prefill(cfg, T, B, head_rows=1)
    pk = peaks()
    tf = flops / (ms / 1e3) / 1e12
    return {
        "value": B * T / (ms / 1e3), "ms": ms, "e2e_value": B * T / (e2e_ms / 1e3),
        "d2h_global": B * cfg.vocab_size * 4, "launches": launches, "batch_per_gpu": B,
        "roofline": {"kernel": "whole step (head-sharded)", "bound": "tensor", "achieved": tf / world,
                     "peak": pk["bf16_tflops_sustained"], "unit": "TFLOP/s",
                     "frac": tf / world / pk["bf16_tflops_sustained"], "traffic": None},
        "phases_ms": None, "step_tflops_per_gpu": tf / world,
        "step_mfu": tf / world / pk["bf16_tflops"], "clocks": clk.summary(), "flops_step": flops,
    }


def run_decode(args, local, B=None, params=None):
    """1.3B cached decode: one CUDA-graph step (all layers + head + argmax)
    replayed; HBM bytes = weights once + state read/write + logits."""
    import torch

    import paper_2603_09555_b200 as m

    cfg = m.named_config(args.decode_model, compute="bf16")
    if params is None:
        params = m.synthetic_init(cfg, seed=7, device=f"cuda:{local}")
    if B is None:
        B = args.decode_batch
    prompt = torch.randint(0, cfg.vocab_size, (B, 16), device=f"cuda:{local}")
    _, cache = m.prefill(params, prompt, cfg, logits=None)
    dec = m.GreedyDecoder(params, cfg, cache, args.decode_steps + 8)
    dec.step()  # capture + first replay
    for _ in range(3):
        dec.step()
    torch.cuda.synchronize()
    n = args.decode_steps
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        dec.step()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / n
    del dec, cache
    nbytes = m.decode_step_bytes(cfg, B)
    gbs = nbytes / (ms / 1e3) / 1e9
    pk = peaks()
    return {
        "model": args.decode_model,
        "batch": B,
        "ms_per_step": ms,
        "tok_per_s": B / (ms / 1e3),
        "hbm_gbs": gbs,
        "hbm_frac": gbs / pk["hbm_gbs"],
        "bytes_per_step": nbytes,
        "note": ("CUDA-graph step: per layer a swapped-operand tensor-core in_proj, the TMA state "
                 "stream (conv + SSM update + gate + sum u^2), out_proj, norm + residual finish; "
                 "head + argmax"),
    }


def run_decode_heads(args, rank, world, local):
    """``--workload decode --shard heads``: one batch of ``--decode-batch`` rows
    decoded by all ranks, each owning n_heads / N SSD heads of every layer; the
    token step (every layer's partial in_proj / state stream / out_proj, ONE
    NCCL all-reduce of [partial | sum u^2] per layer, finish, head, argmax) is
    one captured CUDA graph (shard.HeadShardedGraphDecoder).  Strong scaling:
    value = B / max-over-ranks token-step time."""
    import torch
    import torch.distributed as dist

    import paper_2603_09555_b200 as m
    from paper_2603_09555_b200 import cost, shard

    cfg = m.named_config(args.decode_model, compute="bf16")
    dev = f"cuda:{local}"
    params = shard.synthetic_shard(cfg, rank, world, seed=7, device=dev)
    B, W = args.decode_batch, args.warmup
    n = max(args.steps, 1) * 16
    prompt = torch.randint(0, cfg.vocab_size, (B, 16), generator=torch.Generator().manual_seed(5))
    run = shard.HeadShardedPrefill(params, prompt.to(dev), cfg)
    for i in range(cfg.n_layers):
        buf = run.partial(i)
        if world > 1:
            dist.all_reduce(buf)
        run.finish()
    tok = torch.empty((B,), dtype=torch.int64, device=dev)
    run.logits(argmax=tok)
    gd = shard.HeadShardedGraphDecoder([shard.HeadShardedDecoder.from_prefill(run)],
                                       n + 16 * W + 2,
                                       reduce=shard.nccl_reduce() if world > 1 else None)
    gd.set_token(tok)
    gd.step_idx.fill_(1)
    for _ in range(16 * W):
        gd.step()
    with ClockSampler(local) as clk:
        barrier(world)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(n):
            gd.step()
        e.record()
        torch.cuda.synchronize()
        barrier(world)
    ms = max_over_ranks(s.elapsed_time(e) / n, world)
    loc = params.local
    # this rank's algorithmic bytes: its weight shard (+ the replicated embedding /
    # head), its heads' state read + written, the logits
    nbytes = (cost.decode_step_bytes(cfg, B) - cost.weight_bytes(cfg) - 2 * cost.cache_bytes(cfg, B)
              + sum(t.numel() * t.element_size() for lp in params.layers
                    for t in (lp.W_in, lp.W_out))
              + params.embedding.numel() * 2
              + 2 * cfg.n_layers * B * (loc.n_heads * cfg.head_dim * cfg.d_state
                                        + loc.conv_dim * (cfg.conv_kernel - 1)) * 4)
    gbs = nbytes / (ms / 1e3) / 1e9
    pk = peaks()
    if rank == 0:
        print(json.dumps({
            "metric": f"decode_tokens_per_s[{args.decode_model}]",
            "value": B / (ms / 1e3), "unit": "tok/s", "n_gpus": world, "steps": args.steps,
            "warmup": W, "ms_per_step": ms * 16, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random ids; device-drawn weights with the reference init distributions)",
            "config": {"workload": f"Mamba-2 {args.decode_model} bf16 cached decode, SSD-head-group "
                                   f"sharded (BASELINE configs[2])",
                       "global_batch": B, "heads_per_gpu": loc.n_heads,
                       "step": "16 greedy tokens (one captured CUDA graph per token, the per-layer "
                               "NCCL all-reduce inside it)",
                       "parallelism": f"head-group-sharded x{world}"},
            "ms_per_token": ms,
            "roofline": {"kernel": "head-sharded decode token step (one CUDA graph)", "bound": "hbm",
                         "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": gbs / pk["hbm_gbs"], "traffic": None,
                         "algorithmic_bytes_per_token_step_per_gpu": nbytes},
            "e2e": None, "cpu_baseline": None, "clocks": clk.summary(),
            "gpu_launches": n * (cfg.n_layers * 5 + 5),
        }), flush=True)


def run_decode_workload(args, rank, world, local):
    """``--workload decode``: the decode headline line (BASELINE metric "decode
    tok/s & HBM GB/s"): per-GPU batch ``--decode-batch`` of the 1.3B model, rows
    sharded over ranks (weak scaling, no collective), CUDA-graph steps with the
    state resident in HBM; e2e = the public ``generate`` from a pinned host
    prompt (16 tokens) with the tokens copied back, prefill and graph capture
    included, tokens/s over the generated tokens."""
    import torch

    import paper_2603_09555_b200 as m

    cfg = m.named_config(args.decode_model, compute="bf16")
    dev = f"cuda:{local}"
    params = m.synthetic_init(cfg, seed=7, device=dev)
    B, K, W = args.decode_batch, args.steps, args.warmup
    n_steps = max(K, 1) * 16  # one "step" of the contract = 16 decode tokens per row
    prompt = torch.randint(0, cfg.vocab_size, (B, 16), device=dev)
    _, cache = m.prefill(params, prompt, cfg, logits=None)
    dec = m.GreedyDecoder(params, cfg, cache, n_steps + 16 * W + 8)
    for _ in range(16 * W):
        dec.step()
    with ClockSampler(local) as clk:
        barrier(world)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(n_steps):
            dec.step()
        e.record()
        torch.cuda.synchronize()
        barrier(world)
    ms = max_over_ranks(s.elapsed_time(e) / n_steps, world)
    del dec, cache
    nbytes = m.decode_step_bytes(cfg, B)
    pk = peaks()
    # e2e through the public API with host buffers
    host_prompt = torch.randint(0, cfg.vocab_size, (B, 16)).pin_memory()
    gen = 64
    m.generate(params, host_prompt.to(dev, non_blocking=True), gen, cfg=cfg)  # warm: captures
    torch.cuda.synchronize()
    barrier(world)
    s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s2.record()
    res = m.generate(params, host_prompt.to(dev, non_blocking=True), gen, cfg=cfg)
    toks = res.tokens.to("cpu", non_blocking=True)
    e2.record()
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(s2.elapsed_time(e2), world)
    if rank == 0:
        gbs = nbytes / (ms / 1e3) / 1e9
        line = {
            "metric": f"decode_tokens_per_s[{args.decode_model}]",
            "value": B * world / (ms / 1e3),
            "unit": "tok/s",
            "n_gpus": world,
            "steps": K,
            "warmup": W,
            "ms_per_step": ms * 16,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic (random ids; device-drawn weights with the reference init distributions)",
            "config": {"workload": f"Mamba-2 {args.decode_model} bf16 cached decode (BASELINE configs[2])",
                       "batch_per_gpu": B, "global_batch": B * world,
                       "step": "16 greedy tokens per row (CUDA-graph token steps)",
                       "parallelism": f"batch-sharded x{world} (no data-path collective)",
                       "l2": "weights 2.7 GB + state read/written per token > 126 MB L2; no flush"},
            "ms_per_token": ms,
            "hbm_gbs": gbs,
            "e2e": {"value": B * world * (gen - 1) / (e2e_ms / 1e3), "unit": "tok/s",
                    "h2d_bytes_per_step": int(host_prompt.numel() * 8),
                    "d2h_bytes_per_step": int(toks.numel() * 8),
                    "note": "public generate(): prompt H2D + 16-token prefill + 63 decode steps + "
                            "tokens D2H; the decode graph captured by a warm-up call is reused "
                            "when the cache is <= 8 GB (decode._GRAPH_CACHE), else re-captured"},
            "roofline": {"kernel": "decode token step (one CUDA graph: 48 x [in_proj, state stream, "
                                   "out_proj, finish] + head)",
                         "bound": "hbm", "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": gbs / pk["hbm_gbs"], "traffic": None,
                         "algorithmic_bytes_per_token_step": nbytes},
            "cpu_baseline": None,
            "clocks": clk.summary(),
            "gpu_launches": n_steps * (cfg.n_layers * 4 + 5),
        }
        print(json.dumps(line), flush=True)


def run_serve_workload(args, rank, world, local):
    """``--workload serve`` (BASELINE configs[4], C5): Mamba-2 780M serving, a
    global batch of 64 prompts of 4K tokens, each prefilled and then extended
    by 512 greedy tokens through the public ``generate`` (decode.py:147-194):
    one chunked-SSD prefill, then CUDA-graph token steps with the cache in
    place.  Rows are sharded over ranks (strong scaling: the global batch is
    fixed, no data-path collective).  One step = one whole serving batch.
    ``value`` = (prompt + generated) tokens/s over all ranks with the prompts
    resident in HBM; ``e2e`` = the same call from pinned host prompts with the
    generated tokens copied back.  ``roofline`` = the decode phase (the
    larger share), measured in a separate pass of CUDA-graph token steps
    against the HBM peak; ``phases_ms_per_step`` splits prefill / decode."""
    import torch

    import paper_2603_09555_b200 as m
    from paper_2603_09555_b200 import _abi

    lib = _abi.lib()
    cfg = m.named_config(args.serve_model, compute="bf16")
    dev = f"cuda:{local}"
    if args.serve_batch % world:
        raise ValueError("--serve-batch must divide by the number of GPUs")
    B, P, G = args.serve_batch // world, args.serve_prompt, args.serve_gen
    K, W = args.steps, args.warmup
    params = m.synthetic_init(cfg, seed=11, device=dev)
    gen_t = torch.Generator().manual_seed(1000 + rank)
    host_prompt = torch.randint(0, cfg.vocab_size, (B, P), generator=gen_t).pin_memory()
    dev_prompt = host_prompt.to(dev)

    def serve(prompt):
        return m.generate(params, prompt, G, cfg=cfg)

    for _ in range(W):
        serve(dev_prompt)  # warm-up: the first call captures the decode graph
    torch.cuda.synchronize()
    # prefill share of the step, timed alone on the same prompts
    pf_ms = []
    for _ in range(2):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        m.prefill(params, dev_prompt, cfg, logits="last")
        e.record()
        torch.cuda.synchronize()
        pf_ms.append(s.elapsed_time(e))
    prefill_ms = max_over_ranks(min(pf_ms), world)
    with ClockSampler(local) as clk:
        barrier(world)
        torch.cuda.synchronize()
        n0 = lib.ssd200_launch_count()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(K):
            res = serve(dev_prompt)
        e.record()
        torch.cuda.synchronize()
        barrier(world)
        host_launches = lib.ssd200_launch_count() - n0
    ms = max_over_ranks(s.elapsed_time(e) / K, world)
    out_tokens = res.tokens
    # e2e: pinned host prompts in, generated tokens out, inside the timed region
    host_out = torch.empty(out_tokens.shape, dtype=out_tokens.dtype).pin_memory()
    barrier(world)
    torch.cuda.synchronize()
    s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s2.record()
    for _ in range(K):
        r = serve(host_prompt.to(dev, non_blocking=True))
        host_out.copy_(r.tokens, non_blocking=True)
    e2.record()
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(s2.elapsed_time(e2) / K, world)
    del res, r
    from paper_2603_09555_b200 import decode as mdec

    mdec.clear_graph_cache()
    torch.cuda.empty_cache()
    # decode-phase roofline: CUDA-graph token steps at this batch, separate pass
    dargs = argparse.Namespace(**vars(args))
    dargs.decode_model, dargs.decode_steps = args.serve_model, 64
    dec = run_decode(dargs, local, B=B, params=params)
    pk = peaks()
    tokens = B * world * (P + G)
    if rank == 0:
        line = {
            "metric": f"serve_tokens_per_s[{args.serve_model}]",
            "value": tokens / (ms / 1e3),
            "unit": "tok/s",
            "n_gpus": world,
            "steps": K,
            "warmup": W,
            "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic (random ids; device-drawn weights with the reference init distributions)",
            "config": {"workload": f"Mamba-2 {args.serve_model} serving: prefill {P} + {G}-step greedy "
                                   f"decode (BASELINE configs[4])",
                       "global_batch": B * world, "batch_per_gpu": B, "prompt_len": P,
                       "gen_len": G, "tokens_per_step": tokens,
                       "parallelism": f"batch-sharded x{world} (no data-path collective)",
                       "l2": "weights 1.6 GB + per-row state per token > 126 MB L2; no flush"},
            "generated_tokens_per_s": B * world * G / (ms / 1e3),
            "phases_ms_per_step": {"prefill": prefill_ms, "decode": ms - prefill_ms},
            "e2e": {"value": tokens / (e2e_ms / 1e3), "unit": "tok/s",
                    "h2d_bytes_per_step": int(host_prompt.numel() * 8) * world,
                    "d2h_bytes_per_step": int(host_out.numel() * 8) * world},
            "roofline": {"kernel": f"decode token step at B={B} (one CUDA graph: "
                                   f"{cfg.n_layers} x [in_proj, state stream, out_proj, finish] + head)",
                         "bound": "hbm", "achieved": dec["hbm_gbs"], "peak": pk["hbm_gbs"],
                         "unit": "GB/s", "frac": dec["hbm_frac"], "traffic": None,
                         "algorithmic_bytes_per_token_step": dec["bytes_per_step"],
                         "ms_per_token_step": dec["ms_per_step"]},
            "cpu_baseline": None,
            "clocks": clk.summary(),
            "gpu_launches": int(host_launches + K * (G - 1) * (cfg.n_layers * 4 + 5)),
        }
        print(json.dumps(line), flush=True)


def _weight_gb(model):
    import paper_2603_09555_b200 as m
    from paper_2603_09555_b200 import cost

    return cost.n_params(m.named_config(model, compute="bf16")) * 2 / 1e9


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(self_launch(args))
    from paper_2603_09555_b200 import _abi

    opts = dict(kv.split("=") for kv in args.tune)
    with _abi.tuning(**opts) if opts else _nullctx():
        run(args)


class _nullctx:
    def __enter__(self):
        return None

    def __exit__(self, *a):
        return False


def run(args):
    import torch

    rank, world, local = dist_setup(args.gpus)
    if args.workload in ("decode", "serve"):
        if args.workload == "decode" and args.shard == "heads":
            run_decode_heads(args, rank, world, local)
        else:
            (run_decode_workload if args.workload == "decode" else run_serve_workload)(
                args, rank, world, local)
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
            dist.destroy_process_group()
        return
    heads = args.shard == "heads"
    res = (run_prefill_heads if heads else run_prefill)(args, rank, world, local)
    torch.cuda.empty_cache()
    c2 = dec = cpu = None
    if world == 1 and not args.no_c2:  # extra points at N=1 (the scaling runs stay short)
        c2 = run_prefill_point(args.c2_model, args.c2_batch, args.c2_seqlen, args.steps,
                               args.warmup, local)
    if world == 1 and not args.no_decode:
        import paper_2603_09555_b200 as m

        dcfg = m.named_config(args.decode_model, compute="bf16")
        dparams = m.synthetic_init(dcfg, seed=7, device=f"cuda:{local}")
        sweep = [int(x) for x in args.decode_sweep.split(",") if x.strip()] or [args.decode_batch]
        dec = {"model": args.decode_model, "workload": "BASELINE configs[2]: cached decode, "
               "CUDA-graph token steps", "sweep": []}
        for b in sweep:
            r = run_decode(args, local, B=b, params=dparams)
            dec["sweep"].append({k: r[k] for k in ("batch", "ms_per_step", "tok_per_s",
                                                   "hbm_gbs", "hbm_frac", "bytes_per_step")})
        del dparams
        torch.cuda.empty_cache()
    if rank == 0 and world == 1 and not args.no_cpu:
        # two blocks: ~10 s of host work at 2.7B (one block took 4.8 s on the box)
        v, secs, desc = cpu_prefill_sample(args.model, T=min(args.cpu_seqlen, args.seqlen),
                                           layers=2)
        cpu = {"value": v, "unit": "tok/s", "cores": _NCPU, "kind": "port", "sample": desc,
               "seconds": secs}
    if rank == 0:
        line = {
            "metric": f"prefill_tokens_per_s[{args.model}]",
            "value": res["value"],
            "unit": "tok/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": res["ms"],
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic (random ids; device-drawn weights with the reference init distributions)",
            "config": {
                "workload": f"Mamba-2 {args.model} bf16 chunked-SSD prefill "
                            + ("(BASELINE configs[3], north-star C4)" if args.model.lower() == "2.7b"
                               else "(BASELINE configs[1] point)"),
                "global_batch": args.batch,
                "batch_per_gpu": args.batch if heads else res["batch_per_gpu"],
                "seq_len": args.seqlen,
                "chunk": 256,
                "head": "tied head on the last position only",
                "parallelism": (f"SSD-head-group-sharded x{world} (one NCCL all-reduce per layer)"
                                if heads else f"batch-sharded x{world} (global batch split, no "
                                "data-path collective)"),
                "l2": f"working set > 126 MB L2 (activations + {_weight_gb(args.model):.2f} GB bf16 weights per "
                      "step); no flush",
                "tuning": dict(kv.split("=") for kv in args.tune) or "library defaults",
            },
            "tflops_per_gpu": res["step_tflops_per_gpu"],
            "mfu": res["step_mfu"],
            "e2e": {"value": res["e2e_value"], "unit": "tok/s",
                    "h2d_bytes_per_step": args.batch * args.seqlen * 8,
                    "d2h_bytes_per_step": res["d2h_global"]},
            "roofline": res["roofline"],
            "phases_ms_per_step": res["phases_ms"],
            "cpu_baseline": cpu,
            "c2": c2,
            "decode": dec,
            "clocks": res["clocks"],
            "gpu_launches": int(res["launches"]),
            "world": {"ranks": world, "backend": "nccl" if world > 1 else None,
                      "nccl_version": _nccl_version() if world > 1 else None},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


def _nccl_version():
    try:
        import torch

        v = torch.cuda.nccl.version()
        return ".".join(map(str, v)) if isinstance(v, tuple) else str(v)
    except Exception:  # noqa: BLE001
        return None


if __name__ == "__main__":
    main()
