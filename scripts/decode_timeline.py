"""Launch timeline of one captured decode token step (diagnostic).

Needs the probe build: `make -C paper_2603_09555_b200/csrc trace`, then
  SSD200_LIBRARY=$PWD/paper_2603_09555_b200/libssd200_trace.so \
      python scripts/decode_timeline.py --batch 1 [--model 1.3b] [--layers-shown 3]
Per traced launch (in issue order): when its first / last CTA entered, passed
its dependency wait and left, relative to the first launch's first entry (us).
The per-layer summary is the mean over the middle layers."""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_09555_b200 as m  # noqa: E402
from paper_2603_09555_b200 import _abi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="1.3b")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--layers-shown", type=int, default=3)
    ap.add_argument("--json", default="")
    ap.add_argument("--tune", action="append", default=[], help="tuning field=value")
    args = ap.parse_args()
    kv = dict(t.split("=") for t in args.tune)
    with _abi.tuning(**kv):
        run(args)


def run(args):
    lib = _abi.lib()
    if not hasattr(lib, "ssd200_trace_reset"):
        raise SystemExit("not a probe build (make -C paper_2603_09555_b200/csrc trace)")
    lib.ssd200_trace_reset.argtypes = [ctypes.c_int, ctypes.c_void_p]
    lib.ssd200_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int]
    cfg = m.named_config(args.model, compute="bf16")
    params = m.synthetic_init(cfg, seed=7, device="cuda:0")
    B = args.batch
    prompt = torch.randint(0, cfg.vocab_size, (B, 16), device="cuda:0")
    _, cache = m.prefill(params, prompt, cfg, logits=None)
    dec = m.GreedyDecoder(params, cfg, cache, 64)
    torch.cuda.synchronize()
    lib.ssd200_trace_reset(1, None)  # slots are handed out while the graph is captured
    torch.cuda.synchronize()
    dec.step()  # warm-up body on a side stream + capture + first replay
    for _ in range(5):
        dec.step()
    torch.cuda.synchronize()
    # the warm-up body and the capture each took slots; the replays write the captured ones
    n_max = 2048
    out = np.zeros((n_max, 6), dtype=np.uint64)
    names = ctypes.create_string_buffer(n_max * 32)
    n = lib.ssd200_trace_read(out.ctypes.data, names, n_max)
    nm = [names.raw[i * 32:(i + 1) * 32].split(b"\0")[0].decode() for i in range(n)]
    per = n // 2  # warm-up body, then the captured body
    lib.ssd200_trace_reset(0, None)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    dec.step()
    ev1.record()
    torch.cuda.synchronize()
    step_ms = ev0.elapsed_time(ev1)
    n2 = lib.ssd200_trace_read(out.ctypes.data, names, n_max)
    assert n2 == n
    cyc = np.zeros(16, dtype=np.uint64)
    if hasattr(lib, "ssd200_trace_cycles"):
        lib.ssd200_trace_cycles.argtypes = [ctypes.c_void_p]
        lib.ssd200_trace_cycles(cyc.ctypes.data)
        nt = max(int(cyc[5]), 1)
        print(f"# state stream consumer (warp 0), SM cycles per tile over {nt} tiles: "
              f"wait {cyc[0] / nt:.0f}, B/C conv {cyc[1] / nt:.0f}, x conv + z {cyc[2] / nt:.0f}, "
              f"state rows {cyc[3] / nt:.0f}, y / u / done {cyc[4] / nt:.0f}")
    rows = out[per:n].astype(np.int64)
    names_c = nm[per:n]
    t0 = rows[:, 0].min()
    r = (rows - t0) / 1e3  # us
    print(f"# {args.model} B={B}: step {step_ms * 1e3:.1f} us (event), {len(r)} traced launches")
    print("# launch                 enter(first..last)   waited(first..last)   exit(first..last)  [us]")
    k = 4 if cfg.n_layers * 4 == len(r) else max(1, len(r) // cfg.n_layers)
    shown = args.layers_shown * k
    for i in list(range(min(shown, len(r)))) + list(range(max(shown, len(r) - k), len(r))):
        e = r[i]
        print(f"{i:4d} {names_c[i]:16s} {e[0]:8.1f}..{e[1]:8.1f}  {e[2]:8.1f}..{e[3]:8.1f}  "
              f"{e[4]:8.1f}..{e[5]:8.1f}")
    # per-layer mean durations of the middle layers
    L = len(r) // k
    mid = [r[j * k:(j + 1) * k] for j in range(1, L - 1)]
    keys = []
    for j in range(k):
        keys.append({
            "kernel": names_c[j],
            "enter_after_prev_exit_first": float(np.mean([x[j][0] - (x[j - 1][5] if j else x[0][0])
                                                           for x in mid])),
            "wait_done_after_first_enter": float(np.mean([x[j][3] - x[j][0] for x in mid])),
            "exit_last_after_wait_last": float(np.mean([x[j][5] - x[j][3] for x in mid])),
            "span_first_enter_to_last_exit": float(np.mean([x[j][5] - x[j][0] for x in mid])),
        })
    layer_us = float(np.mean([mid[j + 1][0][0] - mid[j][0][0] for j in range(len(mid) - 1)]))
    print(f"# per layer (mean over middle layers): {layer_us:.2f} us")
    for kk in keys:
        print("#  {kernel:16s} span {span_first_enter_to_last_exit:6.2f}  last wait-done {wait_done_after_first_enter:6.2f} "
              "after first enter, last exit {exit_last_after_wait_last:6.2f} after last wait".format(**kk))
    if args.json:
        with open(args.json, "w") as f:
            json.dump({"model": args.model, "batch": B, "step_us": step_ms * 1e3,
                       "layer_us": layer_us, "kernels": keys,
                       "rows_us": r.tolist(), "names": names_c}, f)


if __name__ == "__main__":
    main()
