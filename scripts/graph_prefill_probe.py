import sys, time
sys.path.insert(0, '/root/repo')
import torch
import paper_2603_09555_b200 as m
for model, B, T in (("370m", 1, 2048), ("370m", 1, 8192), ("370m", 4, 8192)):
    cfg = m.named_config(model, compute="bf16")
    params = m.synthetic_init(cfg, seed=0)
    tok = torch.randint(0, cfg.vocab_size, (B, T), device="cuda")
    for _ in range(3):
        m.prefill(params, tok, cfg, logits="last")
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    t0 = time.perf_counter(); s.record()
    for _ in range(n):
        m.prefill(params, tok, cfg, logits="last")
    e.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
    eager = s.elapsed_time(e) / n
    host = (t1 - t0) / n * 1e3
    # graph
    st = torch.cuda.Stream(); st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        m.prefill(params, tok, cfg, logits="last")
    torch.cuda.current_stream().wait_stream(st)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out, _ = m.prefill(params, tok, cfg, logits="last")
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    s.record()
    for _ in range(n):
        g.replay()
    e.record(); torch.cuda.synchronize()
    gr = s.elapsed_time(e) / n
    print(f"{model} B={B} T={T}: eager {eager:.3f} ms/step (host {host:.3f} ms), graph {gr:.3f} ms -> {B*T/eager*1e3:.0f} vs {B*T/gr*1e3:.0f} tok/s", flush=True)
    del params
    torch.cuda.empty_cache()
