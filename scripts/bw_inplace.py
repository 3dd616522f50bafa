import torch
x = torch.randn(256 * 1024 * 1024, device="cuda")  # 1 GiB f32
for name, fn in [("mul_", lambda: x.mul_(0.999)), ("copy", lambda: y.copy_(x))]:
    y = torch.empty_like(x)
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(10): fn()
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    print(name, f"{2 * x.numel() * 4 / ms / 1e6:.0f} GB/s")
