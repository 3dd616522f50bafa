"""CTA-pair GEMM check: ssd200_gemm_bf16 (F32 epilogue) with option 20 on vs torch."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_09555_b200 import _abi

lib = _abi.lib()
for (M, N, K) in [(8192, 4384, 1024), (32768, 1024, 2048), (9000, 1100, 320)]:
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda", generator=g).to(torch.bfloat16)
    ref = A.float() @ B.float().t()
    for pair in (0, 1):
        lib.ssd200_set_option(20, pair)
        C = torch.full((M, N), float("nan"), device="cuda", dtype=torch.float32)
        _abi.check(lib.ssd200_gemm_bf16(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K,
                                        _abi.stream_handle()), "gemm")
        torch.cuda.synchronize()
        err = (C - ref).abs().max().item()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            lib.ssd200_gemm_bf16(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K,
                                 _abi.stream_handle())
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 10
        print(f"M={M} N={N} K={K} pair={pair} max|err|={err:.3e} ref max {ref.abs().max().item():.1f} "
              f"{ms*1e3:.1f} us {2*M*N*K/ms/1e9:.0f} TF/s", flush=True)
lib.ssd200_set_option(20, 0)
