"""GEMM throughput (CUDA events) of tkb.gemm vs torch.matmul (cuBLAS) at a few shapes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_20399_b200 import attention as A


def t_events(fn, iters=20, warmup=5):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(iters):
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


for M, N, K in ((4096, 4096, 4096), (8192, 8192, 8192), (16384, 4096, 4096), (4096, 12288, 4096)):
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ms = t_events(lambda: A.gemm(a, b, out=c))
    ref = t_events(lambda: torch.matmul(a, b, out=c))
    fl = 2.0 * M * N * K
    print(f"gemm {M}x{N}x{K}: tkb {fl / ms / 1e9:7.1f} TFLOPS  cuBLAS {fl / ref / 1e9:7.1f} TFLOPS", flush=True)
