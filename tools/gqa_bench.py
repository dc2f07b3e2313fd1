"""Grouped-query attention fwd / bwd TFLOPS (FA convention, query-head FLOPs) next to the
multi-head case of the same query shape."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_20399_b200 import attention as A


def t(fn, iters=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


B, H, N, D = 8, 32, 4096, 128
for HKV in (32, 8, 1):
    for causal in (False, True):
        q = torch.empty(B, H, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1)
        k, v = (torch.empty(B, HKV, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1) for _ in range(2))
        do = torch.empty_like(q).uniform_(-1, 1)
        o, lse = A.attention_fwd(q, k, v, causal=causal)
        cf = 0.5 if causal else 1.0
        ms_f = t(lambda: A.attention_fwd(q, k, v, causal=causal, out=o, lse=lse))
        ms_b = t(lambda: A.attention_bwd(q, k, v, o, do, lse, causal=causal))
        print(f"B{B} H{H} Hkv{HKV} N{N} D{D} causal={int(causal)}: fwd {4*B*H*N*N*D*cf/ms_f/1e9:7.1f} TFLOPS"
              f"  bwd {10*B*H*N*N*D*cf/ms_b/1e9:7.1f} TFLOPS")
