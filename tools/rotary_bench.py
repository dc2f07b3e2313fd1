"""Rotary (tkb_rotary_qk) bandwidth: algorithmic bytes (read + write Q and K, the sin/cos
tables) / time, against the measured copy bandwidth."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_20399_b200 import attention as A

for B, H, HKV, N, D in ((16, 16, 16, 4096, 128), (16, 32, 8, 4096, 128), (16, 16, 16, 4096, 64)):
    q = torch.empty(B, H, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1)
    k = torch.empty(B, HKV, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1)
    ang = torch.rand(N, D // 2, device="cuda", dtype=torch.float32)
    sin, cos = ang.sin(), ang.cos()
    f = lambda: A.rotary_qk(q, k, sin, cos)  # noqa
    for _ in range(5): f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(50): f()
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 50
    by = 2 * 2 * (q.numel() + k.numel()) + 2 * 4 * N * D // 2
    print(f"rotary_qk B{B} H{H} Hkv{HKV} N{N} D{D}: {ms:.4f} ms  {by / ms / 1e6:.0f} GB/s")
