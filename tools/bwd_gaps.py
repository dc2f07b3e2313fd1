"""Where the backward step's time goes: per-kernel CUDA events inside a back-to-back
sequence vs one call, and host time per call. python tools/bwd_gaps.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_20399_b200 import attention as A

B, H, N, D = 16, 16, 4096, 128
CAUSAL = bool(int(sys.argv[1])) if len(sys.argv) > 1 else True
q, k, v, do = (torch.empty(B, H, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1) for _ in range(4))
o, lse = A.attention_fwd(q, k, v, causal=CAUSAL)
dq, dk, dv = (torch.empty_like(q) for _ in range(3))
ws = torch.empty(A.bwd_workspace_bytes(B, H, N, D), dtype=torch.uint8, device="cuda")
bwd = lambda: A.attention_bwd(q, k, v, o, do, lse, causal=CAUSAL, dq=dq, dk=dk, dv=dv, workspace=ws)  # noqa
for _ in range(3):
    bwd()
torch.cuda.synchronize()
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa
# 1) whole calls back to back
s, e = ev(), ev()
s.record()
t0 = time.perf_counter()
for _ in range(10):
    bwd()
t1 = time.perf_counter()
e.record()
torch.cuda.synchronize()
print(f"10 bwd calls: {s.elapsed_time(e) / 10:.3f} ms/call on the GPU, host {1e3 * (t1 - t0) / 10:.3f} ms/call")
# 2) the three kernels as separate calls with events between them
marks = [ev() for _ in range(31)]
marks[0].record()
for i in range(10):
    for j, m in enumerate((1, 2, 4)):
        A.debug_set_bwd_phases(m)
        bwd()
        marks[1 + 3 * i + j].record()
A.debug_set_bwd_phases(7)
torch.cuda.synchronize()
tot = [0.0, 0.0, 0.0]
for i in range(10):
    for j in range(3):
        tot[j] += marks[3 * i + j].elapsed_time(marks[3 * i + j + 1])
print("sequence: prep %.3f  dkdv %.3f  dq %.3f  ms (sum %.3f)" % (tot[0] / 10, tot[1] / 10, tot[2] / 10, sum(tot) / 10))
# 3) each kernel alone, 5 reps
for name, m in (("prep", 1), ("dkdv", 2), ("dq", 4)):
    A.debug_set_bwd_phases(m)
    s, e = ev(), ev()
    s.record()
    for _ in range(5):
        bwd()
    e.record()
    torch.cuda.synchronize()
    print(f"{name} alone: {s.elapsed_time(e) / 5:.3f} ms")
A.debug_set_bwd_phases(7)
