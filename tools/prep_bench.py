"""bwd_prep alone (debug phase mask 1) over many calls: ms and algorithmic GB/s."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_20399_b200 import attention as A

B, H, N, D = 16, 16, 4096, 128
q, k, v, do = (torch.empty(B, H, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1) for _ in range(4))
o, lse = A.attention_fwd(q, k, v, causal=True)
dq, dk, dv = (torch.empty_like(q) for _ in range(3))
ws = torch.empty(A.bwd_workspace_bytes(B, H, N, D), dtype=torch.uint8, device="cuda")
A.debug_set_bwd_phases(1)
f = lambda: A.attention_bwd(q, k, v, o, do, lse, causal=True, dq=dq, dk=dk, dv=dv, workspace=ws)  # noqa
for _ in range(10): f()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(200): f()
e.record(); torch.cuda.synchronize()
A.debug_set_bwd_phases(7)
ms = s.elapsed_time(e) / 200
by = 4 * B * H * N * D + 12 * B * H * N
print(f"prep {ms:.4f} ms  {by / ms / 1e6:.0f} GB/s")
