"""One bench-shaped step (fwd + bwd, B16 H16 N4096 D128 causal) for ncu captures."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_20399_b200 import attention as A

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="16,16,4096,128")
ap.add_argument("--causal", type=int, default=1)
ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()
B, H, N, D = map(int, a.shape.split(","))
q, k, v, do = (torch.empty(B, H, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1) for _ in range(4))
ws = torch.empty(A.bwd_workspace_bytes(B, H, N, D), dtype=torch.uint8, device="cuda")
for _ in range(a.steps):
    o, lse = A.attention_fwd(q, k, v, causal=bool(a.causal))
    A.attention_bwd(q, k, v, o, do, lse, causal=bool(a.causal), workspace=ws)
torch.cuda.synchronize()
print("ok")
