"""Forward-only launches for ncu captures: python tools/profile_fwd.py --shape B,H,N,D --causal 0 --iters 2"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_20399_b200 import attention as A

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="4,16,4096,128")
ap.add_argument("--causal", type=int, default=0)
ap.add_argument("--iters", type=int, default=2)
a = ap.parse_args()
B, H, N, D = map(int, a.shape.split(","))
q, k, v = (torch.empty(B, H, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1) for _ in range(3))
for _ in range(a.iters):
    o, lse = A.attention_fwd(q, k, v, causal=bool(a.causal))
torch.cuda.synchronize()
print("ok")
