import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2410_20399_b200 import attention as A
M = N = K = 8192
a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    A.gemm(a, b, out=c); torch.matmul(a, b, out=c)
torch.cuda.synchronize()
