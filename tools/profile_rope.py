"""One plain and one fused-rotary forward (B16 H16 N4096 D128 causal) for an ncu capture."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_20399_b200 import attention as A  # noqa: E402

B, H, N, D = 16, 16, 4096, 128
q, k, v = (torch.empty(B, H, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1) for _ in range(3))
ang = torch.rand(N, D // 2, device="cuda")
tabs = (ang.sin().contiguous(), ang.cos().contiguous())
for _ in range(2):
    A.attention_fwd(q, k, v, causal=True)
    A.attention_fwd(q, k, v, causal=True, rotary_tables=tabs)
torch.cuda.synchronize()
print("ok")
