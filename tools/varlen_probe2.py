"""Probe: fixed-length ragged call alone, and after a variable-length call (sync after each)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2410_20399_b200 import attention as A  # noqa: E402

mode = sys.argv[1]
g = torch.Generator().manual_seed(0)
rnd = lambda *s: (torch.rand(*s, generator=g) * 2 - 1).to("cuda", torch.bfloat16)  # noqa: E731


def fixed(n):
    q, k, v, do = (rnd(1, 2, n, 128) for _ in range(4))
    o, lse = A.attention_fwd(q, k, v, causal=True)
    torch.cuda.synchronize()
    print("fixed fwd ok", n, flush=True)
    A.attention_bwd(q, k, v, o, do, lse, causal=True)
    torch.cuda.synchronize()
    print("fixed bwd ok", n, flush=True)


def varlen(lens):
    T = sum(lens)
    q, k, v, do = (rnd(T, 2, 128) for _ in range(4))
    cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
    o, lse = A.attention_fwd_varlen(q, k, v, cu, max(lens), causal=True)
    torch.cuda.synchronize()
    print("varlen fwd ok", flush=True)
    A.attention_bwd_varlen(q, k, v, o, do, lse, cu, max(lens), causal=True)
    torch.cuda.synchronize()
    print("varlen bwd ok", flush=True)


if mode == "fixed":
    fixed(130)
    fixed(640)
else:
    varlen([130, 0, 640, 1, 255, 384])
    fixed(130)
