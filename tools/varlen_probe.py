"""Probe: does a variable-length call fault when the offset tensor-map base lies before the
allocation (fresh process, first allocations)? Runs fwd and bwd with a sync after each."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2410_20399_b200 import attention as A  # noqa: E402

lens = [300, 1, 128, 0, 513, 129]
H, D = 4, 128
pad_mb = int(sys.argv[1]) if len(sys.argv) > 1 else 0
guard = torch.empty(pad_mb << 20, dtype=torch.uint8, device="cuda") if pad_mb else None
T = sum(lens)
g = torch.Generator().manual_seed(0)
mk = lambda: (torch.rand(T, H, D, generator=g) * 2 - 1).to("cuda", torch.bfloat16)  # noqa: E731
q, k, v, do = mk(), mk(), mk(), mk()
cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
print("q ptr", hex(q.data_ptr()), "offset bytes", max(lens) * H * D * 2, flush=True)
o, lse = A.attention_fwd_varlen(q, k, v, cu, max(lens), causal=True)
torch.cuda.synchronize()
print("fwd ok", flush=True)
dq, dk, dv = A.attention_bwd_varlen(q, k, v, o, do, lse, cu, max(lens), causal=True)
torch.cuda.synchronize()
print("bwd ok", flush=True)
