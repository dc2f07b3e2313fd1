"""Per-kernel times of the variable-length backward (debug phase masks) next to the same
sequences as separate fixed-length problems of similar total work."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_20399_b200 import attention as A  # noqa: E402


def timed(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


rng = np.random.default_rng(1)
H, D = 16, 128
lens = rng.integers(512, 8193, size=32)
T, nmax = int(lens.sum()), int(lens.max())
cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
q, k, v, do = (torch.empty(T, H, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1) for _ in range(4))
for causal in (True, False):
    o, lse = A.attention_fwd_varlen(q, k, v, cu, nmax, causal=causal)
    dq, dk, dv = (torch.empty_like(q) for _ in range(3))
    ws = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
    f = lambda: A.attention_bwd_varlen(q, k, v, o, do, lse, cu, nmax, causal=causal, dq=dq, dk=dk, dv=dv,  # noqa
                                       workspace=ws)
    res = {}
    for name, mask in (("prep", 1), ("dkdv", 2), ("dq", 4), ("all", 7)):
        A.debug_set_bwd_phases(7)
        f()
        A.debug_set_bwd_phases(mask)
        res[name] = timed(f)
    A.debug_set_bwd_phases(7)
    half = 0.5 if causal else 1.0
    n2 = float((lens.astype(np.float64) ** 2).sum())
    fl_kv, fl_q = 8 * H * n2 * D * half, 6 * H * n2 * D * half
    print(f"varlen causal={causal}: prep {res['prep']:.3f} dkdv {res['dkdv']:.3f} ms ({fl_kv / res['dkdv'] / 1e9:.0f} "
          f"TFLOPS executed)  dq {res['dq']:.3f} ms ({fl_q / res['dq'] / 1e9:.0f})  all {res['all']:.3f} ms "
          f"({10 * H * n2 * D * half / res['all'] / 1e9:.0f} FA)", flush=True)
