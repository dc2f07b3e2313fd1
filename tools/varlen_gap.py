"""Where the variable-length backward loses against fixed length: per-kernel times (debug phase
masks) for (a) 32 equal sequences of 4096 through the varlen entry point vs the fixed-length
B=32 N=4096 problem, (b) the r2c random-length batch (32 sequences of 512-8192) in its own
order, (c) the same sequences sorted longest first."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_20399_b200 import attention as A  # noqa: E402

H, D = 16, 128


def timed(fn, iters=10):
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


def kernels(f):
    res = {}
    for name, mask in (("dkdv", 2), ("dq", 4), ("all", 7)):
        A.debug_set_bwd_phases(7)
        f()
        A.debug_set_bwd_phases(mask)
        res[name] = timed(f)
    A.debug_set_bwd_phases(7)
    return res


def varlen(lens, causal=True):
    lens = np.asarray(lens)
    T, nmax = int(lens.sum()), int(lens.max())
    cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
    q, k, v, do = (torch.empty(T, H, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1) for _ in range(4))
    o, lse = A.attention_fwd_varlen(q, k, v, cu, nmax, causal=causal)
    dq, dk, dv = (torch.empty_like(q) for _ in range(3))
    ws = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
    f = lambda: A.attention_bwd_varlen(q, k, v, o, do, lse, cu, nmax, causal=causal, dq=dq, dk=dk, dv=dv,  # noqa
                                       workspace=ws)
    r = kernels(f)
    n2 = float((lens.astype(np.float64) ** 2).sum())
    r["fa_tflops"] = 10 * H * n2 * D * (0.5 if causal else 1.0) / r["all"] / 1e9
    return r


def fixed(B, N, causal=True):
    q, k, v, do = (torch.empty(B, H, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1) for _ in range(4))
    o, lse = A.attention_fwd(q, k, v, causal=causal)
    dq, dk, dv = (torch.empty_like(q) for _ in range(3))
    ws = torch.empty(A.bwd_workspace_bytes(B, H, N, D), dtype=torch.uint8, device="cuda")
    f = lambda: A.attention_bwd(q, k, v, o, do, lse, causal=causal, dq=dq, dk=dk, dv=dv, workspace=ws)  # noqa
    r = kernels(f)
    r["fa_tflops"] = 10 * B * H * N * N * D * (0.5 if causal else 1.0) / r["all"] / 1e9
    return r


def show(name, r):
    print(f"{name:40s} dkdv {r['dkdv']:.3f} ms  dq {r['dq']:.3f} ms  all {r['all']:.3f} ms  "
          f"{r['fa_tflops']:.0f} TFLOPS (FA)", flush=True)


show("fixed B32 N4096", fixed(32, 4096))
show("varlen 32 x 4096", varlen([4096] * 32))
rng = np.random.default_rng(1)
lens = rng.integers(512, 8193, size=32)
show("varlen random (r2c order)", varlen(lens))
show("varlen random, longest first", varlen(np.sort(lens)[::-1]))
show("varlen random, shortest first", varlen(np.sort(lens)))
