"""Variable-length batch throughput (tkb_attn_fwd_varlen / tkb_attn_bwd_varlen) against the
same sequences padded to the longest one through the fixed-length entry points.

FLOPs count only each sequence's own work (FA convention, causal halved), so the padded run
is charged the same useful FLOPs it computes around its padding. CUDA events, inputs resident."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_20399_b200 import attention as A  # noqa: E402


def timed(fn, iters=20, warmup=5):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def run(lens, H, D, causal):
    rng = np.random.default_rng(0)
    T, B, nmax = int(sum(lens)), len(lens), int(max(lens))
    cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
    q, k, v, do = (torch.empty(T, H, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1) for _ in range(4))
    o, lse = A.attention_fwd_varlen(q, k, v, cu, nmax, causal=causal)
    wsf = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    dq, dk, dv = (torch.empty_like(q) for _ in range(3))
    fwd = timed(lambda: A.attention_fwd_varlen(q, k, v, cu, nmax, causal=causal, out=o, lse=lse, workspace=wsf))
    bwd = timed(lambda: A.attention_bwd_varlen(q, k, v, o, do, lse, cu, nmax, causal=causal, dq=dq, dk=dk, dv=dv))
    # padded: [B, H, nmax, D]
    qp, kp, vp, dop = (torch.empty(B, H, nmax, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1)
                       for _ in range(4))
    op, lp = A.attention_fwd(qp, kp, vp, causal=causal)
    dqp, dkp, dvp = (torch.empty_like(qp) for _ in range(3))
    pfwd = timed(lambda: A.attention_fwd(qp, kp, vp, causal=causal, out=op, lse=lp))
    pbwd = timed(lambda: A.attention_bwd(qp, kp, vp, op, dop, lp, causal=causal, dq=dqp, dk=dkp, dv=dvp))
    half = 0.5 if causal else 1.0
    n2 = float(sum(int(n) * int(n) for n in lens))
    ff, fb = 4.0 * H * n2 * D * half, 10.0 * H * n2 * D * half
    del rng
    return {"sequences": B, "tokens": T, "max_len": nmax, "heads": H, "head_dim": D, "causal": causal,
            "varlen_fwd_ms": fwd, "varlen_fwd_tflops": ff / fwd / 1e9, "varlen_bwd_ms": bwd,
            "varlen_bwd_tflops": fb / bwd / 1e9, "padded_fwd_ms": pfwd, "padded_fwd_tflops": ff / pfwd / 1e9,
            "padded_bwd_ms": pbwd, "padded_bwd_tflops": fb / pbwd / 1e9}


if __name__ == "__main__":
    rng = np.random.default_rng(1)
    out = []
    for D in (128, 64):
        lens = rng.integers(512, 8193, size=32)  # 32 sequences of 512 .. 8192 tokens
        for causal in (True, False):
            r = run(lens, 16, D, causal)
            out.append(r)
            print(json.dumps(r), flush=True)
