"""BASELINE configs[3]: D=64 vs D=128 sequence sweep N=768..16384, fwd and bwd, causal and
non-causal (B*H*N held near 256 x 4096 tokens-heads), TFLOPS and the algorithmic HBM GB/s
of each pass. Writes a markdown table to stdout.

  python tools/sweep.py [--ns 768,1024,...]
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_20399_b200 import attention as A


def t_events(fn, iters=10, warmup=3):
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


ap = argparse.ArgumentParser()
ap.add_argument("--ns", default="768,1024,1536,2048,3072,4096,6144,8192,12288,16384")
args = ap.parse_args()
print("| D | N | B x H | causal | fwd ms | fwd TFLOPS | fwd GB/s | bwd ms | bwd TFLOPS | bwd GB/s |")
print("|---|---|---|---|---|---|---|---|---|---|")
for D in (64, 128):
    for N in map(int, args.ns.split(",")):
        BH = max(1, (256 * 4096) // N)
        H = 16
        B = max(1, BH // H)
        q, k, v, do = (torch.empty(B, H, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1) for _ in range(4))
        ws = torch.empty(A.bwd_workspace_bytes(B, H, N, D), dtype=torch.uint8, device="cuda")
        for causal in (False, True):
            o, lse = A.attention_fwd(q, k, v, causal=causal)
            dq, dk, dv = (torch.empty_like(q) for _ in range(3))
            fms = t_events(lambda: A.attention_fwd(q, k, v, causal=causal, out=o, lse=lse))
            bms = t_events(lambda: A.attention_bwd(q, k, v, o, do, lse, causal=causal, dq=dq, dk=dk, dv=dv,
                                                  workspace=ws))
            f = 0.5 if causal else 1.0
            ff = 4 * B * H * N * N * D * f
            bf = 10 * B * H * N * N * D * f
            fbytes = 8 * B * H * N * D + 4 * B * H * N
            bbytes = 16 * B * H * N * D + 8 * B * H * N
            print(f"| {D} | {N} | {B}x{H} | {int(causal)} | {fms:.3f} | {ff / fms / 1e9:.0f} | {fbytes / fms / 1e6:.0f} "
                  f"| {bms:.3f} | {bf / bms / 1e9:.0f} | {bbytes / bms / 1e6:.0f} |", flush=True)
        del q, k, v, do, ws, o, lse, dq, dk, dv
        torch.cuda.empty_cache()
