"""One small call of every device entry point, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): fixed-length fwd + bwd (MHA causal D128 ragged N, D64 non-causal),
grouped-query with the dK/dV head split (MQA), a variable-length batch, the fused rotary
forward, the standalone rotary and the GEMM. Usage:
  compute-sanitizer --tool memcheck python tools/sanitize_small.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_20399_b200 import attention as A  # noqa: E402

dev = "cuda"
CLONE_O = os.environ.get("TKB_SANITIZE_CLONE_O") == "1"
g = torch.Generator(device=dev).manual_seed(0)


def rnd(*shape):
    return torch.empty(*shape, device=dev, dtype=torch.bfloat16).uniform_(-1, 1, generator=g)


for B, H, HKV, N, D, causal in ((1, 2, 2, 300, 128, True), (1, 2, 2, 200, 64, False), (1, 8, 1, 256, 128, True)):
    q, do = rnd(B, H, N, D), rnd(B, H, N, D)
    k, v = rnd(B, HKV, N, D), rnd(B, HKV, N, D)
    o, lse = A.attention_fwd(q, k, v, causal=causal)
    if CLONE_O:  # O re-written by a plain store (initcheck does not track TMA bulk stores)
        o = o.clone()
    A.attention_bwd(q, k, v, o, do, lse, causal=causal)
    torch.cuda.synchronize()
    print("fixed", B, H, HKV, N, D, causal, "ok", flush=True)

lens = [130, 1, 257]
T = sum(lens)
cu = torch.tensor([0, 130, 131, 388], dtype=torch.int32, device=dev)
q, k, v, do = rnd(T, 2, 128), rnd(T, 2, 128), rnd(T, 2, 128), rnd(T, 2, 128)
o, lse = A.attention_fwd_varlen(q, k, v, cu, max(lens), causal=True)
if CLONE_O:
    o = o.clone()
A.attention_bwd_varlen(q, k, v, o, do, lse, cu, max(lens), causal=True)
torch.cuda.synchronize()
print("varlen ok", flush=True)

N, D = 256, 128
q, k, v = rnd(1, 2, N, D), rnd(1, 2, N, D), rnd(1, 2, N, D)
pos = torch.arange(N, device=dev, dtype=torch.float64)[:, None]
freq = 10000.0 ** (-torch.arange(D // 2, device=dev, dtype=torch.float64) / (D // 2))
sin, cos = (f(pos * freq[None, :]).float().contiguous() for f in (torch.sin, torch.cos))
A.attention_fwd(q, k, v, causal=True, rotary_tables=(sin, cos))
A.rotary_qk(q, k, sin, cos)
torch.cuda.synchronize()
print("rotary ok", flush=True)

a, b = rnd(256, 192), rnd(192, 320)
A.gemm(a, b)
torch.cuda.synchronize()
print("gemm ok", flush=True)
