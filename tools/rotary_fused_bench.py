"""Cost of the fused rotary prologue: attention_fwd(rotary_tables=...) (one launch,
tkb_attn_fwd_rotary) against the same forward without rotary and against the two-launch
path (tkb_rotary_qk + tkb_attn_fwd). CUDA-event timing, inputs resident, power-capped clocks
sampled (TFLOPS/GHz is the robust comparison)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml  # noqa: E402
import torch  # noqa: E402

from paper_2410_20399_b200 import attention as A  # noqa: E402

pynvml.nvmlInit()
hnd = pynvml.nvmlDeviceGetHandleByIndex(0)


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = []
    s.record()
    for _ in range(reps):
        fn()
        clk.append(pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM))
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps, sorted(clk)[len(clk) // 2]


out = []
for B, H, HKV, N, D, causal in ((16, 16, 16, 4096, 128, True), (16, 16, 16, 4096, 128, False),
                                (16, 32, 8, 4096, 128, True), (4, 16, 16, 16384, 128, True),
                                (16, 16, 16, 4096, 64, True)):
    q = torch.empty(B, H, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1)
    k = torch.empty(B, HKV, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1)
    v = torch.empty_like(k).uniform_(-1, 1)
    ang = torch.rand(N, D // 2, device="cuda", dtype=torch.float32)
    sin, cos = ang.sin().contiguous(), ang.cos().contiguous()
    o = torch.empty_like(q)
    lse = torch.empty(B, H, N, device="cuda")
    fl = 4.0 * B * H * N * N * D * (0.5 if causal else 1.0)
    plain = timed(lambda: A.attention_fwd(q, k, v, causal=causal, out=o, lse=lse))
    fused = timed(lambda: A.attention_fwd(q, k, v, causal=causal, out=o, lse=lse, rotary_tables=(sin, cos)))

    def two():
        qr, kr = A.rotary_qk(q, k, sin, cos)
        A.attention_fwd(qr, kr, v, causal=causal, out=o, lse=lse)
    sep = timed(two)
    r = {"shape": f"B{B} H{H} Hkv{HKV} N{N} D{D} causal={int(causal)}"}
    for name, (ms, mhz) in (("no_rotary", plain), ("fused", fused), ("two_launch", sep)):
        r[name] = {"ms": round(ms, 4), "tflops": round(fl / ms / 1e9, 1), "sm_mhz": mhz,
                   "tflops_per_ghz": round(fl / ms / 1e9 / (mhz / 1e3), 1)}
    r["fused_cost_pct"] = round(100 * (r["no_rotary"]["tflops_per_ghz"] / r["fused"]["tflops_per_ghz"] - 1), 2)
    r["two_launch_cost_pct"] = round(100 * (r["no_rotary"]["tflops_per_ghz"] / r["two_launch"]["tflops_per_ghz"] - 1), 2)
    print(json.dumps(r), flush=True)
    out.append(r)
    del q, k, v, o, lse
    torch.cuda.empty_cache()
