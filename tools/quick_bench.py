"""Quick kernel timing (CUDA events) of the fwd/bwd kernels at a few shapes."""
import argparse
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_20399_b200 import attention as A

def t_events(fn, iters=20, warmup=5):
    for _ in range(warmup): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for _ in range(iters):
        s.record(); fn(); e.record(); torch.cuda.synchronize(); times.append(s.elapsed_time(e))
    times.sort()
    return times[len(times)//2]

def t_soak(fn, secs):
    """Repeat fn for ~secs seconds; returns (ms per call, median SM clock MHz sampled by NVML
    every 5 ms during the loop). TFLOPS / GHz is then comparable across power-cap states."""
    import threading, statistics, time
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    for _ in range(3): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
    n = max(3, int(secs / max(time.perf_counter() - t0, 1e-4)))
    clocks, stop = [], threading.Event()
    def sample():
        while not stop.is_set():
            clocks.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            time.sleep(0.005)
    th = threading.Thread(target=sample); th.start()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize()
    stop.set(); th.join()
    return s.elapsed_time(e) / n, statistics.median(clocks[len(clocks) // 5:] or clocks)


ap = argparse.ArgumentParser()
ap.add_argument("--bwd", action="store_true")
ap.add_argument("--sdpa", action="store_true")
ap.add_argument("--uniform", action="store_true", help="U(-1,1) inputs (bench.py data) instead of randn")
ap.add_argument("--no-causal", action="store_true")
ap.add_argument("--only-causal", action="store_true")
ap.add_argument("--shapes", default="16,16,4096,128;16,16,4096,64;4,16,16384,128;16,16,1024,128")
ap.add_argument("--pairs", action="store_true", help="D=128 backward dK/dV on CTA pairs")
ap.add_argument("--soak", type=float, default=0.0, help="time each pass over ~SOAK s and report TFLOPS per GHz")
args = ap.parse_args()
if args.pairs:
    A.set_bwd_pairs(True)
for sh in args.shapes.split(";"):
    B, H, N, D = map(int, sh.split(","))
    if args.uniform:
        q, k, v = (torch.empty(B, H, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1) for _ in range(3))
    else:
        q, k, v = (torch.randn(B, H, N, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    for causal in ((False,) if args.no_causal else (True,) if args.only_causal else (False, True)):
        o, lse = A.attention_fwd(q, k, v, causal=causal)
        fwd = lambda: A.attention_fwd(q, k, v, causal=causal, out=o, lse=lse)  # noqa
        fl = 4 * B * H * N * N * D * (0.5 if causal else 1.0)
        if args.soak > 0:
            ms, mhz = t_soak(fwd, args.soak)
            print(f"fwd B{B} H{H} N{N} D{D} causal={int(causal)}: {ms*1e3:8.1f} us  {fl/ms/1e9:7.1f} TFLOPS"
                  f" at {mhz:.0f} MHz = {fl/ms/1e9/(mhz/1e3):6.1f} TFLOPS/GHz", flush=True)
        else:
            ms = t_events(fwd)
        line = f"fwd B{B} H{H} N{N} D{D} causal={int(causal)}: {ms*1e3:8.1f} us  {fl/ms/1e9:7.1f} TFLOPS"
        try:
            if not args.sdpa: raise RuntimeError("skipped")
            ref = t_events(lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=causal))
            line += f"   | torch sdpa {fl/ref/1e9:7.1f} TFLOPS"
        except Exception as ex:
            line += f"   | sdpa err {ex}"
        if args.soak <= 0:
            print(line, flush=True)
        if args.bwd:
            do = torch.randn_like(q)
            ws = torch.empty(A.bwd_workspace_bytes(B, H, N, D), dtype=torch.uint8, device="cuda")
            dq, dk, dv = A.attention_bwd(q, k, v, o, do, lse, causal=causal, workspace=ws)
            bwd = lambda: A.attention_bwd(q, k, v, o, do, lse, causal=causal, dq=dq, dk=dk, dv=dv, workspace=ws)  # noqa
            fl = 10 * B * H * N * N * D * (0.5 if causal else 1.0)
            if args.soak > 0:
                ms, mhz = t_soak(bwd, args.soak)
                print(f"bwd B{B} H{H} N{N} D{D} causal={int(causal)}: {ms*1e3:8.1f} us  {fl/ms/1e9:7.1f} TFLOPS"
                      f" at {mhz:.0f} MHz = {fl/ms/1e9/(mhz/1e3):6.1f} TFLOPS/GHz", flush=True)
                continue
            ms = t_events(bwd)
            line = f"bwd B{B} H{H} N{N} D{D} causal={int(causal)}: {ms*1e3:8.1f} us  {fl/ms/1e9:7.1f} TFLOPS"
            try:
                if not args.sdpa: raise RuntimeError("skipped")
                qr, kr, vr = (x.detach().clone().requires_grad_() for x in (q, k, v))
                out = torch.nn.functional.scaled_dot_product_attention(qr, kr, vr, is_causal=causal)
                ref = t_events(lambda: torch.autograd.grad(out, (qr, kr, vr), do, retain_graph=True))
                line += f"   | torch sdpa bwd {fl/ref/1e9:7.1f} TFLOPS"
            except Exception as ex:
                line += f"   | sdpa bwd err {ex}"
            print(line, flush=True)
