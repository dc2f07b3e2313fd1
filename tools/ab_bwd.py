"""A/B of the backward for variant libraries (TKB_LIB_PATH): per shape, the dK/dV kernel alone
(debug phase mask 2), the dQ kernel alone (4) and the whole backward, CUDA events over many calls,
with the median SM clock (NVML) of the whole-backward loop."""
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml  # noqa: E402
import torch  # noqa: E402

from paper_2410_20399_b200 import attention as A  # noqa: E402

shapes = (sys.argv[1] if len(sys.argv) > 1 else "16,16,4096,128,1;16,16,4096,128,0;64,16,1024,128,1").split(";")
pynvml.nvmlInit()
hd = pynvml.nvmlDeviceGetHandleByIndex(0)


def timed(fn, iters):
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


for sh in shapes:
    B, H, N, D, causal = map(int, sh.split(","))
    q, k, v, do = (torch.empty(B, H, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1) for _ in range(4))
    o, lse = A.attention_fwd(q, k, v, causal=bool(causal))
    dq, dk, dv = (torch.empty_like(q) for _ in range(3))
    ws = torch.empty(A.bwd_workspace_bytes(B, H, N, D), dtype=torch.uint8, device="cuda")
    f = lambda: A.attention_bwd(q, k, v, o, do, lse, causal=bool(causal), dq=dq, dk=dk, dv=dv, workspace=ws)  # noqa
    f()
    res = {}
    for name, mask in (("dkdv", 2), ("dq", 4)):
        A.debug_set_bwd_phases(1)
        f()
        A.debug_set_bwd_phases(mask)
        res[name] = timed(f, 20)
        A.debug_set_bwd_phases(7)
    clk, stop = [], [False]

    def sample():
        while not stop[0]:
            clk.append(pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM))
            time.sleep(0.01)

    th = threading.Thread(target=sample)
    th.start()
    res["bwd"] = timed(f, max(10, int(2000 / max(res["dkdv"] + res["dq"], 0.05) / 10)))
    stop[0] = True
    th.join()
    mhz = statistics.median(clk) if clk else 0
    fl = 10.0 * B * H * N * N * D * (0.5 if causal else 1.0)
    print(f"{os.path.basename(os.environ.get('TKB_LIB_PATH', 'libtkb.so'))} B{B} H{H} N{N} D{D} c{causal}: "
          f"dkdv {res['dkdv']:.3f} ms  dq {res['dq']:.3f} ms  bwd {res['bwd']:.3f} ms = {fl / res['bwd'] / 1e9:.0f} "
          f"TFLOPS at {mhz:.0f} MHz ({fl / res['bwd'] / 1e9 / mhz * 1e3:.1f} TFLOPS/GHz)", flush=True)
