"""dK/dV single-CTA vs CTA-pair kernel (tkb_set_bwd_pairs) at a few shapes: the dK/dV kernel
alone (debug phase mask 2), CUDA events, TFLOPS/GHz under the power cap."""
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml  # noqa: E402
import torch  # noqa: E402

from paper_2410_20399_b200 import attention as A  # noqa: E402

pynvml.nvmlInit()
hd = pynvml.nvmlDeviceGetHandleByIndex(0)
for sh in (sys.argv[1] if len(sys.argv) > 1 else "16,16,4096,128,1;16,16,4096,128,0;8,16,8192,128,1").split(";"):
    B, H, N, D, causal = map(int, sh.split(","))
    q, k, v, do = (torch.empty(B, H, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1) for _ in range(4))
    o, lse = A.attention_fwd(q, k, v, causal=bool(causal))
    dq, dk, dv = (torch.empty_like(q) for _ in range(3))
    ws = torch.empty(A.bwd_workspace_bytes(B, H, N, D), dtype=torch.uint8, device="cuda")
    f = lambda: A.attention_bwd(q, k, v, o, do, lse, causal=bool(causal), dq=dq, dk=dk, dv=dv, workspace=ws)  # noqa
    for pairs in (0, 1, 0, 1):
        A.set_bwd_pairs(bool(pairs))
        A.debug_set_bwd_phases(7)
        f()
        A.debug_set_bwd_phases(2)
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        clk, stop = [], [False]

        def sample():
            while not stop[0]:
                clk.append(pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM))
                time.sleep(0.01)

        th = threading.Thread(target=sample)
        th.start()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(30):
            f()
        e.record()
        torch.cuda.synchronize()
        stop[0] = True
        th.join()
        ms = s.elapsed_time(e) / 30
        mhz = statistics.median(clk)
        fl = 8.0 * B * H * N * N * D * (0.5 if causal else 1.0)
        print(f"pairs={pairs} B{B} H{H} N{N} D{D} c{causal}: dkdv {ms:.3f} ms {fl / ms / 1e9:.0f} TFLOPS at {mhz:.0f} MHz "
              f"({fl / ms / 1e9 / mhz * 1e3:.1f} /GHz)", flush=True)
    A.debug_set_bwd_phases(7)
    A.set_bwd_pairs(False)
