"""A/B timing of the forward (optionally with the fused rotary prologue) for variant libraries
(TKB_LIB_PATH): each call repeated for ~SECS seconds, mean ms per call and the mean SM clock."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml  # noqa: E402
import torch  # noqa: E402

from paper_2410_20399_b200 import attention as A  # noqa: E402

B, H, HKV, N, D, causal, rope = map(int, (sys.argv[1] if len(sys.argv) > 1 else "16,16,16,4096,128,1,1").split(","))
SECS = float(os.environ.get("SECS", "2"))
q = torch.empty(B, H, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1)
k = torch.empty(B, HKV, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1)
v = torch.empty_like(k).uniform_(-1, 1)
ang = torch.rand(N, D // 2, device="cuda")
tabs = (ang.sin().contiguous(), ang.cos().contiguous())
o = torch.empty_like(q)
lse = torch.empty(B, H, N, device="cuda")
if rope == 2:  # the two-launch path: tkb_rotary_qk, then tkb_attn_fwd
    def fn():
        qr, kr = A.rotary_qk(q, k, *tabs)
        A.attention_fwd(qr, kr, v, causal=bool(causal), out=o, lse=lse)
elif rope == 1:  # fused: tkb_attn_fwd_rotary
    def fn():
        A.attention_fwd(q, k, v, causal=bool(causal), out=o, lse=lse, rotary_tables=tabs)
else:
    def fn():
        A.attention_fwd(q, k, v, causal=bool(causal), out=o, lse=lse)
for _ in range(5):
    fn()
torch.cuda.synchronize()
pynvml.nvmlInit()
hd = pynvml.nvmlDeviceGetHandleByIndex(0)
clk, stop = [], [False]


def sample():
    while not stop[0]:
        clk.append(pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM))
        time.sleep(0.02)


th = threading.Thread(target=sample)
th.start()
n, t0 = 0, time.time()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
while time.time() - t0 < SECS:
    for _ in range(10):
        fn()
    n += 10
    torch.cuda.synchronize()
e.record()
torch.cuda.synchronize()
stop[0] = True
th.join()
ms = s.elapsed_time(e) / n
mhz = sum(clk) / max(1, len(clk))
fl = 4.0 * B * H * N * N * D * (0.5 if causal else 1.0)
print(f"{os.path.basename(os.environ.get('TKB_LIB_PATH', 'libtkb.so'))} rope={rope} causal={causal}: {ms:.4f} ms "
      f"{fl / ms / 1e9:.0f} TFLOPS at {mhz:.0f} MHz = {fl / ms / 1e9 / mhz * 1e3:.1f} TFLOPS/GHz")
