"""Probe which call breaks CUDA-graph capture of the attention calls."""
import ctypes
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2410_20399_b200 import attention as A  # noqa: E402

B, H, N, D = 2, 4, 1024, 128
q, k, v, do = (torch.empty((B, H, N, D), device="cuda", dtype=torch.bfloat16).uniform_(-1, 1) for _ in range(4))
A.device_init(0)
o, lse = torch.empty_like(q), torch.empty((B, H, N), dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    A.attention_fwd(q, k, v, causal=True, out=o, lse=lse)
torch.cuda.synchronize()
for mode in ("relaxed", "thread_local", "global"):
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g, stream=s, capture_error_mode=mode):
            try:
                A.attention_fwd(q, k, v, causal=True, out=o, lse=lse)
            except Exception as e:  # noqa: BLE001
                print(mode, "call raised", e)
        g.replay()
        torch.cuda.synchronize()
        print(mode, "ok")
    except Exception as e:  # noqa: BLE001
        print(mode, "capture failed:", str(e).splitlines()[0], "| tkb:", A.lib().tkb_last_error())
        break
