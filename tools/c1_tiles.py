"""BASELINE configs[0] (B1 H8 N1024 D64 non-causal forward) and a few other small problems:
microseconds per forward with one- vs two-tile tasks (tkb_debug_set_fwd_task_tiles), CUDA
events around each call with a 256 MB L2 scrub in between (inputs cold, as in bench.py's C1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_20399_b200 import attention as A  # noqa: E402

scrub = torch.empty(64 << 20, device="cuda", dtype=torch.float32)
for B, H, N, D, causal in ((1, 8, 1024, 64, False), (1, 8, 1024, 128, True), (1, 16, 2048, 128, True),
                           (2, 8, 512, 64, True), (1, 32, 1024, 128, False)):
    q, k, v = (torch.empty(B, H, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1) for _ in range(3))
    o, lse = A.attention_fwd(q, k, v, causal=causal)
    res = {}
    for tiles in (2, 1, 0):
        A.debug_set_fwd_task_tiles(tiles)
        ts = []
        for it in range(60):
            scrub.fill_(1.0)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            A.attention_fwd(q, k, v, causal=causal, out=o, lse=lse)
            e.record()
            torch.cuda.synchronize()
            if it >= 10:
                ts.append(s.elapsed_time(e) * 1e3)
        ts.sort()
        res[tiles] = ts[len(ts) // 2]
    A.debug_set_fwd_task_tiles(0)
    print(f"B{B} H{H} N{N} D{D} causal={int(causal)}: two-tile {res[2]:.1f} us, one-tile {res[1]:.1f} us, "
          f"auto {res[0]:.1f} us", flush=True)
