"""dK/dV task boundaries in the backward's cycle trace (debug knob tkb_debug_set_trace): per
traced CTA, the step periods (MMA warp top-of-step stamps) and where each task's finish sits."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_20399_b200 import attention as A  # noqa: E402

B, H, N, D, causal = map(int, (sys.argv[1] if len(sys.argv) > 1 else "16,16,4096,128,1").split(","))
q, k, v, do = (torch.empty(B, H, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1) for _ in range(4))
o, lse = A.attention_fwd(q, k, v, causal=bool(causal))
A.attention_bwd(q, k, v, o, do, lse, causal=bool(causal))
slots = 4
buf = torch.zeros(slots, 4, 32, 8, dtype=torch.int64, device="cuda")
A.debug_set_trace(buf, 37, slots)
A.debug_set_bwd_phases(3)
A.attention_bwd(q, k, v, o, do, lse, causal=bool(causal))
torch.cuda.synchronize()
A.debug_set_trace(None)
A.debug_set_bwd_phases(7)
t = buf.cpu()
for slot in range(slots):
    tops = [int(t[slot, 0, x, 0]) for x in range(32)]
    sfull = [int(t[slot, 1, x, 0]) for x in range(32)]
    dsd = [int(t[slot, 1, x, 3]) for x in range(32)]
    print(f"=== CTA {slot * 37}")
    print("step top deltas:", [b - a for a, b in zip(tops, tops[1:]) if a and b])
    for n in range(6):
        dkv, fin, nxt = int(t[slot, 1, n, 4]), int(t[slot, 1, n, 6]), int(t[slot, 1, n, 7])
        if dkv:
            print(f"task {n}: dkv_full {dkv}  finish end +{fin - dkv}  next task's first S +{nxt - dkv if nxt else -1}")
    print("s_full:", sfull[:20])
    print("dS done:", dsd[:20])
