"""dQ kernel step periods from the backward's cycle trace (debug knob tkb_debug_set_trace):
consecutive s_full stamps of the compute warps; task boundaries show as longer gaps."""
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
A.debug_set_bwd_phases(5)  # prep + dQ
A.attention_bwd(q, k, v, o, do, lse, causal=bool(causal))
torch.cuda.synchronize()
A.debug_set_trace(None)
A.debug_set_bwd_phases(7)
t = buf.cpu()
for slot in range(slots):
    sf = [int(t[slot, 3, i, 0]) for i in range(32)]
    ds = [int(t[slot, 3, i, 2]) for i in range(32)]
    print(f"=== CTA {slot * 37}: s_full deltas", [b - a for a, b in zip(sf, sf[1:]) if a and b])
    print("   dS-done -> next s_full", [b - a for a, b in zip(ds, sf[1:]) if a and b])

for slot in range(slots):
    for n in range(1, 8):
        e = [int(t[slot, 3, n, i]) for i in (3, 4, 5, 6, 7)]
        if e[0]:
            print(f"CTA {slot * 37} task {n}: finish start, +stage_a {e[1] - e[0]}, +dq_full {e[2] - e[0]}, "
                  f"+staged {e[3] - e[0]}, +stored {e[4] - e[0] if e[4] else -1}")
