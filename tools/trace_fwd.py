"""Per-task cycle timeline of the persistent forward (debug build, TKB_FWD_TRACE=1 via
TKB_LIB_PATH): for a few CTAs, each task's load / MMA / softmax events relative to the
CTA's first stamp. Usage: TKB_LIB_PATH=build/libtkb_ftrace.so python tools/trace_fwd.py B,H,N,D,causal"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_20399_b200 import attention as A  # noqa: E402

B, H, N, D, causal = map(int, (sys.argv[1] if len(sys.argv) > 1 else "64,16,1024,128,1").split(","))
q, k, v = (torch.empty(B, H, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1) for _ in range(3))
for _ in range(3):
    A.attention_fwd(q, k, v, causal=bool(causal))
slots = 4
buf = torch.zeros(slots, 4, 32, 8, dtype=torch.int64, device="cuda")
A.debug_set_trace(buf, 37, slots)  # CTAs 0, 37, 74, 111
A.attention_fwd(q, k, v, causal=bool(causal))
torch.cuda.synchronize()
A.debug_set_trace(None)
t = buf.cpu()
names = {0: ["L.start", "L.Qissued", "L.claimed", "L.lastKV"], 1: ["M.start", "M.firstQK", "M.end", "M.q0full", "M.k0full"],
         2: ["S0.start", "S0.firstS", "S0.loopEnd", "S0.oFull", "S0.finEnd", "S0.enter"],
         3: ["S1.start", "S1.firstS", "S1.loopEnd", "S1.oFull", "S1.finEnd", "S1.enter"]}
for slot in range(slots):
    base = int(t[slot][t[slot] > 0].min()) if (t[slot] > 0).any() else 0
    print(f"=== CTA {slot * 37}")
    for n in range(32):
        row = []
        for role in range(4):
            for e, nm in enumerate(names[role]):
                val = int(t[slot, role, n, e])
                if val:
                    row.append(f"{nm}={val - base}")
        if row:
            print(f"task {n:2d}: " + " ".join(row))
