"""Per-role cycle timeline of the persistent forward kernel (debug build with -DTKB_FWD_TRACE).

  TKB_LIB_PATH=build/libtkb_trace.so python tools/trace_fwd.py B,H,N,D,causal
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_20399_b200 import attention as A

B, H, N, D, causal = map(int, (sys.argv[1] if len(sys.argv) > 1 else "16,16,4096,128,0").split(","))
off = int(sys.argv[2]) if len(sys.argv) > 2 else 0
first = int(sys.argv[3]) if len(sys.argv) > 3 else 6
count = int(sys.argv[4]) if len(sys.argv) > 4 else 4
q, k, v = (torch.empty(B, H, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1) for _ in range(3))
slots = 4
buf = torch.zeros(slots, 4, 32, 8, dtype=torch.int64, device="cuda")
A.attention_fwd(q, k, v, causal=bool(causal))
A.debug_set_trace(buf, 37, slots | (off << 16))
A.attention_fwd(q, k, v, causal=bool(causal))
torch.cuda.synchronize()
A.debug_set_trace(None)
t = buf.cpu()
names = {0: ["m.iter", "m.p0ok", "m.p1ok", "m.pv0", "m.qk0", "m.pv1", "m.qk1"],
         1: ["s0.sfull", "s0.stat", "s0.parr", "s0.ld", "s0.exp"], 2: ["s1.sfull", "s1.stat", "s1.parr", "s1.ld", "s1.exp"],
         3: ["c.st0", "c.p0", "c.st1", "c.p1"]}
for slot in (0,):
    print(f"--- CTA {slot * 37}")
    prev = None
    for it in range(first, first + count):
        ev = []
        for role, nm in names.items():
            for e, n in enumerate(nm):
                val = int(t[slot, role, it, e])
                if val:
                    ev.append((val, n))
        ev.sort()
        if not ev:
            continue
        base = ev[0][0]
        print(f"iter {it + off:2d} (+{base - prev if prev else 0:5d}): " + "  ".join(f"{n}+{v - base}" for v, n in ev))
        prev = base
