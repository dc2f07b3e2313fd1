"""Per-role cycle timeline of the backward kernel (debug): prints steady-state iterations."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_20399_b200 import attention as A

B, H, N, D, causal = map(int, (sys.argv[1] if len(sys.argv) > 1 else "16,16,4096,128,0").split(","))
q, k, v, do = (torch.randn(B, H, N, D, device="cuda", dtype=torch.bfloat16) for _ in range(4))
o, lse = A.attention_fwd(q, k, v, causal=bool(causal))
slots = 8
buf = torch.zeros(slots, 4, 32, 8, dtype=torch.int64, device="cuda")
every = (B * H * ((N + 127) // 128)) // slots
A.attention_bwd(q, k, v, o, do, lse, causal=bool(causal))
A.debug_set_trace(buf, every, slots)
A.attention_bwd(q, k, v, o, do, lse, causal=bool(causal))
torch.cuda.synchronize()
A.debug_set_trace(None)
t = buf.cpu()
names = {0: ["m.qwait", "m.S", "m.dsfull", "m.dQ", "m.dofull", "m.dqempty", "m.pfull", "m.dV"],
         1: ["c.sfull", "c.Pdone", "c.dpfull", "c.dSdone"], 2: ["r.dqfull", "r.empty", "i.start", "i.issued"],
         3: ["T.S", "T.dK", "T.dQ", "T.dP", "T.dV"]}
for slot in (1, 4):
    print(f"--- slot {slot} (item {slot * every})")
    for it in range(8, 12):
        ev = []
        for role in range(4):
            for e, nm in enumerate(names[role]):
                val = int(t[slot, role, it, e])
                if val:
                    ev.append((val, nm))
        ev.sort()
        base = ev[0][0] if ev else 0
        print(f"iter {it}: " + "  ".join(f"{nm}+{v - base}" for v, nm in ev))
    # average iteration period from m.S stamps
    s_stamps = [int(t[slot, 0, i, 1]) for i in range(32) if int(t[slot, 0, i, 1])]
    if len(s_stamps) > 4:
        d = [b - a for a, b in zip(s_stamps, s_stamps[1:])]
        print("iteration period (cycles):", d[2:12])
