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
every = int(os.environ.get("TRACE_EVERY", (B * H * ((N + 127) // 128)) // slots))
A.attention_bwd(q, k, v, o, do, lse, causal=bool(causal))
A.debug_set_trace(buf, every, slots)
A.attention_bwd(q, k, v, o, do, lse, causal=bool(causal))
torch.cuda.synchronize()
A.debug_set_trace(None)
t = buf.cpu()
names = {0: ["kv.m.top", "kv.m.dVissued", "kv.m.Sissued", "kv.m.dKissued", "kv.m.end"],
         1: ["kv.c.sfull", "kv.c.Pdone", "kv.c.dpfull", "kv.c.dSdone"],
         2: ["q.m.dswait", "q.m.dsfull", "q.m.end"], 3: ["q.c.sfull", "q.c.dpfull", "q.c.dSdone"]}
for slot in (1, 4):
    print(f"--- slot {slot} (item {slot * every})")
    for roles in ((0, 1), (2, 3)):
      for it in range(8, 11):
        ev = []
        for role in roles:
            for e, nm in enumerate(names[role]):
                val = int(t[slot, role, it, e])
                if val:
                    ev.append((val, nm))
        ev.sort()
        base = ev[0][0] if ev else 0
        print(f"iter {it}: " + "  ".join(f"{nm}+{v - base}" for v, nm in ev))
    for role, ev_i, nm in ((0, 4, "dkdv"), (2, 2, "dq")):
        st = [int(t[slot, role, i, ev_i]) for i in range(32) if int(t[slot, role, i, ev_i])]
        if len(st) > 4:
            d = [b - a for a, b in zip(st, st[1:])]
            print(f"{nm} iteration period (cycles):", d[2:12])

# CTA timeline: first S^T ready, last step, finish (cycles from CTA start)
for slot in range(slots):
    first = int(t[slot, 1, 0, 0])
    fin = int(t[slot, 1, 31, 7])
    last = max(int(t[slot, 1, it, 3]) for it in range(31))
    if first or fin:
        print(f"slot {slot}: first s_full {first}, last traced dS {last}, finish {fin}")

# persistent dK/dV finish per task n (role 1 events 4-7: dkv_full, dV stored, dK stored, next task's first S)
for slot in range(min(slots, 2)):
    for n in range(1, 6):
        e = [int(t[slot, 1, n, i]) for i in (4, 5, 6, 7)]
        l5, l6 = int(t[slot, 0, n, 5]), int(t[slot, 0, n, 6])
        if e[0]:
            print(f"slot {slot} task {n}: dkv_full {e[0]}  +dV read {l5 - e[0] if l5 else -1}  +dV stored {e[1] - e[0]}"
                  f"  +dK read {l6 - e[0] if l6 else -1}  +dK stored {e[2] - e[0]}  +next S {e[3] - e[0] if e[3] else -1}")
