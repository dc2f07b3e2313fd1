"""Per-step cycle timeline of the persistent backward kernels (debug build knob
tkb_debug_set_trace): for one traced CTA, the MMA-warp and compute-warp event stamps of
the first 32 steps, and the step periods."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_20399_b200 import attention as A  # noqa: E402

B, H, N, D, causal = map(int, (sys.argv[1] if len(sys.argv) > 1 else "16,16,4096,128,1").split(","))
q, k, v, do = (torch.empty(B, H, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1) for _ in range(4))
o, lse = A.attention_fwd(q, k, v, causal=bool(causal))
A.set_bwd_pairs(bool(int(os.environ.get("PAIRS", "0"))))
slots = 4
buf = torch.zeros(slots, 4, 32, 8, dtype=torch.int64, device="cuda")
A.attention_bwd(q, k, v, o, do, lse, causal=bool(causal))
A.debug_set_trace(buf, 37, slots)  # CTAs 0, 37, 74, 111
A.attention_bwd(q, k, v, o, do, lse, causal=bool(causal))
torch.cuda.synchronize()
A.debug_set_trace(None)
t = buf.cpu()
names = {0: ["m.top", "m.dVissued", "m.Sissued", "m.dKissued", "m.end"],
         1: ["c.sfull", "c.Pdone", "c.dpfull", "c.dSdone"],
         2: ["m.dswait", "m.dsfull", "m.end"], 3: ["c.sfull", "c.dpfull", "c.dSdone"]}
for kern, (rm, rc, last) in (("dkdv", (0, 1, 4)), ("dq", (2, 3, 2))):
    print(f"===== {kern}")
    for slot in range(2):
        ends = [int(t[slot, rm, i, last]) for i in range(32)]
        per = [b - a for a, b in zip(ends, ends[1:]) if a and b]
        print(f"slot {slot} step periods:", per)
        for it in range(10, 14):
            ev = []
            for role in (rm, rc):
                for e, nm in enumerate(names[role]):
                    val = int(t[slot, role, it, e])
                    if val:
                        ev.append((val, nm))
            ev.sort()
            base = ev[0][0] if ev else 0
            print(f"  step {it}: " + "  ".join(f"{nm}+{v - base}" for v, nm in ev))
