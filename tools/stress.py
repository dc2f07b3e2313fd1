"""Race / determinism stress: repeated fwd + bwd on several shapes, every output compared
bit for bit with the first run (the backward is deterministic by construction; a lost
barrier phase shows up as a mismatch, a hang as the 20-s mbarrier trap)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_20399_b200 import attention as A

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
shapes = [(2, 8, 2, 1000, 128, True), (4, 16, 16, 2048, 128, True), (3, 6, 3, 777, 64, False),
          (1, 32, 1, 4096, 128, True), (16, 16, 16, 512, 64, True), (2, 4, 4, 129, 128, False)]
t0 = time.time()
bad = 0
for (B, H, HKV, N, D, causal) in shapes:
    g = torch.Generator(device="cuda").manual_seed(N + D)
    q = torch.empty(B, H, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1, generator=g)
    k, v = (torch.empty(B, HKV, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1, generator=g) for _ in range(2))
    do = torch.empty_like(q).uniform_(-1, 1, generator=g)
    for pairs in ((False, True) if D == 128 else (False,)):
        A.set_bwd_pairs(pairs)
        ref = None
        for r in range(reps):
            o, lse = A.attention_fwd(q, k, v, causal=causal)
            outs = (o, lse) + A.attention_bwd(q, k, v, o, do, lse, causal=causal)
            if ref is None:
                ref = [x.clone() for x in outs]
            else:
                for name, a, b in zip(("o", "lse", "dq", "dk", "dv"), ref, outs):
                    if not torch.equal(a, b):
                        bad += 1
                        print("MISMATCH", (B, H, HKV, N, D, causal), "pairs" if pairs else "", name, "rep", r)
        A.set_bwd_pairs(False)
torch.cuda.synchronize()
print(f"stress: {len(shapes)} shapes x {reps} reps, {bad} mismatches, {time.time() - t0:.1f} s")
