"""Seeded random-shape parity sweep on the B200: forward O / L and backward dQ / dK / dV
against the fp64 oracle over shapes the fixed tests do not pin — arbitrary ragged N,
B / H / Hkv combinations (MHA, GQA, MQA), D 64 / 128, causal or not, contiguous [B,H,N,D]
or [B,N,H,D] storage. Same bar as the other parity tests: bf16 outputs max-abs 2e-2 and
rel-L2 1e-2, fp32 L max-abs 1e-3.
"""
import random

import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2410_20399_b200 import attention as A

pytestmark = pytest.mark.gpu

MAX_ABS, REL_L2, L_ABS = 2e-2, 1e-2, 1e-3


def _case(seed):
    r = random.Random(seed)
    hkv = r.choice([1, 2, 3])
    h = hkv * r.choice([1, 2, 4])
    return dict(B=r.choice([1, 2, 3]), H=h, HKV=hkv, N=r.choice([1, 2, 63, 127, 129, 255, 257, 500, 777, 1024, 1311]),
                D=r.choice([64, 128]), causal=r.random() < 0.5, bnhd=r.random() < 0.3)


CASES = [_case(s) for s in range(48)]


@pytest.mark.parametrize("c", CASES, ids=[f"B{c['B']}H{c['H']}kv{c['HKV']}N{c['N']}D{c['D']}"
                                            f"{'c' if c['causal'] else 'n'}{'T' if c['bnhd'] else ''}" for c in CASES])
def test_fuzz_fwd_bwd(cuda_dev, c):
    B, H, HKV, N, D, causal = c["B"], c["H"], c["HKV"], c["N"], c["D"], c["causal"]
    seed = 1000 + N * 7 + D + H * 13 + HKV
    q = orc.fill(seed, B * H * N * D).reshape(B, H, N, D)
    k = orc.fill(seed + 1, B * HKV * N * D).reshape(B, HKV, N, D)
    v = orc.fill(seed + 2, B * HKV * N * D).reshape(B, HKV, N, D)
    do = orc.fill(seed + 3, B * H * N * D).reshape(B, H, N, D)

    def dev(x):
        t = torch.from_numpy(np.ascontiguousarray(x)).to("cuda", torch.bfloat16)
        return t.transpose(1, 2).contiguous().transpose(1, 2) if c["bnhd"] else t

    qd, kd, vd, dod = (dev(x) for x in (q, k, v, do))
    o, lse = A.attention_fwd(qd, kd, vd, causal=causal)
    dq, dk, dv = A.attention_bwd(qd, kd, vd, o, dod, lse, causal=causal)
    torch.cuda.synchronize()
    if D == 128:  # the opt-in CTA-pair dK/dV kernel on the same inputs
        A.set_bwd_pairs(True)
        try:
            _, dk2, dv2 = A.attention_bwd(qd, kd, vd, o, dod, lse, causal=causal)
            torch.cuda.synchronize()
        finally:
            A.set_bwd_pairs(False)
        assert (dk2.float() - dk.float()).abs().max().item() <= 1e-2
        assert (dv2.float() - dv.float()).abs().max().item() <= 1e-2
    g = H // HKV
    ke, ve = np.repeat(k, g, axis=1).reshape(-1, N, D), np.repeat(v, g, axis=1).reshape(-1, N, D)
    ro, rl = orc.attn_fwd(q.reshape(-1, N, D), ke, ve, causal=causal)
    rdq, rdk, rdv = orc.attn_bwd(q.reshape(-1, N, D), ke, ve, do.reshape(-1, N, D), causal=causal)
    rdk = rdk.reshape(B, HKV, g, N, D).sum(axis=2).reshape(-1, N, D)
    rdv = rdv.reshape(B, HKV, g, N, D).sum(axis=2).reshape(-1, N, D)
    for name, got, ref in (("o", o, ro), ("dq", dq, rdq), ("dk", dk, rdk), ("dv", dv, rdv)):
        got = got.float().cpu().numpy().reshape(-1, N, D)
        assert np.isfinite(got).all(), name
        ma, rl2 = orc.max_abs(got, ref), orc.rel_l2(got, ref)
        assert ma <= MAX_ABS and rl2 <= REL_L2, (name, ma, rl2)
    assert orc.max_abs(lse.cpu().numpy().reshape(-1, N), rl) <= L_ABS
