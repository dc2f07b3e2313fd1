"""Grouped-query / multi-query attention on the B200.

The reference has no GQA; parity is anchored on the multi-head oracle
(oracle/attn_oracle.cpp) through the defining identity: GQA with Hkv kv heads equals
multi-head attention with each kv head repeated H / Hkv times, and dK/dV of a kv head
are the sums of the repeated heads' gradients. Same bar as the MHA tests: bf16 outputs
within max-abs 2e-2 and rel-L2 1e-2, fp32 L within 1e-3.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2410_20399_b200 import attention as A

pytestmark = pytest.mark.gpu

MAX_ABS, REL_L2, L_ABS = 2e-2, 1e-2, 1e-3


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", torch.bfloat16)


def _inputs(seed, B, H, HKV, N, D):
    q = orc.fill(seed, B * H * N * D).reshape(B, H, N, D)
    k = orc.fill(seed + 1, B * HKV * N * D).reshape(B, HKV, N, D)
    v = orc.fill(seed + 2, B * HKV * N * D).reshape(B, HKV, N, D)
    do = orc.fill(seed + 3, B * H * N * D).reshape(B, H, N, D)
    return q, k, v, do


def _close(name, got, ref):
    assert np.isfinite(got).all(), name
    ma, rl = orc.max_abs(got, ref), orc.rel_l2(got, ref)
    assert ma <= MAX_ABS and rl <= REL_L2, (name, ma, rl)


@pytest.mark.parametrize("H,HKV", [(8, 2), (8, 1), (4, 4)])
@pytest.mark.parametrize("D", [64, 128])
@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("N", [200, 512])
def test_gqa_fwd_bwd(cuda_dev, H, HKV, D, causal, N):
    B, g = 2, H // HKV
    q, k, v, do = _inputs(40 + H + HKV + D + N, B, H, HKV, N, D)
    qd, kd, vd, dod = (_dev(x) for x in (q, k, v, do))
    o, lse = A.attention_fwd(qd, kd, vd, causal=causal)
    dq, dk, dv = A.attention_bwd(qd, kd, vd, o, dod, lse, causal=causal)
    torch.cuda.synchronize()
    assert tuple(dk.shape) == (B, HKV, N, D) and tuple(dv.shape) == (B, HKV, N, D)
    # multi-head oracle on the repeated kv heads
    ke, ve = np.repeat(k, g, axis=1), np.repeat(v, g, axis=1)
    ro, rl = orc.attn_fwd(q.reshape(-1, N, D), ke.reshape(-1, N, D), ve.reshape(-1, N, D), causal=causal)
    rdq, rdk, rdv = orc.attn_bwd(q.reshape(-1, N, D), ke.reshape(-1, N, D), ve.reshape(-1, N, D),
                                 do.reshape(-1, N, D), causal=causal)
    _close("o", o.float().cpu().numpy().reshape(-1, N, D), ro)
    assert orc.max_abs(lse.cpu().numpy().reshape(-1, N), rl) <= L_ABS
    _close("dq", dq.float().cpu().numpy().reshape(-1, N, D), rdq)
    # dK/dV of a kv head = sum over its query-head group
    rdk = rdk.reshape(B, HKV, g, N, D).sum(axis=2)
    rdv = rdv.reshape(B, HKV, g, N, D).sum(axis=2)
    _close("dk", dk.float().cpu().numpy(), rdk)
    _close("dv", dv.float().cpu().numpy(), rdv)


def test_gqa_deterministic(cuda_dev):
    q, k, v, do = (_dev(x) for x in _inputs(7, 2, 8, 2, 640, 128))
    o, lse = A.attention_fwd(q, k, v, causal=True)
    r1 = A.attention_bwd(q, k, v, o, do, lse, causal=True)
    r2 = A.attention_bwd(q, k, v, o, do, lse, causal=True)
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(r1, r2))


def test_gqa_rejects_bad_group(cuda_dev):
    q, k, v, _ = (_dev(x) for x in _inputs(3, 1, 6, 4, 128, 64))
    with pytest.raises(A.ConfigError):
        A.attention_fwd(q, k, v)


def test_mqa_split_reduce_launches_and_determinism(cuda_dev):
    """Few kv heads: the dK/dV tasks split the query heads (fp32 partials + an ordered reduce
    launch: prep, dK/dV, reduce, dQ); results stay deterministic and match the oracle."""
    B, H, HKV, N, D = 1, 16, 1, 384, 128
    q, k, v, do = _inputs(11, B, H, HKV, N, D)
    qd, kd, vd, dod = (_dev(x) for x in (q, k, v, do))
    o, lse = A.attention_fwd(qd, kd, vd, causal=True)
    r1 = A.attention_bwd(qd, kd, vd, o, dod, lse, causal=True)
    assert A.last_launch_count() == 4
    r2 = A.attention_bwd(qd, kd, vd, o, dod, lse, causal=True)
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(r1, r2))
    ke, ve = np.repeat(k, H, axis=1), np.repeat(v, H, axis=1)
    rdq, rdk, rdv = orc.attn_bwd(q.reshape(-1, N, D), ke.reshape(-1, N, D), ve.reshape(-1, N, D),
                                 do.reshape(-1, N, D), causal=True)
    _close("dk", r1[1].float().cpu().numpy(), rdk.reshape(B, HKV, H, N, D).sum(axis=2))
    _close("dv", r1[2].float().cpu().numpy(), rdv.reshape(B, HKV, H, N, D).sum(axis=2))
