"""Backward dK/dV on CTA pairs (tkb_set_bwd_pairs, D = 128) on the B200.

attn_bwd_dkdv2_kernel runs the four dK/dV GEMMs as tcgen05 cta_group::2 MMAs (M = 256)
over the kv blocks of a cluster of two CTAs. Same bar as test_attn_bwd_gpu.py: bf16
dQ/dK/dV within max-abs 2e-2 and rel-L2 1e-2 of the fp64 oracle. Shapes cover odd kv-block
counts (the grid is rounded up to an even count: the extra CTA's K/V rows are out of
bounds and its stores are clipped), ragged N, causal pairs whose first q block is fully
masked for the odd CTA, and grouped-query heads.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2410_20399_b200 import attention as A

pytestmark = pytest.mark.gpu

MAX_ABS, REL_L2 = 2e-2, 1e-2


@pytest.fixture
def pairs(cuda_dev):
    A.set_bwd_pairs(True)
    yield
    A.set_bwd_pairs(False)


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", torch.bfloat16)


def _close(name, got, ref):
    assert np.isfinite(got).all(), name
    ma, rl = orc.max_abs(got, ref), orc.rel_l2(got, ref)
    assert ma <= MAX_ABS and rl <= REL_L2, (name, ma, rl)


def _inputs(seed, B, H, HKV, N, D=128):
    q = orc.fill(seed, B * H * N * D).reshape(B, H, N, D)
    k = orc.fill(seed + 1, B * HKV * N * D).reshape(B, HKV, N, D)
    v = orc.fill(seed + 2, B * HKV * N * D).reshape(B, HKV, N, D)
    do = orc.fill(seed + 3, B * H * N * D).reshape(B, H, N, D)
    return q, k, v, do


def _check(q, k, v, do, causal):
    B, H, N, D = q.shape
    HKV = k.shape[1]
    g = H // HKV
    qd, kd, vd, dod = (_dev(x) for x in (q, k, v, do))
    o, lse = A.attention_fwd(qd, kd, vd, causal=causal)
    dq, dk, dv = A.attention_bwd(qd, kd, vd, o, dod, lse, causal=causal)
    torch.cuda.synchronize()
    ke, ve = np.repeat(k, g, axis=1), np.repeat(v, g, axis=1)
    rdq, rdk, rdv = orc.attn_bwd(q.reshape(-1, N, D), ke.reshape(-1, N, D), ve.reshape(-1, N, D),
                                 do.reshape(-1, N, D), causal=causal)
    _close("dq", dq.float().cpu().numpy().reshape(-1, N, D), rdq)
    _close("dk", dk.float().cpu().numpy().reshape(-1, N, D), rdk.reshape(B, HKV, g, N, D).sum(axis=2).reshape(-1, N, D))
    _close("dv", dv.float().cpu().numpy().reshape(-1, N, D), rdv.reshape(B, HKV, g, N, D).sum(axis=2).reshape(-1, N, D))


@pytest.mark.parametrize("N", [1, 100, 200, 384, 1000, 1024])
@pytest.mark.parametrize("causal", [False, True])
def test_pairs_mha(pairs, N, causal):
    _check(*_inputs(700 + N, 1, 2, 2, N), causal)


@pytest.mark.parametrize("H,HKV", [(8, 2), (8, 1)])
@pytest.mark.parametrize("causal", [False, True])
def test_pairs_gqa(pairs, H, HKV, causal):
    _check(*_inputs(900 + H + HKV, 2, H, HKV, 384), causal)


def test_pairs_match_single_cta(cuda_dev):
    # both dK/dV kernels accumulate in the same order: the outputs agree to bf16 rounding
    q, k, v, do = (_dev(x) for x in _inputs(11, 2, 4, 4, 2048))
    o, lse = A.attention_fwd(q, k, v, causal=True)
    one = A.attention_bwd(q, k, v, o, do, lse, causal=True)
    A.set_bwd_pairs(True)
    try:
        two = A.attention_bwd(q, k, v, o, do, lse, causal=True)
        again = A.attention_bwd(q, k, v, o, do, lse, causal=True)
    finally:
        A.set_bwd_pairs(False)
    torch.cuda.synchronize()
    for a, b, c in zip(one, two, again):
        assert torch.equal(b, c)  # deterministic
        assert (a.float() - b.float()).abs().max().item() <= 1e-2
