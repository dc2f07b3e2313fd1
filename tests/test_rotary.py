"""Rotary embedding: oracle pinned to the reference on CPU, the
sm_100a kernel against the oracle on the GPU (tests mirror test_kernels.cpp:215-308)."""
import math

import numpy as np
import pytest
import torch

from oracle import oracle as orc


def _tables(seed, n, half, lo=-3.14159, hi=3.14159):
    a = orc.fill(seed, n * half, bf16=False, lo=lo, hi=hi).reshape(n, half)
    return np.sin(a).astype(np.float32), np.cos(a).astype(np.float32), a


# ------------------------------------------------------------------ CPU: oracle pinning
@pytest.mark.skipif(not orc.ref_available(), reason="oracle/_ref not built")
def test_oracle_rotary_matches_reference_oracle():
    x = orc.fill(11, 64 * 128, bf16=False).reshape(64, 128)
    s, c, _ = _tables(12, 64, 64)
    np.testing.assert_allclose(orc.rotary(x, s, c), orc.ref_rotary_oracle(x, s, c), rtol=0, atol=1e-12)


@pytest.mark.skipif(not orc.ref_available(), reason="oracle/_ref not built")
def test_reference_rotary_kernel_matches_oracle():
    # test_kernels.cpp:228-249: the reference kernel vs oracle_rotary within 1e-5
    x = orc.fill(13, 2 * 2 * 64 * 64, bf16=False).reshape(2, 2, 64, 64)
    s, c, _ = _tables(14, 64, 32)
    got = orc.ref_rotary(x, s, c)
    assert np.max(np.abs(got - orc.rotary(x, s, c))) <= 1e-5


def test_oracle_rotary_identity_and_norms():
    x = orc.fill(15, 32 * 64, bf16=False).reshape(32, 64)
    z = np.zeros((32, 32), np.float32)
    np.testing.assert_array_equal(orc.rotary(x, z, np.ones_like(z)), x.astype(np.float64))
    s, c, _ = _tables(16, 32, 32)
    o = orc.rotary(x, s, c)
    np.testing.assert_allclose(np.hypot(o[:, :32], o[:, 32:]), np.hypot(x[:, :32], x[:, 32:]), atol=1e-6)


# ------------------------------------------------------------------ GPU: kernel parity
def _dev(x, dt=torch.bfloat16):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dt)


@pytest.mark.gpu
@pytest.mark.parametrize("B,H,N,D", [(1, 1, 64, 128), (2, 3, 200, 64), (1, 2, 1000, 128), (2, 2, 17, 32)])
def test_rotary_matches_oracle(cuda_dev, B, H, N, D):
    from paper_2410_20399_b200 import attention as A

    x = orc.fill(20 + N, B * H * N * D).reshape(B, H, N, D)
    s, c, _ = _tables(21 + N, N, D // 2)
    got = A.rotary(_dev(x), _dev(s, torch.float32), _dev(c, torch.float32))
    torch.cuda.synchronize()
    ref = orc.rotary(x, s, c)
    # one bf16 rounding of the output: |err| <= |o| 2^-8
    err = np.abs(got.float().cpu().numpy() - ref)
    assert np.all(err <= np.abs(ref) * 2.0 ** -8 + 1e-6)


@pytest.mark.gpu
def test_rotary_identity_and_inplace(cuda_dev):
    from paper_2410_20399_b200 import attention as A

    x = _dev(orc.fill(30, 2 * 2 * 64 * 64).reshape(2, 2, 64, 64))
    zero = torch.zeros(64, 32, device="cuda")
    one = torch.ones(64, 32, device="cuda")
    y = x.clone()
    A.rotary(y, zero, one, out=y)  # in place, identity rotation: bit-exact
    torch.cuda.synchronize()
    assert torch.equal(x, y)


@pytest.mark.gpu
def test_rotary_composes_like_angles(cuda_dev):
    # test_kernels.cpp:251-285 (within the two bf16 roundings of the two-step path)
    from paper_2410_20399_b200 import attention as A

    x = orc.fill(40, 32 * 64).reshape(1, 1, 32, 64)
    a = orc.fill(41, 32 * 32, bf16=False).reshape(32, 32)
    b = orc.fill(42, 32 * 32, bf16=False).reshape(32, 32)
    t = lambda ang: (_dev(np.sin(ang), torch.float32), _dev(np.cos(ang), torch.float32))  # noqa: E731
    two = A.rotary(A.rotary(_dev(x), *t(a)), *t(b))
    one = A.rotary(_dev(x), *t(a + b))
    torch.cuda.synchronize()
    assert torch.max(torch.abs(two.float() - one.float())).item() <= 2 * 2.0 ** -8


@pytest.mark.gpu
@pytest.mark.parametrize("causal", [False, True])
def test_attention_with_rotary_prologue(cuda_dev, causal):
    # O = attention(rope(Q), rope(K), V) against the oracle chain on bf16-rounded rotated inputs
    from paper_2410_20399_b200 import attention as A

    B, H, HKV, N, D = 1, 4, 2, 384, 128
    q = orc.fill(50, B * H * N * D).reshape(B, H, N, D)
    k = orc.fill(51, B * HKV * N * D).reshape(B, HKV, N, D)
    v = orc.fill(52, B * HKV * N * D).reshape(B, HKV, N, D)
    pos = np.arange(N, dtype=np.float64)[:, None]
    freq = 10000.0 ** (-np.arange(D // 2, dtype=np.float64) / (D // 2))
    ang = pos * freq[None, :]
    s, c = np.sin(ang).astype(np.float32), np.cos(ang).astype(np.float32)
    tabs = (_dev(s, torch.float32), _dev(c, torch.float32))
    o, lse = A.attention_fwd(_dev(q), _dev(k), _dev(v), causal=causal, rotary_tables=tabs)
    torch.cuda.synchronize()
    rq = np.asarray(torch.from_numpy(orc.rotary(q, s, c).astype(np.float32)).bfloat16().float())
    rk = np.asarray(torch.from_numpy(orc.rotary(k, s, c).astype(np.float32)).bfloat16().float())
    g = H // HKV
    ro, rl = orc.attn_fwd(rq.reshape(-1, N, D), np.repeat(rk, g, 1).reshape(-1, N, D),
                          np.repeat(v, g, 1).reshape(-1, N, D), causal=causal)
    got = o.float().cpu().numpy().reshape(-1, N, D)
    assert orc.max_abs(got, ro) <= 2e-2 and orc.rel_l2(got, ro) <= 1e-2
    assert orc.max_abs(lse.cpu().numpy().reshape(-1, N), rl) <= 1e-3


@pytest.mark.gpu
@pytest.mark.parametrize("B,H,HKV,N,D,causal", [(2, 4, 4, 1000, 128, True), (1, 8, 2, 200, 64, False),
                                                (2, 8, 1, 4096, 128, True), (1, 2, 2, 129, 64, True)])
def test_fused_rotary_forward_equals_the_two_launch_path(cuda_dev, B, H, HKV, N, D, causal):
    """tkb_attn_fwd_rotary (one launch: the aux warps rotate Q / K block by block while the
    attention of the rotated blocks runs) gives bit-identical rotated Q / K to tkb_rotary_qk
    and bit-identical O / L to tkb_attn_fwd on them; repeated calls (the flag workspace is
    cleared by each call) stay identical."""
    from paper_2410_20399_b200 import attention as A

    g = torch.Generator(device="cuda").manual_seed(N + D)
    q = torch.empty(B, H, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1, generator=g)
    k = torch.empty(B, HKV, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1, generator=g)
    v = torch.empty(B, HKV, N, D, device="cuda", dtype=torch.bfloat16).uniform_(-1, 1, generator=g)
    pos = torch.arange(N, device="cuda", dtype=torch.float64)[:, None]
    freq = 10000.0 ** (-torch.arange(D // 2, device="cuda", dtype=torch.float64) / (D // 2))
    sin, cos = (f(pos * freq[None, :]).float().contiguous() for f in (torch.sin, torch.cos))
    qr, kr = A.rotary_qk(q, k, sin, cos)
    o_ref, l_ref = A.attention_fwd(qr, kr, v, causal=causal)
    for _ in range(3):
        o, lse, q_rot, k_rot = A.attention_fwd(q, k, v, causal=causal, rotary_tables=(sin, cos), return_rotated=True)
        torch.cuda.synchronize()
        assert torch.equal(q_rot, qr) and torch.equal(k_rot, kr)
        assert torch.equal(o, o_ref) and torch.equal(lse, l_ref)


@pytest.mark.gpu
def test_fused_rotary_backward_chain(cuda_dev):
    """Training with the fused prologue: the backward runs on the rotated Q / K the forward
    returned (dQ, dK are gradients w.r.t. the rotated tensors) and matches the oracle."""
    from paper_2410_20399_b200 import attention as A

    B, H, N, D = 1, 2, 300, 64
    q = orc.fill(60, B * H * N * D).reshape(B, H, N, D)
    k = orc.fill(61, B * H * N * D).reshape(B, H, N, D)
    v = orc.fill(62, B * H * N * D).reshape(B, H, N, D)
    do = orc.fill(63, B * H * N * D).reshape(B, H, N, D)
    ang = np.arange(N)[:, None] * (10000.0 ** (-np.arange(D // 2) / (D // 2)))[None, :]
    s, c = np.sin(ang).astype(np.float32), np.cos(ang).astype(np.float32)
    o, lse, qr, kr = A.attention_fwd(_dev(q), _dev(k), _dev(v), causal=True,
                                      rotary_tables=(_dev(s, torch.float32), _dev(c, torch.float32)),
                                      return_rotated=True)
    dq, dk, dv = A.attention_bwd(qr, kr, _dev(v), o, _dev(do), lse, causal=True)
    torch.cuda.synchronize()
    rq, rk = qr.float().cpu().numpy(), kr.float().cpu().numpy()
    rdq, rdk, rdv = orc.attn_bwd(rq, rk, v, do, causal=True)
    for got, ref in ((dq, rdq), (dk, rdk), (dv, rdv)):
        g = got.float().cpu().numpy()
        assert orc.max_abs(g, ref) <= 2e-2 and orc.rel_l2(g, ref) <= 1e-2


@pytest.mark.gpu
@pytest.mark.parametrize("causal,HKV,D", [(True, 4, 128), (False, 2, 128), (True, 1, 64)])
def test_autograd_attention_with_rotary_matches_torch(cuda_dev, causal, HKV, D):
    """attention(q, k, v, rotary_tables=...) — the fused rotary forward, the backward on the
    rotated Q / K, and dQ / dK back through the rotation's transpose (tkb_rotary_qk with -sin) —
    against torch fp64 autograd through rotate -> SDPA on the same bf16 values."""
    from paper_2410_20399_b200 import attention as A

    B, H, N = 2, 4, 300
    g = torch.Generator(device="cuda").manual_seed(7)
    q, k, v = (torch.empty(B, h, N, D, device="cuda").uniform_(-1, 1, generator=g).bfloat16()
               for h in (H, HKV, HKV))
    w = torch.empty(B, H, N, D, device="cuda").uniform_(-1, 1, generator=g)
    pos = torch.arange(N, device="cuda", dtype=torch.float64)[:, None]
    freq = 10000.0 ** (-torch.arange(D // 2, device="cuda", dtype=torch.float64) / (D // 2))
    sin64, cos64 = torch.sin(pos * freq[None, :]), torch.cos(pos * freq[None, :])
    sin, cos = sin64.float().contiguous(), cos64.float().contiguous()
    qa, ka, va = (x.clone().requires_grad_() for x in (q, k, v))
    loss = (A.attention(qa, ka, va, causal=causal, rotary_tables=(sin, cos)).float() * w).sum()
    loss.backward()

    def rot(x):  # oracle_rotary (oracles.hpp:66-90) in fp64
        x1, x2 = x[..., : D // 2], x[..., D // 2:]
        return torch.cat([x1 * cos64 - x2 * sin64, x2 * cos64 + x1 * sin64], dim=-1)

    qr, kr, vr = (x.double().requires_grad_() for x in (q, k, v))
    kre, vre = rot(kr).repeat_interleave(H // HKV, dim=1), vr.repeat_interleave(H // HKV, dim=1)
    ref = torch.nn.functional.scaled_dot_product_attention(rot(qr), kre, vre, is_causal=causal)
    (ref * w.double()).sum().backward()
    for got, want in ((qa.grad, qr.grad), (ka.grad, kr.grad), (va.grad, vr.grad)):
        assert got.dtype == torch.bfloat16 and got.shape == want.shape
        err = (got.double() - want).abs().max().item()
        assert err <= 2e-2 * max(1.0, want.abs().max().item() / 4), err
