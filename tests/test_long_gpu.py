"""Long-sequence, non-default-scale and input-check parity on the B200.

* BASELINE configs[4]'s per-GPU shard at 8 GPUs (B=4 H=32 N=16384 D=128), causal and not:
  the whole shard runs forward + backward on the GPU; O and L of two subsampled heads are
  compared row for row with the fp64 oracle, dQ at 192 query rows and dK / dV at 192 key
  rows of the same heads (oracle/attn_oracle.cpp tkb_oracle_attn_bwd_sampled: the same math
  as the full oracle, evaluated at the sampled rows only). N = 16384 is 128 kv blocks per
  row: the lazy 2^8 rescale, the fp32 row sums and L see their longest runs here.
* N = 8192 at D = 64 and 128 (BASELINE configs[3]'s long end), full heads.
* A non-default softmax_scale in the forward and the backward.
* The backward's non-finite input check (kernels.hpp:277-284 on the backward's inputs).

Bar (north_star): bf16 O/dQ/dK/dV max-abs <= 2e-2 and rel-L2 <= 1e-2; L within 1e-3.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2410_20399_b200 import attention as A

pytestmark = pytest.mark.gpu

MAX_ABS, REL_L2, LSE_TOL = 2e-2, 1e-2, 1e-3


def _assert_close(name, got, ref, tol=MAX_ABS, rel=REL_L2):
    assert np.isfinite(got).all(), name
    ma, rl = orc.max_abs(got, ref), orc.rel_l2(got, ref)
    assert ma <= tol and rl <= rel, (name, ma, rl)
    return ma, rl


def _sample_rows(n, count, seed):
    """Block edges (first / last row of 128-row blocks, both ends of the sequence) plus random rows."""
    rng = np.random.default_rng(seed)
    edges = [0, 1, 127, 128, 255, 256, n // 2 - 1, n // 2, n - 129, n - 128, n - 2, n - 1]
    rest = rng.choice(n, size=count - len(edges), replace=False)
    return np.unique(np.clip(np.concatenate([edges, rest]), 0, n - 1)).astype(np.int32)


def _gpu_inputs(seed, B, H, N, D):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return [torch.empty((B, H, N, D), device="cuda", dtype=torch.bfloat16).uniform_(-1, 1, generator=g)
            for _ in range(4)]


def _heads(t, idx):
    B, H = t.shape[:2]
    return t.reshape(B * H, *t.shape[2:])[idx].float().cpu().numpy()


@pytest.mark.slow
@pytest.mark.parametrize("causal", [True, False])
def test_configs4_shard_n16384(cuda_dev, causal):
    B, H, N, D = 4, 32, 16384, 128
    q, k, v, do = _gpu_inputs(4242 + causal, B, H, N, D)
    o, lse = A.attention_fwd(q, k, v, causal=causal)
    dq, dk, dv = A.attention_bwd(q, k, v, o, do, lse, causal=causal)
    torch.cuda.synchronize()
    idx = np.array([1 * H + 7, 3 * H + 30])  # (b=1, h=7), (b=3, h=30)
    hq, hk, hv, hdo = (_heads(t, idx) for t in (q, k, v, do))
    ro, rl = orc.attn_fwd_rows(hq, hk, hv, causal=causal)
    _assert_close("o", _heads(o, idx), ro)
    assert orc.max_abs(_heads(lse, idx), rl) <= LSE_TOL
    qr, kr = _sample_rows(N, 192, 1), _sample_rows(N, 192, 2)
    rdq, rdk, rdv = orc.attn_bwd_sampled(hq, hk, hv, hdo, qr, kr, causal=causal)
    _assert_close("dq", _heads(dq, idx)[:, qr], rdq)
    _assert_close("dk", _heads(dk, idx)[:, kr], rdk)
    _assert_close("dv", _heads(dv, idx)[:, kr], rdv)


@pytest.mark.parametrize("D", [64, 128])
@pytest.mark.parametrize("causal", [True, False])
def test_n8192(cuda_dev, D, causal):
    B, H, N = 1, 2, 8192
    q, k, v, do = _gpu_inputs(81 + D + causal, B, H, N, D)
    o, lse = A.attention_fwd(q, k, v, causal=causal)
    dq, dk, dv = A.attention_bwd(q, k, v, o, do, lse, causal=causal)
    torch.cuda.synchronize()
    idx = np.arange(B * H)
    hq, hk, hv, hdo = (_heads(t, idx) for t in (q, k, v, do))
    ro, rl = orc.attn_fwd_rows(hq, hk, hv, causal=causal)
    _assert_close("o", _heads(o, idx), ro)
    assert orc.max_abs(_heads(lse, idx), rl) <= LSE_TOL
    qr, kr = _sample_rows(N, 256, 3), _sample_rows(N, 256, 4)
    rdq, rdk, rdv = orc.attn_bwd_sampled(hq, hk, hv, hdo, qr, kr, causal=causal)
    _assert_close("dq", _heads(dq, idx)[:, qr], rdq)
    _assert_close("dk", _heads(dk, idx)[:, kr], rdk)
    _assert_close("dv", _heads(dv, idx)[:, kr], rdv)


@pytest.mark.parametrize("scale", [0.05, 0.2])
@pytest.mark.parametrize("D", [64, 128])
@pytest.mark.parametrize("causal", [True, False])
def test_softmax_scale(cuda_dev, scale, D, causal):
    """desc.softmax_scale feeds both passes (tau in the forward's exponent, L, and the
    backward's P and its dQ / dK scaling)."""
    B, H, N = 1, 2, 1000
    q, k, v = orc.qkv(900 + D, B, H, N, D)
    do = orc.fill(901 + D, B * H * N * D).reshape(B, H, N, D)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to("cuda", torch.bfloat16)  # noqa: E731
    qd, kd, vd, dod = (dev(x) for x in (q, k, v, do))
    o, lse = A.attention_fwd(qd, kd, vd, causal=causal, softmax_scale=scale)
    dq, dk, dv = A.attention_bwd(qd, kd, vd, o, dod, lse, causal=causal, softmax_scale=scale)
    torch.cuda.synchronize()
    ro, rl = orc.attn_fwd(q, k, v, causal=causal, scale=scale)
    _assert_close("o", o.float().cpu().numpy(), ro)
    assert orc.max_abs(lse.cpu().numpy(), rl) <= LSE_TOL
    rdq, rdk, rdv = orc.attn_bwd(q, k, v, do, causal=causal, scale=scale)
    for name, g, r in (("dq", dq, rdq), ("dk", dk, rdk), ("dv", dv, rdv)):
        _assert_close(name, g.float().cpu().numpy(), r)


@pytest.mark.parametrize("which", ["q", "k", "v", "o", "dout"])
def test_bwd_check_finite(cuda_dev, which):
    B, H, N, D = 1, 2, 300, 64
    q, k, v, do = _gpu_inputs(55, B, H, N, D)
    o, lse = A.attention_fwd(q, k, v)
    A.attention_bwd(q, k, v, o, do, lse, check_finite=True)  # finite: passes
    bad = {"q": q, "k": k, "v": v, "o": o, "dout": do}[which].clone()
    bad[0, 1, 123, 7] = float("inf") if which != "v" else float("nan")
    args = dict(q=q, k=k, v=v, o=o, dout=do)
    args[which] = bad
    with pytest.raises(A.ConfigError):
        A.attention_bwd(args["q"], args["k"], args["v"], args["o"], args["dout"], lse, check_finite=True)


def test_python_boundary_rejects_bad_buffers(cuda_dev):
    """The mirror validates every caller-supplied buffer before the kernel writes to it."""
    B, H, N, D = 1, 2, 256, 64
    q, k, v, do = _gpu_inputs(7, B, H, N, D)
    with pytest.raises(A.ShapeError):  # lse of the wrong dtype
        A.attention_fwd(q, k, v, lse=torch.empty((B, H, N), device="cuda", dtype=torch.float16))
    with pytest.raises(A.ShapeError):  # lse of the wrong shape
        A.attention_fwd(q, k, v, lse=torch.empty((B, H, N - 1), device="cuda", dtype=torch.float32))
    o, lse = A.attention_fwd(q, k, v)
    with pytest.raises(A.ConfigError):  # an fp32 dq with bf16-compatible strides
        A.attention_bwd(q, k, v, o, do, lse, dq=torch.empty(q.shape, device="cuda", dtype=torch.float32))
    with pytest.raises(A.ShapeError):  # dk of the wrong shape
        A.attention_bwd(q, k, v, o, do, lse, dk=torch.empty((B, H, N, D // 2), device="cuda", dtype=torch.bfloat16))
    with pytest.raises(A.BoundsError):  # workspace too small
        A.attention_bwd(q, k, v, o, do, lse, workspace=torch.empty(16, device="cuda", dtype=torch.uint8))
    sin = torch.zeros((N, D // 2), device="cuda")
    with pytest.raises(A.ConfigError):  # rotary on fp32 input
        A.rotary_qk(q.float(), k, sin, sin)
    with pytest.raises(A.ShapeError):  # k with a different N than q
        A.rotary_qk(q, k[:, :, : N // 2], sin, sin)


def test_descriptor_cache_hits(cuda_dev):
    """Repeated calls on the same buffers reuse the encoded TMA descriptors."""
    q, k, v, do = _gpu_inputs(8, 1, 2, 512, 128)
    o, lse = A.attention_fwd(q, k, v)
    h0, m0 = A.map_cache_stats()
    for _ in range(3):
        A.attention_fwd(q, k, v, out=o, lse=lse)
    h1, m1 = A.map_cache_stats()
    assert (m1 - m0, h1 - h0) == (0, 12), (h0, m0, h1, m1)  # 4 maps per forward, all hits


@pytest.mark.parametrize("causal", [True, False])
def test_many_heads_task_decode(cuda_dev, causal):
    """B*H = 70000 (> gridDim.y's 65535) at a ragged N: task ids up to ~10^5 through the FastDiv
    task decoders, L2 head groups that do not divide B*H (a short last group), and the
    grid-stride prep / scan kernels; sampled heads against the fp64 oracle."""
    B, H, N, D = 35000, 2, 200, 64
    q, k, v, do = _gpu_inputs(99 + causal, B, H, N, D)
    o, lse = A.attention_fwd(q, k, v, causal=causal)
    dq, dk, dv = A.attention_bwd(q, k, v, o, do, lse, causal=causal)
    torch.cuda.synchronize()
    idx = np.array([0, 1, 12345, 34999 * 2, 69998, 69999])
    qh, kh, vh, doh = (_heads(t, idx) for t in (q, k, v, do))
    ro, rl = orc.attn_fwd(qh, kh, vh, causal=causal)
    rdq, rdk, rdv = orc.attn_bwd(qh, kh, vh, doh, causal=causal)
    _assert_close("o", _heads(o, idx), ro)
    assert orc.max_abs(lse.reshape(B * H, N)[idx].cpu().numpy(), rl) <= LSE_TOL
    for name, got, ref in (("dq", dq, rdq), ("dk", dk, rdk), ("dv", dv, rdv)):
        _assert_close(name, _heads(got, idx), ref)
