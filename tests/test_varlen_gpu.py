"""Variable-length batches on the B200 (the paper guards OOB rows,
PAPER.md:1017,1056): packed [T, H, D] sequences through tkb_attn_fwd_varlen /
tkb_attn_bwd_varlen.

Three bars:
  * every sequence against the fp64 oracle run on that sequence alone (north-star
    tolerances: bf16 O/dQ/dK/dV max-abs 2e-2, rel-L2 1e-2; L 1e-3);
  * bit-identity with the fixed-length entry points run on each sequence as its own
    [1, H, n, D] problem (same tiles, same summation order: nothing of a neighbour leaks in);
  * rows past cu_seqlens[B] are never written (TMA clipping of the offset tensor map).
"""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2410_20399_b200 import attention as A

pytestmark = pytest.mark.gpu

O_MAX_ABS, O_REL_L2, L_ABS = 2e-2, 1e-2, 1e-3


def _packed(seed, lens, H, D, hkv=None, tail=0):
    """q [T, H, D], k / v [T, Hkv, D], dO [T, H, D] (bf16-exact fp32) and int32 cu_seqlens."""
    hkv = hkv or H
    T = int(sum(lens)) + tail
    q = orc.fill(seed, T * H * D).reshape(T, H, D)
    k = orc.fill(seed + 1, T * hkv * D).reshape(T, hkv, D)
    v = orc.fill(seed + 2, T * hkv * D).reshape(T, hkv, D)
    do = orc.fill(seed + 3, T * H * D).reshape(T, H, D)
    cu = np.zeros(len(lens) + 1, dtype=np.int32)
    cu[1:] = np.cumsum(lens)
    return q, k, v, do, cu


def _dev(x, dtype=torch.bfloat16):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dtype)


def _heads(x, s0, s1, group=1):
    """[T, h, D] rows s0:s1 -> [H, n, D] fp32 (kv heads repeated for grouped-query)."""
    y = np.ascontiguousarray(np.transpose(x[s0:s1], (1, 0, 2)))
    return np.repeat(y, group, axis=0) if group > 1 else y


def _run(q, k, v, do, cu, causal, max_len):
    qd, kd, vd, dod = _dev(q), _dev(k), _dev(v), _dev(do)
    cud = _dev(cu, torch.int32)
    o, lse = A.attention_fwd_varlen(qd, kd, vd, cud, max_len, causal=causal)
    dq, dk, dv = A.attention_bwd_varlen(qd, kd, vd, o, dod, lse, cud, max_len, causal=causal)
    torch.cuda.synchronize()
    return o, lse, dq, dk, dv


CASES = [
    # (lens, D, causal, hkv)
    ([300, 1, 128, 0, 513, 129], 128, True, None),
    ([300, 1, 128, 0, 513, 129], 128, False, None),
    ([77, 256, 1000, 64], 64, True, None),
    ([77, 256, 1000, 64], 64, False, None),
    ([200, 384, 33], 128, True, 2),  # grouped-query: 8 query heads over 2 kv heads
]


@pytest.mark.parametrize("lens,D,causal,hkv", CASES)
def test_varlen_vs_oracle(cuda_dev, lens, D, causal, hkv):
    H = 8 if hkv else 4
    group = H // hkv if hkv else 1
    q, k, v, do, cu = _packed(1000 + D + len(lens), lens, H, D, hkv)
    max_len = max(lens)
    o, lse, dq, dk, dv = _run(q, k, v, do, cu, causal, max_len)
    o, dq, dk, dv = (t.float().cpu().numpy() for t in (o, dq, dk, dv))
    lse = lse.cpu().numpy()
    for b, n in enumerate(lens):
        if n == 0:
            continue
        s0, s1 = int(cu[b]), int(cu[b + 1])
        qh, kh, vh, doh = _heads(q, s0, s1), _heads(k, s0, s1, group), _heads(v, s0, s1, group), _heads(do, s0, s1)
        ro, rl = orc.attn_fwd(qh, kh, vh, causal=causal)
        rdq, rdk, rdv = orc.attn_bwd(qh, kh, vh, doh, causal=causal)
        if group > 1:  # dK / dV of a kv head sum over its query heads
            rdk = rdk.reshape(-1, group, n, D).sum(1)
            rdv = rdv.reshape(-1, group, n, D).sum(1)
        got = {"o": (_heads(o, s0, s1), ro), "dq": (_heads(dq, s0, s1), rdq), "dk": (_heads(dk, s0, s1), rdk),
               "dv": (_heads(dv, s0, s1), rdv)}
        for name, (g, r) in got.items():
            assert np.isfinite(g).all(), (b, name)
            ma, rl2 = orc.max_abs(g, r), orc.rel_l2(g, r)
            assert ma <= O_MAX_ABS and rl2 <= O_REL_L2, (b, n, name, ma, rl2)
        assert orc.max_abs(lse[b, :, :n], rl) <= L_ABS, (b, n)


@pytest.mark.parametrize("D,causal", [(128, True), (128, False), (64, True)])
def test_varlen_bitwise_equals_fixed_per_sequence(cuda_dev, D, causal):
    lens = [130, 0, 640, 1, 255, 384]
    H = 2
    q, k, v, do, cu = _packed(7 + D, lens, H, D)
    o, lse, dq, dk, dv = _run(q, k, v, do, cu, causal, max(lens))
    for b, n in enumerate(lens):
        if n == 0:
            continue
        s0, s1 = int(cu[b]), int(cu[b + 1])
        t = [_dev(_heads(x, s0, s1)[None]) for x in (q, k, v, do)]
        fo, fl = A.attention_fwd(t[0], t[1], t[2], causal=causal)
        fdq, fdk, fdv = A.attention_bwd(t[0], t[1], t[2], fo, t[3], fl, causal=causal)
        torch.cuda.synchronize()
        assert torch.equal(o[s0:s1].transpose(0, 1), fo[0]), b
        assert torch.equal(lse[b, :, :n], fl[0]), b
        assert torch.equal(dq[s0:s1].transpose(0, 1), fdq[0]), b
        assert torch.equal(dk[s0:s1].transpose(0, 1), fdk[0]), b
        assert torch.equal(dv[s0:s1].transpose(0, 1), fdv[0]), b


def test_varlen_never_writes_past_the_last_sequence(cuda_dev):
    # T has 200 rows past cu[B]: the TMA maps clip every store at each sequence's end, so
    # the tail keeps its sentinel in O, dQ, dK and dV
    lens, H, D, tail = [100, 300, 17], 2, 128, 200
    q, k, v, do, cu = _packed(31, lens, H, D, tail=tail)
    T = q.shape[0]
    qd, kd, vd, dod = _dev(q), _dev(k), _dev(v), _dev(do)
    cud = _dev(cu, torch.int32)
    sentinel = 12.5
    o = torch.full((T, H, D), sentinel, dtype=torch.bfloat16, device="cuda")
    o, lse = A.attention_fwd_varlen(qd, kd, vd, cud, max(lens), causal=True, out=o)
    grads = [torch.full((T, H, D), sentinel, dtype=torch.bfloat16, device="cuda") for _ in range(3)]
    A.attention_bwd_varlen(qd, kd, vd, o, dod, lse, cud, max(lens), causal=True, dq=grads[0], dk=grads[1],
                           dv=grads[2])
    torch.cuda.synchronize()
    end = int(cu[-1])
    for t in [o] + grads:
        assert bool((t[end:] == sentinel).all())
        assert not bool((t[:end] == sentinel).any())


def test_varlen_deterministic_and_launch_count(cuda_dev):
    lens, H, D = [513, 1000, 3], 4, 128
    q, k, v, do, cu = _packed(99, lens, H, D)
    a = _run(q, k, v, do, cu, True, max(lens))
    assert A.last_launch_count() == 4  # maps, prep, dK/dV, dQ
    b = _run(q, k, v, do, cu, True, max(lens))
    for i, (x, y) in enumerate(zip(a, b)):
        if i == 1:  # L: rows past each sequence's length are never written
            for s, n in enumerate(lens):
                assert torch.equal(x[s, :, :n], y[s, :, :n])
        else:
            assert torch.equal(x, y)


def test_varlen_rejects_bad_layouts(cuda_dev):
    lens, H, D = [10, 20], 2, 64
    q, k, v, do, cu = _packed(5, lens, H, D)
    qd, kd, vd = _dev(q), _dev(k), _dev(v)
    with pytest.raises(A.ShapeError):  # int64 cu_seqlens
        A.attention_fwd_varlen(qd, kd, vd, _dev(cu, torch.int64), 20)
    with pytest.raises(A.ShapeError):  # [B, H, N, D] instead of packed [T, H, D]
        A.attention_fwd_varlen(qd[None], kd[None], vd[None], _dev(cu, torch.int32), 20)


@pytest.mark.parametrize("bad", ["too_long", "decreasing", "start", "past_total"])
def test_varlen_check_finite_validates_offsets(cuda_dev, bad):
    """desc.check_finite (the synchronising input check) also checks cu_seqlens on the host."""
    lens, H, D = [100, 60], 2, 64
    q, k, v, do, cu = _packed(3, lens, H, D)
    qd, kd, vd = _dev(q), _dev(k), _dev(v)
    A.attention_fwd_varlen(qd, kd, vd, _dev(cu, torch.int32), 100, check_finite=True)  # valid
    cu_bad = {"too_long": [0, 100, 160], "decreasing": [0, 120, 100], "start": [1, 100, 160],
              "past_total": [0, 100, 200]}[bad]
    max_len = 60 if bad == "too_long" else 100
    err = A.BoundsError if bad == "past_total" else A.ConfigError
    with pytest.raises(err):
        A.attention_fwd_varlen(qd, kd, vd, _dev(np.asarray(cu_bad, np.int32), torch.int32), max_len,
                               check_finite=True)


def test_varlen_check_finite_rejects_non_finite(cuda_dev):
    lens, H, D = [100, 60], 2, 128
    q, k, v, do, cu = _packed(4, lens, H, D)
    q[150, 1, 7] = np.inf
    with pytest.raises(A.ConfigError):
        A.attention_fwd_varlen(_dev(q), _dev(k), _dev(v), _dev(cu, torch.int32), 100, check_finite=True)
