"""GEMM on the attention machinery: oracle pinned to the reference
(oracle_gemm, gemm_kernel, supergroup_order via oracle/_ref) on CPU; the sm_100a kernel
against the oracle on the GPU (bf16 inputs, fp32 accumulation, bf16 C)."""
import numpy as np
import pytest
import torch

from oracle import oracle as orc


# ------------------------------------------------------------------ CPU: oracle pinning
@pytest.mark.skipif(not orc.ref_available(), reason="oracle/_ref not built")
def test_oracle_gemm_matches_reference_oracle():
    a = orc.fill(1, 64 * 192, bf16=False).reshape(64, 192)
    b = orc.fill(2, 192 * 128, bf16=False).reshape(192, 128)
    np.testing.assert_allclose(orc.gemm(a, b), orc.ref_gemm_oracle(a, b), rtol=0, atol=1e-12)


@pytest.mark.skipif(not orc.ref_available(), reason="oracle/_ref not built")
def test_reference_gemm_kernel_matches_oracle():
    a = orc.fill(3, 256 * 128, bf16=False).reshape(256, 128)
    b = orc.fill(4, 128 * 256, bf16=False).reshape(128, 256)
    assert np.max(np.abs(orc.ref_gemm(a, b) - orc.gemm(a, b))) <= 1e-4


@pytest.mark.skipif(not orc.ref_available(), reason="oracle/_ref not built")
def test_supergroup_order_is_the_references():
    # the device-side task order (gemm_sm100.cu supergroup()) restates grid.hpp:28-47;
    # this pins the Python restatement used to check it
    def mine(r, c, sm):
        sr = (r // sm) * sm
        out = []
        for t in range(r * c):
            if t < sr * c:
                out.append((sm * (t // (sm * c)) + t % sm, (t % (sm * c)) // sm))
            else:
                rem = t - sr * c
                out.append((sr + rem % (r - sr), rem // (r - sr)))
        return out
    for r, c, sm in ((7, 5, 3), (12, 4, 12), (13, 9, 4), (1, 1, 12)):
        rows, cols = orc.ref_supergroup_order(r, c, sm)
        assert mine(r, c, sm) == list(zip(rows.tolist(), cols.tolist()))


def test_gemm_config_validation():
    from paper_2410_20399_b200 import attention as A
    A.GemmConfig(100, 200, 304).validate()  # dense rows: k, n multiples of 8 (16-byte TMA strides)
    with pytest.raises(A.ConfigError):
        A.GemmConfig(0, 64, 64).validate()
    with pytest.raises(A.ShapeError):
        A.lib()  # noqa: B018
        import ctypes
        d = A.GemmConfig(64, 64, 64).desc(lda=60)
        A._check(A.lib().tkb_gemm_validate(ctypes.byref(d)))


# ------------------------------------------------------------------ GPU: kernel parity
def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", torch.bfloat16)


@pytest.mark.gpu
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 512, 1024), (300, 200, 104), (1024, 1024, 4096),
                                   (2048, 768, 512), (129, 296, 80), (520, 136, 72), (4096, 256, 64)])
def test_gemm_matches_oracle(cuda_dev, M, N, K):
    from paper_2410_20399_b200 import attention as A

    a = orc.fill(10 + M, M * K).reshape(M, K)
    b = orc.fill(11 + N, K * N).reshape(K, N)
    c = A.gemm(_dev(a), _dev(b))
    torch.cuda.synchronize()
    ref = orc.gemm(a, b)
    got = c.float().cpu().numpy()
    # fp32 accumulation then one bf16 rounding of C
    assert np.all(np.abs(got - ref) <= np.abs(ref) * 2.0 ** -8 + 1e-3 * np.sqrt(K))


@pytest.mark.gpu
def test_gemm_strided_and_deterministic(cuda_dev):
    from paper_2410_20399_b200 import attention as A

    a_full = _dev(orc.fill(20, 512 * 320).reshape(512, 320))
    b = _dev(orc.fill(21, 256 * 384).reshape(256, 384))
    a = a_full[:, :256]  # lda = 320
    c1 = A.gemm(a, b)
    c2 = A.gemm(a, b)
    torch.cuda.synchronize()
    assert torch.equal(c1, c2)
    ref = orc.gemm(a.float().cpu().numpy(), b.float().cpu().numpy())
    got = c1.float().cpu().numpy()
    assert np.all(np.abs(got - ref) <= np.abs(ref) * 2.0 ** -8 + 1e-3 * np.sqrt(256)), np.max(np.abs(got - ref))
