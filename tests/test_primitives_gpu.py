"""Unit tests of the sm_100a tile primitives (TMA SW128, tcgen05.mma SS/TS, TMEM).

Each selftest variant computes one 128xN fp32 tile on the GPU; the check is a
plain torch fp32 matmul of the same bf16 operands.
"""
import ctypes
import os

import pytest
import torch

from paper_2410_20399_b200 import _lib

pytestmark = pytest.mark.gpu


def _st():
    lib = _lib.load_selftest()
    f = lib.tkb_selftest_umma
    f.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    f.restype = ctypes.c_int
    return f


@pytest.mark.parametrize("variant,n,k", [(0, 128, 128), (0, 128, 64), (1, 128, 128), (1, 64, 128),
                                         (2, 128, 128), (2, 64, 128), (3, 128, 128), (3, 64, 128),
                                         (4, 128, 128), (5, 128, 128), (5, 128, 64)])
def test_umma_variant(cuda_dev, variant, n, k):
    g = torch.Generator().manual_seed(1000 * variant + n + k)
    M = 128
    A = torch.randn(M, k, generator=g).to(torch.bfloat16)
    if variant in (0, 5):
        B = torch.randn(n, k, generator=g).to(torch.bfloat16)
        ref = A.float() @ B.float().t()
    elif variant == 4:
        B = torch.zeros(k, n, dtype=torch.bfloat16)
        ref = A.float()
    else:
        B = torch.randn(k, n, generator=g).to(torch.bfloat16)
        ref = A.float() @ B.float()
    A_dev = A.t().contiguous().to(cuda_dev) if variant == 3 else A.to(cuda_dev)
    A_rowmajor = A.to(cuda_dev)  # the TMEM-staged variants read A row-major
    B_dev = B.to(cuda_dev)
    C = torch.zeros(ref.shape, dtype=torch.float32, device=cuda_dev)
    a_ptr = A_rowmajor.data_ptr() if variant in (2, 4, 5) else A_dev.data_ptr()
    rc = _st()(variant, n, k, a_ptr, B_dev.data_ptr(), C.data_ptr(),
               torch.cuda.current_stream().cuda_stream, 1, None)
    assert rc == 0
    torch.cuda.synchronize()
    err = (C.cpu() - ref).abs().max().item()
    assert err < 1e-3 * max(1.0, ref.abs().max().item()), f"variant {variant}: max err {err}"


@pytest.mark.parametrize("variant", [0, 1, 2, 3])
def test_umma_throughput(cuda_dev, variant):
    """Cycles per 128x128x16 tcgen05.mma for each operand flavour (single CTA, back to back)."""
    n, k, reps = 128, 128, 200
    A = torch.randn(128, k, device=cuda_dev).to(torch.bfloat16)
    B = torch.randn(k, n, device=cuda_dev).to(torch.bfloat16)
    C = torch.zeros(128, n, device=cuda_dev)
    cyc = torch.zeros(1, dtype=torch.int64, device=cuda_dev)
    rc = _st()(variant, n, k, A.data_ptr(), B.data_ptr(), C.data_ptr(),
               torch.cuda.current_stream().cuda_stream, reps, cyc.data_ptr())
    assert rc == 0
    torch.cuda.synchronize()
    per_mma = cyc.item() / (reps * k / 16)
    print(f"variant {variant}: {per_mma:.1f} cycles per 128x128x16 MMA")
    assert per_mma < 1000


def test_tmem_16lane_shapes(cuda_dev):
    """The 16x256b load / 16x128b store register maps the backward's dK/dV compute uses."""
    lib = _lib.load_selftest()
    lib.tkb_selftest_tmem_shapes.argtypes = [ctypes.c_void_p]
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    assert lib.tkb_selftest_tmem_shapes(bad.data_ptr()) == 0
    assert int(bad.item()) == 0
