"""The tile vocabulary (tkb/tile.cuh) on the B200: one 128 x 128 attention tile built only
from the ThunderKittens ops the north star keeps (rt / st / tt / gl, load / store,
mm_ABt / mma_AB, row_max / sub_row / exp2 / row_sum / copy / div_row), checked against a
plain torch fp32 reference of the same op; plus the reference's tile tests that pin the
op semantics (test_tiles.cpp:29-37 bf16 RNE incl. the halfway case; the SW128 round
trip of test_layouts.cpp:60-66)."""
import ctypes

import pytest
import torch

from paper_2410_20399_b200 import _lib

pytestmark = pytest.mark.gpu


def _fn(name, nargs):
    f = getattr(_lib.load_selftest(), name)
    f.argtypes = [ctypes.c_void_p] * nargs
    f.restype = ctypes.c_int
    return f


def test_tile_api_attention_tile(cuda_dev):
    g = torch.Generator().manual_seed(7)
    Q, K, V = (torch.randn(128, 128, generator=g).to(torch.bfloat16) for _ in range(3))
    q, k, v = (x.to(cuda_dev) for x in (Q, K, V))
    O = torch.empty(128, 128, device=cuda_dev)
    m = torch.empty(128, device=cuda_dev)
    l = torch.empty(128, device=cuda_dev)
    P = torch.empty(128, 128, device=cuda_dev)
    qb = torch.empty(128, 128, device=cuda_dev)
    rc = _fn("tkb_selftest_tile_api", 9)(q.data_ptr(), k.data_ptr(), v.data_ptr(), O.data_ptr(), m.data_ptr(),
                                         l.data_ptr(), P.data_ptr(), qb.data_ptr(),
                                         torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    torch.cuda.synchronize()
    # torch fp32 reference of the same sequence of tile ops (exp2 domain, no scale)
    S = Q.float() @ K.float().t()
    ref_m = S.max(dim=1).values
    E = torch.exp2(S - ref_m[:, None])
    ref_l = E.sum(dim=1)
    ref_p = E.to(torch.bfloat16).float()
    ref_o = (ref_p @ V.float()) / ref_l[:, None]
    assert torch.allclose(m.cpu(), ref_m, atol=1e-3 * ref_m.abs().max().item())
    assert torch.allclose(l.cpu(), ref_l, rtol=2e-3)
    assert (P.cpu() - ref_p).abs().max().item() <= 2 ** -7  # bf16 of an ex2.approx value
    assert (O.cpu() - ref_o).abs().max().item() <= 2e-2
    # st_bf::chunk addressing reads back exactly what TMA placed (SW128, layouts.hpp:111-132)
    assert torch.equal(qb.cpu(), Q.float())


def test_copy_is_round_to_nearest_even(cuda_dev):
    # test_tiles.cpp:29-37: 1 + 2^-8 is the halfway case between 1.0 and 1.0078125 -> even (1.0)
    vals = torch.tensor([1.0000001, 1.0, -1.0000001, 1.0078125, 1.00390625, 1.01171875, -3.0e-39, 65504.0],
                        dtype=torch.float32)
    inp = vals.to(cuda_dev)
    out = torch.empty_like(inp)
    rc = _fn("tkb_selftest_rne", 4)(inp.data_ptr(), out.data_ptr(), ctypes.c_void_p(8),
                                    torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    torch.cuda.synchronize()
    want = vals.to(torch.bfloat16).float()  # torch's RNE
    assert torch.equal(out.cpu(), want)
    assert out[0].item() == 1.0 and out[3].item() == 1.0078125 and out[4].item() == 1.0


def test_tile_api_operand_and_transfer_flavours(cuda_dev):
    """global -> register -> shared -> register -> TMEM transfers, the SS mm_AB with a
    swap_layout B, the TS mm_ABt (A in TMEM), the grouped-A mma_AB_groups and the
    warp-collective store_rows, each against a torch fp32 matmul of the same bf16 operands."""
    g = torch.Generator().manual_seed(11)
    A, B = (torch.randn(128, 128, generator=g).to(torch.bfloat16) for _ in range(2))
    a, b = A.to(cuda_dev), B.to(cuda_dev)
    C1, C2, C3 = (torch.empty(128, 128, device=cuda_dev) for _ in range(3))
    C3b = torch.empty(128, 128, device=cuda_dev, dtype=torch.bfloat16)
    rc = _fn("tkb_selftest_tile_api2", 7)(a.data_ptr(), b.data_ptr(), C1.data_ptr(), C2.data_ptr(), C3.data_ptr(),
                                          C3b.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    torch.cuda.synchronize()
    ab = A.float() @ B.float()
    abt = A.float() @ B.float().t()
    tol = 1e-3 * ab.abs().max().item()
    assert (C1.cpu() - ab).abs().max().item() <= tol
    assert (C2.cpu() - abt).abs().max().item() <= tol
    assert (C3.cpu() - ab).abs().max().item() <= tol
    assert torch.equal(C3b.cpu(), C3.cpu().to(torch.bfloat16))
