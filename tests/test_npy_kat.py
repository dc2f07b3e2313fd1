"""Golden KATs in the reference's own .npy format (npy.hpp:18-87).

tests/golden/npy/ holds the dense d=64 case of test_kernels.cpp:128-146 (q, k, v and the
reference kernel's O), written by the reference's writer (oracle/npy_tool, built from
npy.hpp) in tests/golden/make_golden.py. numpy and the reference reader must agree on
them, and the B200 kernel must reproduce O from them within the north-star bar.
"""
import os

import numpy as np
import pytest

from oracle import oracle as orc

NPY = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "npy")
NAMES = ("q", "k", "v", "o_ref")


def _load(name):
    return np.load(os.path.join(NPY, f"dense_d64_{name}.npy"))


def test_npy_kats_are_float32_384x64_and_match_golden():
    arrs = {n: _load(n) for n in NAMES}
    for n, a in arrs.items():
        assert a.dtype == np.float32 and a.shape == (384, 64), n
    g = np.load(os.path.join(os.path.dirname(NPY), "golden.npz"))
    np.testing.assert_array_equal(arrs["o_ref"], g["dense_d64.o_kernel"][0, 0])
    # the inputs are the reference generator's stream (seed 164 = 100 + d, Q then K then V)
    stream = orc.fill(164, 3 * 384 * 64, bf16=False).reshape(3, 384, 64)
    for i, n in enumerate(("q", "k", "v")):
        np.testing.assert_array_equal(arrs[n], stream[i])


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(orc.__file__), "_ref", "npy_tool")),
                    reason="oracle/_ref/npy_tool not built")
def test_reference_reader_and_numpy_agree(tmp_path):
    for n in NAMES:
        data, shape = orc.ref_load_npy(os.path.join(NPY, f"dense_d64_{n}.npy"))
        assert shape == (384, 64)
        np.testing.assert_array_equal(data, _load(n))
    # round trip through the reference writer
    x = np.arange(24, dtype=np.float32).reshape(2, 3, 4)
    p = str(tmp_path / "x.npy")
    orc.ref_save_npy(p, x)
    np.testing.assert_array_equal(np.load(p), x)


@pytest.mark.gpu
def test_kernel_reproduces_npy_kat(cuda_dev):
    import torch

    from paper_2410_20399_b200 import attention as A

    # the reference runs fp32 inputs; the B200 path is bf16: compare against the fp64 oracle on
    # the bf16-rounded inputs (the north-star bar) and against the reference O within bf16 error
    q, k, v, o_ref = (_load(n) for n in NAMES)
    t = lambda x: torch.from_numpy(x[None, None]).to("cuda", torch.bfloat16)  # noqa: E731
    o, _ = A.attention_fwd(t(q), t(k), t(v))
    torch.cuda.synchronize()
    got = o.float().cpu().numpy()[0, 0]
    rb = lambda x: torch.from_numpy(x).bfloat16().float().numpy()  # noqa: E731
    ro, _ = orc.attn_fwd(rb(q), rb(k), rb(v))
    assert orc.max_abs(got, ro) <= 2e-2 and orc.rel_l2(got, ro) <= 1e-2
    assert orc.max_abs(got, o_ref) <= 2e-2
