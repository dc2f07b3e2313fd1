"""CPU tests of the C-ABI boundary (no GPU): the library loads, exports exactly what
include/tkb_attn.h declares, validates like AttentionConfig::validate
(kernels.hpp:188-202), and fails loudly (never falls back to the CPU) without a B200."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2410_20399_b200 import _lib
from paper_2410_20399_b200 import attention as A

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tkb_attn.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"TKB_API\s+[\w\s\*]+?\b(tkb_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("tkb_attn_fwd", "tkb_attn_bwd", "tkb_attn_bwd_workspace_bytes", "tkb_attn_validate",
              "tkb_last_error", "tkb_shard_range"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert set(A.exported_symbols()) == set(declared_symbols())
    assert A.lib().tkb_abi_version() == 4


def test_library_is_built_for_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("B,H,N,D,code", [
    (1, 1, 384, 64, 0), (1, 8, 1024, 64, 0), (2, 3, 200, 128, 0), (1, 1, 1, 64, 0),
    (1, 1, 384, 96, 1),   # D not in {64, 128}: ConfigError, as the reference (test_kernels.cpp:310-327)
    (0, 1, 384, 64, 1), (1, 1, 0, 64, 1),
])
def test_validate_codes(B, H, N, D, code):
    d = A.AttentionConfig(B, H, N, D).desc()
    assert A.lib().tkb_attn_validate(ctypes.byref(d)) == code


def test_validate_matches_reference_on_head_dim():
    gold = np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))
    assert int(gold["validate.d96"]) == 1  # reference: ConfigError
    with pytest.raises(A.ConfigError):
        A.AttentionConfig(1, 1, 384, 96).validate()
    # ragged N is rejected by the reference's stock tiling (N % kv_rows) but supported here
    assert int(gold["validate.n200"]) == 1
    A.AttentionConfig(1, 1, 200, 64).validate()


def test_bad_strides_are_shape_errors():
    d = A.AttentionConfig(1, 2, 64, 64).desc(strides=(64 * 64 * 2, 64 * 64, 60))
    assert A.lib().tkb_attn_validate(ctypes.byref(d)) == 2


def test_workspace_bytes():
    # delta + lse2, fp32 each, rows padded to 128
    assert A.bwd_workspace_bytes(2, 3, 200, 128) == 2 * 6 * 256 * 4
    assert A.bwd_workspace_bytes(1, 1, 128, 64) == 2 * 128 * 4


@pytest.mark.parametrize("units,world", [(256, 1), (256, 8), (1024, 3), (5, 8), (0, 2)])
def test_shard_range_partitions(units, world):
    spans = [A.shard_range(units, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == units
    for (b0, e0), (b1, _) in zip(spans, spans[1:]):
        assert e0 == b1
    sizes = [e - b for b, e in spans]
    assert max(sizes) - min(sizes) <= 1


def test_fwd_without_a_b200_fails_loudly():
    """No CPU fallback: a call with no sm_100 device returns an error, never computes."""
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    d = A.AttentionConfig(1, 1, 128, 64).desc()
    buf = (ctypes.c_uint16 * (128 * 64))()
    rc = A.lib().tkb_attn_fwd(ctypes.byref(d), ctypes.addressof(buf), ctypes.addressof(buf), ctypes.addressof(buf),
                              ctypes.addressof(buf), None, None)
    assert rc in (4, 5)  # TKB_ERR_UNSUPPORTED / TKB_ERR_CUDA
    assert A.lib().tkb_last_error()
    with pytest.raises(A.ConfigError):  # the python mirror refuses CPU tensors outright
        x = torch.zeros(1, 1, 128, 64, dtype=torch.bfloat16)
        A.attention_fwd(x, x, x)


def test_null_pointers_are_bounds_errors():
    d = A.AttentionConfig(1, 1, 128, 64).desc()
    assert A.lib().tkb_attn_fwd(ctypes.byref(d), None, None, None, None, None, None) == 3


def test_kv_heads_must_divide_heads():
    # grouped-query attention: H % Hkv == 0 (ConfigError otherwise), checked without a GPU
    A.AttentionConfig(1, 8, 64, 64, kv_heads=2).validate()
    A.AttentionConfig(1, 8, 64, 64, kv_heads=1).validate()
    with pytest.raises(A.ConfigError):
        A.AttentionConfig(1, 8, 64, 64, kv_heads=3).validate()


def test_desc_layout_matches_header():
    # AttnDesc mirrors tkb_attn_desc (include/tkb_attn.h, ABI 2): 8 x 4-byte fields + 6 x int64
    import ctypes
    assert ctypes.sizeof(A.AttnDesc) == 8 * 4 + 6 * 8
    assert A.AttnDesc.kv_heads.offset == 28 and A.AttnDesc.kv_stride_b.offset == 56


@pytest.mark.parametrize("scale,code", [(0.0, 0), (0.05, 0), (0.2, 0), (-0.1, 1), (float("inf"), 1),
                                        (float("nan"), 1)])
def test_softmax_scale_validation(scale, code):
    """0 selects D^-1/2; a negative or non-finite scale is a ConfigError (never silently replaced)."""
    d = A.AttentionConfig(1, 2, 256, 64).desc()
    d.softmax_scale = scale
    assert A.lib().tkb_attn_validate(ctypes.byref(d)) == code


def test_task_count_bound():
    """The persistent schedulers use 32-bit task ids: B * H * ceil(N / 128) must stay < 2^31
    (B * H beyond gridDim.y's 65535 is fine: the helper kernels walk it grid-stride)."""
    A.AttentionConfig(70000, 2, 128, 64).validate()  # B*H = 140000 > 65535
    with pytest.raises(A.ConfigError):
        A.AttentionConfig(65536, 256, 16384, 128).validate()  # 2^24 heads x 128 blocks = 2^31


def test_device_init_without_a_gpu_fails_cleanly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(A.Error):
        A.device_init(0)



def _varlen_call(d, cu=1 << 12, total=100, ptr=1 << 16, ws=1 << 20, ws_bytes=1 << 20):
    return A.lib().tkb_attn_fwd_varlen(ctypes.byref(d), cu, total, ptr, ptr, ptr, ptr, None, ws, ws_bytes, None)


def test_varlen_validation_without_a_gpu():
    """Variable-length batches (tkb_attn_fwd_varlen): packed [T, H, D] only (batch strides 0),
    cu_seqlens present and aligned, T inside the 32-bit TMA coordinate range — all checked
    before any device work."""
    d = A.AttentionConfig(3, 4, 512, 128).desc()
    d.stride_b = 4 * 128 * 512
    assert _varlen_call(d) == 2  # ShapeError: batch stride on a packed tensor
    d = A.AttentionConfig(3, 4, 512, 128).desc()
    assert A.lib().tkb_attn_fwd_varlen(ctypes.byref(d), None, 100, 1 << 16, 1 << 16, 1 << 16, 1 << 16, None,
                                       1 << 20, 1 << 20, None) == 3  # BoundsError: null cu_seqlens
    assert _varlen_call(d, ws=None) == 3 and _varlen_call(d, ws_bytes=3 * 4 * 128 - 1) == 3  # workspace
    assert _varlen_call(d, ws=(1 << 20) + 64) == 2  # workspace not 128-byte aligned
    # per-sequence maps: 4 (fwd) / 7 (bwd) 128-byte CUtensorMaps per sequence, rounded to 256
    assert A.lib().tkb_attn_fwd_varlen_workspace_bytes(ctypes.byref(d)) == 1536
    assert (A.lib().tkb_attn_bwd_varlen_workspace_bytes(ctypes.byref(d))
            == A.lib().tkb_attn_bwd_workspace_bytes(ctypes.byref(d)) + 2816)
    assert _varlen_call(d, cu=(1 << 12) + 2) == 2  # misaligned cu_seqlens
    assert _varlen_call(d, total=-1) == 1 and _varlen_call(d, total=1 << 31) == 1  # ConfigError
    d.stride_n = 4 * 128 + 4  # token stride not a multiple of 8 elements
    assert _varlen_call(d) == 2
    d = A.AttentionConfig(3, 4, 512, 96).desc()
    assert _varlen_call(d) == 1  # head_dim
    d = A.AttentionConfig(3, 4, 512, 128).desc()
    assert A.lib().tkb_attn_bwd_varlen(ctypes.byref(d), 1 << 12, 100, *([None] * 10), 0, None) == 3


def test_varlen_python_mirror_rejects_cpu_tensors():
    torch = pytest.importorskip("torch")
    x = torch.zeros(10, 2, 64, dtype=torch.bfloat16)
    with pytest.raises(A.ConfigError):
        A.attention_fwd_varlen(x, x, x, torch.tensor([0, 10], dtype=torch.int32), 10)


def test_fastdiv_multiplier_is_exact():
    """The task decoders divide by launch constants through FastDiv (attn_common.cuh): the
    round-up multiplier m = ceil(2^(31 + ceil(log2 d)) / d), q = umulhi(n, m) >> (p - 32).
    Same arithmetic in Python: exact for every tested divisor over dividends up to 2^31 - 1."""
    import random

    def fastdiv(n, d):
        if d == 1:
            return n
        l = (d - 1).bit_length()  # ceil(log2 d)
        p = 31 + l
        m = ((1 << p) + d - 1) // d
        assert m < (1 << 32)
        return ((n * m) >> 32) >> (p - 32)

    rng = random.Random(7)
    divisors = list(range(1, 300)) + [2 ** k + o for k in range(2, 31) for o in (-1, 0, 1)] + \
        [rng.randrange(1, 2 ** 31) for _ in range(200)]
    for d in divisors:
        ns = [0, 1, d - 1, d, d + 1, 2 ** 31 - 1, 2 ** 31 - 2] + [rng.randrange(0, 2 ** 31) for _ in range(50)]
        for n in ns:
            if 0 <= n < 2 ** 31:
                assert fastdiv(n, d) == n // d, (n, d)


def test_workspace_bytes_grouped_query_split():
    """Grouped-query dK/dV with few kv heads splits the query heads over tasks (bwd_kv_split,
    attn_common.cuh: doubling while (kv blocks x B x Hkv) x split < 4 x 148) and reserves fp32
    dV / dK partials per chunk in the backward workspace."""
    def ws(B, H, hkv, N, D):
        d = A.AttentionConfig(B, H, N, D, kv_heads=hkv).desc()
        return A.lib().tkb_attn_bwd_workspace_bytes(ctypes.byref(d))

    base = lambda B, H, N: 2 * B * H * ((N + 127) // 128 * 128) * 4  # noqa: E731 - delta + lse2
    assert ws(2, 8, 8, 512, 128) == base(2, 8, 512)           # multi-head: no split
    # MQA, B=2, N=512: 4 kv blocks x 2 units = 8 tasks -> split 8 (the whole group)
    assert ws(2, 8, 1, 512, 128) == base(2, 8, 512) + 2 * 8 * 2 * 512 * 128 * 4
    # B=8 H=32 Hkv=1 N=4096: 32 x 8 = 256 tasks -> split 4 (256 x 4 >= 592)
    assert ws(8, 32, 1, 4096, 128) == base(8, 32, 4096) + 2 * 4 * 8 * 4096 * 128 * 4
    # plenty of kv heads: 16 x 64 x 8 = 8192 tasks -> no split
    assert ws(16, 64, 8, 1024, 64) == base(16, 64, 1024)
    # the Python helper takes kv_heads too
    assert A.bwd_workspace_bytes(2, 8, 512, 128, kv_heads=1) == ws(2, 8, 1, 512, 128)
    assert A.bwd_workspace_bytes(2, 8, 512, 128) == ws(2, 8, 8, 512, 128)


def test_fwd_task_tiles_knob_validates():
    assert A.lib().tkb_debug_set_fwd_task_tiles(3) == 1  # TKB_ERR_CONFIG
    assert A.lib().tkb_debug_set_fwd_task_tiles(-1) == 1
    for t in (1, 2, 0):
        assert A.lib().tkb_debug_set_fwd_task_tiles(t) == 0
