"""ctypes front-end of the CPU oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module, and only as the checker or the timed CPU
baseline. The product package (paper_2410_20399_b200) never imports it.

  liboracle.so          fp64 restatement (oracle/attn_oracle.cpp), built by oracle/Makefile
  _ref/libkittensim_ref.so  the UNMODIFIED reference attention path compiled from
                        /root/reference/proj/include (oracle/ref_shim.cpp); prebuilt here,
                        travels to the GPU box (git-ignored, not gpurun-ignored)
"""
import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libkittensim_ref.so")

_F = ctypes.POINTER(ctypes.c_float)
_D = ctypes.POINTER(ctypes.c_double)
_cache = {}


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _ptr(a, t):
    return a.ctypes.data_as(t)


def lib():
    if "o" not in _cache:
        if not os.path.exists(ORACLE_SO):
            build()
        L = ctypes.CDLL(ORACLE_SO)
        L.tkb_oracle_fill.argtypes = [ctypes.c_uint32, ctypes.c_float, ctypes.c_float, ctypes.c_int, _F,
                                      ctypes.c_int64]
        L.tkb_oracle_round_bf16.argtypes = [ctypes.c_float]
        L.tkb_oracle_round_bf16.restype = ctypes.c_float
        L.tkb_oracle_attn_fwd.argtypes = [_F, _F, _F, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_double, _D, _D, ctypes.c_int]
        L.tkb_oracle_attn_bwd.argtypes = [_F, _F, _F, _F, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_double, _D, _D, _D, ctypes.c_int]
        L.tkb_oracle_attn_fwd_rows.argtypes = L.tkb_oracle_attn_fwd.argtypes
        _I = ctypes.POINTER(ctypes.c_int)
        L.tkb_oracle_attn_bwd_sampled.argtypes = [_F, _F, _F, _F, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                                  ctypes.c_int, ctypes.c_double, _I, ctypes.c_int, _I, ctypes.c_int,
                                                  _D, _D, _D, ctypes.c_int]
        L.tkb_oracle_rotary.argtypes = [_F, _F, _F, ctypes.c_int64, ctypes.c_int, ctypes.c_int, _D]
        L.tkb_oracle_gemm.argtypes = [_F, _F, ctypes.c_int, ctypes.c_int, ctypes.c_int, _D, ctypes.c_int]
        _cache["o"] = L
    return _cache["o"]


def ref_available():
    return os.path.exists(REF_SO)


def ref_lib():
    if "r" not in _cache:
        L = ctypes.CDLL(REF_SO)
        L.kref_validate.argtypes = [ctypes.c_int] * 6 + [ctypes.c_char_p, ctypes.c_int]
        L.kref_kv_tile_rows.argtypes = [ctypes.c_int]
        L.kref_temperature_scale.argtypes = [ctypes.c_int]
        L.kref_temperature_scale.restype = ctypes.c_double
        L.kref_round_to_bf16.argtypes = [ctypes.c_float]
        L.kref_round_to_bf16.restype = ctypes.c_float
        L.kref_attention_fwd.argtypes = [ctypes.c_int] * 8 + [ctypes.c_uint64, _F, _F, _F, _F, ctypes.c_char_p,
                                                              ctypes.c_int]
        L.kref_oracle_attention.argtypes = [_D, _D, _D, ctypes.c_int, ctypes.c_int, ctypes.c_int, _D]
        L.kref_fill.argtypes = [ctypes.c_uint32, ctypes.c_float, ctypes.c_float, ctypes.c_int, _F, ctypes.c_int64]
        L.kref_oracle_rotary.argtypes = [_D, _D, _D, ctypes.c_int, ctypes.c_int, _D]
        L.kref_rotary.argtypes = [ctypes.c_int] * 5 + [_F, _F, _F, _F, ctypes.c_char_p, ctypes.c_int]
        L.kref_oracle_gemm.argtypes = [_D, _D, ctypes.c_int, ctypes.c_int, ctypes.c_int, _D]
        L.kref_gemm.argtypes = [ctypes.c_int] * 7 + [_F, _F, _F, ctypes.c_char_p, ctypes.c_int]
        _I = ctypes.POINTER(ctypes.c_int)
        L.kref_supergroup_order.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _I, _I]
        _cache["r"] = L
    return _cache["r"]


def threads():
    return max(1, os.cpu_count() or 1)


# ------------------------------------------------------------------ generators


def fill(seed, total, bf16=True, lo=-1.0, hi=1.0):
    """fill_uniform (report.hpp:57-61) over one mt19937(seed) stream of `total` values."""
    out = np.empty(total, dtype=np.float32)
    lib().tkb_oracle_fill(seed, lo, hi, int(bf16), _ptr(out, _F), total)
    return out


def qkv(seed, B, H, N, D, bf16=True, scale_qk=1.0):
    """Q then K then V from one stream, as the reference tests do (test_kernels.cpp:134-137).
    scale_qk > 1 gives the 'peaky' distribution; values stay bf16-exact
    for power-of-two scales."""
    n = B * H * N * D
    a = fill(seed, 3 * n, bf16).reshape(3, B, H, N, D)
    q, k, v = a[0].copy(), a[1].copy(), a[2].copy()
    if scale_qk != 1.0:
        q *= scale_qk
        k *= scale_qk
    return q, k, v


# ------------------------------------------------------------------ oracle


def attn_fwd(q, k, v, causal=False, scale=None, nthreads=None):
    """fp64 O [.., N, D] and L [.., N] for float32 inputs of shape [..., N, D]."""
    q = np.ascontiguousarray(q, dtype=np.float32)
    k = np.ascontiguousarray(k, dtype=np.float32)
    v = np.ascontiguousarray(v, dtype=np.float32)
    N, D = q.shape[-2:]
    heads = int(np.prod(q.shape[:-2])) if q.ndim > 2 else 1
    scale = scale if scale else 1.0 / np.sqrt(D)
    o = np.empty(q.shape, dtype=np.float64)
    lse = np.empty(q.shape[:-1], dtype=np.float64)
    lib().tkb_oracle_attn_fwd(_ptr(q, _F), _ptr(k, _F), _ptr(v, _F), heads, N, D, int(causal), scale, _ptr(o, _D),
                              _ptr(lse, _D), nthreads or threads())
    return o, lse


def attn_bwd(q, k, v, dout, causal=False, scale=None, nthreads=None):
    q, k, v, dout = (np.ascontiguousarray(x, dtype=np.float32) for x in (q, k, v, dout))
    N, D = q.shape[-2:]
    heads = int(np.prod(q.shape[:-2])) if q.ndim > 2 else 1
    scale = scale if scale else 1.0 / np.sqrt(D)
    dq, dk, dv = (np.empty(q.shape, dtype=np.float64) for _ in range(3))
    lib().tkb_oracle_attn_bwd(_ptr(q, _F), _ptr(k, _F), _ptr(v, _F), _ptr(dout, _F), heads, N, D, int(causal), scale,
                              _ptr(dq, _D), _ptr(dk, _D), _ptr(dv, _D), nthreads or threads())
    return dq, dk, dv


def attn_fwd_rows(q, k, v, causal=False, scale=None, nthreads=None):
    """attn_fwd with every (head, row) an independent work item (long sequences, few heads)."""
    q, k, v = (np.ascontiguousarray(x, dtype=np.float32) for x in (q, k, v))
    N, D = q.shape[-2:]
    heads = int(np.prod(q.shape[:-2])) if q.ndim > 2 else 1
    scale = scale if scale else 1.0 / np.sqrt(D)
    o = np.empty(q.shape, dtype=np.float64)
    lse = np.empty(q.shape[:-1], dtype=np.float64)
    lib().tkb_oracle_attn_fwd_rows(_ptr(q, _F), _ptr(k, _F), _ptr(v, _F), heads, N, D, int(causal), scale,
                                   _ptr(o, _D), _ptr(lse, _D), nthreads or threads())
    return o, lse


def attn_bwd_sampled(q, k, v, dout, qrows, krows, causal=False, scale=None, nthreads=None):
    """dQ at query rows `qrows` and dK / dV at key rows `krows` of every head ([..., len, D])."""
    q, k, v, dout = (np.ascontiguousarray(x, dtype=np.float32) for x in (q, k, v, dout))
    N, D = q.shape[-2:]
    lead = q.shape[:-2]
    heads = int(np.prod(lead)) if q.ndim > 2 else 1
    scale = scale if scale else 1.0 / np.sqrt(D)
    qr = np.ascontiguousarray(qrows, dtype=np.int32)
    kr = np.ascontiguousarray(krows, dtype=np.int32)
    _I = ctypes.POINTER(ctypes.c_int)
    dq = np.empty(lead + (len(qr), D), dtype=np.float64)
    dk = np.empty(lead + (len(kr), D), dtype=np.float64)
    dv = np.empty(lead + (len(kr), D), dtype=np.float64)
    lib().tkb_oracle_attn_bwd_sampled(_ptr(q, _F), _ptr(k, _F), _ptr(v, _F), _ptr(dout, _F), heads, N, D,
                                      int(causal), scale, _ptr(qr, _I), len(qr), _ptr(kr, _I), len(kr), _ptr(dq, _D),
                                      _ptr(dk, _D), _ptr(dv, _D), nthreads or threads())
    return dq, dk, dv


# ------------------------------------------------------------------ reference (oracle/_ref)


def ref_attention_fwd(q, k, v, kv_rows=0, workers=0, bf16=True, threaded=True, seed=0):
    """The reference kernel path execute_functional(attention_fwd_kernel(cfg, g)) on [B,H,N,D] fp32."""
    B, H, N, D = q.shape
    q, k, v = (np.ascontiguousarray(x, dtype=np.float32) for x in (q, k, v))
    o = np.empty_like(q)
    err = ctypes.create_string_buffer(512)
    rc = ref_lib().kref_attention_fwd(B, H, N, D, kv_rows, workers, int(bf16), int(threaded), seed, _ptr(q, _F),
                                      _ptr(k, _F), _ptr(v, _F), _ptr(o, _F), err, 512)
    if rc != 0:
        raise RuntimeError(f"reference error {rc}: {err.value.decode()}")
    return o


def ref_oracle_attention(q, k, v):
    """The reference fp64 oracle_attention for one head [N, D]."""
    q, k, v = (np.ascontiguousarray(x, dtype=np.float64) for x in (q, k, v))
    out = np.empty_like(q)
    rc = ref_lib().kref_oracle_attention(_ptr(q, _D), _ptr(k, _D), _ptr(v, _D), q.shape[0], k.shape[0], q.shape[1],
                                         _ptr(out, _D))
    assert rc == 0
    return out


def ref_fill(seed, total, bf16=True, lo=-1.0, hi=1.0):
    out = np.empty(total, dtype=np.float32)
    ref_lib().kref_fill(seed, lo, hi, int(bf16), _ptr(out, _F), total)
    return out


# ------------------------------------------------------------------ metrics


def max_abs(got, ref):
    return float(np.max(np.abs(np.asarray(got, dtype=np.float64) - ref))) if np.size(ref) else 0.0


def rel_l2(got, ref):
    ref = np.asarray(ref, dtype=np.float64)
    den = np.linalg.norm(ref)
    return float(np.linalg.norm(np.asarray(got, dtype=np.float64) - ref) / (den if den > 0 else 1.0))


# ------------------------------------------------------------------ rotary / GEMM


def rotary(x, sin_tab, cos_tab):
    """fp64 oracle_rotary (oracles.hpp:66-90) on x [..., N, hd] with [N, hd/2] tables."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    n, hd = x.shape[-2:]
    s = np.ascontiguousarray(sin_tab, dtype=np.float32)
    c = np.ascontiguousarray(cos_tab, dtype=np.float32)
    out = np.empty(x.shape, dtype=np.float64)
    lib().tkb_oracle_rotary(_ptr(x, _F), _ptr(s, _F), _ptr(c, _F), x.size // hd, n, hd, _ptr(out, _D))
    return out


def gemm(a, b, nthreads=None):
    """fp64 oracle_gemm (oracles.hpp:17-30): C = A B for row-major A [M, K], B [K, N]."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    m, k = a.shape
    n = b.shape[1]
    c = np.empty((m, n), dtype=np.float64)
    lib().tkb_oracle_gemm(_ptr(a, _F), _ptr(b, _F), m, n, k, _ptr(c, _D), nthreads or threads())
    return c


def ref_rotary_oracle(x, sin_tab, cos_tab):
    """The reference's own oracle_rotary on one [N, hd] head (oracle/_ref)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    n, hd = x.shape
    out = np.empty_like(x)
    rc = ref_lib().kref_oracle_rotary(_ptr(x, _D), _ptr(np.ascontiguousarray(sin_tab, np.float64), _D),
                                      _ptr(np.ascontiguousarray(cos_tab, np.float64), _D), n, hd, _ptr(out, _D))
    assert rc == 0
    return out


def ref_rotary(x, sin_tab, cos_tab, workers=4):
    """The reference rotary_kernel through execute_functional (fp32), x [B, H, N, hd]."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    B, H, N, hd = x.shape
    out = np.empty_like(x)
    err = ctypes.create_string_buffer(256)
    rc = ref_lib().kref_rotary(B, H, N, hd, workers, _ptr(x, _F), _ptr(np.ascontiguousarray(sin_tab, np.float32), _F),
                               _ptr(np.ascontiguousarray(cos_tab, np.float32), _F), _ptr(out, _F), err, 256)
    if rc:
        raise RuntimeError(err.value.decode())
    return out


def ref_gemm_oracle(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    m, k = a.shape
    n = b.shape[1]
    c = np.empty((m, n), dtype=np.float64)
    assert ref_lib().kref_oracle_gemm(_ptr(a, _D), _ptr(b, _D), m, n, k, _ptr(c, _D)) == 0
    return c


def ref_gemm(a, b, m_block=2, n_block=4, super_m=12, bf16=False):
    """The reference gemm_kernel through execute_functional."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    m, k = a.shape
    n = b.shape[1]
    c = np.empty((m, n), dtype=np.float32)
    err = ctypes.create_string_buffer(256)
    rc = ref_lib().kref_gemm(m, n, k, m_block, n_block, super_m, int(bf16), _ptr(a, _F), _ptr(b, _F), _ptr(c, _F),
                             err, 256)
    if rc:
        raise RuntimeError(err.value.decode())
    return c


def ref_supergroup_order(r_blocks, c_blocks, super_m):
    rows = np.empty(r_blocks * c_blocks, dtype=np.int32)
    cols = np.empty_like(rows)
    _I = ctypes.POINTER(ctypes.c_int)
    assert ref_lib().kref_supergroup_order(r_blocks, c_blocks, super_m, rows.ctypes.data_as(_I),
                                           cols.ctypes.data_as(_I)) == 0
    return rows, cols


def _npy_tool():
    return os.path.join(HERE, "_ref", "npy_tool")


def ref_save_npy(path, arr):
    """Write float32 `arr` with the reference's own .npy writer (npy.hpp:18-49)."""
    import subprocess
    import tempfile

    a = np.ascontiguousarray(arr, dtype=np.float32)
    with tempfile.NamedTemporaryFile(suffix=".bin") as f:
        a.tofile(f.name)
        subprocess.run([_npy_tool(), "save", f.name, path] + [str(d) for d in a.shape], check=True)


def ref_load_npy(path):
    """Read a float32 .npy with the reference's own reader (npy.hpp:51-87) -> (data, shape)."""
    import subprocess
    import tempfile

    with tempfile.NamedTemporaryFile(suffix=".bin") as f:
        r = subprocess.run([_npy_tool(), "load", path, f.name], check=True, capture_output=True, text=True)
        shape = tuple(int(x) for x in r.stdout.split())
        return np.fromfile(f.name, dtype=np.float32).reshape(shape), shape
