"""Host-side mirror of the reference's attention interface, over the C ABI.

Reference (kittensim, /root/reference/proj/include/kittensim):
  AttentionConfig + validate()      kernels.hpp:168-203  -> AttentionConfig below
  AttentionGlobals {q,k,v,o}        kernels.hpp:205-213  -> torch tensors [B,H,N,D] bf16
  attention_fwd_kernel + execute_functional              -> attention_fwd()
  exception taxonomy                errors.hpp:9-46      -> the classes below
New (absent from the reference): causal masking, saved L,
attention_bwd() producing dQ/dK/dV from L.

Every call goes to the sm_100a kernels in libtkb.so through ctypes; there is no
CPU or PyTorch fallback — a missing library or a non-B200 device raises.
"""
import ctypes
import math
from dataclasses import dataclass
from typing import Optional

from . import _lib

# ---------------------------------------------------------------- errors.hpp:9-46


class Error(RuntimeError):
    """kittensim::Error"""


class ConfigError(Error):
    """kittensim::ConfigError — bad shape / dim / non-finite input."""


class ShapeError(Error):
    """kittensim::ShapeError — layout not supported."""


class BoundsError(Error):
    """kittensim::BoundsError — null pointer / workspace too small."""


class ContractViolation(Error):
    """kittensim::ContractViolation"""


class UnsupportedDevice(Error):
    """Device is not a B200 (sm_100)."""


class CudaError(Error):
    """CUDA runtime / driver error."""


_CODES = {1: ConfigError, 2: ShapeError, 3: BoundsError, 4: UnsupportedDevice, 5: CudaError, 6: ContractViolation}


class AttnDesc(ctypes.Structure):
    """tkb_attn_desc (include/tkb_attn.h)."""

    _fields_ = [
        ("batches", ctypes.c_int32),
        ("heads", ctypes.c_int32),
        ("seq", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("causal", ctypes.c_int32),
        ("check_finite", ctypes.c_int32),
        ("softmax_scale", ctypes.c_float),
        ("kv_heads", ctypes.c_int32),
        ("stride_b", ctypes.c_int64),
        ("stride_h", ctypes.c_int64),
        ("stride_n", ctypes.c_int64),
        ("kv_stride_b", ctypes.c_int64),
        ("kv_stride_h", ctypes.c_int64),
        ("kv_stride_n", ctypes.c_int64),
    ]


class GemmDesc(ctypes.Structure):
    """tkb_gemm_desc (include/tkb_attn.h)."""

    _fields_ = [("m", ctypes.c_int32), ("n", ctypes.c_int32), ("k", ctypes.c_int32), ("super_m", ctypes.c_int32),
                ("lda", ctypes.c_int64), ("ldb", ctypes.c_int64), ("ldc", ctypes.c_int64)]


_VP = ctypes.c_void_p
_SIGS = {
    "tkb_attn_desc_init": (None, [ctypes.POINTER(AttnDesc)] + [ctypes.c_int32] * 5),
    "tkb_attn_validate": (ctypes.c_int, [ctypes.POINTER(AttnDesc)]),
    "tkb_attn_fwd": (ctypes.c_int, [ctypes.POINTER(AttnDesc), _VP, _VP, _VP, _VP, _VP, _VP]),
    "tkb_attn_bwd_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(AttnDesc)]),
    "tkb_attn_fwd_rotary_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(AttnDesc)]),
    "tkb_attn_fwd_rotary": (ctypes.c_int, [ctypes.POINTER(AttnDesc)] + [_VP] * 10 + [ctypes.c_size_t, _VP]),
    "tkb_attn_bwd": (ctypes.c_int, [ctypes.POINTER(AttnDesc)] + [_VP] * 10 + [ctypes.c_size_t, _VP]),
    "tkb_attn_fwd_varlen_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(AttnDesc)]),
    "tkb_attn_bwd_varlen_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(AttnDesc)]),
    "tkb_attn_fwd_varlen": (ctypes.c_int, [ctypes.POINTER(AttnDesc), _VP, ctypes.c_int64] + [_VP] * 6
                            + [ctypes.c_size_t, _VP]),
    "tkb_attn_bwd_varlen": (ctypes.c_int, [ctypes.POINTER(AttnDesc), _VP, ctypes.c_int64] + [_VP] * 10
                            + [ctypes.c_size_t, _VP]),
    "tkb_rotary": (ctypes.c_int, [ctypes.POINTER(AttnDesc), _VP, _VP, _VP, _VP, _VP]),
    "tkb_rotary_qk": (ctypes.c_int, [ctypes.POINTER(AttnDesc), _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "tkb_gemm_validate": (ctypes.c_int, [ctypes.POINTER(GemmDesc)]),
    "tkb_gemm": (ctypes.c_int, [ctypes.POINTER(GemmDesc), _VP, _VP, _VP, _VP]),
    "tkb_shard_range": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]),
    "tkb_device_init": (ctypes.c_int, [ctypes.c_int]),
    "tkb_debug_map_cache_stats": (ctypes.c_int, [ctypes.POINTER(ctypes.c_ulonglong), ctypes.POINTER(ctypes.c_ulonglong)]),
    "tkb_last_launch_count": (ctypes.c_int, []),
    "tkb_debug_set_trace": (ctypes.c_int, [_VP, ctypes.c_int, ctypes.c_int]),
    "tkb_debug_set_bwd_phases": (ctypes.c_int, [ctypes.c_int]),
    "tkb_set_bwd_pairs": (ctypes.c_int, [ctypes.c_int]),
    "tkb_debug_set_fwd_task_tiles": (ctypes.c_int, [ctypes.c_int]),
    "tkb_last_error": (ctypes.c_char_p, []),
    "tkb_abi_version": (ctypes.c_int, []),
}


def lib():
    L = _lib.load()
    if not getattr(L, "_tkb_typed", False):
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        L._tkb_typed = True
    return L


def exported_symbols():
    return list(_SIGS)


def _check(rc):
    if rc != 0:
        msg = lib().tkb_last_error().decode(errors="replace")
        raise _CODES.get(rc, Error)(msg)


# ---------------------------------------------------------------- kernels.hpp:168-203


@dataclass
class AttentionConfig:
    """The reference AttentionConfig minus its CPU-model knobs (kv_rows, qo_rows,
    num_workers are compile-time tile shapes of the sm_100a kernels)."""

    batches: int = 1
    heads: int = 1
    seq: int = 0
    head_dim: int = 0
    causal: bool = False
    softmax_scale: Optional[float] = None
    check_finite: bool = False
    kv_heads: int = 0  # grouped-query attention: 0 = heads

    def temperature_scale(self) -> float:
        """tau = softmax_scale * log2(e) (kernels.hpp:184-186)."""
        s = self.softmax_scale if self.softmax_scale else 1.0 / math.sqrt(self.head_dim)
        return s * 1.44269504089

    def desc(self, strides=None, kv_strides=None) -> AttnDesc:
        d = AttnDesc()
        lib().tkb_attn_desc_init(ctypes.byref(d), self.batches, self.heads, self.seq, self.head_dim,
                                 int(bool(self.causal)))
        d.softmax_scale = float(self.softmax_scale or 0.0)
        d.check_finite = int(bool(self.check_finite))
        d.kv_heads = int(self.kv_heads or 0)
        if strides is not None:
            d.stride_b, d.stride_h, d.stride_n = strides
        if kv_strides is not None:
            d.kv_stride_b, d.kv_stride_h, d.kv_stride_n = kv_strides
        return d

    def validate(self):
        _check(lib().tkb_attn_validate(ctypes.byref(self.desc())))


def _stream(torch_mod, dev):
    return torch_mod.cuda.current_stream(dev).cuda_stream


def _bhnd(t, name):
    if t.dim() != 4:
        raise ShapeError(f"{name} must be [B, H, N, D]")
    if t.stride(3) != 1:
        raise ShapeError(f"{name}: head_dim must be contiguous")
    return t.stride(0), t.stride(1), t.stride(2)


def _check_kv(q, k, v):
    """q [B, H, N, D]; k, v [B, Hkv, N, D] with H % Hkv == 0 (Hkv == H: multi-head)."""
    if k.shape != v.shape:
        raise ShapeError("k and v must have the same shape")
    B, H, N, D = q.shape
    if k.dim() != 4 or k.shape[0] != B or k.shape[2] != N or k.shape[3] != D:
        raise ShapeError("k, v must be [B, Hkv, N, D] matching q's B, N, D")
    hkv = k.shape[1]
    if hkv < 1 or H % hkv:
        raise ConfigError(f"heads ({H}) must be a multiple of kv heads ({hkv})")
    kst = _bhnd(k, "k")
    if _bhnd(v, "v") != kst:
        raise ShapeError("k and v must share strides")
    return hkv, kst


def _tables(sin_tab, cos_tab, N, D, device):
    import torch

    for t in (sin_tab, cos_tab):
        if not t.is_cuda or t.dtype != torch.float32 or tuple(t.shape) != (N, D // 2) or not t.is_contiguous():
            raise ShapeError("sin / cos tables must be contiguous fp32 CUDA tensors [N, D/2]")
        if t.device != device:
            raise ConfigError("sin / cos tables must be on the tensors' device")


def _bf16_cuda(t, name, device=None):
    import torch

    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.bfloat16:
        raise ConfigError(f"{name} must be a bf16 CUDA tensor (no CPU fallback)")
    if device is not None and t.device != device:
        raise ConfigError(f"{name} must be on {device}")


def _out_like(t, name, ref_shape, ref_strides, device):
    """A caller-supplied output: bf16, on `device`, with the expected shape and strides."""
    _bf16_cuda(t, name, device)
    if tuple(t.shape) != tuple(ref_shape) or _bhnd(t, name) != ref_strides:
        raise ShapeError(f"{name} must have shape {tuple(ref_shape)} and the matching input's strides")


def rotary(x, sin_tab, cos_tab, out=None):
    """Rotary position embedding (the reference rotary_kernel, kernels.hpp:357-513): pairs
    (x[..., p, i], x[..., p, i + D/2]) rotated by the [N, D/2] sin / cos table angles."""
    import torch

    _bf16_cuda(x, "x")
    st = _bhnd(x, "x")
    B, H, N, D = x.shape
    _tables(sin_tab, cos_tab, N, D, x.device)
    if out is None:
        out = torch.empty_strided(x.shape, x.stride(), dtype=torch.bfloat16, device=x.device)
    else:
        _out_like(out, "out", x.shape, st, x.device)
    d = AttentionConfig(B, H, N, D).desc(strides=st)
    _check(lib().tkb_rotary(ctypes.byref(d), x.data_ptr(), sin_tab.data_ptr(), cos_tab.data_ptr(), out.data_ptr(),
                            _stream(torch, x.device)))
    return out


def rotary_qk(q, k, sin_tab, cos_tab):
    """The attention prologue: rotated copies of Q and K from one launch."""
    import torch

    _bf16_cuda(q, "q")
    _bf16_cuda(k, "k", q.device)
    st = _bhnd(q, "q")
    kst = _bhnd(k, "k")
    B, H, N, D = q.shape
    if k.shape[0] != B or k.shape[2] != N or k.shape[3] != D:
        raise ShapeError("k must be [B, Hkv, N, D] matching q's B, N, D")
    hkv = k.shape[1]
    if hkv < 1 or H % hkv:
        raise ConfigError(f"heads ({H}) must be a multiple of kv heads ({hkv})")
    _tables(sin_tab, cos_tab, N, D, q.device)
    qr = torch.empty_strided(q.shape, q.stride(), dtype=torch.bfloat16, device=q.device)
    kr = torch.empty_strided(k.shape, k.stride(), dtype=torch.bfloat16, device=q.device)
    d = AttentionConfig(B, H, N, D, kv_heads=hkv).desc(strides=st, kv_strides=kst)
    _check(lib().tkb_rotary_qk(ctypes.byref(d), q.data_ptr(), k.data_ptr(), sin_tab.data_ptr(), cos_tab.data_ptr(),
                               qr.data_ptr(), kr.data_ptr(), _stream(torch, q.device)))
    return qr, kr


_rope_ws = {}


def _rope_workspace(device, stream, nbytes):
    """The fused rotary forward's block flags (cleared by each call on its stream; one buffer
    per (device, stream), so calls sharing it are stream-ordered as the ABI requires)."""
    import torch

    key = (device, stream)
    ws = _rope_ws.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=device)
        _rope_ws[key] = ws
    return ws


def attention_fwd(q, k, v, causal=False, softmax_scale=None, out=None, lse=None, return_lse=True,
                  check_finite=False, rotary_tables=None, return_rotated=False):
    """O = softmax(scale * Q K^T [causal]) V on the B200; returns (O, L) with L fp32 [B, H, N].
    k, v may carry fewer heads than q (grouped-query / multi-query attention).
    rotary_tables=(sin, cos) ([N, D/2] fp32) applies the rotary embedding to Q and K inside
    the same launch (tkb_attn_fwd_rotary); return_rotated=True also returns the rotated
    (Q, K) — the tensors the backward differentiates against."""
    import torch

    _bf16_cuda(q, "q")
    _bf16_cuda(k, "k", q.device)
    _bf16_cuda(v, "v", q.device)
    st = _bhnd(q, "q")
    hkv, kst = _check_kv(q, k, v)
    B, H, N, D = q.shape
    if out is None:
        out = torch.empty_strided(q.shape, q.stride(), dtype=torch.bfloat16, device=q.device)
    else:
        _out_like(out, "out", q.shape, st, q.device)
    if (return_lse or rotary_tables is not None) and lse is None:
        lse = torch.empty((B, H, N), dtype=torch.float32, device=q.device)
    if lse is not None:
        _check_lse(lse, B, H, N, q.device)
    cfg = AttentionConfig(B, H, N, D, causal, softmax_scale, check_finite, kv_heads=hkv)
    d = cfg.desc(strides=st, kv_strides=kst)
    stream = _stream(torch, q.device)
    if rotary_tables is not None:
        sin_tab, cos_tab = rotary_tables
        _tables(sin_tab, cos_tab, N, D, q.device)
        q_rot = torch.empty_strided(q.shape, q.stride(), dtype=torch.bfloat16, device=q.device)
        k_rot = torch.empty_strided(k.shape, k.stride(), dtype=torch.bfloat16, device=q.device)
        nbytes = int(lib().tkb_attn_fwd_rotary_workspace_bytes(ctypes.byref(d)))
        ws = _rope_workspace(q.device, stream, nbytes)
        _check(lib().tkb_attn_fwd_rotary(ctypes.byref(d), q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                         sin_tab.data_ptr(), cos_tab.data_ptr(), q_rot.data_ptr(), k_rot.data_ptr(),
                                         out.data_ptr(), lse.data_ptr(), ws.data_ptr(), ws.numel(), stream))
        res = (out, lse) if return_lse else (out,)
        if return_rotated:
            res = res + (q_rot, k_rot)
        return res if len(res) > 1 else res[0]
    _check(lib().tkb_attn_fwd(ctypes.byref(d), q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                              lse.data_ptr() if lse is not None else None, stream))
    return (out, lse) if return_lse else out


def _check_lse(lse, B, H, N, device):
    import torch

    if (not isinstance(lse, torch.Tensor) or not lse.is_cuda or lse.device != device or lse.dtype != torch.float32
            or tuple(lse.shape) != (B, H, N) or not lse.is_contiguous()):
        raise ShapeError(f"lse must be a contiguous fp32 CUDA tensor [B, H, N] = {(B, H, N)} on {device}")


def bwd_workspace_bytes(B, H, N, D, causal=False, kv_heads=None):
    """Bytes of the backward's workspace (tkb_attn_bwd_workspace_bytes); with few kv heads the
    grouped-query dK/dV split adds fp32 partials, so pass kv_heads for k / v with fewer heads."""
    cfg = AttentionConfig(B, H, N, D, causal, kv_heads=kv_heads or H)
    return int(lib().tkb_attn_bwd_workspace_bytes(ctypes.byref(cfg.desc())))


def attention_bwd(q, k, v, o, dout, lse, causal=False, softmax_scale=None, dq=None, dk=None, dv=None,
                  workspace=None, check_finite=False):
    """dQ, dK, dV from the saved L (deterministic). With grouped-query k/v, dK/dV sum the
    contributions of every query head of the group (in TMEM, no atomics)."""
    import torch

    for t, name in ((q, "q"), (k, "k"), (v, "v"), (o, "o"), (dout, "dout")):
        _bf16_cuda(t, name, q.device)
    st = _bhnd(q, "q")
    hkv, kst = _check_kv(q, k, v)
    for t, name in ((o, "o"), (dout, "dout")):
        if t.shape != q.shape or _bhnd(t, name) != st:
            raise ShapeError(f"{name} must match q's shape and strides")
    B, H, N, D = q.shape
    _check_lse(lse, B, H, N, q.device)
    if dq is None:
        dq = torch.empty_strided(q.shape, q.stride(), dtype=torch.bfloat16, device=q.device)
    if dk is None:
        dk = torch.empty_strided(k.shape, k.stride(), dtype=torch.bfloat16, device=q.device)
    if dv is None:
        dv = torch.empty_strided(k.shape, k.stride(), dtype=torch.bfloat16, device=q.device)
    _out_like(dq, "dq", q.shape, st, q.device)
    _out_like(dk, "dk", k.shape, kst, q.device)
    _out_like(dv, "dv", k.shape, kst, q.device)
    cfg = AttentionConfig(B, H, N, D, causal, softmax_scale, check_finite, kv_heads=hkv)
    d = cfg.desc(strides=st, kv_strides=kst)
    ws_bytes = int(lib().tkb_attn_bwd_workspace_bytes(ctypes.byref(d)))
    if workspace is None:
        workspace = torch.empty(ws_bytes, dtype=torch.uint8, device=q.device)
    elif (not workspace.is_cuda or workspace.device != q.device or not workspace.is_contiguous()
          or workspace.numel() * workspace.element_size() < ws_bytes):
        raise BoundsError(f"workspace must be a contiguous CUDA buffer of >= {ws_bytes} bytes on {q.device}")
    _check(lib().tkb_attn_bwd(ctypes.byref(d), q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                              dout.data_ptr(), lse.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(),
                              workspace.data_ptr(), ws_bytes, _stream(torch, q.device)))
    return dq, dk, dv


# ------------------------------------------------- variable-length batches


def _thd(t, name):
    """A packed token-major [T, H, D] tensor: (head stride, token stride), D contiguous."""
    if t.dim() != 3:
        raise ShapeError(f"{name} must be [T, H, D] (packed variable-length batch)")
    if t.stride(2) != 1:
        raise ShapeError(f"{name}: head_dim must be contiguous")
    return t.stride(1), t.stride(0)


def _varlen_args(q, k, v, cu_seqlens, max_seqlen):
    import torch

    _bf16_cuda(q, "q")
    _bf16_cuda(k, "k", q.device)
    _bf16_cuda(v, "v", q.device)
    qs = _thd(q, "q")
    ks = _thd(k, "k")
    if _thd(v, "v") != ks or tuple(v.shape) != tuple(k.shape):
        raise ShapeError("k and v must share shape and strides")
    T, H, D = q.shape
    if k.shape[0] != T or k.shape[2] != D:
        raise ShapeError("k, v must be [T, Hkv, D] matching q's T and D")
    hkv = k.shape[1]
    if hkv < 1 or H % hkv:
        raise ConfigError(f"heads ({H}) must be a multiple of kv heads ({hkv})")
    if (not isinstance(cu_seqlens, torch.Tensor) or not cu_seqlens.is_cuda or cu_seqlens.device != q.device
            or cu_seqlens.dtype != torch.int32 or cu_seqlens.dim() != 1 or not cu_seqlens.is_contiguous()
            or cu_seqlens.numel() < 2):
        raise ShapeError("cu_seqlens must be a contiguous int32 CUDA tensor [B + 1] on q's device")
    B = cu_seqlens.numel() - 1
    if int(max_seqlen) < 1:
        raise ConfigError("max_seqlen must be >= 1")
    return T, B, H, D, hkv, qs, ks


def _varlen_desc(B, H, max_seqlen, D, causal, softmax_scale, check_finite, hkv, qs, ks):
    cfg = AttentionConfig(B, H, int(max_seqlen), D, causal, softmax_scale, check_finite, kv_heads=hkv)
    d = cfg.desc()
    d.stride_b, d.stride_h, d.stride_n = 0, qs[0], qs[1]
    d.kv_stride_b, d.kv_stride_h, d.kv_stride_n = 0, ks[0], ks[1]
    return d


def _workspace(workspace, nbytes, device):
    import torch

    if workspace is None:
        return torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
    if (not workspace.is_cuda or workspace.device != device or not workspace.is_contiguous()
            or workspace.numel() * workspace.element_size() < nbytes or workspace.data_ptr() % 128):
        raise BoundsError(f"workspace must be a contiguous 128-byte aligned CUDA buffer of >= {nbytes} bytes "
                          f"on {device}")
    return workspace


def attention_fwd_varlen(q, k, v, cu_seqlens, max_seqlen, causal=False, softmax_scale=None, out=None, lse=None,
                         return_lse=True, check_finite=False, workspace=None):
    """Forward over a packed variable-length batch: sequence b is rows [cu[b], cu[b+1]) of
    q [T, H, D] and k, v [T, Hkv, D]; it attends only to itself (causal: within the
    sequence). Returns (O [T, H, D], L fp32 [B, H, max_seqlen]); L rows past a sequence's
    length are not written. max_seqlen must be >= every length (tkb_attn_fwd_varlen)."""
    import torch

    T, B, H, D, hkv, qs, ks = _varlen_args(q, k, v, cu_seqlens, max_seqlen)
    if out is None:
        out = torch.empty_strided(q.shape, q.stride(), dtype=torch.bfloat16, device=q.device)
    else:
        _bf16_cuda(out, "out", q.device)
        if tuple(out.shape) != tuple(q.shape) or _thd(out, "out") != qs:
            raise ShapeError("out must match q's shape and strides")
    if return_lse and lse is None:
        lse = torch.empty((B, H, int(max_seqlen)), dtype=torch.float32, device=q.device)
    if lse is not None:
        _check_lse(lse, B, H, int(max_seqlen), q.device)
    d = _varlen_desc(B, H, max_seqlen, D, causal, softmax_scale, check_finite, hkv, qs, ks)
    ws_bytes = int(lib().tkb_attn_fwd_varlen_workspace_bytes(ctypes.byref(d)))
    workspace = _workspace(workspace, ws_bytes, q.device)
    _check(lib().tkb_attn_fwd_varlen(ctypes.byref(d), cu_seqlens.data_ptr(), T, q.data_ptr(), k.data_ptr(),
                                     v.data_ptr(), out.data_ptr(), lse.data_ptr() if lse is not None else None,
                                     workspace.data_ptr(), ws_bytes, _stream(torch, q.device)))
    return (out, lse) if return_lse else out


def attention_bwd_varlen(q, k, v, o, dout, lse, cu_seqlens, max_seqlen, causal=False, softmax_scale=None,
                         dq=None, dk=None, dv=None, workspace=None, check_finite=False):
    """dQ, dK, dV of a packed variable-length batch from the saved L [B, H, max_seqlen]
    (tkb_attn_bwd_varlen); deterministic like attention_bwd."""
    import torch

    T, B, H, D, hkv, qs, ks = _varlen_args(q, k, v, cu_seqlens, max_seqlen)
    for t, name in ((o, "o"), (dout, "dout")):
        _bf16_cuda(t, name, q.device)
        if tuple(t.shape) != tuple(q.shape) or _thd(t, name) != qs:
            raise ShapeError(f"{name} must match q's shape and strides")
    _check_lse(lse, B, H, int(max_seqlen), q.device)
    if dq is None:
        dq = torch.empty_strided(q.shape, q.stride(), dtype=torch.bfloat16, device=q.device)
    if dk is None:
        dk = torch.empty_strided(k.shape, k.stride(), dtype=torch.bfloat16, device=q.device)
    if dv is None:
        dv = torch.empty_strided(k.shape, k.stride(), dtype=torch.bfloat16, device=q.device)
    for t, name, ref, rs in ((dq, "dq", q, qs), (dk, "dk", k, ks), (dv, "dv", k, ks)):
        _bf16_cuda(t, name, q.device)
        if tuple(t.shape) != tuple(ref.shape) or _thd(t, name) != rs:
            raise ShapeError(f"{name} must match the shape and strides of its input")
    d = _varlen_desc(B, H, max_seqlen, D, causal, softmax_scale, check_finite, hkv, qs, ks)
    ws_bytes = int(lib().tkb_attn_bwd_varlen_workspace_bytes(ctypes.byref(d)))
    workspace = _workspace(workspace, ws_bytes, q.device)
    _check(lib().tkb_attn_bwd_varlen(ctypes.byref(d), cu_seqlens.data_ptr(), T, q.data_ptr(), k.data_ptr(),
                                     v.data_ptr(), o.data_ptr(), dout.data_ptr(), lse.data_ptr(), dq.data_ptr(),
                                     dk.data_ptr(), dv.data_ptr(), workspace.data_ptr(), ws_bytes,
                                     _stream(torch, q.device)))
    return dq, dk, dv


# ------------------------------------------------- PyTorch autograd (a training-step caller)


def _autograd_fn():
    import torch

    class _Attention(torch.autograd.Function):
        """O = attention(q, k, v) whose backward is tkb_attn_bwd from the saved L. With rotary
        tables the forward is the fused rotary launch (tkb_attn_fwd_rotary), the backward runs
        on the rotated Q / K it returned and takes dQ / dK back through the rotation's transpose
        — the rotation by -theta, i.e. tkb_rotary_qk with the sin table negated."""

        @staticmethod
        def forward(ctx, q, k, v, causal, softmax_scale, sin_tab, cos_tab):
            ctx.rope = sin_tab is not None
            if ctx.rope:
                o, lse, q, k = attention_fwd(q, k, v, causal=causal, softmax_scale=softmax_scale,
                                             rotary_tables=(sin_tab, cos_tab), return_rotated=True)
                ctx.save_for_backward(q, k, v, o, lse, sin_tab, cos_tab)
            else:
                o, lse = attention_fwd(q, k, v, causal=causal, softmax_scale=softmax_scale)
                ctx.save_for_backward(q, k, v, o, lse)
            ctx.causal, ctx.softmax_scale = causal, softmax_scale
            return o

        @staticmethod
        def backward(ctx, do):
            q, k, v, o, lse = ctx.saved_tensors[:5]
            do = do if do.stride() == o.stride() else do.contiguous()
            if do.stride() != q.stride():  # dO must share q's layout: bring both to contiguous
                q, o, do = q.contiguous(), o.contiguous(), do.contiguous()
            dq, dk, dv = attention_bwd(q, k, v, o, do, lse, causal=ctx.causal, softmax_scale=ctx.softmax_scale)
            if ctx.rope:  # d(R x)/dx = R: the gradient goes back through R^T = R(-theta)
                sin_tab, cos_tab = ctx.saved_tensors[5:]
                dq, dk = rotary_qk(dq, dk, -sin_tab, cos_tab)
            return dq, dk, dv, None, None, None, None

    return _Attention


_ATTN_FN = None


def attention(q, k, v, causal=False, softmax_scale=None, rotary_tables=None):
    """Differentiable attention for PyTorch code: O = softmax(scale q k^T [causal]) v with the
    B200 forward, and a backward (dQ, dK, dV) from the saved L — one tkb_attn_fwd launch
    forward, tkb_attn_bwd backward; bf16 CUDA tensors [B, H, N, D] (k, v may be grouped-query).
    rotary_tables=(sin, cos) ([N, D/2] fp32) rotates q and k inside the forward launch; their
    gradients come back through the inverse rotation (one tkb_rotary_qk launch)."""
    global _ATTN_FN
    if _ATTN_FN is None:
        _ATTN_FN = _autograd_fn()
    sin_tab, cos_tab = rotary_tables if rotary_tables is not None else (None, None)
    return _ATTN_FN.apply(q, k, v, bool(causal), softmax_scale, sin_tab, cos_tab)


@dataclass
class GemmConfig:
    """The reference GemmConfig (kernels.hpp:23-46) minus its CPU-model knobs (m_block /
    n_block are the compile-time 128 x 256 tile); super_m keeps its meaning (grid.hpp:28-47)."""

    m: int = 0
    n: int = 0
    k: int = 0
    super_m: int = 12

    def desc(self, lda=0, ldb=0, ldc=0) -> GemmDesc:
        return GemmDesc(self.m, self.n, self.k, self.super_m, lda, ldb, ldc)

    def validate(self):
        _check(lib().tkb_gemm_validate(ctypes.byref(self.desc())))


def gemm(a, b, out=None, super_m=12):
    """C = A B (bf16 row-major [M, K] x [K, N] -> [M, N], fp32 accumulation) on tcgen05."""
    import torch

    for t, name in ((a, "a"), (b, "b")):
        if not t.is_cuda or t.dtype != torch.bfloat16 or t.dim() != 2 or t.stride(1) != 1:
            raise ConfigError(f"{name} must be a row-major bf16 CUDA matrix")
    M, K = a.shape
    if b.shape[0] != K:
        raise ShapeError("inner dimensions differ")
    N = b.shape[1]
    if out is None:
        out = torch.empty((M, N), dtype=torch.bfloat16, device=a.device)
    elif tuple(out.shape) != (M, N) or out.stride(1) != 1 or out.dtype != torch.bfloat16:
        raise ShapeError("out must be a row-major bf16 [M, N] matrix")
    d = GemmConfig(M, N, K, super_m).desc(a.stride(0), b.stride(0), out.stride(0))
    _check(lib().tkb_gemm(ctypes.byref(d), a.data_ptr(), b.data_ptr(), out.data_ptr(), _stream(torch, a.device)))
    return out


def shard_range(units, rank, world):
    """Contiguous balanced [begin, end) of the flattened batch x head grid for `rank`."""
    b, e = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().tkb_shard_range(units, rank, world, ctypes.byref(b), ctypes.byref(e)))
    return b.value, e.value


def debug_set_trace(buf=None, every=1, slots=0):
    """Enable the backward kernel's per-role cycle timeline into a device int64 tensor
    [slots, 4, 32, 8] (debug only); buf=None disables."""
    lib().tkb_debug_set_trace(buf.data_ptr() if buf is not None else None, every, slots)


def debug_set_fwd_task_tiles(tiles=0):
    """Forward query tiles per task for later calls from this thread: 0 = by problem size, 1 or 2
    forced (tkb_debug_set_fwd_task_tiles; the results are the same bits)."""
    _check(lib().tkb_debug_set_fwd_task_tiles(int(tiles)))


def debug_set_bwd_phases(mask=7):
    """Profiling only: run a subset of the backward stages (1 prep, 2 dK/dV, 4 dQ)."""
    lib().tkb_debug_set_bwd_phases(int(mask))


def set_bwd_pairs(on=True):
    """D = 128 backward: run dK/dV on CTA pairs (cta_group::2 clusters) instead of one CTA
    per kv block. Applies to this host thread's later calls; results match the oracle
    either way."""
    lib().tkb_set_bwd_pairs(1 if on else 0)


def device_init(device=0):
    """One-time per-device library state (the schedulers' counter pool); optional."""
    _check(lib().tkb_device_init(int(device)))


def map_cache_stats():
    """(hits, misses) of this thread's TMA descriptor cache."""
    h, m = ctypes.c_ulonglong(), ctypes.c_ulonglong()
    lib().tkb_debug_map_cache_stats(ctypes.byref(h), ctypes.byref(m))
    return h.value, m.value


def last_launch_count():
    return int(lib().tkb_last_launch_count())
