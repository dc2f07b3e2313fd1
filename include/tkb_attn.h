/*
 * tkb_attn.h — C ABI of the B200-native (sm_100a) attention hot path.
 *
 * This is the drop-in boundary for the reference's attention entry points
 * (reference = kittensim, /root/reference/proj/include/kittensim):
 *
 *   tkb_attn_fwd    replaces  attention_fwd_kernel(cfg, globals)      kernels.hpp:250-343
 *                   + execute_functional(spec, pipeline_cfg, opts)   lcsf.hpp:779-819
 *                   + attention_pipeline_config(cfg)                 kernels.hpp:345-355
 *                   (paper entry: lcf::kernel<attn_fwd_template<D>>)
 *   tkb_attn_validate replaces AttentionConfig::validate()            kernels.hpp:188-202
 *   tkb_attn_bwd    new: the reference has no backward; it follows
 *                   the restated oracle (oracle/attn_oracle.cpp) — dQ/dK/dV from saved L
 *   error codes     mirror the exception taxonomy                     errors.hpp:9-46
 *
 * Conventions
 *   - Tensors are row-major [B, H, N, D] bf16 (optionally strided over B, H, N;
 *     D must be contiguous), as GlobalTensor::index (tiles.hpp:106-108); with
 *     grouped-query attention (desc.kv_heads) k/v/dk/dv are [B, Hkv, N, D].
 *   - O is bf16 (the reference keeps fp32 O, kernels.hpp:212).
 *   - lse is fp32 [B, H, N], contiguous: L_i = ln sum_j exp(scale * q_i . k_j)
 *     over the unmasked keys (natural log).
 *   - causal: key j is visible to query i iff j <= i (top-left aligned).
 *   - All entry points are asynchronous on `stream` (a cudaStream_t), never
 *     throw, and are safe to call from several host threads, on any mix of
 *     devices and streams. The last error message of the calling thread is
 *     returned by tkb_last_error().
 *   - Allocation: the library owns one 64 KB block per device (the persistent
 *     schedulers' task counters, one slot per stream), made by tkb_device_init()
 *     or by the first call on that device; nothing else is ever allocated.
 *     Call tkb_device_init() up front to keep the first call capturable in a
 *     CUDA graph. Calls captured into a graph get a counter slot of their own
 *     for the graph's lifetime; a graph must not be replayed concurrently with
 *     itself (its kernels share that slot). check_finite is not capturable.
 *   - check_finite (desc) reads its result back and synchronises the stream.
 */
#ifndef TKB_ATTN_H
#define TKB_ATTN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TKB_ABI_VERSION 4

#if defined(__GNUC__)
#define TKB_API __attribute__((visibility("default")))
#else
#define TKB_API
#endif

/* Error codes (errors.hpp:9-46). */
enum tkb_status {
    TKB_OK = 0,
    TKB_ERR_CONFIG = 1,      /* ConfigError: bad shape/dim, non-finite input when checked */
    TKB_ERR_SHAPE = 2,       /* ShapeError: strides / layout not supported            */
    TKB_ERR_BOUNDS = 3,      /* BoundsError: null pointer / workspace too small        */
    TKB_ERR_UNSUPPORTED = 4, /* device is not sm_100 (B200)                            */
    TKB_ERR_CUDA = 5,        /* CUDA runtime / driver error                            */
    TKB_ERR_CONTRACT = 6     /* ContractViolation: internal invariant broken           */
};

/* Problem descriptor — the AttentionConfig of kernels.hpp:168-176, minus the
 * CPU-model knobs (kv_rows/qo_rows/num_workers are compile-time tile shapes here). */
typedef struct tkb_attn_desc {
    int32_t batches;      /* B >= 1 */
    int32_t heads;        /* H >= 1 */
    int32_t seq;          /* N >= 1 (query and key/value length) */
    int32_t head_dim;     /* D in {64, 128} */
    int32_t causal;       /* 0 / 1 */
    int32_t check_finite; /* 1: scan inputs first and fail with TKB_ERR_CONFIG on inf/nan
                             (kernels.hpp:277-284); synchronises the stream */
    float softmax_scale;  /* 0: D^-1/2; must be finite and >= 0 */
    int32_t kv_heads;     /* Hkv: 0 = H (multi-head); H % Hkv == 0 (grouped-query, Hkv = 1: multi-query).
                             k/v/dk/dv are [B, Hkv, N, D]; query head h reads kv head h / (H / Hkv) */
    /* element strides of q/o/do/dq; 0 = contiguous [B,H,N,D] */
    int64_t stride_b;
    int64_t stride_h;
    int64_t stride_n;
    /* element strides of k/v/dk/dv; all 0 = contiguous [B,Hkv,N,D] (or q's strides when Hkv == H) */
    int64_t kv_stride_b;
    int64_t kv_stride_h;
    int64_t kv_stride_n;
} tkb_attn_desc;

/* Fill `desc` with a contiguous problem and default scale. */
TKB_API void tkb_attn_desc_init(tkb_attn_desc* desc, int32_t batches, int32_t heads, int32_t seq, int32_t head_dim,
                        int32_t causal);

/* AttentionConfig::validate(): TKB_OK or TKB_ERR_CONFIG/SHAPE with a message. No device work. */
TKB_API int tkb_attn_validate(const tkb_attn_desc* desc);

/* Forward: o = softmax(scale * q k^T [+ causal mask]) v ; lse saved for the backward.
 * lse may be NULL (inference). */
TKB_API int tkb_attn_fwd(const tkb_attn_desc* desc, const void* q, const void* k, const void* v, void* o, float* lse,
                 void* stream);

/* Rotary embedding fused into the forward (one launch): q and k are rotated by the fp32
 * [seq, head_dim/2] sin / cos tables (the pair (x[p][i], x[p][i + D/2]), as tkb_rotary) into
 * q_rot ([B, H, N, D], q's strides) and k_rot ([B, Hkv, N, D], k's strides) — which the
 * backward then takes as its q / k — while the attention of the rotated q, k and v runs in
 * the same kernel. The workspace (tkb_attn_fwd_rotary_workspace_bytes) holds per-block
 * flags, cleared on the stream before each launch (any initial contents; capturable in a
 * CUDA graph); calls that share a workspace must be stream-ordered. */
TKB_API size_t tkb_attn_fwd_rotary_workspace_bytes(const tkb_attn_desc* desc);
TKB_API int tkb_attn_fwd_rotary(const tkb_attn_desc* desc, const void* q, const void* k, const void* v,
                                const float* sin_tab, const float* cos_tab, void* q_rot, void* k_rot, void* o,
                                float* lse, void* workspace, size_t workspace_bytes, void* stream);

/* Bytes of caller-provided device workspace the backward needs: two fp32 [B*H, N_pad]
 * vectors, delta = rowsum(dO * O) and -L log2(e) (N_pad = N rounded up to 128). */
TKB_API size_t tkb_attn_bwd_workspace_bytes(const tkb_attn_desc* desc);

/* Backward from the saved lse: dq, dk, dv (bf16, same layout as q). Deterministic:
 * repeated calls on the same inputs produce bit-identical outputs. */
TKB_API int tkb_attn_bwd(const tkb_attn_desc* desc, const void* q, const void* k, const void* v, const void* o,
                 const void* dout, const float* lse, void* dq, void* dk, void* dv, void* workspace,
                 size_t workspace_bytes, void* stream);

/* Variable-length batches (the paper guards out-of-bounds rows,
 * PAPER.md:1017,1056): B sequences of different lengths packed token-major. Sequence b is
 * rows [cu_seqlens[b], cu_seqlens[b+1]) of
 *   q, o, dout, dq   [T, H, D]    (desc.stride_n / stride_h: token / head strides, 0 = H*D / D)
 *   k, v, dk, dv     [T, Hkv, D]  (desc.kv_stride_n / kv_stride_h, 0 = Hkv*D / D)
 * with T = total_tokens >= cu_seqlens[B]; desc.batches = B, desc.seq = the maximum length
 * (every cu_seqlens[b+1] - cu_seqlens[b] must be <= desc.seq; 0 is allowed); stride_b and
 * kv_stride_b must be 0. cu_seqlens: int32 device array [B + 1], non-decreasing, cu[0] = 0.
 * Each sequence attends only to itself (causal: top-left aligned within the sequence). Every
 * sequence gets its own TMA maps (built on the device into the workspace, one extra small
 * launch), so a tile never reads or writes a neighbouring sequence's rows: rows past a
 * sequence's end are zero-filled on load and clipped on store. lse is fp32 [B, H, desc.seq];
 * rows past a sequence's length are left untouched. Workspaces: 128-byte aligned, of
 * tkb_attn_fwd_varlen_workspace_bytes / tkb_attn_bwd_varlen_workspace_bytes(desc) bytes
 * (no zero-fill needed; calls sharing one must be stream-ordered). Results equal the
 * fixed-length entry points run on each sequence alone, bit for bit. With desc.check_finite
 * the call also reads cu_seqlens back and rejects bad offsets (TKB_ERR_CONFIG / _BOUNDS);
 * otherwise they are preconditions. */
TKB_API size_t tkb_attn_fwd_varlen_workspace_bytes(const tkb_attn_desc* desc);
TKB_API int tkb_attn_fwd_varlen(const tkb_attn_desc* desc, const int32_t* cu_seqlens, int64_t total_tokens,
                                const void* q, const void* k, const void* v, void* o, float* lse, void* workspace,
                                size_t workspace_bytes, void* stream);
TKB_API size_t tkb_attn_bwd_varlen_workspace_bytes(const tkb_attn_desc* desc);
TKB_API int tkb_attn_bwd_varlen(const tkb_attn_desc* desc, const int32_t* cu_seqlens, int64_t total_tokens,
                                const void* q, const void* k, const void* v, const void* o, const void* dout,
                                const float* lse, void* dq, void* dk, void* dv, void* workspace,
                                size_t workspace_bytes, void* stream);

/* Rotary position embedding (replaces rotary_kernel, kernels.hpp:357-513; oracle
 * oracles.hpp:66-90): for position p and i < D/2 the pair (x[p][i], x[p][i + D/2]) is
 * rotated by the angle whose sin / cos are sin_tab / cos_tab [seq, D/2] (fp32, contiguous,
 * shared by every batch and head). x, out: [B, H, N, D] bf16 with desc's strides; out may
 * alias x. D must be a multiple of 16 here (any seq). The rotation's transpose — the
 * backward of the rotary prologue, taking dQ / dK of the rotated Q / K back to the inputs —
 * is the same call with sin_tab negated (rotation by -angle). */
TKB_API int tkb_rotary(const tkb_attn_desc* desc, const void* x, const float* sin_tab, const float* cos_tab,
                       void* out, void* stream);

/* The attention prologue: Q ([B, H, N, D]) and K ([B, Hkv, N, D], desc.kv_heads / kv strides)
 * rotated in one launch into q_out / k_out (may alias q / k). */
TKB_API int tkb_rotary_qk(const tkb_attn_desc* desc, const void* q, const void* k, const float* sin_tab,
                          const float* cos_tab, void* q_out, void* k_out, void* stream);

/* GEMM on the same tcgen05 / TMA machinery (replaces gemm_kernel, kernels.hpp:21-164;
 * oracle oracles.hpp:17-30): C[m, n] = A[m, k] B[k, n], bf16 row-major, fp32 accumulation,
 * bf16 C. Tasks (128 x 256 blocks of C) run in the reference's supergrouped order
 * (grid.hpp:28-47). Leading dimensions in elements, 0 = dense; multiples of 8. */
typedef struct tkb_gemm_desc {
    int32_t m, n, k;
    int32_t super_m; /* supergroup height (GemmConfig::super_m, kernels.hpp:29); 0 = 12 */
    int64_t lda, ldb, ldc;
} tkb_gemm_desc;

TKB_API int tkb_gemm_validate(const tkb_gemm_desc* desc);
TKB_API int tkb_gemm(const tkb_gemm_desc* desc, const void* a, const void* b, void* c, void* stream);

/* Multi-GPU sharding of the flattened batch x head grid:
 * contiguous, balanced [begin, end) of `units` for `rank` of `world`. No collective. */
TKB_API int tkb_shard_range(int64_t units, int32_t rank, int32_t world, int64_t* begin, int64_t* end);

/* One-time per-device state (SM count, the schedulers' counter pool). Optional: the first
 * call on a device does it otherwise. Thread-safe. */
TKB_API int tkb_device_init(int device);

/* Debug timeline of the kernels (the reference's Timeline, lcsf.hpp:165-224): device
 * buffer of slots x 4 roles x 32 iterations x 8 events int64 cycle stamps; the backward
 * traces every `every`-th work item, the persistent forward every `every`-th CTA.
 * NULL disables. Applies to later calls from the calling host thread only. */
TKB_API int tkb_debug_set_trace(void* device_buf, int every, int slots);

/* Debug / profiling: run only some backward stages (bit 0 prep, bit 1 dK/dV kernel,
 * bit 2 dQ kernel; default 7). Results are only complete with 7. Applies to later calls
 * from the calling host thread only. */
TKB_API int tkb_debug_set_bwd_phases(int mask);

/* Backward dK/dV kernel selection at D = 128 (calling host thread only): 0 = one CTA
 * per kv block (default), 1 = CTA pairs (clusters of 2, tcgen05 cta_group::2, M = 256
 * MMAs over two kv blocks; half the per-SM operand traffic). Same results, bit for bit
 * within each variant's own summation order. */
TKB_API int tkb_set_bwd_pairs(int on);

/* Debug / testing: query tiles per forward task (calling host thread only). 0 (default) picks
 * by problem size — two 128-row tiles sharing each K / V block, or one when two-tile tasks
 * would leave SMs idle; 1 or 2 force it. Results are the same bits either way. */
TKB_API int tkb_debug_set_fwd_task_tiles(int tiles);

/* Hits / misses of the calling thread's TMA descriptor cache (debug, tests). */
TKB_API int tkb_debug_map_cache_stats(unsigned long long* hits, unsigned long long* misses);

/* Number of kernels the last successful fwd / bwd call on this thread launched. */
TKB_API int tkb_last_launch_count(void);

TKB_API const char* tkb_last_error(void);
TKB_API int tkb_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TKB_ATTN_H */
