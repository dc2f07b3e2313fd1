// attn_common.cuh — parameter blocks shared by the C-ABI layer and the kernels.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

namespace tkb {

// Opt a kernel into `bytes` of dynamic shared memory on the CURRENT device. The attribute
// is per device (cuKernelSetAttribute takes a CUdevice), so it is tracked per device
// ordinal in a lock-free bit mask owned by the caller (one per kernel instantiation);
// concurrent first calls from several host threads both set it, which is idempotent.
template <class Kern>
inline int ensure_smem(Kern kern, int bytes, std::atomic<unsigned long long>& done_mask) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return (int)e;
    const unsigned long long bit = dev < 64 ? (1ull << dev) : 0ull;  // ordinals >= 64: set on every launch
    if (bit && (done_mask.load(std::memory_order_acquire) & bit)) return 0;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return (int)e;
    done_mask.fetch_or(bit, std::memory_order_release);
    return 0;
}

// Division by a launch-constant divisor without the integer-division sequence (whose
// MUFU.RCP queues behind the softmax warps' exponentials on the same SM sub-partition: a task
// decode cost ~1.2 k clk there). Round-up multiplier (Granlund-Montgomery, as CUTLASS's
// FastDivmod): q = umulhi(n, mul) >> shr, exact for 0 <= n < 2^31 and 1 <= d < 2^31.
struct FastDiv {
    uint32_t mul = 0, shr = 0, d = 1;
    FastDiv() = default;
    explicit FastDiv(uint32_t divisor) : d(divisor < 1 ? 1 : divisor) {
        if (d != 1) {
            uint32_t l = 0;
            while ((1ull << l) < d) ++l;  // ceil(log2 d)
            const uint32_t p = 31 + l;
            mul = (uint32_t)(((1ull << p) + d - 1) / d);
            shr = p - 32;
        }
    }
    __device__ __forceinline__ int div(int n) const {
        return d == 1 ? n : (int)(__umulhi((uint32_t)n, mul) >> shr);
    }
};

// Tile shapes (compile time; the reference's runtime AttentionConfig knobs
// kv_rows / qo_rows / num_workers, kernels.hpp:168-176, become these).
constexpr int kBlockM = 128;   // query rows per tcgen05 M tile (one softmax warpgroup)
constexpr int kBlockN = 128;   // key/value rows per KV tile
constexpr int kQStages = 2;    // query tiles per CTA (ping-pong softmax warpgroups)
constexpr int kRowsPerCta = kBlockM * kQStages;

// Variable-length batches (tkb_attn_fwd_varlen / tkb_attn_bwd_varlen): sequence b is rows
// [cu[b], cu[b+1]) of packed [T, H, D] tensors. Each sequence gets its own TMA maps
// ({D, n_b, H, 1} over base + cu[b] sn, written on the device by varlen_maps_kernel with
// tensormap.replace into the caller's workspace, [B][kMaps] CUtensorMaps): a tile past a
// sequence's end is zero-filled on load and clipped on store exactly like the ragged tail of
// a fixed-length head, so no tile reads or writes a neighbouring sequence's rows.
// Fixed-length problems (cu == nullptr): n = n_max, bcoord = batch, off = 0, maps = null
// (the kernel-parameter maps over [B, H, N, D]).
struct SeqView {
    int n;                    // rows of this sequence
    int bcoord;               // TMA outermost coordinate (batch; 0 with per-sequence maps)
    int off;                  // first packed row of the sequence (cu[b]; 0 fixed-length)
    const CUtensorMap* maps;  // this sequence's maps (varlen) or null
    // Run f(const CUtensorMap*) on map idx of this sequence (varlen) or on the kernel-parameter
    // map `fixed`. Two call sites, not one pointer select: a descriptor pointer that may be
    // either a parameter or a global address makes the compiler materialise the parameter's
    // address generically, and the fixed-length TMA through it faulted (illegal instruction).
    template <class F>
    __device__ __forceinline__ void with_map(const CUtensorMap& fixed, int idx, F&& f) const {
        if (maps != nullptr)
            f(maps + idx);
        else
            f(&fixed);
    }
};
__device__ __forceinline__ SeqView seq_view(const int* cu, const CUtensorMap* vmaps, int kmaps, int n_max, int b) {
    SeqView v;
    if (cu == nullptr) {
        v.n = n_max, v.bcoord = b, v.off = 0, v.maps = nullptr;
    } else {
        const int s0 = __ldg(cu + b), s1 = __ldg(cu + b + 1);
        v.n = s1 - s0, v.bcoord = 0, v.off = s0, v.maps = vmaps + (size_t)b * kmaps;
    }
    return v;
}
// per-sequence map slots
constexpr int kFwdMaps = 4;  // q, k, v, o
constexpr int kBwdMaps = 7;  // q, k, v, do, dq, dk, dv
enum { kMapQ = 0, kMapK = 1, kMapV = 2, kMapO = 3, kMapDo = 3, kMapDq = 4, kMapDk = 5, kMapDv = 6 };

// Builds [B][nmaps] per-sequence maps from host-encoded templates over the packed tensors
// ({D, n_max, H, 1}): base += cu[b] * row_bytes, rows = n_b.
struct VarlenMapTemplates {
    CUtensorMap tmpl[kBwdMaps];
    unsigned long long base[kBwdMaps];
    long long row_bytes[kBwdMaps];
    int nmaps;
};
int launch_varlen_maps(const VarlenMapTemplates& t, const int* cu, int batches, CUtensorMap* out, cudaStream_t stream);

struct FwdParams {
    CUtensorMap tm_q, tm_k, tm_v, tm_o;  // 4-D {D, N, H, B}, box {64, 128, 1, 1}, SW128
    float* lse;                          // [B*H, N] fp32, may be null
    const int* cu_seqlens;               // varlen: [B + 1] packed row offsets (null: fixed N)
    const CUtensorMap* vmaps;            // varlen: [B][kFwdMaps] per-sequence maps (workspace)
    int* sched;                          // persistent task counter pair (self-resetting)
    long long* trace;                    // optional per-role cycle timeline (tkb_debug_set_trace)
    int trace_every;
    int trace_slots;
    int n;                               // sequence length (varlen: the maximum)
    int heads;
    int group;                           // query heads per kv head (grouped-query attention; 1 = MHA)
    int bh;                              // batches * heads          (set by launch_attn_fwd)
    int m_blocks;                        // query blocks of task_tiles * 128 rows (set by launch_attn_fwd)
    int task_tiles;                      // query tiles per task: 2, or 1 when 2-tile tasks would
                                         //   leave SMs idle (set by launch_attn_fwd)
    int tasks;                           // bh * m_blocks            (set by launch_attn_fwd;
                                         //   tkb_attn_validate keeps B*H*ceil(N/128) < 2^31)
    int head_group;                      // heads per L2 group       (set by launch_attn_fwd)
    FastDiv fd_sec, fd_group, fd_grem, fd_heads;  // task decode divisors (set by launch_attn_fwd)
    float scale_log2;                    // softmax_scale * log2(e)
    // Fused rotary prologue (attn_fwd_template<D, Causal, true>): the two aux warps of every
    // CTA rotate 128-row blocks of Q and K from q_src / k_src into q_rot / k_rot (same
    // strides; tm_q / tm_k map the rotated copies) and publish each block with a flag set to
    // `epoch`; the load warp waits for a block's flag before its TMA reads it.
    const float* sin_tab;                // [N, D/2] fp32
    const float* cos_tab;
    const void* q_src;                   // bf16, strides q_sb / q_sh / q_sn
    const void* k_src;                   // bf16, strides k_sb / k_sh / k_sn
    void* q_rot;
    void* k_rot;
    long long q_sb, q_sh, q_sn, k_sb, k_sh, k_sn;
    unsigned* flags;                     // [B * Hkv * nq128] K blocks, then [B * H * nq128] Q blocks
    unsigned epoch;                      // this launch's flag value (never 0)
};

struct BwdParams {
    CUtensorMap tm_q, tm_k, tm_v, tm_do;  // 4-D {D, N, H, B}, box {64, 128, 1, 1}, SW128 (loads)
    CUtensorMap tm_dq, tm_dk, tm_dv;      // same layout (stores)
    CUtensorMap tm_q64, tm_do64;          // Q / dO with a {64, 64, 1, 1} box (CTA-pair query halves)
    const float* lse2;                    // [B*H, Npad] -L * log2(e); -inf on padded rows (workspace)
    const float* delta;                   // [B*H, Npad] rowsum(dO * O) (workspace)
    const int* cu_seqlens;                // varlen: [B + 1] packed row offsets (null: fixed N)
    const CUtensorMap* vmaps;             // varlen: [B][kBwdMaps] per-sequence maps (workspace)
    long long* trace;                     // optional per-role cycle timeline (tkb_debug_set_trace)
    int trace_every;                      // trace CTAs with linear id % trace_every == 0
    int trace_slots;
    int n;
    int n_pad;
    int heads;         // query heads
    int group;         // query heads per kv head (grouped-query attention; 1 = MHA)
    int bh;            // batches * heads (persistent task count = bh * n_pad / 128)
    int head_group;    // heads per L2 group of the persistent task order
    int num_sms;       // persistent grid size
    int pairs;         // D = 128: dK/dV on CTA pairs (attn_bwd_dkdv2_kernel)
    int kv_G;          // (batch, kv head) units per L2 group of the dK/dV task order
    int kv_units;      // dK/dV task units = B * Hkv * kv_split
    int kv_split;      // grouped-query: query-head chunks per (batch, kv head) (bwd_kv_split)
    float* dkv_part;   // kv_split > 1: fp32 dV / dK partials [2][kv_split][B * Hkv][n_pad][D] (workspace)
    // task decode divisors (set by the host: fill_bwd_divisors)
    FastDiv kv_sec, kv_g, kv_grem, kv_nq, kv_hkv, kv_c;  // dK/dV: G*nq, G, last-group size, nq, Hkv, split
    FastDiv q_sec, q_g, q_grem, q_heads;           // dQ: head_group*nq, head_group, last-group size, H
    void* dk;          // dK / dV base pointers and element strides (persistent dK/dV kernel:
    void* dv;          //   direct row stores from registers)
    long long kv_sb, kv_sh, kv_sn;
    void* dq;          // dQ base and element strides (dQ kernel: direct row stores)
    long long q_sb, q_sh, q_sn;
    int* sched;        // persistent task counter pair (self-resetting, lcsf::queue_exit)
    float scale;       // softmax_scale
    float scale_log2;  // softmax_scale * log2(e)
};

// Grouped-query dK/dV with few kv heads: a (kv block, kv head) task walks all `group` query
// heads, and with fewer than ~4 such tasks per SM the last wave leaves SMs idle (MQA causal: one
// j = 0 task holds 32 query heads' work). The query heads are then split into kv_split chunks,
// each task writes fp32 dV / dK partials and a reduce kernel sums them in chunk order
// (deterministic). A function of the problem alone (B200's 148 SMs), so the workspace size does
// not depend on the device; never for variable-length batches.
constexpr int kSplitSms = 148;
inline int bwd_kv_split(long long units, int group, int nq, bool varlen) {
    if (varlen || group < 2) return 1;
    const long long tasks = (long long)nq * units;
    int c = 1;
    while (c < group && group % (2 * c) == 0 && tasks * c < 4ll * kSplitSms) c *= 2;
    return c;
}

// The backward's task-decode divisors (after bh, heads, group, n_pad, head_group, num_sms and
// kv_split are set).
inline void fill_bwd_divisors(BwdParams& p) {
    const int nq = p.n_pad / 128;
    const int hkv = p.heads / p.group;
    const int hb = hkv * (p.bh / p.heads) * p.kv_split;  // task units: (batch, kv head, chunk)
    const long long tasks = (long long)nq * hb;
    // few tasks per SM (or a grouped-query split, which only happens then): one group spanning
    // everything, i.e. longest-first over the whole causal queue
    int G = (tasks < 4ll * p.num_sms || p.kv_split > 1) ? hb : p.head_group / (p.group > 1 ? p.group : 1);
    G = G < 1 ? 1 : (G > hb ? hb : G);
    p.kv_G = G;
    p.kv_units = hb;
    p.kv_sec = FastDiv((uint32_t)(G * nq));
    p.kv_g = FastDiv((uint32_t)G);
    p.kv_grem = FastDiv((uint32_t)(hb % G ? hb % G : G));
    p.kv_nq = FastDiv((uint32_t)nq);
    p.kv_hkv = FastDiv((uint32_t)hkv);
    p.kv_c = FastDiv((uint32_t)p.kv_split);
    p.q_sec = FastDiv((uint32_t)(p.head_group * nq));
    p.q_g = FastDiv((uint32_t)p.head_group);
    p.q_grem = FastDiv((uint32_t)(p.bh % p.head_group ? p.bh % p.head_group : p.head_group));
    p.q_heads = FastDiv((uint32_t)p.heads);
}

// Per-role cycle timeline (the Timeline of lcsf.hpp:165-224, recorded on the device):
// trace[slot][role][iter][event] = clock64() - CTA start, roles MMA / COMPUTE / REDUCE.
constexpr int kTraceIters = 32;
constexpr int kTraceEvents = 8;
constexpr int kTraceRoles = 4;

// GEMM (gemm_sm100.cu): C[m, n] = A[m, k] B[k, n], bf16 row-major, fp32 accumulation.
struct GemmParams {
    CUtensorMap tm_a;  // 2-D {k, m}, box {64, 128}, SW128
    CUtensorMap tm_b;  // 2-D {n, k}, box {64, 64}, SW128 (MN-major B panels)
    CUtensorMap tm_c;  // 2-D {n, m}, box {64, 128}, SW128
    int m, n, k;
    int super_m;       // supergroup height of the task order (grid.hpp:28-47)
};
int launch_gemm(const GemmParams& p, int num_sms, cudaStream_t stream);

// Rotary embedding (rotary_sm100.cu): up to two tensors (Q, K) per launch.
namespace rope {
struct Tensor {
    const void* x;       // bf16 [B, heads, N, hd]
    void* o;             // bf16, may alias x
    int64_t xb, xh, xn;  // element strides of x
    int64_t ob, oh, on;  // element strides of o
    int heads;
    int64_t items;       // B * heads * N * (hd / 16); 0 = unused slot
};
struct Params {
    Tensor t[2];
    const float* sin_tab;  // [N, hd/2] fp32
    const float* cos_tab;
    int n, hd;
};
}  // namespace rope
int launch_rotary(const rope::Params& p, int num_sms, cudaStream_t stream);

// Launchers (return cudaError_t as int).
int launch_attn_fwd(int head_dim, bool causal, FwdParams p, int batches, int num_sms, cudaStream_t stream,
                    bool rope = false);

}  // namespace tkb
