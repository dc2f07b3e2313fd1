// attn_fwd_sm100.cu — attention forward for B200 (sm_100a): TMA -> tcgen05 -> TMEM.
//
// Reference: kittensim attention_fwd_kernel (kernels.hpp:250-343) and the
// paper's H100 listing attn_fwd_template<D>. Same math
// (online softmax in the exp2 domain with tau = scale * log2 e, fp32 row
// normaliser summed over fp32 P, bf16 P into the PV product, kernels.hpp:
// 315-332), re-built for Blackwell as a warp-specialised CTA — the LCSF
// template (lcsf.hpp:112-161) in hardware:
//
//   warp 8      LOAD     (producer worker): TMA Q once, then K_i / V_i into an
//                        N-slot SMEM ring guarded by full/empty mbarriers
//   warp 9      MMA      (consumer, tensor part): one thread issues
//                        S_s = Q_s K_i^T (SS, both K-major) and
//                        O_s += P_s V_i (TS: P from TMEM, V MN-major)
//   warps 0-3   SOFTMAX0 (consumer, query tile 0: rows q0 .. q0+127)
//   warps 4-7   SOFTMAX1 (consumer, query tile 1: rows q0+128 .. q0+255)
//                        each thread owns one query row: tcgen05.ld of S,
//                        row max, exp2, row sum, bf16 P written back into TMEM
//                        (aliasing the upper half of S), lazy O rescale,
//                        then the FINISH stage: O / l -> bf16 -> SMEM -> TMA
//                        store, and L = ln2 * (m + log2 l).
//
// TMEM (512 columns): S0 [0,128) S1 [128,256) O0 [256,256+D) O1 [256+D,256+2D);
// P_s = bf16 pairs in columns [S_s+64, S_s+128).
//
// Tensor-core ordering: tcgen05.mma ops of one thread execute in issue order,
// so issuing PV_{i-1}(s) before QK_i(s) makes "S_i(s) full" imply "PV_{i-1}(s)
// done": the softmax may then rescale O_s and overwrite P_s safely.
#include <cuda.h>
#include <cuda_runtime.h>

#include "attn_common.cuh"
#include "tkb/tcgen05.cuh"
#include "tkb/tma.cuh"

namespace tkb {
namespace fwd {

template <int D>
struct Cfg {
    static constexpr int kAtoms = D / 64;                 // 128-byte-wide column blocks
    static constexpr int kAtomBytes = kBlockM * 128;      // one atom of a 128-row tile
    static constexpr int kTileBytes = kBlockM * D * 2;    // one 128 x D bf16 tile
    static constexpr int kKvSlots = (D == 128) ? 4 : 8;
    static constexpr int kSmemQ = kQStages * kTileBytes;
    static constexpr int kSmemKv = kKvSlots * kTileBytes;
    static constexpr int kSmemBytes = kSmemQ + kSmemKv + 1024;  // + alignment slack
    static __device__ __forceinline__ constexpr uint32_t tmem_s(int s) { return s * 128u; }
    static __device__ __forceinline__ constexpr uint32_t tmem_o(int s) { return 256u + s * D; }
    static constexpr int kThreads = 320;
    static constexpr int kWarpLoad = 8;
    static constexpr int kWarpMma = 9;
};

constexpr float kRescaleThreshold = 8.0f;  // log2 units: defer O rescale while max grows < 2^8
constexpr float kLn2 = 0.69314718055994530942f;

TKB_DEVICE void advance(int& slot, uint32_t& phase, int nslots) {
    if (++slot == nslots) {
        slot = 0;
        phase ^= 1u;
    }
}

template <int D, bool CAUSAL>
__global__ void __launch_bounds__(320, 1) attn_fwd_kernel(const __grid_constant__ FwdParams p) {
    using C = Cfg<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;
    uint8_t* sKV = smem + C::kSmemQ;

    __shared__ mbarrier q_full[kQStages], s_full[kQStages], p_full[kQStages], o_full[kQStages];
    __shared__ mbarrier kv_full[C::kKvSlots], kv_empty[C::kKvSlots];
    __shared__ uint32_t tmem_slot;

    const int warp = warpid();
    const int lane = laneid();
    const int mblk = CAUSAL ? (int)(gridDim.x - 1 - blockIdx.x) : (int)blockIdx.x;  // heavy causal tiles first
    const int head = blockIdx.y;
    const int batch = blockIdx.z;
    const int q0 = mblk * kRowsPerCta;
    const int n = p.n;
    int nkv = (n + kBlockN - 1) / kBlockN;
    if (CAUSAL) {
        const int last_row = min(q0 + kRowsPerCta, n) - 1;
        nkv = min(nkv, last_row / kBlockN + 1);
    }

    if (warp == C::kWarpLoad && lane == 0) {
        for (int s = 0; s < kQStages; ++s) {
            mbar_init(&q_full[s], 1);
            mbar_init(&s_full[s], 1);
            mbar_init(&p_full[s], WARPGROUP_THREADS);
            mbar_init(&o_full[s], 1);
        }
        for (int i = 0; i < C::kKvSlots; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        fence_barrier_init();
        tma::prefetch_desc(&p.tm_q);
        tma::prefetch_desc(&p.tm_k);
        tma::prefetch_desc(&p.tm_v);
        tma::prefetch_desc(&p.tm_o);
    }
    if (warp == C::kWarpMma) tmem::alloc<512>(&tmem_slot);
    tmem::fence_before();
    __syncthreads();
    tmem::fence_after();
    const uint32_t tbase = tmem_slot;

    if (warp == C::kWarpLoad) {
        // ----------------------------- LOAD (LCSF load stage) -----------------------------
        if (lane == 0) {
            const uint64_t pol_q = tma::policy_evict_first();
            const uint64_t pol_kv = tma::policy_evict_last();
            for (int s = 0; s < kQStages; ++s) {
                mbar_arrive_expect_tx(&q_full[s], C::kTileBytes);
                for (int a = 0; a < C::kAtoms; ++a)
                    tma::load_4d(sQ + s * C::kTileBytes + a * C::kAtomBytes, &p.tm_q, &q_full[s], a * 64,
                                 q0 + s * kBlockM, head, batch, pol_q);
            }
            int slot = 0;
            uint32_t phase = 0;
            for (int i = 0; i < nkv; ++i) {
#pragma unroll
                for (int kv = 0; kv < 2; ++kv) {
                    mbar_wait(&kv_empty[slot], phase ^ 1u);
                    mbar_arrive_expect_tx(&kv_full[slot], C::kTileBytes);
                    for (int a = 0; a < C::kAtoms; ++a)
                        tma::load_4d(sKV + slot * C::kTileBytes + a * C::kAtomBytes, kv == 0 ? &p.tm_k : &p.tm_v,
                                     &kv_full[slot], a * 64, i * kBlockN, head, batch, pol_kv);
                    advance(slot, phase, C::kKvSlots);
                }
            }
        }
    } else if (warp == C::kWarpMma) {
        // ----------------------------- MMA (LCSF compute, tensor part) ---------------------
        if (lane == 0) {
            constexpr uint32_t idesc_qk = umma::idesc_bf16<kBlockM, kBlockN, false, false>();
            constexpr uint32_t idesc_pv = umma::idesc_bf16<kBlockM, D, false, true>();
            auto qk = [&](int s, int kslot) {  // S_s = Q_s K^T   (mm_ABt, tiles.hpp:349)
                const uint32_t qa = smem_u32(sQ + s * C::kTileBytes);
                const uint32_t kb = smem_u32(sKV + kslot * C::kTileBytes);
#pragma unroll
                for (int k = 0; k < D / 16; ++k) {
                    const uint32_t off = (k / 4) * C::kAtomBytes + (k % 4) * 32;
                    umma::mma_ss(tbase + C::tmem_s(s), umma::desc_kmajor(qa + off), umma::desc_kmajor(kb + off),
                                 idesc_qk, k > 0);
                }
            };
            auto pv = [&](int s, int vslot, bool acc) {  // O_s += P_s V   (mma_AB, tiles.hpp:350-352)
                const uint32_t vb = smem_u32(sKV + vslot * C::kTileBytes);
#pragma unroll
                for (int k = 0; k < kBlockN / 16; ++k)
                    umma::mma_ts(tbase + C::tmem_o(s), tbase + C::tmem_s(s) + 64 + k * 8,
                                 umma::desc_mnmajor(vb + k * 16 * 128, C::kAtomBytes), idesc_pv, (acc || k > 0));
            };
            mbar_wait(&q_full[0], 0);
            mbar_wait(&q_full[1], 0);
            int slot = 0;
            uint32_t phase = 0;
            mbar_wait(&kv_full[slot], phase);
            tmem::fence_after();
            qk(0, slot);
            umma::commit(&s_full[0]);
            qk(1, slot);
            umma::commit(&s_full[1]);
            umma::commit(&kv_empty[slot]);
            advance(slot, phase, C::kKvSlots);
            for (int i = 1; i < nkv; ++i) {
                const int vslot = slot;
                mbar_wait(&kv_full[vslot], phase);
                advance(slot, phase, C::kKvSlots);
                const int kslot = slot;
                const uint32_t pphase = (uint32_t)((i - 1) & 1);
#pragma unroll
                for (int s = 0; s < kQStages; ++s) {
                    mbar_wait(&p_full[s], pphase);
                    tmem::fence_after();
                    pv(s, vslot, i > 1);
                    if (s == 0) {
                        mbar_wait(&kv_full[kslot], phase);
                        tmem::fence_after();
                    }
                    qk(s, kslot);
                    umma::commit(&s_full[s]);
                }
                umma::commit(&kv_empty[vslot]);
                umma::commit(&kv_empty[kslot]);
                advance(slot, phase, C::kKvSlots);
            }
            const int vslot = slot;
            mbar_wait(&kv_full[vslot], phase);
            const uint32_t pphase = (uint32_t)((nkv - 1) & 1);
#pragma unroll
            for (int s = 0; s < kQStages; ++s) {
                mbar_wait(&p_full[s], pphase);
                tmem::fence_after();
                pv(s, vslot, nkv > 1);
                umma::commit(&o_full[s]);
            }
            umma::commit(&kv_empty[vslot]);
        }
    } else {
        // ----------------------------- SOFTMAX + FINISH ------------------------------------
        const int s = warp / 4;                    // query tile of this warpgroup
        const int wq = warp % 4;                   // TMEM lane quarter
        const int row_in_tile = wq * 32 + lane;    // == TMEM lane
        const int row = q0 + s * kBlockM + row_in_tile;
        const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
        const uint32_t tS = tbase + lane_off + C::tmem_s(s);
        const uint32_t tP = tS + 64;
        const uint32_t tO = tbase + lane_off + C::tmem_o(s);
        const float tau = p.scale_log2;

        float m = -INFINITY;  // running max of tau * S (the value actually subtracted)
        float l = 0.f;        // running normaliser (fp32 sum of fp32 P, kernels.hpp:324)
        for (int i = 0; i < nkv; ++i) {
            mbar_wait(&s_full[s], (uint32_t)(i & 1));
            tmem::fence_after();
            float x[kBlockN];
            tmem::ldw_32x32b_x128(tS, reinterpret_cast<uint32_t*>(x));
            const int kv0 = i * kBlockN;
            const bool need_mask = CAUSAL ? (kv0 + kBlockN - 1 > q0 + s * kBlockM) : (kv0 + kBlockN > n);
            if (need_mask) {
                const int lim = CAUSAL ? min(row - kv0, n - 1 - kv0) : (n - 1 - kv0);  // last visible column
#pragma unroll
                for (int j = 0; j < kBlockN; ++j)
                    if (j > lim) x[j] = -INFINITY;
            }
            // row_max (accumulating form, tiles.hpp:290-298)
            float mx0 = x[0], mx1 = x[1], mx2 = x[2], mx3 = x[3];
#pragma unroll
            for (int j = 4; j < kBlockN; j += 4) {
                mx0 = fmaxf(mx0, x[j]);
                mx1 = fmaxf(mx1, x[j + 1]);
                mx2 = fmaxf(mx2, x[j + 2]);
                mx3 = fmaxf(mx3, x[j + 3]);
            }
            const float m_new = fmaxf(m, fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3)) * tau);
            // Rescale lazily: only when some row of the warp grew by > 2^8 (warp-uniform
            // because tcgen05.ld/st are warp-collective). The final O / l is unchanged.
            if (__any_sync(0xffffffffu, m_new > m + kRescaleThreshold)) {
                const float alpha = ex2_approx(m - m_new);  // exp2(-inf) = 0 on the first tile
                m = m_new;
                l *= alpha;
                if (i > 0) {  // mul_row(o, o, alpha) (tiles.hpp:282-287); PV_{i-1} is complete
#pragma unroll
                    for (int c = 0; c < D; c += 32) {
                        uint32_t o[32];
                        tmem::ldw_32x32b_x32(tO + c, o);
#pragma unroll
                        for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * alpha);
                        tmem::st_32x32b_x32(tO + c, o);
                    }
                }
            }
            // P = exp2(tau * S - m) (exp2, tiles.hpp:217-219); row_sum (tiles.hpp:301-309)
            const float neg_m = -m;
            float l0 = 0.f, l1 = 0.f, l2 = 0.f, l3 = 0.f;
            uint32_t pk[kBlockN / 2];
#pragma unroll
            for (int j = 0; j < kBlockN; j += 4) {
                const float p0 = ex2_approx(fmaf(x[j], tau, neg_m));
                const float p1 = ex2_approx(fmaf(x[j + 1], tau, neg_m));
                const float p2 = ex2_approx(fmaf(x[j + 2], tau, neg_m));
                const float p3 = ex2_approx(fmaf(x[j + 3], tau, neg_m));
                l0 += p0;
                l1 += p1;
                l2 += p2;
                l3 += p3;
                pk[j / 2] = pack_bf16x2(p0, p1);  // copy(att_mma, att) bf16 RNE (tiles.hpp:195-200)
                pk[j / 2 + 1] = pack_bf16x2(p2, p3);
            }
            l += (l0 + l1) + (l2 + l3);
            tmem::st_32x32b_x64(tP, pk);
            tmem::wait_st();
            tmem::fence_before();
            mbar_arrive(&p_full[s]);
        }

        // FINISH (kernels.hpp:335-342): O / l, store; plus L for the backward.
        mbar_wait(&o_full[s], 0);
        tmem::fence_after();
        const float inv_l = 1.f / l;
        if (p.lse != nullptr && row < n)
            p.lse[(size_t)(batch * p.heads + head) * n + row] = (m + __log2f(l)) * kLn2;
        uint8_t* stage = sQ + s * C::kTileBytes;  // Q_s is dead: every QK(s) completed before o_full
#pragma unroll
        for (int a = 0; a < C::kAtoms; ++a) {
#pragma unroll
            for (int c = 0; c < 64; c += 32) {
                uint32_t o[32];
                tmem::ldw_32x32b_x32(tO + a * 64 + c, o);
#pragma unroll
                for (int q = 0; q < 4; ++q) {  // four 16-byte chunks
                    uint4 v;
                    v.x = pack_bf16x2(__uint_as_float(o[q * 8 + 0]) * inv_l, __uint_as_float(o[q * 8 + 1]) * inv_l);
                    v.y = pack_bf16x2(__uint_as_float(o[q * 8 + 2]) * inv_l, __uint_as_float(o[q * 8 + 3]) * inv_l);
                    v.z = pack_bf16x2(__uint_as_float(o[q * 8 + 4]) * inv_l, __uint_as_float(o[q * 8 + 5]) * inv_l);
                    v.w = pack_bf16x2(__uint_as_float(o[q * 8 + 6]) * inv_l, __uint_as_float(o[q * 8 + 7]) * inv_l);
                    const int chunk = c / 8 + q;
                    *reinterpret_cast<uint4*>(stage + a * C::kAtomBytes + row_in_tile * 128 +
                                              ((chunk ^ (row_in_tile & 7)) * 16)) = v;
                }
            }
        }
        tma::fence_async_smem();
        named_sync(1 + s, WARPGROUP_THREADS);
        if (wq == 0 && lane == 0) {
            for (int a = 0; a < C::kAtoms; ++a)
                tma::store_4d(&p.tm_o, stage + a * C::kAtomBytes, a * 64, q0 + s * kBlockM, head, batch);
            tma::commit_group();
            tma::wait_group_read<0>();
        }
    }

    tmem::fence_before();
    __syncthreads();
    if (warp == C::kWarpMma) tmem::dealloc<512>(tbase);
}

template <int D, bool CAUSAL>
int launch(const FwdParams& p, int batches, cudaStream_t stream) {
    using C = Cfg<D>;
    auto kern = attn_fwd_kernel<D, CAUSAL>;
    static bool configured = false;  // per instantiation; attribute setting is idempotent
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
        if (e != cudaSuccess) return (int)e;
        configured = true;
    }
    dim3 grid((p.n + kRowsPerCta - 1) / kRowsPerCta, p.heads, batches);
    kern<<<grid, C::kThreads, C::kSmemBytes, stream>>>(p);
    return (int)cudaGetLastError();
}

}  // namespace fwd

int launch_attn_fwd(int head_dim, bool causal, const FwdParams& p, int batches, cudaStream_t stream) {
    if (head_dim == 128) return causal ? fwd::launch<128, true>(p, batches, stream) : fwd::launch<128, false>(p, batches, stream);
    return causal ? fwd::launch<64, true>(p, batches, stream) : fwd::launch<64, false>(p, batches, stream);
}

}  // namespace tkb
