// attn_bwd_sm100.cu — attention backward for B200 (sm_100a), dQ/dK/dV from the saved L.
//
// The reference has no backward; the math follows the restated
// oracle (oracle/attn_oracle.cpp, bwd_head):
//   P = exp(S - L), dV = P^T dO, dP = dO V^T, Delta = rowsum(dO o O),
//   dS = P o (dP - Delta), dQ = scale dS K, dK = scale dS^T Q
//
// Three launches:
//   bwd_prep    Delta = rowsum(dO o O), lse2 = L log2(e) (padded with +inf),
//               reset the dQ ordering semaphores
//   bwd_main    KV-stationary warp-specialised CTA (one 128-row K/V block per CTA,
//               iterating over 128-row Q blocks), 5 tcgen05 GEMMs per tile pair:
//                 S^T  = K Q^T       (SS)            -> TMEM S
//                 dP^T = V dO^T      (SS)            -> TMEM dP
//                 dV  += P^T dO      (TS, P in TMEM) -> TMEM dV
//                 dK  += dS^T Q      (TS, dS in TMEM)-> TMEM dK
//                 dQ_i = dS K        (SS, dS in SMEM)-> TMEM (aliases dP)
//               dQ_i is reduced into an fp32 accumulator by TMA bulk stores/adds in a
//               FIXED order per Q block (ordering semaphores) -> deterministic.
//   bwd_convert dQ fp32 -> bf16
//
// Warp roles (512 threads):
//   warps 0-7   COMPUTE: thread = (kv row r = TMEM lane, q half h); P, dS; dK/dV epilogue
//   warps 8-11  REDUCE : thread = q row of dQ_i; TMEM -> regs -> SMEM -> TMA add
//   warp 12     MMA    : one thread issues all tcgen05.mma
//   warp 13     LOAD   : TMA K, V once; Q_i (+lse2) and dO_i (+Delta) rings
//   warps 14-15 idle (complete the warpgroup for setmaxnreg)
//
// TMEM columns: S [0,128) | dV [128,128+D) | dP/dS/dQ [128+D, 256+D) | dK [256+D, 256+2D)
// P^T (bf16) lives in S columns [32,96), dS^T in dP columns [32,96): each q half h
// writes only inside the S/dP columns it has itself read ([64h, 64h+64)).
//
// Deterministic dQ order: CTA (bh, kv block j) visits Q blocks in the order
//   causal:     i = j + t,            t = 0 .. nq-1-j
//   non-causal: i = (j + t) mod nq,   t = 0 .. nq-1
// so for every Q block the contributor at visit t is unique; it waits until the
// block's semaphore equals t, stores (t == 0) or adds (t > 0), and bumps it.
#include <cuda.h>
#include <cuda_runtime.h>

#include "attn_common.cuh"
#include "tkb/tcgen05.cuh"
#include "tkb/tma.cuh"

namespace tkb {
namespace bwd {

template <int D>
struct Cfg {
    static constexpr int kAtoms = D / 64;
    static constexpr int kAtomBytes = 128 * 128;        // 128 rows x 128 B
    static constexpr int kTileBytes = 128 * D * 2;      // 128 x D bf16
    static constexpr int kDoStages = (D == 128) ? 1 : 2;  // D=128: smem goes to dQ staging
    static constexpr int kDqStageBytes = 128 * 32 * 4;    // 128 rows x 32 fp32 columns
    static constexpr int kDqStages = 2;
    // smem carve-up (all 1024-aligned)
    static constexpr int kOffK = 0;
    static constexpr int kOffV = kOffK + kTileBytes;
    static constexpr int kOffQ = kOffV + kTileBytes;                    // 2 stages
    static constexpr int kOffDo = kOffQ + 2 * kTileBytes;               // kDoStages
    static constexpr int kOffDs = kOffDo + kDoStages * kTileBytes;      // 128 x 128 bf16
    static constexpr int kOffDq = kOffDs + 128 * 128 * 2;               // kDqStages staging buffers
    static constexpr int kOffLse = kOffDq + kDqStages * kDqStageBytes;  // 2 Q stages x 128 fp32
    static constexpr int kOffDelta = kOffLse + 2 * 128 * 4;             // 2 Q stages x 128 fp32
    static constexpr int kOffBar = kOffDelta + 2 * 128 * 4;             // mbarriers + TMEM slot
    // No alignment slack: the dynamic smem window starts 1 KB-aligned (after the driver's
    // 1 KB reservation); checked at run time.
    static constexpr int kSmemBytes = kOffBar + 256;  // 32 mbarrier slots
    static_assert(kSmemBytes <= 232448, "exceeds 227 KB of shared memory");
    static __device__ __forceinline__ constexpr uint32_t tmem_s() { return 0u; }
    static __device__ __forceinline__ constexpr uint32_t tmem_dv() { return 128u; }
    static __device__ __forceinline__ constexpr uint32_t tmem_dp() { return 128u + D; }
    static __device__ __forceinline__ constexpr uint32_t tmem_dk() { return 256u + D; }
};

constexpr int kThreads = 512;
constexpr int kWarpReduce0 = 8;
constexpr int kWarpMma = 12;
constexpr int kWarpLoad = 13;
constexpr int kWarpIssue0 = 14;  // warps 14, 15: dQ TMA issuers
constexpr int kComputeThreads = 256;
constexpr int kReduceThreads = 128;
constexpr int kBarCompute = 1;
constexpr int kBarReduce = 2;

TKB_DEVICE int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
TKB_DEVICE void red_release_add(int* p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int D, bool CAUSAL>
__global__ void __launch_bounds__(kThreads, 1) attn_bwd_kernel(const __grid_constant__ BwdParams p) {
    using C = Cfg<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw;
    if (smem_u32(smem) & 1023) __trap();  // SW128 tiles need 1 KB alignment
    uint8_t* sK = smem + C::kOffK;
    uint8_t* sV = smem + C::kOffV;
    uint8_t* sQ = smem + C::kOffQ;
    uint8_t* sDo = smem + C::kOffDo;
    uint8_t* sDs = smem + C::kOffDs;
    uint8_t* sDq = smem + C::kOffDq;
    float* sLse = reinterpret_cast<float*>(smem + C::kOffLse);
    float* sDelta = reinterpret_cast<float*>(smem + C::kOffDelta);

    // barriers live in dynamic smem (static smem would push D=128 past 227 KB)
    mbarrier* bars = reinterpret_cast<mbarrier*>(smem + C::kOffBar);
    mbarrier& kv_full = bars[0];
    mbarrier* q_full = bars + 1;    // [2]
    mbarrier* q_empty = bars + 3;   // [2]
    mbarrier* do_full = bars + 5;   // [kDoStages <= 2]
    mbarrier* do_empty = bars + 7;  // [kDoStages <= 2]
    mbarrier& s_full = bars[9];
    mbarrier& p_full = bars[10];
    mbarrier& dp_full = bars[11];
    mbarrier& ds_full = bars[12];
    mbarrier& dq_full = bars[13];
    mbarrier& dq_empty = bars[14];
    mbarrier& dkv_full = bars[15];
    uint32_t& tmem_slot = *reinterpret_cast<uint32_t*>(bars + 20);
    mbarrier* chunk_full = bars + 16;   // [2] dQ staging buffer written (reduce warps)
    mbarrier* chunk_empty = bars + 18;  // [2] dQ staging buffer read by TMA (issuers)
    volatile int* issued = reinterpret_cast<volatile int*>(bars + 21);  // chunks handed to TMA

    const int warp = warpid();
    const int lane = laneid();
    // Work item from a start-order ticket rather than blockIdx: a CTA only ever waits (dQ
    // ordering) on CTAs of its own head, and tickets guarantee every head is started
    // contiguously, whatever order the hardware dispatches blocks in.
    volatile int* ticket_slot = reinterpret_cast<volatile int*>(bars + 22);
    if (threadIdx.x == 0) *ticket_slot = atomicAdd(p.ticket, 1);
    __syncthreads();
    const int item = *ticket_slot;
    const int nkv_blocks = p.n_pad / 128;
    const int bh = item / nkv_blocks;
    const int j = item % nkv_blocks;  // kv block (heavy causal blocks first)
    const int head = bh % p.heads;
    const int batch = bh / p.heads;
    // optional timeline (debug): one slot per traced work item
    long long* tr = nullptr;
    const long long t_start = clock64();
    if (p.trace != nullptr && item % p.trace_every == 0 && item / p.trace_every < p.trace_slots)
        tr = p.trace + (size_t)(item / p.trace_every) * kTraceRoles * kTraceIters * kTraceEvents;
#define TKB_TR(role, t, ev)                                                                      \
    do {                                                                                         \
        if (tr != nullptr && (t) < kTraceIters)                                                  \
            tr[((role) * kTraceIters + (t)) * kTraceEvents + (ev)] = clock64() - t_start;        \
    } while (0)
    const int kv0 = j * 128;
    const int nq = p.n_pad / 128;
    const int T = CAUSAL ? (nq - j) : nq;  // q blocks visited by this CTA
    auto qblock = [&](int t) { return CAUSAL ? (j + t) : ((j + t) % nq); };

    if (warp == kWarpLoad && lane == 0) {
        mbar_init(&kv_full, 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(&q_full[s], 1);
            mbar_init(&q_empty[s], 1);
        }
        for (int s = 0; s < C::kDoStages; ++s) {
            mbar_init(&do_full[s], 1);
            mbar_init(&do_empty[s], 1);  // MMA commit after dV
        }
        mbar_init(&s_full, 1);
        mbar_init(&p_full, kComputeThreads);
        mbar_init(&dp_full, 1);
        mbar_init(&ds_full, kComputeThreads);
        mbar_init(&dq_full, 1);
        mbar_init(&dq_empty, kReduceThreads);
        mbar_init(&dkv_full, 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(&chunk_full[b], kReduceThreads);
            mbar_init(&chunk_empty[b], 1);
        }
        *issued = 0;
        fence_barrier_init();
        tma::prefetch_desc(&p.tm_q);
        tma::prefetch_desc(&p.tm_k);
        tma::prefetch_desc(&p.tm_v);
        tma::prefetch_desc(&p.tm_do);
    }
    if (warp == kWarpMma) tmem::alloc<512>(&tmem_slot);
    tmem::fence_before();
    __syncthreads();
    tmem::fence_after();
    const uint32_t tbase = tmem_slot;

    if (warp >= kWarpMma) {
        setmaxnreg_dec<56>();
        if (warp == kWarpLoad && lane == 0) {
            // ------------------------------------------------------------- LOAD
            const uint64_t pol_stream = tma::policy_evict_first();
            const uint64_t pol_keep = tma::policy_evict_last();
            mbar_arrive_expect_tx(&kv_full, 2 * C::kTileBytes);
            for (int a = 0; a < C::kAtoms; ++a) {
                tma::load_4d(sK + a * C::kAtomBytes, &p.tm_k, &kv_full, a * 64, kv0, head, batch, pol_stream);
                tma::load_4d(sV + a * C::kAtomBytes, &p.tm_v, &kv_full, a * 64, kv0, head, batch, pol_stream);
            }
            // Issue order follows the order in which slots free up (dO_t after dV_t, Q_t after
            // dK_t): dO_{t+1} is requested before Q_{t+2}, so neither waits behind the other.
            auto load_q = [&](int t) {
                const int i = qblock(t), qs = t & 1;
                mbar_wait(&q_empty[qs], ((t >> 1) & 1) ^ 1);
                mbar_arrive_expect_tx(&q_full[qs], C::kTileBytes + 1024);
                for (int a = 0; a < C::kAtoms; ++a)
                    tma::load_4d(sQ + qs * C::kTileBytes + a * C::kAtomBytes, &p.tm_q, &q_full[qs], a * 64, i * 128,
                                 head, batch, pol_keep);
                tma::load_1d(sLse + qs * 128, p.lse2 + (size_t)bh * p.n_pad + i * 128, 512, &q_full[qs]);
                tma::load_1d(sDelta + qs * 128, p.delta + (size_t)bh * p.n_pad + i * 128, 512, &q_full[qs]);
            };
            auto load_do = [&](int t) {
                const int i = qblock(t), ds = t % C::kDoStages;
                mbar_wait(&do_empty[ds], ((t / C::kDoStages) & 1) ^ 1);
                mbar_arrive_expect_tx(&do_full[ds], C::kTileBytes);
                for (int a = 0; a < C::kAtoms; ++a)
                    tma::load_4d(sDo + ds * C::kTileBytes + a * C::kAtomBytes, &p.tm_do, &do_full[ds], a * 64,
                                 i * 128, head, batch, pol_keep);
            };
            load_q(0);
            load_do(0);
            if (T > 1) load_q(1);
            for (int t = 1; t < T; ++t) {
                load_do(t);
                if (t + 1 < T) load_q(t + 1);
            }
        } else if (warp >= kWarpIssue0 && lane == 0) {
            // ------------------------------------------------------------- dQ TMA ISSUERS
            // Two threads alternate Q blocks, so one can wait for its adds to land in L2
            // (required before the ordering semaphore is released) while the other keeps
            // draining staging chunks. Chunks are consumed strictly in order (hand-off on
            // `issued`): an mbarrier parity wait cannot look more than one phase ahead.
            constexpr int NC = D / 32;
            int* sema = p.dq_sema + (size_t)bh * nq;
            for (int t = warp - kWarpIssue0; t < T; t += 2) {
                const int i = qblock(t);
                // visit t of block i is the t-th contributor; a lost contributor traps
                // (~4 s) instead of hanging the GPU (DeadlockError analogue, lcsf.hpp:486-489)
                for (long long t0 = clock64(); ld_acquire(sema + i) != t;)
                    if (clock64() - t0 > (1ll << 33)) __trap();
                tma::fence_async_global();
                while (*issued < t * NC) {
                }
                if (warp == kWarpIssue0) TKB_TR(2, t, 2);
                for (int c = 0; c < NC; ++c) {
                    const int g = t * NC + c;
                    const int b = g & 1;
                    mbar_wait(&chunk_full[b], (g >> 1) & 1);
                    const uint8_t* buf = sDq + b * C::kDqStageBytes;
                    if (t == 0)
                        tma::store_3d(&p.tm_dqacc, buf, c * 32, i * 128, bh);
                    else
                        tma::reduce_add_3d(&p.tm_dqacc, buf, c * 32, i * 128, bh);
                    tma::commit_group();
                    tma::wait_group_read<0>();
                    mbar_arrive(&chunk_empty[b]);
                    *issued = g + 1;
                }
                if (warp == kWarpIssue0) TKB_TR(2, t, 3);
                tma::wait_group<0>();  // the adds have been performed
                tma::fence_async_global();
                __threadfence();
                red_release_add(sema + i, 1);
            }
        } else if (warp == kWarpMma && lane == 0) {
            // ------------------------------------------------------------- MMA
            constexpr uint32_t id_s = umma::idesc_bf16<128, 128, false, false>();  // S^T, dP^T
            constexpr uint32_t id_kv = umma::idesc_bf16<128, D, false, true>();    // dV, dK (A in TMEM)
            constexpr uint32_t id_q = umma::idesc_bf16<128, D, true, true>();      // dQ (A = dS MN-major)
            const uint32_t aK = smem_u32(sK), aV = smem_u32(sV), aDs = smem_u32(sDs);
            constexpr uint32_t HI = umma::desc_hi_sw128(1024);  // SBO = 8 rows x 128 B
            // X^T = A B^T with A = K or V [kv][D] and B = Q or dO [q][D], both K-major
            auto mm_abt = [&](uint32_t dst, uint32_t a, uint32_t b) {
                a = umma::opaque(a);
                b = umma::opaque(b);
#pragma unroll
                for (int k = 0; k < D / 16; ++k) {
                    const uint32_t off = (k / 4) * C::kAtomBytes + (k % 4) * 32;
                    umma::mma_ss_split(tbase + dst, umma::desc_lo(a + off, 16), HI, umma::desc_lo(b + off, 16), HI,
                                       id_s, k > 0);
                }
            };
            // acc += A[tmem] B with B = dO or Q [q][D] (MN-major)
            auto mma_tb = [&](uint32_t dst, uint32_t a_tmem, uint32_t b, bool acc) {
                b = umma::opaque(b);
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    umma::mma_ts_split(tbase + dst, tbase + a_tmem + k * 8, umma::desc_lo(b + k * 2048, C::kAtomBytes),
                                       HI, id_kv, acc || k > 0);
            };
            auto mm_dq = [&]() {  // dQ = dS K : A = dS^T smem [kv][q] (MN-major), B = K [kv][D] (MN-major)
                const uint32_t a = umma::opaque(aDs), b = umma::opaque(aK);
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    umma::mma_ss_split(tbase + C::tmem_dp(), umma::desc_lo(a + k * 2048, C::kAtomBytes), HI,
                                       umma::desc_lo(b + k * 2048, C::kAtomBytes), HI, id_q, k > 0);
            };
            auto qaddr = [&](int t) { return smem_u32(sQ + (t & 1) * C::kTileBytes); };
            auto doaddr = [&](int t) { return smem_u32(sDo + (t % C::kDoStages) * C::kTileBytes); };

            mbar_wait(&kv_full, 0);
            // prologue: S_0, dP_0, dV_0
            mbar_wait(&q_full[0], 0);
            tmem::fence_after();
            mm_abt(C::tmem_s(), aK, qaddr(0));
            umma::commit(&s_full);
            mbar_wait(&do_full[0], 0);
            tmem::fence_after();
            mm_abt(C::tmem_dp(), aV, doaddr(0));
            umma::commit(&dp_full);
            mbar_wait(&p_full, 0);
            tmem::fence_after();
            mma_tb(C::tmem_dv(), C::tmem_s() + 32, doaddr(0), false);
            umma::commit(&do_empty[0]);
            for (int t = 0; t < T - 1; ++t) {
                const uint32_t ph = (uint32_t)(t & 1);
                const int t1 = t + 1;
                // (1) S_{t+1}
                TKB_TR(0, t, 0);
                mbar_wait(&q_full[t1 & 1], (t1 >> 1) & 1);
                tmem::fence_after();
                mm_abt(C::tmem_s(), aK, qaddr(t1));
                umma::commit(&s_full);
                TKB_TR(0, t, 1);
                // (2) dK += dS_t^T Q_t ; (3) dQ_t = dS_t K
                mbar_wait(&ds_full, ph);
                TKB_TR(0, t, 2);
                tmem::fence_after();
                mma_tb(C::tmem_dk(), C::tmem_dp() + 32, qaddr(t), t > 0);
                umma::commit(&q_empty[t & 1]);
                mm_dq();
                umma::commit(&dq_full);
                TKB_TR(0, t, 3);
                // (4) dP_{t+1} once the reduce warps drained dQ_t
                mbar_wait(&do_full[t1 % C::kDoStages], (t1 / C::kDoStages) & 1);
                TKB_TR(0, t, 4);
                mbar_wait(&dq_empty, ph);
                TKB_TR(0, t, 5);
                tmem::fence_after();
                mm_abt(C::tmem_dp(), aV, doaddr(t1));
                umma::commit(&dp_full);
                // (5) dV += P_{t+1}^T dO_{t+1}
                mbar_wait(&p_full, t1 & 1);
                TKB_TR(0, t, 6);
                tmem::fence_after();
                mma_tb(C::tmem_dv(), C::tmem_s() + 32, doaddr(t1), true);
                umma::commit(&do_empty[t1 % C::kDoStages]);
                TKB_TR(0, t, 7);
            }
            // tail: dK, dQ of the last block
            const int tl = T - 1;
            mbar_wait(&ds_full, tl & 1);
            tmem::fence_after();
            mma_tb(C::tmem_dk(), C::tmem_dp() + 32, qaddr(tl), tl > 0);
            umma::commit(&q_empty[tl & 1]);
            mm_dq();
            umma::commit(&dq_full);
            umma::commit(&dkv_full);
        }
    } else if (warp >= kWarpReduce0) {
        // ----------------------------------------------------------------- REDUCE (dQ)
        // TMEM -> registers (frees the dP/dQ columns at once) -> double-buffered SMEM
        // chunks of 128 x 32 fp32, drained by the TMA issuer threads (warps 14, 15).
        setmaxnreg_inc<152>();
        const int wq = warp - kWarpReduce0;
        const int r = wq * 32 + lane;  // q row within the block == TMEM lane
        const uint32_t tdq = tbase + ((uint32_t)(wq * 32) << 16) + C::tmem_dp();
        const bool leader = (threadIdx.x == kWarpReduce0 * 32);
        for (int t = 0; t < T; ++t) {
            mbar_wait(&dq_full, t & 1);
            if (leader) TKB_TR(2, t, 0);
            tmem::fence_after();
            uint32_t acc[D];
#pragma unroll
            for (int c = 0; c < D; c += 32) tmem::ld_32x32b_x32(tdq + c, acc + c);
#pragma unroll
            for (int c = 0; c < D; c += 32) tmem::wait_ld_x32(acc + c);
            tmem::fence_before();
            mbar_arrive(&dq_empty);
            if (leader) TKB_TR(2, t, 1);
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
                const int g = t * (D / 32) + c;
                const int b = g & 1;
                mbar_wait(&chunk_empty[b], ((g >> 1) & 1) ^ 1);
                uint8_t* buf = sDq + b * C::kDqStageBytes;
#pragma unroll
                for (int q = 0; q < 8; ++q)  // 8 chunks of 4 fp32 = one 128-B row (SW128)
                    *reinterpret_cast<uint4*>(buf + r * 128 + ((q ^ (r & 7)) * 16)) =
                        make_uint4(acc[c * 32 + q * 4 + 0], acc[c * 32 + q * 4 + 1], acc[c * 32 + q * 4 + 2],
                                   acc[c * 32 + q * 4 + 3]);
                tma::fence_async_smem();
                mbar_arrive(&chunk_full[b]);
            }
        }
    } else {
        // ----------------------------------------------------------------- COMPUTE
        setmaxnreg_inc<152>();
        const int wq = warp & 3;
        const int h = warp >> 2;       // q half: columns [64h, 64h+64)
        const int r = wq * 32 + lane;  // kv row == TMEM lane
        const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
        const uint32_t tS = tbase + lane_off + C::tmem_s();
        const uint32_t tDp = tbase + lane_off + C::tmem_dp();
        const float tau = p.scale_log2;
        const float scale = p.scale;
        for (int t = 0; t < T; ++t) {
            const int i = qblock(t);
            const int qs = t & 1;
            const bool diag = CAUSAL && (i == j);
            const float* lse = sLse + qs * 128 + 64 * h;
            const float* dlt = sDelta + qs * 128 + 64 * h;
            // P^T = exp2(tau S^T - lse2)
            mbar_wait(&q_full[qs], (t >> 1) & 1);
            mbar_wait(&s_full, t & 1);
            if (threadIdx.x == 0) TKB_TR(1, t, 0);
            tmem::fence_after();
            float pf[64];
            tmem::ld_32x32b_x32(tS + 64 * h, reinterpret_cast<uint32_t*>(pf));
            tmem::ld_32x32b_x32(tS + 64 * h + 32, reinterpret_cast<uint32_t*>(pf) + 32);
            tmem::wait_ld_x32(reinterpret_cast<uint32_t*>(pf));
            tmem::wait_ld_x32(reinterpret_cast<uint32_t*>(pf) + 32);
            uint32_t pk[32];
#pragma unroll
            for (int c = 0; c < 64; c += 2) {
                float p0 = ex2_approx(fmaf(pf[c], tau, -lse[c]));
                float p1 = ex2_approx(fmaf(pf[c + 1], tau, -lse[c + 1]));
                if (diag) {  // causal: key kv0 + r visible to query q0 + 64h + c iff r <= 64h + c
                    if (64 * h + c < r) p0 = 0.f;
                    if (64 * h + c + 1 < r) p1 = 0.f;
                }
                pf[c] = p0;
                pf[c + 1] = p1;
                pk[c / 2] = pack_bf16x2(p0, p1);
            }
            tmem::st_32x32b_x32(tS + 32 + 32 * h, pk);
            tmem::wait_st();
            tmem::fence_before();
            mbar_arrive(&p_full);
            if (threadIdx.x == 0) TKB_TR(1, t, 1);
            // dS^T = P^T o (dP^T - Delta) * scale
            mbar_wait(&dp_full, t & 1);
            if (threadIdx.x == 0) TKB_TR(1, t, 2);
            tmem::fence_after();
            uint8_t* dsrow = sDs + h * C::kAtomBytes + r * 128;
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                uint32_t dpv[32];
                tmem::ldw_32x32b_x32(tDp + 64 * h + 32 * half, dpv);
#pragma unroll
                for (int c = 0; c < 32; c += 2) {
                    const int cc = 32 * half + c;
                    const float d0 = pf[cc] * (__uint_as_float(dpv[c]) - dlt[cc]) * scale;
                    const float d1 = pf[cc + 1] * (__uint_as_float(dpv[c + 1]) - dlt[cc + 1]) * scale;
                    pk[cc / 2] = pack_bf16x2(d0, d1);
                }
            }
            tmem::st_32x32b_x32(tDp + 32 + 32 * h, pk);
#pragma unroll
            for (int q = 0; q < 8; ++q)
                *reinterpret_cast<uint4*>(dsrow + ((q ^ (r & 7)) * 16)) =
                    make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
            tmem::wait_st();
            tmem::fence_before();
            tma::fence_async_smem();
            mbar_arrive(&ds_full);
            if (threadIdx.x == 0) TKB_TR(1, t, 3);
        }
        // FINISH: dV, dK (TMEM fp32) -> bf16 -> SMEM (Q ring is free) -> TMA store
        mbar_wait(&dkv_full, 0);
        tmem::fence_after();
        uint8_t* stage_v = sQ;
        uint8_t* stage_k = sQ + C::kTileBytes;
#pragma unroll
        for (int which = 0; which < 2; ++which) {
            const uint32_t tsrc = tbase + lane_off + (which == 0 ? C::tmem_dv() : C::tmem_dk());
            uint8_t* stg = which == 0 ? stage_v : stage_k;
#pragma unroll
            for (int c = 0; c < D / 2; c += 32) {
                const int col = h * (D / 2) + c;
                uint32_t v[32];
                tmem::ldw_32x32b_x32(tsrc + col, v);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int gc = col / 8 + q;  // global 16-byte chunk index within the row
                    const int atom = gc / 8, ch = gc % 8;
                    uint4 u;
                    u.x = pack_bf16x2(__uint_as_float(v[8 * q + 0]), __uint_as_float(v[8 * q + 1]));
                    u.y = pack_bf16x2(__uint_as_float(v[8 * q + 2]), __uint_as_float(v[8 * q + 3]));
                    u.z = pack_bf16x2(__uint_as_float(v[8 * q + 4]), __uint_as_float(v[8 * q + 5]));
                    u.w = pack_bf16x2(__uint_as_float(v[8 * q + 6]), __uint_as_float(v[8 * q + 7]));
                    *reinterpret_cast<uint4*>(stg + atom * C::kAtomBytes + r * 128 + ((ch ^ (r & 7)) * 16)) = u;
                }
            }
        }
        tma::fence_async_smem();
        named_sync(kBarCompute, kComputeThreads);
        if (threadIdx.x == 0) {
            for (int a = 0; a < C::kAtoms; ++a) {
                tma::store_4d(&p.tm_dv, stage_v + a * C::kAtomBytes, a * 64, kv0, head, batch);
                tma::store_4d(&p.tm_dk, stage_k + a * C::kAtomBytes, a * 64, kv0, head, batch);
            }
            tma::commit_group();
            tma::wait_group_read<0>();
        }
    }

    tmem::fence_before();
    __syncthreads();
    if (warp == kWarpMma) tmem::dealloc<512>(tbase);
#undef TKB_TR
}

// Delta = rowsum(dO o O), lse2 = L log2 e (+inf / 0 on padded rows), semaphores = 0.
template <int D>
__global__ void __launch_bounds__(256) bwd_prep_kernel(const __nv_bfloat16* __restrict__ o,
                                                       const __nv_bfloat16* __restrict__ dout,
                                                       const float* __restrict__ lse, float* __restrict__ lse2,
                                                       float* __restrict__ delta, int* __restrict__ sema, int* __restrict__ ticket, int heads,
                                                       int n, int n_pad, int64_t sb, int64_t sh, int64_t sn) {
    constexpr int kLanesPerRow = D / 8;
    constexpr int kRowsPerBlock = 256 / kLanesPerRow;
    const int bh = blockIdx.y;
    const int b = bh / heads, hh = bh % heads;
    const int row = blockIdx.x * kRowsPerBlock + threadIdx.x / kLanesPerRow;
    const int c = (threadIdx.x % kLanesPerRow) * 8;
    float acc = 0.f;
    if (row < n) {
        const int64_t off = b * sb + hh * sh + (int64_t)row * sn + c;
        const uint4 ov = *reinterpret_cast<const uint4*>(o + off);
        const uint4 dv = *reinterpret_cast<const uint4*>(dout + off);
        const __nv_bfloat162* o2 = reinterpret_cast<const __nv_bfloat162*>(&ov);
        const __nv_bfloat162* d2 = reinterpret_cast<const __nv_bfloat162*>(&dv);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float2 a = __bfloat1622float2(o2[k]);
            const float2 g = __bfloat1622float2(d2[k]);
            acc = fmaf(a.x, g.x, acc);
            acc = fmaf(a.y, g.y, acc);
        }
    }
#pragma unroll
    for (int s = kLanesPerRow / 2; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
    if (row < n_pad && (threadIdx.x % kLanesPerRow) == 0) {
        const size_t idx = (size_t)bh * n_pad + row;
        delta[idx] = row < n ? acc : 0.f;
        lse2[idx] = row < n ? lse[(size_t)bh * n + row] * 1.44269504088896340736f : INFINITY;
    }
    if (blockIdx.x == 0)
        for (int k = threadIdx.x; k < n_pad / 128; k += blockDim.x) sema[(size_t)bh * (n_pad / 128) + k] = 0;
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *ticket = 0;
}

// dq (bf16, user layout) = dq_accum (fp32 [bh][n_pad][D])
template <int D>
__global__ void __launch_bounds__(256) bwd_convert_kernel(const float* __restrict__ acc, __nv_bfloat16* __restrict__ dq,
                                                          int heads, int n, int n_pad, int64_t sb, int64_t sh,
                                                          int64_t sn, int64_t total_chunks) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total_chunks;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(g % (D / 8)) * 8;
        const int64_t rowg = g / (D / 8);
        const int row = (int)(rowg % n);
        const int bh = (int)(rowg / n);
        const float* src = acc + ((size_t)bh * n_pad + row) * D + c;
        const float4 a = *reinterpret_cast<const float4*>(src);
        const float4 bq = *reinterpret_cast<const float4*>(src + 4);
        uint4 u;
        u.x = pack_bf16x2(a.x, a.y);
        u.y = pack_bf16x2(a.z, a.w);
        u.z = pack_bf16x2(bq.x, bq.y);
        u.w = pack_bf16x2(bq.z, bq.w);
        const int b = bh / heads, hh = bh % heads;
        *reinterpret_cast<uint4*>(dq + b * sb + hh * sh + (int64_t)row * sn + c) = u;
    }
}

template <int D, bool CAUSAL>
int launch_main(const BwdParams& p, int batches, cudaStream_t stream) {
    using C = Cfg<D>;
    auto kern = attn_bwd_kernel<D, CAUSAL>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
        if (e != cudaSuccess) return (int)e;
        configured = true;
    }
    dim3 grid((p.n_pad / 128) * p.heads * batches);
    kern<<<grid, kThreads, C::kSmemBytes, stream>>>(p);
    return (int)cudaGetLastError();
}

template <int D>
int launch_all(bool causal, const BwdParams& p, int batches, const void* o, const void* dout, const float* lse,
               float* lse2, float* delta, float* dq_accum, int64_t sb, int64_t sh, int64_t sn, void* dq,
               cudaStream_t stream, int* launches) {
    constexpr int kRowsPerBlock = 256 / (D / 8);
    const int bhs = batches * p.heads;
    dim3 g1((p.n_pad + kRowsPerBlock - 1) / kRowsPerBlock, bhs);
    bwd_prep_kernel<D><<<g1, 256, 0, stream>>>(reinterpret_cast<const __nv_bfloat16*>(o),
                                              reinterpret_cast<const __nv_bfloat16*>(dout), lse, lse2, delta,
                                              p.dq_sema, p.ticket, p.heads, p.n, p.n_pad, sb, sh, sn);
    int e = (int)cudaGetLastError();
    if (e) return e;
    e = causal ? launch_main<D, true>(p, batches, stream) : launch_main<D, false>(p, batches, stream);
    if (e) return e;
    const int64_t chunks = (int64_t)bhs * p.n * (D / 8);
    const int blocks = (int)((chunks + 255) / 256 < 148 * 16 ? (chunks + 255) / 256 : 148 * 16);
    bwd_convert_kernel<D><<<blocks, 256, 0, stream>>>(dq_accum, reinterpret_cast<__nv_bfloat16*>(dq), p.heads, p.n,
                                                      p.n_pad, sb, sh, sn, chunks);
    e = (int)cudaGetLastError();
    if (e) return e;
    *launches = 3;
    return 0;
}

}  // namespace bwd

int launch_attn_bwd(int head_dim, bool causal, const BwdParams& p, int batches, const void* o, const void* dout,
                    const float* lse, float* lse2, float* delta, float* dq_accum, int64_t sb, int64_t sh, int64_t sn,
                    void* dq, cudaStream_t stream, int* launches) {
    if (head_dim == 128)
        return bwd::launch_all<128>(causal, p, batches, o, dout, lse, lse2, delta, dq_accum, sb, sh, sn, dq, stream,
                                    launches);
    return bwd::launch_all<64>(causal, p, batches, o, dout, lse, lse2, delta, dq_accum, sb, sh, sn, dq, stream,
                               launches);
}

}  // namespace tkb
