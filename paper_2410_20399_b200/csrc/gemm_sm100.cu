// gemm_sm100.cu — C = A B on the same tcgen05 / TMA / LCSF machinery as attention
// (the QKV / output projections either side of the attention).
//
// Reference: kittensim gemm_kernel (kernels.hpp:76-149) — one task computes a block of C
// walking K in 64-wide panels through the LCSF ring, tasks in the supergrouped launch
// order (supergroup_order, grid.hpp:28-47), oracle_gemm (oracles.hpp:17-30). Here:
//   tile        128 x 256 of C per task, K panels of 64 (A: 128 x 64 K-major SW128 tile,
//               B: 64 x 256 MN-major = four SW128 atoms), fp32 accumulation in TMEM
//   warp 0      LOAD: TMA of the A / B panels into a 4-stage lcsf::ring (48 KB / stage)
//   warp 1      MMA: converged warp, elected lane issues tcgen05.mma M=128 N=256 K=16
//               (mma_ABt-style A descriptor, B MN-major = the reference's mma_AB with
//               B row-major, kernels.hpp:124-138)
//   warps 4-7   FINISH: TMEM -> fp32 regs -> bf16 -> SMEM atom -> TMA store, while the
//               MMA warp already accumulates the next task into the other TMEM buffer
//               (2 x 256 columns)
// Persistent grid (one CTA per SM); task t -> (row block, col block) by the reference's
// supergroup order, so concurrently running CTAs share A row panels / B column panels
// in L2. Any M, N, K >= 1 (TMA zero-fills / clips the ragged edges); row strides must be
// multiples of 8 elements.
#include <cuda.h>
#include <cuda_runtime.h>

#include "attn_common.cuh"
#include "tkb/cluster.cuh"
#include "tkb/lcsf.cuh"
#include "tkb/tile.cuh"

namespace tkb {
namespace gemm {

constexpr int BM = 128, BN = 256, BK = 64;
constexpr int kStages = 4;
constexpr int kATile = BM * BK * 2;            // 16 KB
constexpr int kBTile = BK * BN * 2;            // 32 KB: 4 atoms of 64 K rows x 64 N cols
constexpr int kBAtom = BK * 128;               // 8 KB
constexpr int kStage = kATile + kBTile;
constexpr int kStaging = BM * 128;             // one 128 x 64 bf16 output atom
constexpr int kOffBar = kStages * kStage + kStaging;
constexpr int kSmemBytes = kOffBar + 256 + 1024;
static_assert(kSmemBytes <= 232448, "smem");
constexpr int kThreads = 256;  // warp 0 load, warp 1 MMA, warps 4-7 epilogue
constexpr int kBarEpi = 1;

// supergroup_order (grid.hpp:28-47): walk super_m rows down each column strip, then the
// remainder rows column by column.
TKB_DEVICE void supergroup(int task, int r_blocks, int c_blocks, int super_m, int& row, int& col) {
    const int super_rows = (r_blocks / super_m) * super_m;
    const int super_repeat = super_m * c_blocks;
    if (task < super_rows * c_blocks) {
        row = super_m * (task / super_repeat) + task % super_m;
        col = (task % super_repeat) / super_m;
    } else {
        const int final_rows = r_blocks - super_rows;
        const int rem = task - super_rows * c_blocks;
        row = super_rows + rem % final_rows;
        col = rem / final_rows;
    }
}

__global__ void __launch_bounds__(kThreads, 1) gemm_kernel(const __grid_constant__ GemmParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    auto sA = [&](int s) { return st_bf<BM, BK>{smem + s * kStage}; };
    auto sB = [&](int s) { return smem + s * kStage + kATile; };  // MN-major [BK rows][BN], 4 atoms
    uint8_t* stage_c = smem + kStages * kStage;
    struct Bars {
        lcsf::ring<kStages> ab;
        mbarrier acc_full[2], acc_empty[2];
        uint32_t tmem_slot;
    };
    Bars& bar = *reinterpret_cast<Bars*>(smem + kOffBar);
    static_assert(sizeof(Bars) <= 256, "barrier area");

    const int warp = warpid();
    const int lane = laneid();
    const int r_blocks = (p.m + BM - 1) / BM, c_blocks = (p.n + BN - 1) / BN;
    const int tasks = r_blocks * c_blocks;
    const int k_tiles = (p.k + BK - 1) / BK;

    if (warp == 0 && lane == 0) {
        bar.ab.init(1, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bar.acc_full[i], 1);
            mbar_init(&bar.acc_empty[i], WARPGROUP_THREADS);
        }
        fence_barrier_init();
        tma::prefetch_desc(&p.tm_a);
        tma::prefetch_desc(&p.tm_b);
        tma::prefetch_desc(&p.tm_c);
    }
    if (warp == 1) tmem::alloc<512>(&bar.tmem_slot);
    tmem::fence_before();
    __syncthreads();
    tmem::fence_after();
    const uint32_t tbase = bar.tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------------------------------------------------------- LOAD
            const uint64_t pol = tma::policy_evict_last();
            lcsf::ring_state<kStages> st;
            for (int t = blockIdx.x; t < tasks; t += gridDim.x) {
                int rb, cb;
                supergroup(t, r_blocks, c_blocks, p.super_m, rb, cb);
                for (int kt = 0; kt < k_tiles; ++kt) {
                    bar.ab.wait_empty(st);
                    mbar_arrive_expect_tx(&bar.ab.full[st.slot], kStage);
                    tma::load_2d(sA(st.slot).ptr, &p.tm_a, &bar.ab.full[st.slot], kt * BK, rb * BM);
#pragma unroll
                    for (int a = 0; a < BN / 64; ++a)
                        tma::load_2d(sB(st.slot) + a * kBAtom, &p.tm_b, &bar.ab.full[st.slot], cb * BN + a * 64,
                                     kt * BK);
                    st.advance();
                }
            }
            (void)pol;
        }
    } else if (warp == 1) {
        // -------------------------------------------------------------------- MMA
        lcsf::ring_state<kStages> st;
        int n = 0;
        for (int t = blockIdx.x; t < tasks; t += gridDim.x, ++n) {
            const int buf = n & 1;
            mbar_wait(&bar.acc_empty[buf], ((n >> 1) & 1) ^ 1u);  // the epilogue drained this buffer
            tmem::fence_after();
            const uint32_t acc = tbase + buf * BN;
            for (int kt = 0; kt < k_tiles; ++kt) {
                bar.ab.wait_full(st);
                tmem::fence_after();
                // C (+)= A B: A K-major, B = swap_layout of the [BK rows][BN] panel (mma_AB)
                mma_AB(tt_fl<BN>{acc}, sA(st.slot), swap_layout(st_bf<BK, BN>{sB(st.slot)}), kt > 0);
                mma_commit(&bar.ab.empty[st.slot]);  // panel consumed -> the producer may refill it
                st.advance();
            }
            mma_commit(&bar.acc_full[buf]);
        }
    } else if (warp >= 4) {
        // -------------------------------------------------------------------- FINISH
        const int wq = warp & 3;
        const int r = wq * 32 + lane;
        const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
        const bool leader = (warp == 4 && lane == 0);
        const st_bf<BM, 64> stage{stage_c};
        int n = 0;
        for (int t = blockIdx.x; t < tasks; t += gridDim.x, ++n) {
            int rb, cb;
            supergroup(t, r_blocks, c_blocks, p.super_m, rb, cb);
            const int buf = n & 1;
            mbar_wait(&bar.acc_full[buf], (n >> 1) & 1);
            tmem::fence_after();
            const uint32_t acc = tbase + lane_off + buf * BN;
#pragma unroll 1
            for (int a = 0; a < BN / 64; ++a) {
                rt_fl<32> v0, v1;
                load(v0, acc + a * 64);
                load(v1, acc + a * 64 + 32);
                load_wait(v0);
                load_wait(v1);
                if (a == BN / 64 - 1) {  // accumulator drained: the MMA warp may reuse it
                    tmem::fence_before();
                    mbar_arrive(&bar.acc_empty[buf]);
                }
                rt_bf<32> b0, b1;
                copy(b0, v0);
                copy(b1, v1);
                if (leader) tma::wait_group_read<0>();  // staging atom free again
                named_sync(kBarEpi, WARPGROUP_THREADS);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    sts_v4(smem_u32(stage.chunk(r, q)), make_uint4(b0.v[4 * q], b0.v[4 * q + 1], b0.v[4 * q + 2],
                                                                   b0.v[4 * q + 3]));
                    sts_v4(smem_u32(stage.chunk(r, 4 + q)), make_uint4(b1.v[4 * q], b1.v[4 * q + 1],
                                                                       b1.v[4 * q + 2], b1.v[4 * q + 3]));
                }
                tma::fence_async_smem();
                named_sync(kBarEpi, WARPGROUP_THREADS);
                if (leader) {
                    tma::store_2d(&p.tm_c, stage.ptr, cb * BN + a * 64, rb * BM);
                    tma::commit_group();
                }
            }
        }
        if (leader) tma::wait_group<0>();
    }

    tmem::fence_before();
    __syncthreads();
    if (warp == 1) tmem::dealloc<512>(tbase);
}

// ------------------------------------------------------------------ CTA pairs (cta_group::2)
// The same GEMM on 2-CTA clusters: a pair computes a 256 x 256 block of C with M = 256 pair
// MMAs (tkb/cluster.cuh). Each CTA holds its 128 rows of the A panel and its 128-column half
// of the B panel (32 KB per stage instead of 48), so per SM a K = 16 step reads 4 + 4 KB of
// SMEM instead of 4 + 8 and the TMA moves a third less: six stages fit where four did.
// Both CTAs' TMA complete on the leader's full barrier; the leader's MMA warp issues for the
// pair and commits multicast (ring slots to both producers, accumulators to both epilogues);
// each CTA's epilogue drains its own TMEM rows and arrives on the leader's acc_empty.
namespace pair2 {
constexpr int BM = 128, BN = 256, BK = 64;  // per CTA: 128 rows; pair tile 256 x 256
#ifndef TKB_GEMM2_STAGES
#define TKB_GEMM2_STAGES 6
#endif
#ifndef TKB_GEMM2_STAGING
#define TKB_GEMM2_STAGING 2
#endif
constexpr int kStages = TKB_GEMM2_STAGES;
constexpr int kStagingAtoms = TKB_GEMM2_STAGING;  // output atoms staged in flight (epilogue)
constexpr int kATile = BM * BK * 2;         // 16 KB
constexpr int kBHalf = BK * (BN / 2) * 2;   // 16 KB: 2 atoms of 64 K rows x 64 N cols
constexpr int kBAtom = BK * 128;            // 8 KB
constexpr int kStage = kATile + kBHalf;
constexpr int kStaging = BM * 128;
constexpr int kOffBar = kStages * kStage + kStagingAtoms * kStaging;
constexpr int kSmemBytes = kOffBar + 256 + 1024;
static_assert(kSmemBytes <= 232448, "smem");
constexpr int kThreads = 256;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm2_kernel(const __grid_constant__ GemmParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    auto sA = [&](int s) { return st_bf<BM, BK>{smem + s * kStage}; };
    auto sB = [&](int s) { return smem + s * kStage + kATile; };  // this CTA's [BK][BN/2] MN-major half
    uint8_t* stage_c = smem + kStages * kStage;
    struct Bars {
        mbarrier full[kStages], empty[kStages];
        mbarrier acc_full[2], acc_empty[2];
        uint32_t tmem_slot;
    };
    Bars& bar = *reinterpret_cast<Bars*>(smem + kOffBar);
    static_assert(sizeof(Bars) <= 256, "barrier area");

    const int warp = warpid();
    const int lane = laneid();
    const uint32_t rank = cluster::ctarank();
    const bool leader = rank == 0;
    const int r_blocks = (p.m + 2 * BM - 1) / (2 * BM), c_blocks = (p.n + BN - 1) / BN;
    const int tasks = r_blocks * c_blocks;
    const int k_tiles = (p.k + BK - 1) / BK;
    const int pair_id = blockIdx.x >> 1, pairs = gridDim.x >> 1;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&bar.full[s], 1);
            mbar_init(&bar.empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bar.acc_full[i], 1);
            mbar_init(&bar.acc_empty[i], 2 * 4);  // one lane per epilogue warp, both CTAs
        }
        fence_barrier_init();
        tma::prefetch_desc(&p.tm_a);
        tma::prefetch_desc(&p.tm_b);
        tma::prefetch_desc(&p.tm_c);
    }
    if (warp == 1) tmem::alloc2<512>(&bar.tmem_slot);
    tmem::fence_before();
    cluster::sync();  // both CTAs' barriers initialised before any remote arrive / complete_tx
    tmem::fence_after();
    const uint32_t tbase = bar.tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------------------------------------------------------- LOAD (both CTAs)
            lcsf::ring_state<kStages> st;
            for (int t = pair_id; t < tasks; t += pairs) {
                int rb, cb;
                supergroup(t, r_blocks, c_blocks, p.super_m, rb, cb);
                const int row0 = rb * 2 * BM + (int)rank * BM, col0 = cb * BN + (int)rank * (BN / 2);
                for (int kt = 0; kt < k_tiles; ++kt) {
                    mbar_wait(&bar.empty[st.slot], st.phase ^ 1u);
                    const uint32_t fb = cluster::map(&bar.full[st.slot], 0);
                    if (leader) mbar_arrive_expect_tx(&bar.full[st.slot], 2 * kStage);
                    cluster::load_2d(sA(st.slot).ptr, &p.tm_a, fb, kt * BK, row0);
#pragma unroll
                    for (int a = 0; a < BN / 128; ++a)
                        cluster::load_2d(sB(st.slot) + a * kBAtom, &p.tm_b, fb, col0 + a * 64, kt * BK);
                    st.advance();
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {
            // -------------------------------------------------------------------- MMA (leader)
            constexpr uint32_t idesc = umma::idesc_bf16_m256<BN, false, true>();
            constexpr uint32_t hi = umma::desc_hi_sw128(1024);
            lcsf::ring_state<kStages> st;
            int n = 0;
            for (int t = pair_id; t < tasks; t += pairs, ++n) {
                const int buf = n & 1;
                cluster::wait(&bar.acc_empty[buf], ((n >> 1) & 1) ^ 1u);  // both epilogues drained it
                tmem::fence_after();
                const uint32_t acc = tbase + buf * BN;
                for (int kt = 0; kt < k_tiles; ++kt) {
                    cluster::wait(&bar.full[st.slot], st.phase);
                    tmem::fence_after();
                    const uint32_t a0 = sA(st.slot).addr(), b0 = smem_u32(sB(st.slot));
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)  // C (+)= A B: A K-major, B MN-major (its N half per CTA)
                        umma::mma2_ss_e(acc, umma::desc_lo(a0 + k * 32, 16), hi, umma::desc_lo(b0 + k * 16 * 128, kBAtom),
                                        hi, idesc, (kt > 0 || k > 0) ? 1u : 0u);
                    pair::mma_commit(&bar.empty[st.slot]);  // both CTAs may refill this slot
                    st.advance();
                }
                pair::mma_commit(&bar.acc_full[buf]);
            }
        }
    } else if (warp >= 4) {
        // -------------------------------------------------------------------- FINISH (both CTAs)
        const int wq = warp & 3;
        const int r = wq * 32 + lane;
        const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
        const bool lead_thr = (warp == 4 && lane == 0);
        const uint32_t empty_remote[2] = {cluster::map(&bar.acc_empty[0], 0), cluster::map(&bar.acc_empty[1], 0)};
        int n = 0;
        for (int t = pair_id; t < tasks; t += pairs, ++n) {
            int rb, cb;
            supergroup(t, r_blocks, c_blocks, p.super_m, rb, cb);
            const int buf = n & 1;
            cluster::wait(&bar.acc_full[buf], (n >> 1) & 1);
            tmem::fence_after();
            const uint32_t acc = tbase + lane_off + buf * BN;
#pragma unroll 1
            for (int a = 0; a < BN / 64; ++a) {
                rt_fl<32> v0, v1;
                load(v0, acc + a * 64);
                load(v1, acc + a * 64 + 32);
                load_wait(v0);
                load_wait(v1);
                if (a == BN / 64 - 1) {  // accumulator drained: the leader's MMA may reuse it
                    tmem::fence_before();
                    __syncwarp();
                    if (lane == 0) cluster::arrive_remote(empty_remote[buf]);
                }
                rt_bf<32> b0, b1;
                copy(b0, v0);
                copy(b1, v1);
                // rotating staging atoms: the one written now was last stored kStagingAtoms
                // stores ago; wait until at most kStagingAtoms - 1 stores are still reading
                const st_bf<BM, 64> stage{stage_c + (a % kStagingAtoms) * kStaging};
                if (lead_thr) tma::wait_group_read<kStagingAtoms - 1>();
                named_sync(kBarEpi, WARPGROUP_THREADS);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    sts_v4(smem_u32(stage.chunk(r, q)), make_uint4(b0.v[4 * q], b0.v[4 * q + 1], b0.v[4 * q + 2],
                                                                   b0.v[4 * q + 3]));
                    sts_v4(smem_u32(stage.chunk(r, 4 + q)), make_uint4(b1.v[4 * q], b1.v[4 * q + 1],
                                                                       b1.v[4 * q + 2], b1.v[4 * q + 3]));
                }
                tma::fence_async_smem();
                named_sync(kBarEpi, WARPGROUP_THREADS);
                if (lead_thr) {
                    tma::store_2d(&p.tm_c, stage.ptr, cb * BN + a * 64, rb * 2 * BM + (int)rank * BM);
                    tma::commit_group();
                }
            }
        }
        if (lead_thr) tma::wait_group<0>();
    }

    tmem::fence_before();
    cluster::sync();  // the peer's TMEM / barriers stay live until both CTAs are done
    if (warp == 1) tmem::dealloc2<512>(tbase);
}
}  // namespace pair2

}  // namespace gemm

#ifndef TKB_GEMM_PAIRS
#define TKB_GEMM_PAIRS 1
#endif

int launch_gemm(const GemmParams& p, int num_sms, cudaStream_t stream) {
    static std::atomic<unsigned long long> smem_set{0}, smem_set2{0};  // per device
    if (TKB_GEMM_PAIRS && p.m > gemm::BM) {  // CTA pairs: a 256 x 256 block of C per cluster
        if (int e = ensure_smem(gemm::pair2::gemm2_kernel, gemm::pair2::kSmemBytes, smem_set2)) return e;
        const int tasks = ((p.m + 2 * gemm::BM - 1) / (2 * gemm::BM)) * ((p.n + gemm::BN - 1) / gemm::BN);
        const int pairs = tasks < num_sms / 2 ? tasks : num_sms / 2;
        gemm::pair2::gemm2_kernel<<<2 * pairs, gemm::pair2::kThreads, gemm::pair2::kSmemBytes, stream>>>(p);
        return (int)cudaGetLastError();
    }
    if (int e = ensure_smem(gemm::gemm_kernel, gemm::kSmemBytes, smem_set)) return e;
    const int tasks = ((p.m + gemm::BM - 1) / gemm::BM) * ((p.n + gemm::BN - 1) / gemm::BN);
    const int grid = tasks < num_sms ? tasks : num_sms;
    gemm::gemm_kernel<<<grid, gemm::kThreads, gemm::kSmemBytes, stream>>>(p);
    return (int)cudaGetLastError();
}

}  // namespace tkb
