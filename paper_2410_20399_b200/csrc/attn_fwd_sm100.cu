// attn_fwd_sm100.cu — attention forward for B200 (sm_100a): TMA -> tcgen05 -> TMEM,
// persistent and warp-specialised.
//
// Reference: kittensim attention_fwd_kernel (kernels.hpp:250-343) and the paper's
// H100 listing attn_fwd_template<D>. Same math (online softmax in
// the exp2 domain with tau = scale * log2 e, fp32 row normaliser summed over fp32 P,
// bf16 P into the PV product, kernels.hpp:315-332), re-built as the LCSF template
// (lcsf.hpp:112-161) in hardware, written with the tile vocabulary of tkb/tile.cuh:
//
//   warp 13     LOAD (producer): claims tasks from the persistent queue, TMA of the two
//               Q tiles of a task, then K_j / V_j through a K/V ring (4 slots at D=128)
//   warp 12     MMA (one thread): S_s = Q_s K_j^T (mm_ABt, both K-major in SMEM) and
//               O_s += P_s V_j (mma_AB, P from TMEM, V MN-major)
//   warps 0-3   SOFTMAX tile 0 (query rows q0 .. q0+127), warps 4-7 SOFTMAX tile 1:
//               one thread per row: tcgen05.ld of S, row_max, exp2 (MUFU plus a
//               polynomial share on the FMA pipe), row_sum, bf16 P into TMEM over S
//   warps 8-11  CORRECTION + FINISH: rescales O when a row max moved by more than 2^8
//               (lazy rescale), and the finish stage O / l -> bf16 -> SMEM -> TMA store
//
// A task is (batch, head, 256-query block). Tasks are claimed dynamically (heavy causal
// blocks first inside L2-sized groups of heads, whose K/V stay resident in the 126 MB
// L2 while their query blocks run), so one CTA per SM streams tasks back to back: the
// next task's Q is prefetched into L2 when it is claimed and its first K/V tiles load
// while the current task drains.
//
// TMEM (512 columns): S0 [0,128) S1 [128,256) O0 [256,256+D) O1 [256+D,256+2D);
// P_s = bf16 pairs in columns [S_s+64, S_s+128).
//
// Ordering: tcgen05.mma ops of the one issuing thread execute in order, so issuing
// PV_{j-1}(s) before QK_j(s) makes "S_j(s) full" imply "PV_{j-1}(s) done": the softmax
// may then overwrite P_s and the correction warps may rescale O_s with no extra barrier.
#include <cuda.h>
#include <cuda_runtime.h>

#include "attn_common.cuh"
#include "tkb/lcsf.cuh"
#include "tkb/tile.cuh"

namespace tkb {
namespace fwd {

#ifndef TKB_FWD_POLY128
#define TKB_FWD_POLY128 2
#endif
#ifndef TKB_FWD_POLY64
#define TKB_FWD_POLY64 3
#endif

template <int D>
struct Cfg {
    using Tile = st_bf<128, D>;                            // Q, K, V, O tiles
    static constexpr int kTile = Tile::kBytes;
    static constexpr int kKvSlots = (D == 128) ? 4 : 8;     // K and V alternate in the ring
    static constexpr int kPolyPairs = (D == 128) ? TKB_FWD_POLY128 : TKB_FWD_POLY64;  // of every 8 exp2 pairs
    static constexpr int kOffQ = 0;
    static constexpr int kOffKV = kOffQ + 2 * kTile;
    static constexpr int kOffO = kOffKV + kKvSlots * kTile;  // finish staging: one 128 x D tile
    static constexpr int kOffAlpha = kOffO + kTile;         // [2][128] rescale factors
    static constexpr int kOffInvL = kOffAlpha + 1024;       // [2][128] 1 / l
    static constexpr int kOffNeed = kOffInvL + 1024;        // [2][4] per-warp rescale flags
    static constexpr int kOffBar = kOffNeed + 64;
    static constexpr int kBarBytes = 512;
    // The dynamic SMEM window starts 1024-byte aligned when the kernel has no static SMEM
    // (checked at run time: a misaligned base traps); D=64 keeps the slack anyway.
    static constexpr int kSlack = (kOffBar + kBarBytes + 1024 <= 232448) ? 1024 : 0;
    static constexpr int kSmemBytes = kOffBar + kBarBytes + kSlack;
    static_assert(kSmemBytes <= 232448, "smem");
    static TKB_DEVICE constexpr uint32_t tmem_s(int s) { return s * 128u; }
    static TKB_DEVICE constexpr uint32_t tmem_o(int s) { return 256u + s * D; }
};

constexpr int kThreads = 512;
constexpr int kWarpMma = 12;
constexpr int kWarpLoad = 13;
constexpr int kWarpCorr0 = 8;
constexpr int kBarEpi = 3;
constexpr int kPChunks = 4;                // P chunks of 32 keys (16 TMEM columns) per tile                 // named barrier of the correction warpgroup
constexpr float kRescaleThreshold = 8.0f;  // log2 units: defer the O rescale while max grows < 2^8
constexpr float kLn2 = 0.69314718055994530942f;

template <int KV_SLOTS>
struct Barriers {
    lcsf::work_queue queue;
    lcsf::ring<KV_SLOTS> kv;
    mbarrier q_full[2], q_empty[2];
    mbarrier s_full[2], o_full[2], stat_full[2], fin_full[2];
    mbarrier p_full[2][kPChunks];  // P in 32-column chunks: PV starts while the softmax still runs
    uint32_t tmem_slot;
};

struct Task {
    int mblk, bh, nkv;
};

// task id -> (256-row query block, batch*head, kv blocks visited). Heads are taken in groups
// of p.head_group; inside a group the heavy (late) causal query blocks come first.
template <bool CAUSAL>
TKB_DEVICE Task decode(const FwdParams& p, int t) {
    const int M = p.m_blocks;
    const int G = p.head_group;
    const int sec = t / (G * M);
    const int r = t - sec * G * M;
    const int gs = min(G, p.bh - sec * G);
    const int mi = r / gs;
    Task w;
    w.bh = sec * G + (r - mi * gs);
    w.mblk = CAUSAL ? (M - 1 - mi) : mi;
    int nkv = (p.n + kBlockN - 1) / kBlockN;
    if (CAUSAL) nkv = min(nkv, (min(w.mblk * kRowsPerCta + kRowsPerCta, p.n) - 1) / kBlockN + 1);
    w.nkv = nkv;
    return w;
}

// Per-role cycle timeline (debug builds with -DTKB_FWD_TRACE; see tkb_debug_set_trace).
#ifdef TKB_FWD_TRACE
#define TKB_FTR(role, it, ev)                                                                        \
    do {                                                                                             \
        const int ti_ = (it) - tr_off;                                                               \
        if (tr != nullptr && ti_ >= 0 && ti_ < kTraceIters)                                          \
            tr[((role) * kTraceIters + ti_) * kTraceEvents + (ev)] = clock64() - t_start;            \
    } while (0)
#else
#define TKB_FTR(role, it, ev) \
    do {                      \
    } while (0)
#endif

template <int D, bool CAUSAL>
__global__ void __launch_bounds__(kThreads, 1) attn_fwd_kernel(const __grid_constant__ FwdParams p) {
    using C = Cfg<D>;
    using Tile = typename C::Tile;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    if constexpr (C::kSlack == 0) {
        if ((smem_u32(smem_raw) & 1023u) != 0) __trap();  // SW128 tiles need a 1024-byte aligned base
    }
    const uint32_t sAlpha = smem_u32(smem + C::kOffAlpha);  // [2][128] f32 (shared-space addresses)
    const uint32_t sInvL = smem_u32(smem + C::kOffInvL);    // [2][128] f32
    const uint32_t sNeed = smem_u32(smem + C::kOffNeed);    // [2][4] u32
    auto& bar = *reinterpret_cast<Barriers<C::kKvSlots>*>(smem + C::kOffBar);
    static_assert(sizeof(Barriers<C::kKvSlots>) <= C::kBarBytes, "barrier area");
    const Tile sQ[2] = {Tile{smem + C::kOffQ}, Tile{smem + C::kOffQ + C::kTile}};
    auto sKV = [&](int slot) { return Tile{smem + C::kOffKV + slot * C::kTile}; };
    const Tile sO{smem + C::kOffO};
    const gl gQ{&p.tm_q}, gK{&p.tm_k}, gV{&p.tm_v}, gO{&p.tm_o};

    const int warp = warpid();
    const int lane = laneid();
#ifdef TKB_FWD_TRACE
    long long* tr = nullptr;
    const int tr_off = p.trace_slots >> 16;  // first traced iteration (debug: slots | offset << 16)
    if (p.trace != nullptr && (int)blockIdx.x % p.trace_every == 0 &&
        (int)blockIdx.x / p.trace_every < (p.trace_slots & 0xffff))
        tr = p.trace + (size_t)((int)blockIdx.x / p.trace_every) * kTraceRoles * kTraceIters * kTraceEvents;
    const long long t_start = clock64();
#endif

    if (warp == kWarpLoad && lane == 0) {
        bar.queue.init(1 + 8 + 4);  // MMA, 8 softmax warps, 4 correction warps
        bar.kv.init(1, 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bar.q_full[s], 1);
            mbar_init(&bar.q_empty[s], 1);
            mbar_init(&bar.s_full[s], 1);
            mbar_init(&bar.p_full[s][0], 2 * WARPGROUP_THREADS);  // softmax + correction (O rescaled)
            for (int c = 1; c < kPChunks; ++c) mbar_init(&bar.p_full[s][c], WARPGROUP_THREADS);
            mbar_init(&bar.o_full[s], 1);
            mbar_init(&bar.stat_full[s], WARPGROUP_THREADS);
            mbar_init(&bar.fin_full[s], WARPGROUP_THREADS);
        }
        fence_barrier_init();
        gQ.prefetch();
        gK.prefetch();
        gV.prefetch();
        gO.prefetch();
    }
    if (warp == kWarpMma) tmem::alloc<512>(&bar.tmem_slot);
    tmem::fence_before();
    __syncthreads();
    tmem::fence_after();
    // each role re-reads the TMEM base after its register reconfiguration (a value live
    // across setmaxnreg is spilled by ptxas)
    auto tmem_base = [&]() { return *reinterpret_cast<volatile uint32_t*>(&bar.tmem_slot); };

    if (warp >= 12) {
        setmaxnreg_dec<80>();
        const uint32_t tbase = tmem_base();
        if (warp == kWarpLoad && lane == 0) {
            // ------------------------------------------------------------ LOAD (producer)
            const uint64_t pol_q = tma::policy_evict_first();
            const uint64_t pol_kv = tma::policy_evict_last();
            lcsf::ring_state<C::kKvSlots> st;
            int n = 0;
            int t = bar.queue.claim(0, p.sched, p.tasks);
            while (t >= 0) {
                const Task w = decode<CAUSAL>(p, t);
                const int b = w.bh / p.heads, h = w.bh - b * p.heads;
                const int q0 = w.mblk * kRowsPerCta;
                for (int s = 0; s < 2; ++s) {
                    mbar_wait(&bar.q_empty[s], (n & 1) ^ 1u);
                    mbar_arrive_expect_tx(&bar.q_full[s], C::kTile);
                    load_async(sQ[s], gQ, &bar.q_full[s], q0 + s * kBlockM, h, b, pol_q);
                }
                // claim the next task now and warm its Q in L2 while this one runs
                const int t_next = bar.queue.claim(n + 1, p.sched, p.tasks);
                if (t_next >= 0) {
                    const Task w2 = decode<CAUSAL>(p, t_next);
                    const int b2 = w2.bh / p.heads, h2 = w2.bh - b2 * p.heads;
                    for (int s = 0; s < 2; ++s)
                        for (int a = 0; a < Tile::kAtoms; ++a)
                            tma::prefetch_4d(gQ.tm, a * 64, w2.mblk * kRowsPerCta + s * kBlockM, h2, b2);
                }
                for (int j = 0; j < w.nkv; ++j) {
#pragma unroll
                    for (int which = 0; which < 2; ++which) {
                        bar.kv.wait_empty(st);
                        mbar_arrive_expect_tx(&bar.kv.full[st.slot], C::kTile);
                        load_async(sKV(st.slot), which == 0 ? gK : gV, &bar.kv.full[st.slot], j * kBlockN, h, b,
                                   pol_kv);
                        st.advance();
                    }
                }
                t = t_next;
                ++n;
            }
        } else if (warp == kWarpMma) {
            // ------------------------------------------------------------ MMA (tensor part of compute)
            // the whole warp runs this loop converged; one elected lane issues each tcgen05 op
            lcsf::ring_state<C::kKvSlots> st;
            uint32_t it = 0;  // p_full completions so far (one per task iteration)
            // O_s (+)= P_s V: chunk c (keys 32c .. 32c+31) is issued as soon as the softmax stored it
            auto pv_chunks = [&](int s, int vslot, bool acc, uint32_t iter) {
                const Tile v = sKV(vslot);
#pragma unroll
                for (int c = 0; c < kPChunks; ++c) {
                    mbar_wait(&bar.p_full[s][c], iter & 1);
                    tmem::fence_after();
                    mma_AB_k<D, 32>(tt_fl<D>{tbase + C::tmem_o(s)}, tt_bf<16>{tbase + C::tmem_s(s) + 64 + 16 * c},
                                    v, 32 * c, acc || c > 0);
                }
            };
            // One flat stream of iterations that runs across task boundaries: iteration
            // (PV_s(block j of task n), QK_s(next block)) where the next block may be block 0
            // of task n+1, so the next task's S = Q K^T overlaps the last softmax of this one.
            int n = 0;
            int t = bar.queue.get(0);
            if (lane == 0) bar.queue.release(0);
            if (t >= 0) {
                Task w = decode<CAUSAL>(p, t);
                mbar_wait(&bar.q_full[0], 0);
                mbar_wait(&bar.q_full[1], 0);
                bar.kv.wait_full(st);
                tmem::fence_after();
                const int k0 = st.slot;
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    mm_ABt(tt_fl<128>{tbase + C::tmem_s(s)}, sQ[s], sKV(k0));
                    umma::commit_e(&bar.s_full[s]);
                    if (w.nkv == 1) umma::commit_e(&bar.q_empty[s]);
                }
                umma::commit_e(&bar.kv.empty[k0]);
                st.advance();
                int j = 0;  // block whose PV is issued next
                for (;;) {
                    // what follows block j: block j+1 of this task, or block 0 of the next task
                    const bool last = (j == w.nkv - 1);
                    int t_next = t;
                    Task w_next = w;
                    if (last) {
                        t_next = bar.queue.get(n + 1);
                        if (lane == 0) bar.queue.release(n + 1);
                        if (t_next >= 0) w_next = decode<CAUSAL>(p, t_next);
                    }
                    const bool has_next = !last || t_next >= 0;
                    const int jn = last ? 0 : j + 1;
                    const int vslot = st.slot;  // V_j
                    bar.kv.wait_full(st);
                    st.advance();
                    const int kslot = st.slot;  // K of the next block
                    TKB_FTR(0, (int)it, 0);
#pragma unroll
                    for (int s = 0; s < 2; ++s) {
                        pv_chunks(s, vslot, j > 0, it);
                        TKB_FTR(0, (int)it, 3 + 2 * s);
                        if (last) umma::commit_e(&bar.o_full[s]);
                        if (has_next) {
                            if (s == 0) bar.kv.wait_full(st);
                            if (last) mbar_wait(&bar.q_full[s], (n + 1) & 1);
                            tmem::fence_after();
                            mm_ABt(tt_fl<128>{tbase + C::tmem_s(s)}, sQ[s], sKV(kslot));
                            TKB_FTR(0, (int)it, 4 + 2 * s);
                            umma::commit_e(&bar.s_full[s]);
                            if (jn == w_next.nkv - 1) umma::commit_e(&bar.q_empty[s]);
                        }
                    }
                    umma::commit_e(&bar.kv.empty[vslot]);
                    ++it;
                    if (!has_next) break;
                    umma::commit_e(&bar.kv.empty[kslot]);
                    st.advance();
                    if (last) {
                        ++n;
                        t = t_next;
                        w = w_next;
                    }
                    j = jn;
                }
            }
        }
    } else if (warp < 8) {
        // ---------------------------------------------------------------- SOFTMAX (compute)
        setmaxnreg_inc<176>();
        const uint32_t tbase = tmem_base();
        const int s = warp >> 2;        // query tile of this warpgroup
        const int wq = warp & 3;        // TMEM lane quarter
        const int r = wq * 32 + lane;   // row within the tile == TMEM lane
        const uint32_t tS = tbase + ((uint32_t)(wq * 32) << 16) + C::tmem_s(s);
        const float tau = p.scale_log2;
        uint32_t sc = 0;  // s_full completions seen
        for (int n = 0;; ++n) {
            const int t = bar.queue.get(n);
            __syncwarp();
            if (lane == 0) bar.queue.release(n);
            if (t < 0) break;
            const Task w = decode<CAUSAL>(p, t);
            const int q0 = w.mblk * kRowsPerCta + s * kBlockM;
            const int row = q0 + r;
            float m = -INFINITY;  // running max of tau * S (the value subtracted)
            float l = 0.f;        // running normaliser (fp32 sum of fp32 P, kernels.hpp:324)
            for (int j = 0; j < w.nkv; ++j) {
                mbar_wait(&bar.s_full[s], sc & 1);
                ++sc;
                if (threadIdx.x % 128 == 0) TKB_FTR(1 + s, (int)(sc - 1), 0);
                tmem::fence_after();
                rt_fl<128> x;
                load(x, tS);
                load_wait(x);
                if (threadIdx.x % 128 == 0) TKB_FTR(1 + s, (int)(sc - 1), 3);
                const int kv0 = j * kBlockN;
                const bool need_mask = CAUSAL ? (kv0 + kBlockN - 1 > q0) : (kv0 + kBlockN > p.n);
                if (need_mask) {
                    const int lim = CAUSAL ? min(row - kv0, p.n - 1 - kv0) : (p.n - 1 - kv0);  // last visible
#pragma unroll
                    for (int c = 0; c < kBlockN; ++c)
                        if (c > lim) x.v[c] = -INFINITY;
                }
                float mx = -INFINITY;
                row_max(mx, x);
                const float m_new = fmaxf(m, mx * tau);
                // lazy rescale, warp-uniform (the correction warp works on whole lane quarters)
                const bool need = __any_sync(0xffffffffu, m_new > m + kRescaleThreshold);
                if (need) {
                    const float alpha = ex2_approx(m - m_new);  // exp2(-inf) = 0 on the first tile
                    m = m_new;
                    l *= alpha;
                    sts_f32(sAlpha + (s * 128 + r) * 4, alpha);
                }
                if (j > 0) {  // the correction warps rescale O_s before PV_s(j) (nothing to do at j = 0)
                    if (lane == 0) sts_u32(sNeed + (s * 4 + wq) * 4, need ? 1u : 0u);
                    mbar_arrive(&bar.stat_full[s]);
                }
                if (threadIdx.x % 128 == 0) TKB_FTR(1 + s, (int)(sc - 1), 1);
                // P = exp2(tau S - m): MUFU ex2, kPolyPairs of every 8 pairs as a polynomial on the
                // FMA pipe; row_sum over fp32 P; P -> bf16 (RNE) into TMEM over S
                const float2 tau2 = make_float2(tau, tau), nm2 = make_float2(-m, -m);
                float2 acc[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
                uint32_t pk[2][16];  // double-buffered P chunk: st of chunk c overlaps exp of chunk c+1
#pragma unroll
                for (int ch = 0; ch < kPChunks; ++ch) {
#pragma unroll
                    for (int c = 32 * ch; c < 32 * ch + 32; c += 2) {
                        const float2 xv = fma2(make_float2(x.v[c], x.v[c + 1]), tau2, nm2);
                        float2 pv;
                        if (((c / 2) % 8) < C::kPolyPairs) {
                            pv = ex2_poly2(xv);
                        } else {
                            pv.x = ex2_approx(xv.x);
                            pv.y = ex2_approx(xv.y);
                        }
                        acc[(c / 2) % 4] = add2(acc[(c / 2) % 4], pv);
                        pk[ch & 1][(c / 2) % 16] = pack_bf16x2(pv.x, pv.y);
                    }
                    if (ch > 0) {  // chunk ch-1 is in TMEM: hand it to the MMA warp
                        tmem::wait_st();
                        tmem::fence_before();
                        mbar_arrive(&bar.p_full[s][ch - 1]);
                    }
                    tmem::st_32x32b_x16(tS + 64 + 16 * ch, pk[ch & 1]);
                }
                l += ((acc[0].x + acc[0].y) + (acc[1].x + acc[1].y)) + ((acc[2].x + acc[2].y) + (acc[3].x + acc[3].y));
                if (threadIdx.x % 128 == 0) TKB_FTR(1 + s, (int)(sc - 1), 4);
                tmem::wait_st();
                tmem::fence_before();
                mbar_arrive(&bar.p_full[s][kPChunks - 1]);
                if (threadIdx.x % 128 == 0) TKB_FTR(1 + s, (int)(sc - 1), 2);
            }
            // finish statistics: L = ln2 (m + log2 l) (the natural-log LSE of S * scale) and 1 / l
            if (p.lse != nullptr && row < p.n) p.lse[(size_t)w.bh * p.n + row] = (m + __log2f(l)) * kLn2;
            sts_f32(sInvL + (s * 128 + r) * 4, 1.f / l);
            // a barrier of its own: on stat_full the next task's first arrival could otherwise
            // run two phases ahead of the correction warps (phase-parity aliasing)
            mbar_arrive(&bar.fin_full[s]);
        }
    } else {
        // ---------------------------------------------------------------- CORRECTION + FINISH
        setmaxnreg_dec<80>();
        const uint32_t tbase = tmem_base();
        const int wq = warp - kWarpCorr0;  // TMEM lane quarter (same as softmax warps wq, 4 + wq)
        const int r = wq * 32 + lane;
        const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
        const bool leader = (threadIdx.x == kWarpCorr0 * 32);
        uint32_t stc[2] = {0, 0};
        uint32_t ci = 0;
        for (int n = 0;; ++n) {
            const int t = bar.queue.get(n);
            __syncwarp();
            if (lane == 0) bar.queue.release(n);
            if (t < 0) break;
            const Task w = decode<CAUSAL>(p, t);
            // j = 0 needs no rescale (O is overwritten by the first PV): its p_full arrival came
            // with the previous task's drain of O (or here, for the first task), and stat_full
            // only carries j >= 1 so the softmax can never run two phases ahead of this warp.
            if (n == 0) {
#pragma unroll
                for (int s = 0; s < 2; ++s) mbar_arrive(&bar.p_full[s][0]);
            }
            for (int j = 1; j < w.nkv; ++j, ++ci) {
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    mbar_wait(&bar.stat_full[s], stc[s] & 1);
                    ++stc[s];
                    if (leader) TKB_FTR(3, (int)ci, 2 * s);
                    if (lds_u32(sNeed + (s * 4 + wq) * 4) != 0) {  // mul_row(o, o, alpha) (tiles.hpp:282-287)
                        const float alpha = lds_f32(sAlpha + (s * 128 + r) * 4);
                        const uint32_t tO = tbase + lane_off + C::tmem_o(s);
                        tmem::fence_after();
#pragma unroll
                        for (int c = 0; c < D; c += 32) {
                            rt_fl<32> o;
                            load(o, tO + c);
                            load_wait(o);
                            mul(o, alpha);
                            tmem::st_32x32b_x32(tO + c, reinterpret_cast<const uint32_t*>(o.v));
                        }
                        tmem::wait_st();
                    }
                    tmem::fence_before();
                    mbar_arrive(&bar.p_full[s][0]);
                    if (leader) TKB_FTR(3, (int)ci, 2 * s + 1);
                }
            }
            // FINISH (kernels.hpp:335-342): O / l -> bf16 -> SMEM -> TMA store
            const int b = w.bh / p.heads, h = w.bh - b * p.heads;
#pragma unroll 1
            for (int s = 0; s < 2; ++s) {
                mbar_wait(&bar.fin_full[s], n & 1);
                mbar_wait(&bar.o_full[s], n & 1);
                tmem::fence_after();
                const float inv_l = lds_f32(sInvL + (s * 128 + r) * 4);
                const uint32_t tO = tbase + lane_off + C::tmem_o(s);
                if (leader) tma::wait_group_read<0>();  // the staging tile is free again
                named_sync(kBarEpi, WARPGROUP_THREADS);
#pragma unroll
                for (int c = 0; c < D; c += 32) {
                    rt_fl<32> o;
                    load(o, tO + c);
                    load_wait(o);
                    mul(o, inv_l);
                    rt_bf<32> ob;
                    copy(ob, o);
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        sts_v4(smem_u32(sO.chunk(r, c / 8 + q)),
                               make_uint4(ob.v[4 * q], ob.v[4 * q + 1], ob.v[4 * q + 2], ob.v[4 * q + 3]));
                }
                // O_s is drained: the next task's first PV_s may overwrite it (its j = 0 arrival)
                tmem::fence_before();
                mbar_arrive(&bar.p_full[s][0]);
                tma::fence_async_smem();
                named_sync(kBarEpi, WARPGROUP_THREADS);
                if (leader) {
                    store_async(gO, sO, w.mblk * kRowsPerCta + s * kBlockM, h, b);
                    tma::commit_group();
                }
            }
        }
        if (leader) tma::wait_group<0>();
    }

    tmem::fence_before();
    __syncthreads();
    if (warp == kWarpMma) tmem::dealloc<512>(tmem_base());
    if (threadIdx.x == 0) lcsf::queue_exit(p.sched);
}
#undef TKB_FTR

template <int D, bool CAUSAL>
int launch(const FwdParams& p, int num_sms, cudaStream_t stream) {
    using C = Cfg<D>;
    auto kern = attn_fwd_kernel<D, CAUSAL>;
    static bool configured = false;  // per instantiation; attribute setting is idempotent
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
        if (e != cudaSuccess) return (int)e;
        configured = true;
    }
    const int grid = p.tasks < num_sms ? p.tasks : num_sms;
    kern<<<grid, kThreads, C::kSmemBytes, stream>>>(p);
    return (int)cudaGetLastError();
}

}  // namespace fwd

// Fills the scheduling fields of p (tasks, m_blocks, bh, head_group) and launches the
// persistent grid (one CTA per SM).
int launch_attn_fwd(int head_dim, bool causal, FwdParams p, int batches, int num_sms, cudaStream_t stream) {
    p.bh = batches * p.heads;
    p.m_blocks = (p.n + kRowsPerCta - 1) / kRowsPerCta;
    p.tasks = p.bh * p.m_blocks;
    // heads whose K/V (4 N D bytes each) fit in ~48 MB of L2 run together
    const long long kv_bytes = 4ll * p.n * head_dim;
    long long g = (48ll << 20) / (kv_bytes > 0 ? kv_bytes : 1);
    if (g < 1) g = 1;
    if (g > p.bh) g = p.bh;
    p.head_group = (int)g;
    if (head_dim == 128)
        return causal ? fwd::launch<128, true>(p, num_sms, stream) : fwd::launch<128, false>(p, num_sms, stream);
    return causal ? fwd::launch<64, true>(p, num_sms, stream) : fwd::launch<64, false>(p, num_sms, stream);
}

}  // namespace tkb
