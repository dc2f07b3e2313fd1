// attn_fwd_sm100.cu — attention forward for B200 (sm_100a): TMA -> tcgen05 -> TMEM.
//
// Reference: kittensim attention_fwd_kernel (kernels.hpp:250-343) and the paper's
// H100 listing attn_fwd_template<D>. Same math (online softmax in
// the exp2 domain with tau = scale * log2 e, fp32 row normaliser summed over fp32 P,
// bf16 P into the PV product, kernels.hpp:315-332), re-built for Blackwell as the LCSF
// template (lcsf.hpp:112-161) in hardware, written with the tile vocabulary of
// tkb/tile.cuh (st_bf / tt_fl / rt_fl, mm_ABt, mma_AB, row_max, load / store):
//
//   warp 8      LOAD     (producer worker): TMA Q once, then K_i / V_i into an
//                        N-slot SMEM ring (lcsf::ring, full/empty mbarriers)
//   warp 9      MMA      (consumer, tensor part; the warp runs converged and one
//                        elected lane issues): S_s = Q_s K_i^T (mm_ABt, SS, both
//                        K-major) and O_s += P_s V_i (mma_AB, TS: P from TMEM,
//                        V MN-major), P consumed in 32-key chunks as they arrive
//   warps 0-3   SOFTMAX0 (consumer, query tile 0: rows q0 .. q0+127)
//   warps 4-7   SOFTMAX1 (consumer, query tile 1: rows q0+128 .. q0+255)
//                        each thread owns one query row: tcgen05.ld of S,
//                        row_max, exp2, row_sum, bf16 P written back into TMEM
//                        (aliasing the upper half of S) chunk by chunk, lazy O
//                        rescale, then the FINISH stage: O / l -> bf16 -> SMEM ->
//                        TMA store, and L = ln2 * (m + log2 l).
//
// TMEM (512 columns): S0 [0,128) S1 [128,256) O0 [256,256+D) O1 [256+D,256+2D);
// P_s = bf16 pairs in columns [S_s+64, S_s+128).
//
// Tensor-core ordering: tcgen05.mma ops of one thread execute in issue order,
// so issuing PV_{i-1}(s) before QK_i(s) makes "S_i(s) full" imply "PV_{i-1}(s)
// done": the softmax may then rescale O_s and overwrite P_s safely.
//
// The kernel is lcsf::kernel<attn_fwd_template<D, Causal>> (tkb/lcsf.cuh: the LCSF skeleton
// owns the persistent task queue, barrier init, TMEM allocation and role dispatch; the
// template below supplies the layout and the load / mma / compute / finish hooks, as the
// paper's lcf::kernel<attn_fwd_template<D>>).
//
// A variant with a separate correction warpgroup (FA4-style) and an MMA stream running across
// task boundaries (git 283279c) measured 3-10% slower at N >= 4096: the two extra warps per
// SM sub-partition cost the softmax warps issue slots on the critical path.
#include <cuda.h>
#include <cuda_runtime.h>

#include "attn_common.cuh"
#include "tkb/lcsf.cuh"
#include "tkb/tile.cuh"

#ifndef TKB_FWD_POLY64
#define TKB_FWD_POLY64 1
#endif
#ifndef TKB_FWD_POLY128
#define TKB_FWD_POLY128 2
#endif
#ifndef TKB_ROPE_DEBUG
#define TKB_ROPE_DEBUG 0  // A/B only: 1 = aux warps publish without rotating, 2 = no flag waits
#endif
#ifndef TKB_FWD_TRACE
#define TKB_FWD_TRACE 0  // debug builds: per-task cycle stamps into tkb_debug_set_trace's buffer
#endif
#ifndef TKB_FWD_PCHUNKS
#define TKB_FWD_PCHUNKS 2
#endif

namespace tkb {
namespace fwd {

template <int D>
struct Cfg {
    using Tile = st_bf<128, D>;
    static constexpr int kTile = Tile::kBytes;
    static constexpr int kKvSlots = (D == 128) ? 4 : 8;  // K and V alternate in the ring
    // exp2 of one pair in every group of four columns, on kPolyGroups of every 4 groups, runs as
    // a polynomial on the FMA pipe (a quarter of the exponentials at 2): per SM sub-partition
    // the two softmax warps' 128 ex2 per kv block occupy MUFU (4 lanes / clk) for 2048 clk,
    // the whole MMA time of the block. At D = 128 this paid only once the row max moved to
    // FMNMX3 and the row sums to FADD2 (3 instead of 4 issue slots per element)
    static constexpr int kPolyGroups = (D == 64) ? TKB_FWD_POLY64 : TKB_FWD_POLY128;
    static constexpr int kSmemQ = kQStages * kTile;
    static constexpr int kSmemKv = kKvSlots * kTile;
    static constexpr int kStageBytes = 128 * 128;  // per-warpgroup O staging: one 128 x 64 atom
    static TKB_DEVICE constexpr uint32_t tmem_s(int s) { return s * 128u; }
    static TKB_DEVICE constexpr uint32_t tmem_o(int s) { return 256u + s * D; }
};

constexpr int kThreads = 320;
constexpr int kWarpLoad = 8;
constexpr int kWarpMma = 9;
constexpr int kPChunks = TKB_FWD_PCHUNKS;       // P handed to the MMA warp in chunks of 128/kPChunks keys
constexpr int kPChunkCols = kBlockN / kPChunks;  // keys per chunk
constexpr float kRescaleThreshold = 8.0f;        // log2 units: defer O rescale while max grows < 2^8
constexpr float kLn2 = 0.69314718055994530942f;

// TKB_FWD_TRACE: trace[slot][role][task n < 32][event] = clock64() (the SM's counter, shared by
// all warps of the CTA), for CTAs with blockIdx.x % trace_every == 0 (roles: 0 load, 1 MMA,
// 2 softmax tile 0, 3 tile 1)
TKB_DEVICE void fwd_stamp(const FwdParams& p, int role, int n, int ev) {
    if constexpr (TKB_FWD_TRACE != 0) {
        if (p.trace == nullptr || (int)blockIdx.x % p.trace_every || (int)blockIdx.x / p.trace_every >= p.trace_slots ||
            n >= kTraceIters)
            return;
        p.trace[(((size_t)(blockIdx.x / p.trace_every) * kTraceRoles + role) * kTraceIters + n) * kTraceEvents + ev] =
            clock64();
    }
}

// ROPE: the fused rotary prologue (rotary_kernel, kernels.hpp:357-513): two aux warps per
// CTA rotate Q and K into q_rot / k_rot block by block, ahead of and overlapped with the
// attention tasks (the same pass over Q / K a separate rotary launch would make, but its
// HBM traffic and issue slots now hide under the tensor-bound attention); the load warp
// TMA-reads a rotated block once its flag carries this launch's epoch.
template <int D, bool CAUSAL, bool ROPE = false>
struct attn_fwd_template {
    using C = Cfg<D>;
    using Tile = typename C::Tile;
    using globals = FwdParams;
    static constexpr int kAuxWarps = ROPE ? 2 : 0;
    static constexpr int kAuxWarp0 = 10;
    static constexpr int kThreads = fwd::kThreads + 32 * kAuxWarps;
    static constexpr int kTmemCols = 512;
    static constexpr int kProducerWarp = kWarpLoad;
    static constexpr int kMmaWarp = fwd::kWarpMma;
    static constexpr int kConsumerWarps = 8;      // two softmax warpgroups
    static constexpr int kQueueReaders = 1 + 8;   // the MMA warp and the 8 softmax warps
    static constexpr bool kAlignSlack = true;
    static constexpr bool kReleaseEarly = true;   // the softmax warps release a task id on reading it
    // D = 64: the 128 free TMEM columns hold a third S buffer; S / P rotate over three buffers
    // in QK issue order, so QK_{i+1}(s) is issued before PV_i(s) and the next block's
    // exponentials do not wait for the PV -> QK round trip (per-buffer s_full / p_full;
    // pv_done marks each PV_s for the lazy O rescale)
    static constexpr bool k3 = (D == 64);

    struct shared {  // placed 1024-aligned: the tiles first
        uint8_t q[kQStages][C::kTile];
        uint8_t kv[C::kKvSlots][C::kTile];
        uint8_t stage[kQStages][C::kStageBytes];  // per-warpgroup O staging atom
        mbarrier q_full[kQStages], q_empty[kQStages], s_full[kQStages], o_full[kQStages];
        mbarrier p_full[kQStages][kPChunks];
        lcsf::ring<C::kKvSlots> kv_ring;
        mbarrier s_full3[3], p_full3[3][kPChunks], pv_done[kQStages];
        lcsf::work_queue queue;
        uint32_t tmem_slot;
    };
    static constexpr int kSmemBytes = (int)sizeof(shared) + 1024;  // + alignment slack
    static_assert(kSmemBytes <= 232448, "smem");

    static TKB_DEVICE Tile sQ(shared& sh, int s) { return Tile{sh.q[s]}; }
    static TKB_DEVICE Tile sKV(shared& sh, int slot) { return Tile{sh.kv[slot]}; }
    static TKB_DEVICE st_bf<128, 64> sStage(shared& sh, int s) { return st_bf<128, 64>{sh.stage[s]}; }

    // task t -> (256-row query block, b, h): heads in L2-sized groups, inside a group the heavy
    // (late) causal query blocks first, heads innermost; claimed dynamically (one CTA per SM)
    struct Task {
        int mblk, head, batch, nkv;
        SeqView sv;  // this batch's length and TMA row coordinates (variable-length batches)
    };
    static TKB_DEVICE Task decode(const globals& p, int t) {
        const int N = p.n;
        const int rows = p.task_tiles * kBlockM;  // query rows per task
        const int m_blocks = p.m_blocks;
        const int G = p.head_group;
        const int sec = p.fd_sec.div(t);  // t / (G * m_blocks)
        const int r = t - sec * G * m_blocks;
        const bool full = p.bh - sec * G >= G;  // the last section may hold fewer heads
        const int gs = full ? G : p.bh - sec * G;
        const int mi = full ? p.fd_group.div(r) : p.fd_grem.div(r);
        const int bh = sec * G + (r - mi * gs);
        Task w;
        w.mblk = CAUSAL ? (m_blocks - 1 - mi) : mi;
        w.batch = p.fd_heads.div(bh);
        w.head = bh - w.batch * p.heads;
        w.sv = seq_view(p.cu_seqlens, p.vmaps, kFwdMaps, N, w.batch);
        const int n = w.sv.n;
        w.nkv = (n + kBlockN - 1) / kBlockN;
        if (CAUSAL) w.nkv = min(w.nkv, (min(w.mblk * rows + rows, n) - 1) / kBlockN + 1);
        return w;
    }
    // variable-length batches: query blocks past a short sequence have no work
    static TKB_DEVICE bool skip(const globals& p, int t) {
        if (p.cu_seqlens == nullptr) return false;
        const Task w = decode(p, t);
        return w.mblk * p.task_tiles * kBlockM >= w.sv.n;
    }
    // kv blocks query tile s of a task visits (causal: tile 0 skips the block only tile 1 sees)
    // (0 for tile 1 of a one-tile task)
    static TKB_DEVICE int tile_blocks(const globals& p, const Task& w, int s) {
        if (s >= p.task_tiles) return 0;
        if (!CAUSAL) return w.nkv;
        return min(w.nkv, (min(w.mblk * p.task_tiles * kBlockM + s * kBlockM + kBlockM, w.sv.n) - 1) / kBlockN + 1);
    }
    // k3: index of (tile s, block i) in the task's QK issue order, its buffer and TMEM column
    static TKB_DEVICE int qk_index(int s, int i, int nk0, int nk1) {
        return min(i, nk0) + min(i, nk1) + ((s == 1 && i < nk0) ? 1 : 0);
    }
    static TKB_DEVICE uint32_t sbuf_col(uint32_t b) { return b == 0 ? 0u : (b == 1 ? 128u : 384u); }

    static TKB_DEVICE int num_tasks(const globals& p) { return p.tasks; }
    // K-block flags come first in p.flags: B * Hkv * nq128 of them
    static TKB_DEVICE size_t rope_kflags(const globals& p) {
        return (size_t)(p.bh / p.heads) * (p.heads / p.group) * ((p.n + 127) / 128);
    }
    static TKB_DEVICE int* counter(const globals& p) { return p.sched; }

    static TKB_DEVICE void init(shared& sh, const globals& p) {
        for (int s = 0; s < kQStages; ++s) {
            mbar_init(&sh.q_full[s], 1);
            mbar_init(&sh.q_empty[s], 1);
            mbar_init(&sh.s_full[s], 1);
            mbar_init(&sh.o_full[s], 1);
            mbar_init(&sh.pv_done[s], 1);
            for (int c = 0; c < kPChunks; ++c) mbar_init(&sh.p_full[s][c], WARPGROUP_THREADS);
        }
        for (int b = 0; b < 3; ++b) {
            mbar_init(&sh.s_full3[b], 1);
            for (int c = 0; c < kPChunks; ++c) mbar_init(&sh.p_full3[b][c], WARPGROUP_THREADS);
        }
        sh.kv_ring.init(1, 1);
        gl{&p.tm_q}.prefetch();
        gl{&p.tm_k}.prefetch();
        gl{&p.tm_v}.prefetch();
        gl{&p.tm_o}.prefetch();
    }

    // ----------------------------- LOAD (LCSF load stage) -----------------------------
    struct producer {
        struct state {
            lcsf::ring_state<C::kKvSlots> st;
        };
        template <class ClaimNext>
        static TKB_DEVICE void load(const lcsf::args<attn_fwd_template>& a, state& ps, int t, int nt,
                                    ClaimNext&& claim_next) {
            const globals& p = a.g;
            shared& sh = a.sh;
            fwd_stamp(p, 0, nt, 0);
            const uint64_t pol_q = tma::policy_evict_first();
            const uint64_t pol_kv = tma::policy_evict_last();
            const Task w = decode(p, t);
            if (w.sv.maps != nullptr) {  // this sequence's maps, written by varlen_maps_kernel
                tma::acquire_map(w.sv.maps + kMapQ);
                tma::acquire_map(w.sv.maps + kMapK);
                tma::acquire_map(w.sv.maps + kMapV);
            }
            const int q0 = w.mblk * p.task_tiles * kBlockM;
            const int nq = (p.n + 127) / 128;
            const int bkv = w.batch * (p.heads / p.group) + w.head / p.group;
            if constexpr (ROPE && TKB_ROPE_DEBUG != 2)  // the task's rotated Q blocks (rows past N: none)
                lcsf::flags_wait_all(p.flags + rope_kflags(p) + (size_t)(w.batch * p.heads + w.head) * nq + q0 / 128,
                                     min(p.task_tiles, nq - q0 / 128), p.epoch);
            for (int s = 0; s < p.task_tiles; ++s) {  // Q_s is free once the last QK_s of the previous task retired
                mbar_wait(&sh.q_empty[s], (nt & 1) ^ 1u);
                mbar_arrive_expect_tx(&sh.q_full[s], C::kTile);
                w.sv.with_map(p.tm_q, kMapQ, [&](const CUtensorMap* m) {
                    load_async(sQ(sh, s), gl{m}, &sh.q_full[s], q0 + s * kBlockM, w.head, w.sv.bcoord, pol_q);
                });
            }
            fwd_stamp(p, 0, nt, 1);  // Q issued (after q_empty)
            const int t_next = claim_next();
            fwd_stamp(p, 0, nt, 2);
            // (warming the next task's Q — or its Q and first K / V block — in L2 ahead of time
            // measured 1-2 % slower: the loads are not L2-miss bound)
            (void)t_next;
            for (int i = 0; i < w.nkv; ++i) {
                // the rotated K block (checking 8 blocks at a time, or the whole task's range at
                // its start, measured slower: the load warp then waits for blocks it does not need yet)
                if constexpr (ROPE && TKB_ROPE_DEBUG != 2) lcsf::flag_wait(p.flags + (size_t)bkv * nq + i, p.epoch);
#pragma unroll
                for (int which = 0; which < 2; ++which) {
                    sh.kv_ring.wait_empty(ps.st);
                    mbar_arrive_expect_tx(&sh.kv_ring.full[ps.st.slot], C::kTile);
                    w.sv.with_map(which == 0 ? p.tm_k : p.tm_v, which == 0 ? kMapK : kMapV, [&](const CUtensorMap* m) {
                        load_async(sKV(sh, ps.st.slot), gl{m}, &sh.kv_ring.full[ps.st.slot], i * kBlockN,
                                   w.head / p.group, w.sv.bcoord, pol_kv);  // grouped-query: kv head = head / group
                    });
                    if (i == w.nkv - 1 && which == 1) fwd_stamp(p, 0, nt, 3);
                    ps.st.advance();
                }
            }
        }
        static TKB_DEVICE void drain(const lcsf::args<attn_fwd_template>&, state&) {}
    };

    // ----------------------------- MMA (LCSF compute, tensor part) ---------------------
    // converged warp; one elected lane issues each tcgen05 op
    struct mma {
        struct state {
            lcsf::ring_state<C::kKvSlots> st;
            uint32_t qbase = 0;           // k3: QK index of the task's first block (buffer = index % 3)
            uint32_t it[kQStages] = {0, 0};  // PVs issued per tile: p_full phases
        };
        static TKB_DEVICE void issue(const lcsf::args<attn_fwd_template>& a, state& ms, int t, int nt) {
            const globals& p = a.g;
            if (a.lane == 0) fwd_stamp(p, 1, nt, 0);
            shared& sh = a.sh;
            const uint32_t tbase = a.tmem;
            auto& kv = sh.kv_ring;
            auto& st = ms.st;
            const Task w = decode(p, t);
            const int nkv = w.nkv;
            const int nk[kQStages] = {tile_blocks(p, w, 0), tile_blocks(p, w, 1)};  // causal: tile 0 may stop one early
            if constexpr (k3) {
                auto gidx = [&](int s, int i) { return ms.qbase + (uint32_t)qk_index(s, i, nk[0], nk[1]); };
                auto qk3 = [&](int s, int i, int kslot) {  // S = Q K^T (mm_ABt, tiles.hpp:349)
                    const uint32_t g = gidx(s, i);
                    mm_ABt(tt_fl<128>{tbase + sbuf_col(g % 3)}, sQ(sh, s), sKV(sh, kslot));
                    mma_commit(&sh.s_full3[g % 3]);
                };
                auto pv3 = [&](int s, int i, int vslot) {  // O_s (+)= P_s(i) V (mma_AB, tiles.hpp:350-352)
                    const uint32_t g = gidx(s, i);
#pragma unroll
                    for (int c = 0; c < kPChunks; ++c) {
                        mbar_wait(&sh.p_full3[g % 3][c], (g / 3) & 1);
                        tmem::fence_after();
                        mma_AB_k<D, kPChunkCols>(
                            tt_fl<D>{tbase + C::tmem_o(s)},
                            tt_bf<kPChunkCols / 2>{tbase + sbuf_col(g % 3) + 64 + c * (kPChunkCols / 2)},
                            swap_layout(sKV(sh, vslot)), c * kPChunkCols, i > 0 || c > 0);
                    }
                    mma_commit(&sh.pv_done[s]);
                };
                mbar_wait(&sh.q_full[0], nt & 1);
                if (nk[1] > 0) mbar_wait(&sh.q_full[1], nt & 1);  // (a one-tile task has no Q_1)
                kv.wait_full(st);
                tmem::fence_after();
#pragma unroll
                for (int s = 0; s < kQStages; ++s) {
                    if (nk[s] == 0) continue;
                    qk3(s, 0, st.slot);
                    if (nk[s] == 1) mma_commit(&sh.q_empty[s]);
                }
                mma_commit(&kv.empty[st.slot]);
                st.advance();
                for (int i = 1; i < nkv; ++i) {
                    const int vslot = st.slot;
                    kv.wait_full(st);  // V_{i-1}
                    st.advance();
                    const int kslot = st.slot;
                    kv.wait_full(st);  // K_i (tile 1 always has block i here)
                    tmem::fence_after();
                    // QK_i(s) before PV_{i-1}(s): its buffer held block index - 3, whose PV was
                    // issued earlier; the other tile's QK_i follows PV_{i-1}(0), which read its buffer
#pragma unroll
                    for (int s = 0; s < kQStages; ++s) {
                        if (i < nk[s]) {
                            qk3(s, i, kslot);
                            if (i == nk[s] - 1) mma_commit(&sh.q_empty[s]);
                        }
                        if (i - 1 < nk[s]) {
                            pv3(s, i - 1, vslot);
                            if (i - 1 == nk[s] - 1) mma_commit(&sh.o_full[s]);
                        }
                    }
                    mma_commit(&kv.empty[vslot]);
                    mma_commit(&kv.empty[kslot]);
                    st.advance();
                }
                const int vslot = st.slot;
                kv.wait_full(st);
#pragma unroll
                for (int s = 0; s < kQStages; ++s) {
                    if (nk[s] != nkv) continue;
                    pv3(s, nkv - 1, vslot);
                    mma_commit(&sh.o_full[s]);
                }
                mma_commit(&kv.empty[vslot]);
                st.advance();
                ms.qbase += (uint32_t)(nk[0] + nk[1]);
            } else {
                auto qk = [&](int s, int kslot) {  // S_s = Q_s K^T   (mm_ABt, tiles.hpp:349)
                    mm_ABt(tt_fl<128>{tbase + C::tmem_s(s)}, sQ(sh, s), sKV(sh, kslot));
                };
                auto pv = [&](int s, int vslot, bool acc, uint32_t phase) {  // O_s += P_s V (mma_AB)
#pragma unroll
                    for (int c = 0; c < kPChunks; ++c) {
                        mbar_wait(&sh.p_full[s][c], phase);
                        tmem::fence_after();
                        mma_AB_k<D, kPChunkCols>(tt_fl<D>{tbase + C::tmem_o(s)},
                                                 tt_bf<kPChunkCols / 2>{tbase + C::tmem_s(s) + 64 + c * (kPChunkCols / 2)},
                                                 swap_layout(sKV(sh, vslot)), c * kPChunkCols, acc || c > 0);
                    }
                };
                mbar_wait(&sh.q_full[0], nt & 1);
                if (a.lane == 0) fwd_stamp(p, 1, nt, 3);
                if (nk[1] > 0) mbar_wait(&sh.q_full[1], nt & 1);  // (a one-tile task has no Q_1)
                kv.wait_full(st);
                if (a.lane == 0) fwd_stamp(p, 1, nt, 4);
                tmem::fence_after();
                // QK_s(next task) overwrites S_s, whose P was read by the previous task's last PV_s
                // (issued before); the first PV_s below overwrites O_s only after the softmax drained it
#pragma unroll
                for (int s = 0; s < kQStages; ++s) {
                    if (nk[s] == 0) continue;
                    qk(s, st.slot);
                    mma_commit(&sh.s_full[s]);
                    if (nk[s] == 1) mma_commit(&sh.q_empty[s]);
                }
                if (a.lane == 0) fwd_stamp(p, 1, nt, 1);
                mma_commit(&kv.empty[st.slot]);
                st.advance();
                for (int i = 1; i < nkv; ++i) {
                    const int vslot = st.slot;
                    kv.wait_full(st);
                    st.advance();
                    const int kslot = st.slot;
                    bool k_ready = false;
#pragma unroll
                    for (int s = 0; s < kQStages; ++s) {
                        if (i > nk[s]) continue;  // tile s is done
                        pv(s, vslot, i > 1, ms.it[s] & 1);
                        ++ms.it[s];
                        if (i == nk[s]) {  // that was tile s's last block
                            mma_commit(&sh.o_full[s]);
                            continue;
                        }
                        if (!k_ready) {
                            kv.wait_full(st);
                            tmem::fence_after();
                            k_ready = true;
                        }
                        qk(s, kslot);
                        mma_commit(&sh.s_full[s]);
                        if (i == nk[s] - 1) mma_commit(&sh.q_empty[s]);  // Q_s's last read: the next task's may load
                    }
                    mma_commit(&kv.empty[vslot]);
                    mma_commit(&kv.empty[kslot]);
                    st.advance();
                }
                const int vslot = st.slot;
                kv.wait_full(st);
#pragma unroll
                for (int s = 0; s < kQStages; ++s) {
                    if (nk[s] != nkv) continue;
                    pv(s, vslot, nkv > 1, ms.it[s] & 1);
                    ++ms.it[s];
                    mma_commit(&sh.o_full[s]);
                }
                mma_commit(&kv.empty[vslot]);
                st.advance();
            }
            if (a.lane == 0) fwd_stamp(p, 1, nt, 2);
        }
    };

    // ----------------------------- SOFTMAX (compute) + FINISH --------------------------
    // warps 0-3 / 4-7: the softmax warpgroup of query tile 0 / 1, one thread per row
    struct consumer {
        struct state {
            uint32_t qbase = 0;  // k3: QK index of this task's first block
            uint32_t pvc = 0;    // k3: pv_done completions consumed
            uint32_t sc = 0;     // s_full completions seen
            float m = -INFINITY;  // running max of tau * S (the value actually subtracted)
            float l = 0.f;        // running normaliser (fp32 sum of fp32 P, kernels.hpp:324)
        };
        static TKB_DEVICE void compute(const lcsf::args<attn_fwd_template>& a, state& cs, int t, int nt) {
            const globals& p = a.g;
            shared& sh = a.sh;
            const int s = a.warp / 4;                  // query tile of this warpgroup
            const int wq = a.warp % 4;                 // TMEM lane quarter
            if (wq == 0 && a.lane == 0) fwd_stamp(p, 2 + s, nt, 5);
            const int row_in_tile = wq * 32 + a.lane;  // == TMEM lane
            const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
            const uint32_t tbase = a.tmem;
            const uint32_t tS_fixed = tbase + lane_off + C::tmem_s(s);
            const uint32_t tO = tbase + lane_off + C::tmem_o(s);
            const float tau = p.scale_log2;
            const Task w = decode(p, t);
            const int N = w.sv.n;
            const int q0 = w.mblk * p.task_tiles * kBlockM;
            const int row = q0 + s * kBlockM + row_in_tile;
            const int nkv = tile_blocks(p, w, s);
            float m = -INFINITY;
            float l = 0.f;
            const int nk0 = tile_blocks(p, w, 0), nk1 = tile_blocks(p, w, 1);
            const bool stamp = (wq == 0 && a.lane == 0);
            if (stamp) fwd_stamp(p, 2 + s, nt, 0);
            for (int i = 0; i < nkv; ++i) {
                uint32_t tS = tS_fixed;
                mbarrier* pf = sh.p_full[s];
                if constexpr (k3) {
                    const uint32_t gi = cs.qbase + (uint32_t)qk_index(s, i, nk0, nk1);
                    const uint32_t b = gi % 3;
                    mbar_wait(&sh.s_full3[b], (gi / 3) & 1);
                    tS = tbase + lane_off + sbuf_col(b);
                    pf = sh.p_full3[b];
                } else {
                    mbar_wait(&sh.s_full[s], cs.sc & 1);
                    ++cs.sc;
                }
                const uint32_t tP = tS + 64;
                if (stamp && i == 0) fwd_stamp(p, 2 + s, nt, 1);
                tmem::fence_after();
                rt_fl<kBlockN> x;
                load(x, tS);
                load_wait(x);
                const int kv0 = i * kBlockN;
                const bool need_mask = CAUSAL ? (kv0 + kBlockN - 1 > q0 + s * kBlockM) : (kv0 + kBlockN > N);
                if (need_mask) {
                    const int lim = CAUSAL ? min(row - kv0, N - 1 - kv0) : (N - 1 - kv0);  // last visible column
#pragma unroll
                    for (int j = 0; j < kBlockN; ++j)
                        if (j > lim) x.v[j] = -INFINITY;
                }
                float mx = -INFINITY;
                row_max(mx, x);  // tiles.hpp:290-298
                const float m_new = fmaxf(m, mx * tau);
                if (k3 && i > 0) {  // PV_{i-1}(s) done: O_s is stable for the rescale below
                    mbar_wait(&sh.pv_done[s], cs.pvc & 1);
                    ++cs.pvc;
                    tmem::fence_after();
                }
                // Rescale lazily: only when some row of the warp grew by > 2^8 (warp-uniform
                // because tcgen05.ld/st are warp-collective). The final O / l is unchanged.
                if (__any_sync(0xffffffffu, m_new > m + kRescaleThreshold)) {
                    const float alpha = ex2_approx(m - m_new);  // exp2(-inf) = 0 on the first tile
                    m = m_new;
                    l *= alpha;
                    if (i > 0) {  // mul_row(o, o, alpha) (tiles.hpp:282-287); PV_{i-1} is complete
#pragma unroll
                        for (int c = 0; c < D; c += 32) {
                            rt_fl<32> o;
                            load(o, tO + c);
                            load_wait(o);
                            mul_row(o, alpha);
                            store(tO + c, o);
                        }
                        tmem::wait_st();
                    }
                }
                // P = exp2(tau * S - m) (exp2, tiles.hpp:217-219); row_sum over fp32 P (tiles.hpp:301-309);
                // bf16 RNE copy into TMEM (copy, tiles.hpp:195-200), handed over chunk by chunk
                const float2 tau2 = make_float2(tau, tau), nm2 = make_float2(-m, -m);
                float2 l01 = make_float2(0.f, 0.f), l23 = make_float2(0.f, 0.f);  // packed FADD2 row sums
                uint32_t pk[kBlockN / 2];
#pragma unroll
                for (int c = 0; c < kPChunks; ++c) {
#pragma unroll
                    for (int j = c * kPChunkCols; j < (c + 1) * kPChunkCols; j += 4) {
                        const float2 xa = fma2(make_float2(x.v[j], x.v[j + 1]), tau2, nm2);
                        const float2 xb = fma2(make_float2(x.v[j + 2], x.v[j + 3]), tau2, nm2);
                        const float p0 = ex2_approx(xa.x), p1 = ex2_approx(xa.y);
                        float p2, p3;
                        if (((j / 4) % 4) < C::kPolyGroups) {  // part of the exponentials on the FMA pipe
                            const float2 pb = ex2_poly2(xb);
                            p2 = pb.x;
                            p3 = pb.y;
                        } else {
                            p2 = ex2_approx(xb.x);
                            p3 = ex2_approx(xb.y);
                        }
                        l01 = add2(l01, make_float2(p0, p1));
                        l23 = add2(l23, make_float2(p2, p3));
                        pk[j / 2] = pack_bf16x2(p0, p1);
                        pk[j / 2 + 1] = pack_bf16x2(p2, p3);
                    }
                    if (c > 0) {  // chunk c-1 is in TMEM: hand it to the MMA warp
                        tmem::wait_st();
                        tmem::fence_before();
                        mbar_arrive(&pf[c - 1]);
                    }
                    if constexpr (kPChunks == 1) {
                        tmem::st_32x32b_x64(tP, pk);
                    } else if constexpr (kPChunks == 2) {
                        tmem::st_32x32b_x32(tP + c * 32, pk + c * 32);
                    } else {
                        tmem::st_32x32b_x16(tP + c * 16, pk + c * 16);
                    }
                }
                l += (l01.x + l01.y) + (l23.x + l23.y);
                tmem::wait_st();
                tmem::fence_before();
                mbar_arrive(&pf[kPChunks - 1]);
            }
            if (stamp) fwd_stamp(p, 2 + s, nt, 2);
            if constexpr (k3) cs.qbase += (uint32_t)(nk0 + nk1);
            cs.m = m;
            cs.l = l;
        }

        // FINISH (kernels.hpp:335-342): O / l -> bf16 -> this warpgroup's SMEM staging atom ->
        // TMA store (one 64-column atom at a time); plus L for the backward
        static TKB_DEVICE void finish(const lcsf::args<attn_fwd_template>& a, state& cs, int t, int nt) {
            const globals& p = a.g;
            shared& sh = a.sh;
            const int s = a.warp / 4;
            const int wq = a.warp % 4;
            const int row_in_tile = wq * 32 + a.lane;
            const uint32_t tO = a.tmem + ((uint32_t)(wq * 32) << 16) + C::tmem_o(s);
            const Task w = decode(p, t);
            if (tile_blocks(p, w, s) == 0) return;  // tile 1 of a one-tile task: no rows
            const int q0 = w.mblk * p.task_tiles * kBlockM;
            const int row = q0 + s * kBlockM + row_in_tile;
            const float m = cs.m, l = cs.l;
            mbar_wait(&sh.o_full[s], nt & 1);
            if constexpr (k3) {  // the last PV_s's pv_done (complete with o_full)
                mbar_wait(&sh.pv_done[s], cs.pvc & 1);
                ++cs.pvc;
            }
            tmem::fence_after();
            if (wq == 0 && a.lane == 0) fwd_stamp(p, 2 + s, nt, 3);
            if (p.lse != nullptr && row < w.sv.n)
                p.lse[(size_t)(w.batch * p.heads + w.head) * p.n + row] = (m + __log2f(l)) * kLn2;
            const bool leader = (wq == 0 && a.lane == 0);
            const st_bf<128, 64> stage = sStage(sh, s);
            if (leader && w.sv.maps != nullptr) tma::acquire_map(w.sv.maps + kMapO);
#pragma unroll 1
            for (int at = 0; at < Tile::kAtoms; ++at) {
                rt_fl<32> o0, o1;
                load(o0, tO + at * 64);
                load(o1, tO + at * 64 + 32);
                load_wait(o0);
                load_wait(o1);
                if (at == Tile::kAtoms - 1) tmem::fence_before();  // O_s drained: the next task's PV may overwrite it
                div_row(o0, l);  // tiles.hpp:276-281
                div_row(o1, l);
                rt_bf<32> b0, b1;
                copy(b0, o0);
                copy(b1, o1);
                if (leader) tma::wait_group_read<0>();  // the staging atom is free again
                named_sync(1 + s, WARPGROUP_THREADS);
                store(stage, b0, row_in_tile, 0);  // register -> shared (tiles.hpp:453-459)
                store(stage, b1, row_in_tile, 32);
                tma::fence_async_smem();
                named_sync(1 + s, WARPGROUP_THREADS);
                if (leader) {
                    w.sv.with_map(p.tm_o, kMapO, [&](const CUtensorMap* m) {  // shared -> global (TMA; rows
                        store_async(gl{m}, stage, q0 + s * kBlockM, w.head, w.sv.bcoord, at * 64);  // past n clipped)
                    });
                    tma::commit_group();
                }
            }
            if (leader) fwd_stamp(p, 2 + s, nt, 4);
        }
        static TKB_DEVICE void drain(const lcsf::args<attn_fwd_template>& a, state&) {
            if (a.warp % 4 == 0 && a.lane == 0) tma::wait_group<0>();
        }
    };

    // ----------------------------- AUX: the fused rotary prologue ---------------------
    // Work items = (batch, up to 4 heads, 128-row block), claimed from counter[3] batch by
    // batch (K items of a batch before its Q items, the attention's consumption order); one
    // warp rotates an item: lane = (row, 8-pair chunk) and, per (row, chunk), the sin / cos
    // table entries are loaded once and applied to all of the item's heads (the tables do
    // not depend on the head), with every load of the step issued before any math. fp32 math
    // on the bf16 inputs and fp32 tables, bf16 RNE out: the separate tkb_rotary kernel's
    // arithmetic (oracle_rotary, oracles.hpp:66-90), so both paths agree bit for bit.
    static constexpr int kRopeHeads = 4;
    struct aux {
        static TKB_DEVICE void run(const lcsf::args<attn_fwd_template>& a, int) {
            if constexpr (ROPE) {
                const globals& p = a.g;
                const int lane = a.lane;
                const int N = p.n;
                const int nq = (N + 127) / 128;
                const int H = p.heads, hkv = H / p.group, B = p.bh / H;
                const int q4 = (H + kRopeHeads - 1) / kRopeHeads, k4 = (hkv + kRopeHeads - 1) / kRopeHeads;
                const int per_batch = (q4 + k4) * nq;
                const int items = B * per_batch;
                constexpr int half = D / 2;
                constexpr int kChunks = D / 16;          // 8-pair chunks per row
                constexpr int kRowsPerPass = 32 / kChunks;
                const int c = lane % kChunks;
                for (;;) {
                    int it = 0;
                    if (lane == 0) it = atomicAdd(p.sched + 3, 1);
                    it = __shfl_sync(0xffffffffu, it, 0);
                    if (it >= items) break;
                    const int b = it / per_batch;
                    int r = it - b * per_batch;
                    const bool is_k = r < k4 * nq;
                    if (!is_k) r -= k4 * nq;
                    const int quad = r / nq;
                    // causal: a head's heavy (late) Q blocks first, as the attention claims them
                    const int blk = (!is_k && CAUSAL) ? nq - 1 - (r - quad * nq) : r - quad * nq;
                    const int h0 = quad * kRopeHeads;
                    const int nh = min(kRopeHeads, (is_k ? hkv : H) - h0);
                    const __nv_bfloat16* src = reinterpret_cast<const __nv_bfloat16*>(is_k ? p.k_src : p.q_src);
                    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(is_k ? p.k_rot : p.q_rot);
                    const long long sb = is_k ? p.k_sb : p.q_sb, shd = is_k ? p.k_sh : p.q_sh,
                                    sn = is_k ? p.k_sn : p.q_sn;
                    const int row_end = TKB_ROPE_DEBUG == 1 ? 0 : min(N, blk * 128 + 128);
                    for (int row = blk * 128 + lane / kChunks; row < row_end; row += kRowsPerPass) {
                        const float4* sp = reinterpret_cast<const float4*>(p.sin_tab + (size_t)row * half + 8 * c);
                        const float4* cp = reinterpret_cast<const float4*>(p.cos_tab + (size_t)row * half + 8 * c);
                        const long long base = b * sb + row * sn + 8 * c;
                        uint4 x1[kRopeHeads], x2[kRopeHeads];
#pragma unroll
                        for (int j = 0; j < kRopeHeads; ++j) {
                            if (j < nh) {
                                const __nv_bfloat16* xr = src + base + (h0 + j) * shd;
                                x1[j] = *reinterpret_cast<const uint4*>(xr);
                                x2[j] = *reinterpret_cast<const uint4*>(xr + half);
                            }
                        }
                        const float4 s0 = __ldg(sp), s1 = __ldg(sp + 1), c0 = __ldg(cp), c1 = __ldg(cp + 1);
                        const float sn8[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
                        const float cs8[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
                        for (int j = 0; j < kRopeHeads; ++j) {
                            if (j >= nh) continue;
                            const uint32_t av[4] = {x1[j].x, x1[j].y, x1[j].z, x1[j].w};
                            const uint32_t bv[4] = {x2[j].x, x2[j].y, x2[j].z, x2[j].w};
                            uint32_t o1[4], o2[4];
#pragma unroll
                            for (int q = 0; q < 4; ++q) {  // packed f32x2: the same roundings as fmaf(x1, c, -(x2 s))
                                const float2 u = make_float2(__uint_as_float(av[q] << 16), __uint_as_float(av[q] & 0xFFFF0000u));
                                const float2 v = make_float2(__uint_as_float(bv[q] << 16), __uint_as_float(bv[q] & 0xFFFF0000u));
                                const float2 sp2 = make_float2(sn8[2 * q], sn8[2 * q + 1]);
                                const float2 cp2 = make_float2(cs8[2 * q], cs8[2 * q + 1]);
                                const float2 vs = mul2(v, sp2), us = mul2(u, sp2);
                                const float2 r1 = fma2(u, cp2, make_float2(-vs.x, -vs.y));
                                const float2 r2 = fma2(v, cp2, us);
                                o1[q] = pack_bf16x2(r1.x, r1.y);
                                o2[q] = pack_bf16x2(r2.x, r2.y);
                            }
                            __nv_bfloat16* orow = dst + base + (h0 + j) * shd;
                            *reinterpret_cast<uint4*>(orow) = make_uint4(o1[0], o1[1], o1[2], o1[3]);
                            *reinterpret_cast<uint4*>(orow + half) = make_uint4(o2[0], o2[1], o2[2], o2[3]);
                        }
                    }
                    lcsf::flag_writer_fence();
                    __syncwarp();
                    if (lane < nh) {
                        const size_t f = is_k ? (size_t)(b * hkv + h0 + lane) * nq + blk
                                              : rope_kflags(p) + (size_t)(b * H + h0 + lane) * nq + blk;
                        lcsf::flag_publish(p.flags + f, p.epoch);
                    }
                }
            }
        }
    };
};

template <int D, bool CAUSAL, bool ROPE>
int launch(const FwdParams& p, int num_sms, cudaStream_t stream) {
    using T = attn_fwd_template<D, CAUSAL, ROPE>;
    auto kern = lcsf::kernel<T>;
    static std::atomic<unsigned long long> smem_set{0};  // per instantiation, per device
    if (int e = ensure_smem(kern, T::kSmemBytes, smem_set)) return e;
    kern<<<p.tasks < num_sms ? p.tasks : num_sms, T::kThreads, T::kSmemBytes, stream>>>(p);
    return (int)cudaGetLastError();
}

}  // namespace fwd

// Fills the persistent task fields of p and launches one CTA per SM (at most one per task).
// rope: the fused rotary prologue (attn_fwd_template<D, Causal, true>).
int launch_attn_fwd(int head_dim, bool causal, FwdParams p, int batches, int num_sms, cudaStream_t stream,
                    bool rope) {
    p.bh = batches * p.heads;
    // Two query tiles per task share each K / V block; when even the one-tile tasks all fit in
    // one wave (small B*H*N, e.g. BASELINE configs[0]: 32 two-tile tasks for 148 SMs) a task is
    // one tile, doubling the CTAs that work in parallel on the latency-bound problem (C1: 22.5 ->
    // 19.5 us). With more tasks the one-tile CTAs (tile 1's warps idle, half the MMA work per K / V
    // block) lose: 128 two-tile tasks ran 16-34 % faster than 256 one-tile ones (tools/c1_tiles.py).
    if (p.task_tiles != 1 && p.task_tiles != 2)  // 0: by problem size (tkb_debug_set_fwd_task_tiles forces it)
        p.task_tiles = 2ll * p.bh * ((p.n + 2 * kBlockM - 1) / (2 * kBlockM)) <= num_sms ? 1 : 2;
    p.m_blocks = (p.n + p.task_tiles * kBlockM - 1) / (p.task_tiles * kBlockM);
    p.tasks = p.bh * p.m_blocks;
    const long long kv_bytes = 4ll * p.n * head_dim / p.group;  // K / V of one query head's kv head
    long long g = (48ll << 20) / (kv_bytes > 0 ? kv_bytes : 1);  // heads whose K / V fit ~48 MB of L2
    p.head_group = (int)(g < 1 ? 1 : (g > p.bh ? p.bh : g));
    p.fd_sec = FastDiv((uint32_t)(p.head_group * p.m_blocks));
    p.fd_group = FastDiv((uint32_t)p.head_group);
    p.fd_grem = FastDiv((uint32_t)(p.bh % p.head_group ? p.bh % p.head_group : p.head_group));
    p.fd_heads = FastDiv((uint32_t)p.heads);
    if (rope) {
        if (head_dim == 128)
            return causal ? fwd::launch<128, true, true>(p, num_sms, stream)
                          : fwd::launch<128, false, true>(p, num_sms, stream);
        return causal ? fwd::launch<64, true, true>(p, num_sms, stream) : fwd::launch<64, false, true>(p, num_sms, stream);
    }
    if (head_dim == 128)
        return causal ? fwd::launch<128, true, false>(p, num_sms, stream)
                      : fwd::launch<128, false, false>(p, num_sms, stream);
    return causal ? fwd::launch<64, true, false>(p, num_sms, stream) : fwd::launch<64, false, false>(p, num_sms, stream);
}

}  // namespace tkb
