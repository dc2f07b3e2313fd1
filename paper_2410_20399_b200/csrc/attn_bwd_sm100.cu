// attn_bwd_sm100.cu — attention backward for B200 (sm_100a), dQ/dK/dV from the saved L.
//
// The reference has no backward; the math follows the restated
// oracle (oracle/attn_oracle.cpp, bwd_head):
//   P = exp(S - L), dV = P^T dO, dP = dO V^T, Delta = rowsum(dO o O),
//   dS = P o (dP - Delta), dQ = scale dS K, dK = scale dS^T Q
//
// Design: atomic-free, deterministic by construction. Three launches:
//   bwd_prep   Delta = rowsum(dO o O) and -lse2 = -L log2(e) (-inf on padded rows)
//   bwd_dkdv   KV-stationary: one 128-row K/V block per CTA, streaming Q/dO blocks;
//              4 tcgen05 GEMMs per tile pair, dK/dV accumulate in TMEM:
//                S^T  = K Q^T    (SS)            -> TMEM S
//                dP^T = V dO^T   (SS)            -> TMEM dP
//                dV  += P^T dO   (TS, P in TMEM)
//                dK  += dS^T Q   (TS, dS in TMEM)
//   bwd_dq     Q-stationary: one 128-row Q/dO block per CTA, streaming K/V blocks;
//              3 GEMMs per tile pair, dQ accumulates in TMEM:
//                S   = Q K^T     (TS, Q in TMEM) -> TMEM S
//                dP  = dO V^T    (TS, dO in TMEM)-> TMEM dP
//                dQ += dS K      (TS, dS in TMEM)
//              (all three read only B from SMEM: an SS GEMM would need the full 128 B/clk
//               of SMEM bandwidth and stall behind the TMA traffic)
// A fused single kernel needs an fp32 reduction of a 128 x D dQ partial per tile pair
// through L2; measured on this B200 the chip-wide fp32 add-reduce ceiling is ~5.6 TB/s
// (tools/reduce_bench.py), which caps 128-row KV tiles well below the tensor rate.
// Recomputing S and dP in bwd_dq (7 GEMMs instead of 5) costs less than that.
//
// Both main kernels: warps 0-15 COMPUTE, thread = (TMEM lane row, column group g of 32),
// four warps per SM sub-partition so the exp / FMA / MUFU work of a 128 x 128 tile is
// spread over four instruction streams; warp 16 MMA (converged, one elected lane issues);
// warp 17 LOAD (TMA). bf16 P / dS live in TMEM next to the fp32 values they replace:
// group g writes packed columns [32g, 32g + 16) of the S / dP region, inside the 32
// columns it has itself read, and hands its 32-wide K chunk to the MMA warp at once.
// Tensor ops issued by one thread run in order, so a GEMM that overwrites a region is
// always issued after the GEMM reading it.
#include <cuda.h>
#include <cuda_runtime.h>

#include "attn_common.cuh"
#include "tkb/cluster.cuh"
#include "tkb/lcsf.cuh"
#include "tkb/tile.cuh"

#ifndef TKB_BWD_POLY
#define TKB_BWD_POLY 1  // exponential pairs of every four on the FMA-pipe polynomial (1: a quarter)
#endif

namespace tkb {
namespace bwd {

constexpr int kGroups = 4;                          // 32-column groups per 128-wide tile
constexpr int kComputeThreads = kGroups * 128;      // warps 0-15
constexpr int kWarpMma = 16;
constexpr int kWarpLoad = 17;
constexpr int kThreads = kComputeThreads + 64;      // 576
constexpr int kBarCompute = 1;
constexpr int kAtomBytes = 128 * 128;  // 128 rows x 128 B (one SW128 column block)

template <int D>
struct Tiles {
    static constexpr int kAtoms = D / 64;
    static constexpr int kTileBytes = 128 * D * 2;  // 128 x D bf16
};

// ------------------------------------------------------------------------------ helpers

template <int D>
using Tile = st_bf<128, D>;  // a 128-row K / V / Q / dO block in SMEM (SW128)

// SW128 SMEM tile row r, columns [g D/4, (g+1) D/4) -> TMEM A-operand columns (bf16 pairs):
// shared -> register -> TMEM (a TS-MMA operand staged once per task)
template <int D>
TKB_DEVICE void smem_rows_to_tmem_a(const Tile<D>& tile, uint32_t tdst, int r, int g) {
    rt_bf<D / 4> f;
    load(f, tile, r, g * (D / 4));
    store(tdst + g * (D / 8), f);
}

// TMEM fp32 [lane r][D/4 columns of group g] (x mul) -> bf16 -> SW128 SMEM tile row r
template <int D>
TKB_DEVICE void tmem_rows_to_smem_bf16(uint32_t tsrc, const Tile<D>& stage, int r, int g, float m = 1.f) {
    rt_fl<D / 4> f;
    load(f, tsrc + g * (D / 4));
    load_wait(f);
    mul(f, m);
    rt_bf<D / 4> h;
    copy(h, f);
    store(stage, h, r, g * (D / 4));
}

TKB_DEVICE long long* trace_slot(const BwdParams& p, int lin, int kernel) {
    if (p.trace == nullptr || lin % p.trace_every != 0 || lin / p.trace_every >= p.trace_slots) return nullptr;
    // slot layout [slot][role][iter][event]; kernel 0 (dkdv) uses roles 0-1, kernel 1 (dq) roles 2-3
    return p.trace + (size_t)(lin / p.trace_every) * kTraceRoles * kTraceIters * kTraceEvents +
           (size_t)kernel * 2 * kTraceIters * kTraceEvents;
}

#define TKB_TR(role, t, ev)                                                               \
    do {                                                                                  \
        if (tr != nullptr && (t) < kTraceIters)                                           \
            tr[((role) * kTraceIters + (t)) * kTraceEvents + (ev)] = clock64() - t_start; \
    } while (0)

TKB_DEVICE float4 lds_f4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}

// P chunk: p = exp2(tau * s + nlse) for 32 columns; a quarter of the exponentials run as
// a polynomial on the FMA pipe (MUFU relief). nlse4 holds -lse2 per column (dkdv) or the
// row's -lse2 broadcast (dq, ROWCONST).
template <bool ROWCONST>
TKB_DEVICE void exp_chunk(float* pf, float tau, uint32_t nlse4, float nlse_r) {
#pragma unroll
    for (int c = 0; c < 32; c += 4) {
        const float4 l4 = ROWCONST ? make_float4(nlse_r, nlse_r, nlse_r, nlse_r) : lds_f4(nlse4 + 4 * c);
        const float2 x01 = fma2(make_float2(pf[c], pf[c + 1]), make_float2(tau, tau), make_float2(l4.x, l4.y));
        const float2 x23 = fma2(make_float2(pf[c + 2], pf[c + 3]), make_float2(tau, tau), make_float2(l4.z, l4.w));
        if (((c / 2) & 3) >= 4 - TKB_BWD_POLY) {  // pair index c / 2
            const float2 p01 = ex2_poly2(x01);
            pf[c] = p01.x;
            pf[c + 1] = p01.y;
        } else {
            pf[c] = ex2_approx(x01.x);
            pf[c + 1] = ex2_approx(x01.y);
        }
        float2 p23;
        if (((c / 2 + 1) & 3) >= 4 - TKB_BWD_POLY) {  // pair index c / 2 + 1
            p23 = ex2_poly2(x23);
        } else {
            p23.x = ex2_approx(x23.x);
            p23.y = ex2_approx(x23.y);
        }
        pf[c + 2] = p23.x;
        pf[c + 3] = p23.y;
    }
}

// ---- the dK/dV compute thread's view of a column group (S^T / dP^T: lanes = kv rows,
// columns = queries). A warp of lane quarter wq and column group g reads its 32 lanes x 32
// columns as two tcgen05.ld.16x256b.x4 (lane blocks 0 and 16 of the quarter): element
//   e = 16 h2 + 4 r + 2 h + b   (h2, h, b < 2; r < 4)
// sits at lane 32 wq + 16 h2 + lane / 4 + 8 h, column 32 g + 2 (lane % 4) + 8 r + b. A thread
// thus touches only 8 distinct columns (queries) — against 32 for one-row-per-thread 32x32b
// — so it needs 8 lse / Delta values per step instead of 32. Packed bf16 pairs k = e / 2 go
// back with tcgen05.st.16x128b.x4 (register 2 r + h of block h2 -> lane 16 h2 + lane / 4 + 8 h,
// packed column (lane % 4) + 4 r = queries 2 (lane % 4) + 8 r + {0, 1}): the TS-MMA A-operand
// layout of the group's 32-query K chunk, in the group's first 16 columns.
TKB_DEVICE void grp_load(uint32_t taddr, float* v) {  // taddr: lane 32 wq, column 32 g
    tmem::ld_16x256b_x4(taddr, reinterpret_cast<uint32_t*>(v));
    tmem::ld_16x256b_x4(taddr + (16u << 16), reinterpret_cast<uint32_t*>(v) + 16);
    tmem::wait_ld_x32(reinterpret_cast<uint32_t*>(v));
}
TKB_DEVICE void grp_store_packed(uint32_t taddr, const uint32_t* pk) {  // pk[k] = bf16x2(v[2k], v[2k+1])
    tmem::st_16x128b_x4(taddr, pk);
    tmem::st_16x128b_x4(taddr + (16u << 16), pk + 8);
}
TKB_DEVICE constexpr int grp_row(int e) { return 16 * (e >> 4) + 8 * ((e >> 1) & 1); }  // + lane / 4
TKB_DEVICE constexpr int grp_col(int e) { return 8 * ((e >> 2) & 3) + (e & 1); }         // + 2 (lane % 4)
TKB_DEVICE constexpr int grp_vec(int e) { return 2 * ((e >> 2) & 3) + (e & 1); }         // index in its 8 columns
// Per-column vectors (-lse2, Delta) are stored with each 32-column group permuted so that a
// thread's 8 columns are contiguous: column 2 j + 8 r + b -> position 8 j + 2 r + b.
TKB_DEVICE constexpr int perm32(int i) {
    return (i & ~31) | (((i >> 1) & 3) << 3) | (((i >> 3) & 3) << 1) | (i & 1);
}
// the 8 values of this thread's columns (lane % 4 = j): positions [8 j, 8 j + 8) of its group
TKB_DEVICE void grp_vec_load(uint32_t group_base, float* out) {
    const uint32_t a = group_base + 32u * (laneid() & 3);
    const float4 lo = lds_f4(a), hi = lds_f4(a + 16);
    out[0] = lo.x, out[1] = lo.y, out[2] = lo.z, out[3] = lo.w;
    out[4] = hi.x, out[5] = hi.y, out[6] = hi.z, out[7] = hi.w;
}
// P^T = exp2(tau S^T - lse2) over the group view; a quarter of the exponentials (the last
// pair of every four) run as a polynomial on the FMA pipe (MUFU relief)
TKB_DEVICE void grp_exp(float* v, float tau, const float* nlse) {
#pragma unroll
    for (int e = 0; e < 32; e += 2) {
        const int c = grp_vec(e);
        const float2 x = fma2(make_float2(v[e], v[e + 1]), make_float2(tau, tau), make_float2(nlse[c], nlse[c + 1]));
        float2 y;
        if (((e >> 1) & 3) >= 4 - TKB_BWD_POLY) {
            y = ex2_poly2(x);
        } else {
            y.x = ex2_approx(x.x);
            y.y = ex2_approx(x.y);
        }
        v[e] = y.x;
        v[e + 1] = y.y;
    }
}
// dS^T = P^T o (dP^T - Delta) packed to bf16 pairs (the softmax scale is applied at the finish)
TKB_DEVICE void grp_ds(const float* pf, const uint32_t* dpv, const float* dlt, uint32_t* pk) {
#pragma unroll
    for (int e = 0; e < 32; e += 2) {
        const int c = grp_vec(e);
        const float2 gg = sub2(make_float2(__uint_as_float(dpv[e]), __uint_as_float(dpv[e + 1])),
                               make_float2(dlt[c], dlt[c + 1]));
        const float2 d = mul2(make_float2(pf[e], pf[e + 1]), gg);
        pk[e / 2] = pack_bf16x2(d.x, d.y);
    }
}

// ================================================================== bwd_dkdv (KV-stationary)
// TMEM of the dK/dV kernels: S^T | dV | dP^T (P^T / dS^T packed into S^T / dP^T) | dK.
template <int D>
struct TmemKV {
    static __device__ __forceinline__ constexpr uint32_t tmem_s() { return 0u; }
    static __device__ __forceinline__ constexpr uint32_t tmem_dv() { return 128u; }
    static __device__ __forceinline__ constexpr uint32_t tmem_dp() { return 128u + D; }
    static __device__ __forceinline__ constexpr uint32_t tmem_dk() { return 256u + D; }
};

// ================================================================== bwd_dkdv, persistent
// bwd_dkdv with one CTA per SM walking (kv block, kv head, batch) tasks from the atomic
// queue, so that a task's prologue / finish overlap its neighbours instead of costing a CTA
// turnover (~4000 clk start-up + ~4400 clk finish per CTA, ~9 % of a 32-step task):
//   - K (V) of the next task is loaded as soon as this task's last S^T (dP^T) retired
//     (k_empty / v_empty), i.e. under its last dV / dK GEMMs and finish; the next task's first
//     S^T waits for K only (k_full / v_full; measured neutral against one K+V barrier: the
//     ~3 k clk from this task's last dK to the next first S^T is the 64 KB reload itself);
//   - the Q / dO rings and the per-step barriers run on a step counter continuous across
//     tasks, so the next task's first S^T / dP^T GEMMs are issued right behind this task's
//     last dV / dK (they write the S / dP regions, which hold nothing live by then);
//   - the finish reads dV / dK out of TMEM, releases them at once (dv_free / dk_free: the
//     next task's first dV / dK overwrite them) and stages them in two ring slots for a TMA
//     store issued by the load warp (see FINISH below).
struct KvTask {
    int j, head, batch;
    int chunk;   // query-head chunk (kv_split > 1: grouped-query heads split over tasks)
    SeqView sv;  // this batch's length and TMA row coordinates (variable-length batches)
};

// SMEM of the persistent dK/dV kernel. Q_{t+1} is needed by S_{t+1}, issued right after dV_t;
// its slot is the one dK_{t+1-SQ} frees. With SQ = 2 only dP_t and dV_t (1024 clk) separate
// the two and the L2 -> SMEM latency of the 33 KB reload shows; SQ = 3 gives it a step more.
// dO_{t+1} (first read by dP_{t+1}, late in step t) and lse / delta need only 2 slots.
//
// The kernel is lcsf::kernel<attn_bwd_dkdv_template<D, Causal>> (tkb/lcsf.cuh).
template <int D, bool CAUSAL>
struct attn_bwd_dkdv_template {
    using CT = TmemKV<D>;
    using TL = Tiles<D>;
    using globals = BwdParams;
    static constexpr int SQ = (D == 128) ? 3 : 4;  // Q ring
    static constexpr int SD = (D == 128) ? 2 : 3;  // dO ring
    static constexpr int SA = 2;                   // lse / delta ring
    static constexpr int kThreads = bwd::kThreads;
    static constexpr int kTmemCols = 512;
    static constexpr int kProducerWarp = kWarpLoad;
    static constexpr int kMmaWarp = bwd::kWarpMma;
    static constexpr int kConsumerWarps = 16;
    static constexpr int kQueueReaders = 1 + 16;
    static constexpr bool kAlignSlack = false;  // no static SMEM: the dynamic window starts 1024-aligned
    static constexpr bool kReleaseEarly = false;
    static constexpr int kAuxWarps = 0, kAuxWarp0 = 0;
    // D = 64 leaves 128 TMEM columns free: S^T is double-buffered there (the second buffer at
    // column 384), so S^T_{t+1} is issued before dV_t and the exponentials of step t+1 do not
    // wait for the dV GEMM that reads P_t (the D = 64 step is bound by that chain, not by
    // its 1024 clk of MMA). Per-buffer s_full / p_full keep the phases one apart.
    static constexpr bool kDS = (D == 64);

    struct shared {
        uint8_t k[TL::kTileBytes];
        uint8_t v[TL::kTileBytes];
        uint8_t q[SQ][TL::kTileBytes];
        uint8_t dO[SD][TL::kTileBytes];
        float lse[SA][128];  // -lse2 per query (perm32 order)
        float delta[SA][128];
        mbarrier k_full, v_full;     // K / V of a task in SMEM (separately: S^T needs only K)
        mbarrier k_empty, v_empty;   // the task's last S^T (K) / dP^T (V) retired: the next task's may load
        mbarrier s_full[2];          // [buffer] (one buffer unless kDS)
        mbarrier dp_full;
        mbarrier dv_free, dk_free;   // the finish has read dV / dK out of TMEM
        mbarrier dkv_full;
        mbarrier staged_full;        // a finish has staged dV / dK in two ring slots
        mbarrier q_full[SQ], q_empty[SQ];
        mbarrier do_full[SD], do_empty[SD];
        mbarrier aux_full[SA], aux_empty[SA];
        mbarrier p_full[2][kGroups];  // [buffer][column group]
        mbarrier ds_full[kGroups];
        lcsf::work_queue queue;
        uint32_t tmem_slot;
    };
    static constexpr int kSmemBytes = (int)sizeof(shared);
    static_assert(kSmemBytes <= 232448, "smem");

    static TKB_DEVICE uint32_t s_buf(int x) { return kDS ? ((x & 1) ? 384u : 0u) : CT::tmem_s(); }
    static TKB_DEVICE int buf_of(int x) { return (kDS && (x & 1)) ? 1 : 0; }
    static TKB_DEVICE uint32_t ph_of(int x) { return kDS ? ((x >> 1) & 1) : (x & 1); }  // per-buffer phase

    // Task order. Non-causal: kv block fastest, so the CTAs running together share heads and
    // their Q / dO stay in L2. Causal: kv (batch, head) units in L2-sized groups (p.head_group,
    // as the dQ kernel), inside a group the long tasks (small kv block index) first, so the
    // queue ends on short tasks; with fewer than 4 tasks per SM (grouped-query heads: a task
    // walks its group's query heads) one group spans everything — longest-first overall.
    static TKB_DEVICE int num_tasks(const globals& p) { return (p.n_pad / 128) * p.kv_units; }
    static TKB_DEVICE int* counter(const globals& p) { return p.sched; }
    static TKB_DEVICE KvTask decode(const globals& p, int id) {
        const int nq = p.n_pad / 128;
        const int hkv = p.kv_hkv.d;
        const int hb = p.kv_units;  // (batch, kv head, query-head chunk) units
        const int G = p.kv_G;  // fill_bwd_divisors: all units when < 4 tasks per SM, else L2-sized groups
        KvTask w;
        int unit;
        if (CAUSAL) {  // divisions through FastDiv: no MUFU.RCP behind the compute warps' exponentials
            const int sec = p.kv_sec.div(id);
            const int r = id - sec * G * nq;
            const bool full = hb - sec * G >= G;
            const int gs = full ? G : hb - sec * G;
            w.j = full ? p.kv_g.div(r) : p.kv_grem.div(r);
            unit = sec * G + (r - w.j * gs);
        } else {
            unit = p.kv_nq.div(id);
            w.j = id - unit * nq;
        }
        const int bu = p.kv_c.div(unit);  // the chunk runs fastest: a kv head's chunks run together
        w.chunk = unit - bu * p.kv_split;
        w.batch = p.kv_hkv.div(bu);
        w.head = bu - w.batch * hkv;
        w.sv = seq_view(p.cu_seqlens, p.vmaps, kBwdMaps, p.n, w.batch);
        return w;
    }
    static TKB_DEVICE int q_blocks(const KvTask& w) {  // query blocks a task visits per query head
        const int nb = (w.sv.n + 127) / 128;              // query blocks of this sequence
        return CAUSAL ? (nb - w.j) : nb;
    }
    static TKB_DEVICE int heads_per_task(const globals& p) { return p.kv_c.d == 1 ? p.group : p.group / p.kv_c.d; }
    static TKB_DEVICE int steps(const globals& p, const KvTask& w) { return q_blocks(w) * heads_per_task(p); }
    // variable-length batches: kv blocks past a short sequence have no work
    static TKB_DEVICE bool skip(const globals& p, int id) {
        if (p.cu_seqlens == nullptr) return false;
        const KvTask w = decode(p, id);
        return w.j * 128 >= w.sv.n;
    }
    static TKB_DEVICE Tile<D> tQ(shared& sh, int x) { return Tile<D>{sh.q[x % SQ]}; }
    static TKB_DEVICE Tile<D> tDo(shared& sh, int x) { return Tile<D>{sh.dO[x % SD]}; }

    static TKB_DEVICE void init(shared& sh, const globals& p) {
        mbar_init(&sh.k_full, 1);
        mbar_init(&sh.v_full, 1);
        mbar_init(&sh.k_empty, 1);
        mbar_init(&sh.v_empty, 1);
        mbar_init(&sh.s_full[0], 1);
        mbar_init(&sh.s_full[1], 1);
        mbar_init(&sh.dp_full, 1);
        mbar_init(&sh.dv_free, kComputeThreads);
        mbar_init(&sh.dkv_full, 1);
        mbar_init(&sh.dk_free, kComputeThreads);
        mbar_init(&sh.staged_full, kComputeThreads);
        for (int g = 0; g < kGroups; ++g) {
            mbar_init(&sh.p_full[0][g], 128);
            mbar_init(&sh.p_full[1][g], 128);
            mbar_init(&sh.ds_full[g], 128);
        }
        for (int s = 0; s < SQ; ++s) {
            mbar_init(&sh.q_full[s], 1);
            mbar_init(&sh.q_empty[s], 1);
        }
        for (int s = 0; s < SD; ++s) {
            mbar_init(&sh.do_full[s], 1);
            mbar_init(&sh.do_empty[s], 1);
        }
        for (int s = 0; s < SA; ++s) {
            mbar_init(&sh.aux_full[s], 1);
            mbar_init(&sh.aux_empty[s], 1);
        }
        tma::prefetch_desc(&p.tm_q);
        tma::prefetch_desc(&p.tm_k);
        tma::prefetch_desc(&p.tm_v);
        tma::prefetch_desc(&p.tm_do);
    }

    // ------------------------------------------------------------- LOAD
    struct producer {
        struct state {
            int x = 0;       // global step (ring position)
            int staged = 0;  // staged finishes stored
            KvTask prev{};
        };
        template <class ClaimNext>
        static TKB_DEVICE void load(const lcsf::args<attn_bwd_dkdv_template>& a, state& ps, int id, int n,
                                    ClaimNext&&) {
            const globals& p = a.g;
            shared& sh = a.sh;
            const uint64_t pol_stream = tma::policy_evict_first();
            const uint64_t pol_keep = tma::policy_evict_last();
            const KvTask w = decode(p, id);
            const int T = steps(p, w), T1 = q_blocks(w);
            const int kv0 = w.j * 128;
            if (w.sv.maps != nullptr) {  // this sequence's maps (varlen_maps_kernel); dV / dK: its finish
                for (int m = 0; m < kBwdMaps; ++m) tma::acquire_map(w.sv.maps + m);
            }
            // K as soon as the previous task's last S^T retired, V once its last dP^T did (one
            // GEMM later): the next task's first S^T needs only K
            mbar_wait(&sh.k_empty, (n & 1) ^ 1u);
            mbar_arrive_expect_tx(&sh.k_full, TL::kTileBytes);
            w.sv.with_map(p.tm_k, kMapK, [&](const CUtensorMap* m) {
                load_async(Tile<D>{sh.k}, gl{m}, &sh.k_full, kv0, w.head, w.sv.bcoord, pol_stream);
            });
            mbar_wait(&sh.v_empty, (n & 1) ^ 1u);
            mbar_arrive_expect_tx(&sh.v_full, TL::kTileBytes);
            w.sv.with_map(p.tm_v, kMapV, [&](const CUtensorMap* m) {
                load_async(Tile<D>{sh.v}, gl{m}, &sh.v_full, kv0, w.head, w.sv.bcoord, pol_stream);
            });
            const bool after_staged = n > 0 && T >= 3 && p.kv_split == 1;  // the previous finish staged in our slots
            int ti = 0, hq = w.head * p.group + w.chunk * heads_per_task(p);  // step t = (query head hq, block ti)
            for (int t = 0; t < T; ++t, ++ps.x) {
                const int x = ps.x;
                const int i = (CAUSAL ? w.j : 0) + ti;
                const size_t bhq = (size_t)w.batch * p.heads + hq;
                // in pipe order of the GEMMs that free the slots: dK_{x-SQ}, dV_{x-SD}, dK_{x-SA}
                const int sq = x % SQ, sd = x % SD, sa = x % SA;
                mbar_wait(&sh.q_empty[sq], ((x / SQ) & 1) ^ 1);
                mbar_arrive_expect_tx(&sh.q_full[sq], TL::kTileBytes);
                w.sv.with_map(p.tm_q, kMapQ, [&](const CUtensorMap* m) {
                    load_async(tQ(sh, x), gl{m}, &sh.q_full[sq], i * 128, hq, w.sv.bcoord, pol_keep);
                });
                if (after_staged && t == 1) {
                    // the previous task's finish staged dV / dK in the dO slot of step 1 and the
                    // Q slot of step 2: store them (this warp, off the compute warps' path)
                    // and refill the slots once the store has read them
                    mbar_wait(&sh.staged_full, ps.staged & 1);
                    ++ps.staged;
                    const int prow = ps.prev.j * 128;
                    const KvTask& pw = ps.prev;
                    pw.sv.with_map(p.tm_dv, kMapDv, [&](const CUtensorMap* m) {
                        store_async(gl{m}, tQ(sh, x + 1), prow, pw.head, pw.sv.bcoord);
                    });
                    pw.sv.with_map(p.tm_dk, kMapDk, [&](const CUtensorMap* m) {
                        store_async(gl{m}, tDo(sh, x), prow, pw.head, pw.sv.bcoord);
                    });
                    tma::commit_group();
                    tma::wait_group_read<0>();
                }
                mbar_wait(&sh.do_empty[sd], ((x / SD) & 1) ^ 1);
                mbar_arrive_expect_tx(&sh.do_full[sd], TL::kTileBytes);
                w.sv.with_map(p.tm_do, kMapDo, [&](const CUtensorMap* m) {
                    load_async(tDo(sh, x), gl{m}, &sh.do_full[sd], i * 128, hq, w.sv.bcoord, pol_keep);
                });
                if (++ti == T1) ti = 0, ++hq;
                mbar_wait(&sh.aux_empty[sa], ((x / SA) & 1) ^ 1);
                mbar_arrive_expect_tx(&sh.aux_full[sa], 1024);
                tma::load_1d(sh.lse[sa], p.lse2 + bhq * p.n_pad + i * 128, 512, &sh.aux_full[sa]);
                tma::load_1d(sh.delta[sa], p.delta + bhq * p.n_pad + i * 128, 512, &sh.aux_full[sa]);
            }
            ps.prev = w;
        }
        static TKB_DEVICE void drain(const lcsf::args<attn_bwd_dkdv_template>&, state&) { tma::wait_group<0>(); }
    };

    // ------------------------------------------------------------- MMA (converged warp)
    struct mma {
        struct state {
            int x0 = 0;  // first global step of the task
            long long t_start = 0;
        };
        static TKB_DEVICE void issue(const lcsf::args<attn_bwd_dkdv_template>& a, state& ms, int id, int n) {
            const globals& p = a.g;
            shared& sh = a.sh;
            const uint32_t tbase = a.tmem;
            long long* tr = trace_slot(p, (int)blockIdx.x, 0);
            if (n == 0) ms.t_start = clock64();
            const long long t_start = ms.t_start;
            const Tile<D> tK{sh.k}, tV{sh.v};
            const int T = steps(p, decode(p, id));
            const int x0 = ms.x0;
            const int x_last = x0 + T - 1;
            auto issue_s = [&](int x) {  // S^T = K Q^T
                mbar_wait(&sh.q_full[x % SQ], (x / SQ) & 1);
                tmem::fence_after();
                mm_ABt(tt_fl<128>{tbase + s_buf(x)}, tK, tQ(sh, x));
                mma_commit(&sh.s_full[buf_of(x)]);
                if (x == x_last) mma_commit(&sh.k_empty);  // the task's last S^T: K may reload
            };
            auto issue_dp = [&](int x) {  // dP^T = V dO^T
                mbar_wait(&sh.do_full[x % SD], (x / SD) & 1);
                tmem::fence_after();
                mm_ABt(tt_fl<128>{tbase + CT::tmem_dp()}, tV, tDo(sh, x));
                mma_commit(&sh.dp_full);
                if (x == x_last) mma_commit(&sh.v_empty);  // the task's last dP^T: V may reload
            };
            mbar_wait(&sh.k_full, n & 1);
            issue_s(x0);
            mbar_wait(&sh.v_full, n & 1);
            issue_dp(x0);
            for (int t = 0; t < T; ++t) {
                const int x = x0 + t;
                const uint32_t ph = x & 1;
                TKB_TR(0, x, 0);
                if (t == 0 && n > 0) mbar_wait(&sh.dv_free, (n - 1) & 1);  // previous task's dV read out
                if (kDS && t + 1 < T) issue_s(x + 1);  // other buffer: its P_{t-1} went to dV_{t-1}, issued before
                // dV += P^T dO (mma_AB: P^T chunks in TMEM as they land, dO read MN-major)
                mma_AB_groups(tt_fl<D>{tbase + CT::tmem_dv()}, tt_bf<128>{tbase + s_buf(x)}, swap_layout(tDo(sh, x)),
                              t > 0, [&](int g) {
                                  mbar_wait(&sh.p_full[buf_of(x)][g], ph_of(x));
                                  tmem::fence_after();
                              });
                TKB_TR(0, x, 1);
                mma_commit(&sh.do_empty[x % SD]);
                if (!kDS && t + 1 < T) issue_s(x + 1);  // overwrites P_t, read by dV_t issued before
                TKB_TR(0, x, 2);
                if (t == 0 && n > 0) mbar_wait(&sh.dk_free, (n - 1) & 1);
                // dK += dS^T Q
                mma_AB_groups(tt_fl<D>{tbase + CT::tmem_dk()}, tt_bf<128>{tbase + CT::tmem_dp()},
                              swap_layout(tQ(sh, x)), t > 0, [&](int g) {
                                  mbar_wait(&sh.ds_full[g], ph);
                                  tmem::fence_after();
                              });
                TKB_TR(0, x, 3);
                mma_commit(&sh.q_empty[x % SQ]);
                mma_commit(&sh.aux_empty[x % SA]);  // dK_x waited for the last dS of step x
                if (t + 1 < T) issue_dp(x + 1);  // overwrites dS_t, read by dK_t issued before
                TKB_TR(0, x, 4);
            }
            mma_commit(&sh.dkv_full);
            ms.x0 += T;
        }
    };

    // ------------------------------------------------------------- COMPUTE + FINISH
    struct consumer {
        struct state {
            int x0 = 0;
            long long t_start = 0;
        };
        static TKB_DEVICE void compute(const lcsf::args<attn_bwd_dkdv_template>& a, state& cs, int id, int n) {
            const globals& p = a.g;
            shared& sh = a.sh;
            const int wq = a.warp & 3;
            const int g = a.warp >> 2;
            const int lane = a.lane;
            const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
            const uint32_t tS0 = a.tmem + lane_off + 32 * g;  // + s_buf(x)
            const uint32_t tDp = a.tmem + lane_off + CT::tmem_dp() + 32 * g;
            const float tau = p.scale_log2;
            long long* tr = trace_slot(p, (int)blockIdx.x, 0);
            if (n == 0) cs.t_start = clock64();
            const long long t_start = cs.t_start;
            const KvTask w = decode(p, id);
            const int T = steps(p, w), T1 = q_blocks(w);
            for (int t = 0, ti = 0; t < T; ++t, ti = (ti + 1 == T1) ? 0 : ti + 1) {
                const int x = cs.x0 + t;
                const int sa = x % SA;
                const bool diag = CAUSAL && ti == 0;  // q block i == j
                mbar_wait(&sh.aux_full[sa], (x / SA) & 1);
                float nlse[8], dlt[8];
                grp_vec_load(smem_u32(&sh.lse[sa][32 * g]), nlse);
                grp_vec_load(smem_u32(&sh.delta[sa][32 * g]), dlt);
                mbar_wait(&sh.s_full[buf_of(x)], ph_of(x));
                const uint32_t tS = tS0 + s_buf(x);
                if (threadIdx.x == 0) TKB_TR(1, x, 0);
                if (threadIdx.x == 0 && t == 0 && n > 0) TKB_TR(1, n - 1, 7);  // next task's first S
                tmem::fence_after();
                float pf[32];
                grp_load(tS, pf);
                grp_exp(pf, tau, nlse);
                if (diag) {  // query 32 g + col < kv row: masked
#pragma unroll
                    for (int e = 0; e < 32; ++e)
                        pf[e] = (32 * g + grp_col(e) + 2 * (lane & 3) < 32 * wq + grp_row(e) + (lane >> 2)) ? 0.f
                                                                                                   : pf[e];
                }
                uint32_t pk[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) pk[k] = pack_bf16x2(pf[2 * k], pf[2 * k + 1]);
                grp_store_packed(tS, pk);
                tmem::wait_st();
                tmem::fence_before();
                mbar_arrive(&sh.p_full[buf_of(x)][g]);
                if (threadIdx.x == 0) TKB_TR(1, x, 1);
                mbar_wait(&sh.dp_full, x & 1);
                if (threadIdx.x == 0) TKB_TR(1, x, 2);
                tmem::fence_after();
                uint32_t dpv[32];
                grp_load(tDp, reinterpret_cast<float*>(dpv));
                grp_ds(pf, dpv, dlt, pk);
                grp_store_packed(tDp, pk);
                tmem::wait_st();
                tmem::fence_before();
                mbar_arrive(&sh.ds_full[g]);
                if (threadIdx.x == 0) TKB_TR(1, x, 3);
            }
            cs.x0 += T;
        }
        // FINISH. When the next task has >= 3 steps, dV / dK are staged (bf16, SW128) in the
        // ring slots its step-2 Q and step-1 dO will use — both slots' last data (this task's
        // final step) are consumed — and TMA-stored by the load warp, which refills those two
        // slots only after the store has read them. The compute warps are back on the next
        // task's exponentials after ~500 clk. Otherwise rows are stored from registers.
        static TKB_DEVICE void finish(const lcsf::args<attn_bwd_dkdv_template>& a, state& cs, int id, int n) {
            const globals& p = a.g;
            shared& sh = a.sh;
            const int wq = a.warp & 3;
            const int g = a.warp >> 2;
            const int r = wq * 32 + a.lane;
            const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
            const uint32_t tbase = a.tmem;
            long long* tr = trace_slot(p, (int)blockIdx.x, 0);
            const long long t_start = cs.t_start;
            const KvTask w = decode(p, id);
            const int kv0 = w.j * 128;
            mbar_wait(&sh.dkv_full, n & 1);
            if (threadIdx.x == 0) TKB_TR(1, n, 4);
            tmem::fence_after();
            const int id_next = a.queue.get_warp(n + 1);
            const bool staged = p.kv_split == 1 && id_next >= 0 && steps(p, decode(p, id_next)) >= 3;
            if (p.kv_split > 1) {
                // grouped-query split: this chunk's fp32 partials, reduced by dkv_reduce_kernel
                const size_t u = (size_t)(w.batch * (p.heads / p.group) + w.head);
                const size_t plane = (size_t)p.kv_units / p.kv_split * p.n_pad * D;  // one chunk of one tensor
                float* part = p.dkv_part + ((size_t)w.chunk * (p.kv_units / p.kv_split) + u) * p.n_pad * D +
                              (size_t)(kv0 + r) * D + g * (D / 4);
                rt_fl<D / 4> f;
                load(f, tbase + lane_off + CT::tmem_dv() + g * (D / 4));
                load_wait(f);
                tmem::fence_before();
                mbar_arrive(&sh.dv_free);
#pragma unroll
                for (int c = 0; c < D / 4; c += 4)
                    *reinterpret_cast<float4*>(part + c) = make_float4(f.v[c], f.v[c + 1], f.v[c + 2], f.v[c + 3]);
                load(f, tbase + lane_off + CT::tmem_dk() + g * (D / 4));
                load_wait(f);
                tmem::fence_before();
                mbar_arrive(&sh.dk_free);
                part += plane * p.kv_split;  // the dK planes follow the dV planes
#pragma unroll
                for (int c = 0; c < D / 4; c += 4)
                    *reinterpret_cast<float4*>(part + c) = make_float4(f.v[c], f.v[c + 1], f.v[c + 2], f.v[c + 3]);
            } else if (staged) {
                tmem_rows_to_smem_bf16<D>(tbase + lane_off + CT::tmem_dv(), tQ(sh, cs.x0 + 2), r, g);
                tmem::fence_before();
                mbar_arrive(&sh.dv_free);
                tmem_rows_to_smem_bf16<D>(tbase + lane_off + CT::tmem_dk(), tDo(sh, cs.x0 + 1), r, g, p.scale);
                tmem::fence_before();
                mbar_arrive(&sh.dk_free);
                tma::fence_async_smem();
                mbar_arrive(&sh.staged_full);  // the load warp stores them
            } else {
                // dV / dK rows from registers (register -> global, warp-transposed)
                const int row0 = kv0 + wq * 32;  // row of lane 0
                // variable-length batches: the sequence's first packed row is the base, batch 0
                const size_t base = (size_t)w.sv.off * p.kv_sn;
                const int bidx = p.cu_seqlens ? 0 : w.batch;
                const gv<__nv_bfloat16> gdv{reinterpret_cast<__nv_bfloat16*>(p.dv) + base, p.kv_sb, p.kv_sh, p.kv_sn};
                const gv<__nv_bfloat16> gdk{reinterpret_cast<__nv_bfloat16*>(p.dk) + base, p.kv_sb, p.kv_sh, p.kv_sn};
                rt_fl<D / 4> f;
                rt_bf<D / 4> h;
                load(f, tbase + lane_off + CT::tmem_dv() + g * (D / 4));
                load_wait(f);
                tmem::fence_before();
                mbar_arrive(&sh.dv_free);
                copy(h, f);
                store_rows(gdv, h, bidx, w.head, row0, g * (D / 4), w.sv.n - row0);
                load(f, tbase + lane_off + CT::tmem_dk() + g * (D / 4));
                load_wait(f);
                tmem::fence_before();
                mbar_arrive(&sh.dk_free);
                mul(f, p.scale);  // dK = scale dS^T Q
                copy(h, f);
                store_rows(gdk, h, bidx, w.head, row0, g * (D / 4), w.sv.n - row0);
            }
            if (threadIdx.x == 0) TKB_TR(1, n, 6);
        }
        static TKB_DEVICE void drain(const lcsf::args<attn_bwd_dkdv_template>&, state&) {}
    };
};

// ================================================================== bwd_dkdv on CTA pairs (D = 128)
// The single-CTA bwd_dkdv moves 256 KB through each SM's shared-memory port per step (the
// SS GEMMs S^T / dP^T read 8 KB per MMA, the TS GEMMs 4 KB, TMA writes 64 KB of Q / dO) —
// more than the 128 B/clk port delivers in the 2048 clk the 32 MMAs need. A cluster of two
// CTAs (kv blocks 2p, 2p + 1) runs every GEMM as one M = 256 pair MMA over their 256 kv rows
// (cluster.cuh): B is split between the CTAs, so per SM an S^T / dP^T MMA reads 4 + 2 KB and
// a dV / dK MMA 2 KB, and the step costs 192 KB of SMEM traffic. The two CTAs stream the
// same Q / dO blocks; each holds
//   Q_s  its 64-query half of the block, all D   (B of S^T  = K Q^T, N = queries)
//   Q_t  its 64-column half of D, all 128 queries (B of dK += dS^T Q, N = D)
// (and dO likewise). Causal: the pair visits q blocks >= 2p; block 2p is fully masked for
// the odd CTA (P = 0 there).
// TMEM per CTA: S^T (P^T packed into it) | dV | dP^T (dS^T packed into it) | dK.
struct CfgKV2 {
    static constexpr int D = 128;
    static constexpr int kTile = 128 * D * 2;   // K / V: 32 KB
    static constexpr int kHalf = kTile / 2;     // Q_s, Q_t, dO_s, dO_t: 16 KB
    static constexpr int kStages = 2;
    static constexpr int kOffK = 0;
    static constexpr int kOffV = kOffK + kTile;
    static constexpr int kOffQ = kOffV + kTile;               // [S] x (Q_s | Q_t)
    static constexpr int kOffDo = kOffQ + kStages * kTile;    // [S] x (dO_s | dO_t)
    static constexpr int kOffLse = kOffDo + kStages * kTile;  // [S] x 128 fp32
    static constexpr int kOffDelta = kOffLse + kStages * 512;
    static constexpr int kOffBar = kOffDelta + kStages * 512;
    static constexpr int kSmemBytes = kOffBar + 512 + 1024;
    static_assert(kSmemBytes <= 232448, "smem");
    static __device__ __forceinline__ constexpr uint32_t tmem_s() { return 0u; }
    static __device__ __forceinline__ constexpr uint32_t tmem_dv() { return 128u; }
    static __device__ __forceinline__ constexpr uint32_t tmem_dp() { return 256u; }
    static __device__ __forceinline__ constexpr uint32_t tmem_dk() { return 384u; }
};

template <bool CAUSAL>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    attn_bwd_dkdv2_kernel(const __grid_constant__ BwdParams p) {
    using C = CfgKV2;
    constexpr int S = C::kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sK = smem + C::kOffK;
    uint8_t* sV = smem + C::kOffV;
    uint8_t* sQ = smem + C::kOffQ;
    uint8_t* sDo = smem + C::kOffDo;
    float* sLse = reinterpret_cast<float*>(smem + C::kOffLse);
    float* sDelta = reinterpret_cast<float*>(smem + C::kOffDelta);
    mbarrier* bars = reinterpret_cast<mbarrier*>(smem + C::kOffBar);
    mbarrier& kv_full = bars[0];     // leader: K / V of both CTAs
    mbarrier& s_full = bars[1];      // both (multicast commit)
    mbarrier& dp_full = bars[3];     // both
    mbarrier& dkv_full = bars[5];    // both
    // operand rings, full on the leader (both CTAs' TMA), empty on both (multicast commit):
    // the S^T / dP^T operands (Q_s, dO_s) are released as soon as that GEMM retires, a step
    // before the dK / dV operands (Q_t, dO_t), so the next S^T's Q is loaded early
    mbarrier* qs_full = bars + 8;     // [S]
    mbarrier* qs_empty = bars + 10;   // [S]
    mbarrier* qt_full = bars + 12;    // [S]
    mbarrier* qt_empty = bars + 14;   // [S]
    mbarrier* dos_full = bars + 16;   // [S]
    mbarrier* dos_empty = bars + 18;  // [S]
    mbarrier* dot_full = bars + 20;   // [S]
    mbarrier* dot_empty = bars + 22;  // [S]
    mbarrier* aux_full = bars + 24;   // [S] own: lse2 / delta of the q block
    mbarrier* p_full = bars + 32;    // [kGroups] leader: P^T chunks of both CTAs
    mbarrier* ds_full = bars + 36;   // [kGroups] leader: dS^T chunks
    uint32_t& tmem_slot = *reinterpret_cast<uint32_t*>(bars + 28);

    const int warp = warpid();
    const int lane = laneid();
    const uint32_t rank = cluster::ctarank();
    const bool leader = rank == 0;
    const int j = blockIdx.x;  // kv block; the pair is (j0, j0 + 1)
    const int j0 = j & ~1;
    const int head = blockIdx.y;
    const int batch = blockIdx.z;
    const int kv0 = j * 128;
    const int nq = p.n_pad / 128;
    const int T1 = CAUSAL ? (nq - j0) : nq;
    const int T = T1 * p.group;
    auto qblock = [&](int t) { return CAUSAL ? (j0 + t % T1) : t % T1; };
    auto qhead = [&](int t) { return head * p.group + t / T1; };
    long long* tr = trace_slot(p, (batch * gridDim.y + head) * gridDim.x + j, 0);
    const long long t_start = clock64();

    if (warp == kWarpLoad && lane == 0) {
        mbar_init(&kv_full, 1);
        mbar_init(&s_full, 1);
        mbar_init(&dp_full, 1);
        mbar_init(&dkv_full, 1);
        for (int g = 0; g < kGroups; ++g) {
            mbar_init(&p_full[g], 2 * 4);  // the 4 warps of one column group, both CTAs
            mbar_init(&ds_full[g], 2 * 4);
        }
        for (int s = 0; s < S; ++s) {
            mbar_init(&qs_full[s], 1);
            mbar_init(&qs_empty[s], 1);
            mbar_init(&qt_full[s], 1);
            mbar_init(&qt_empty[s], 1);
            mbar_init(&dos_full[s], 1);
            mbar_init(&dos_empty[s], 1);
            mbar_init(&dot_full[s], 1);
            mbar_init(&dot_empty[s], 1);
            mbar_init(&aux_full[s], 1);
        }
        fence_barrier_init();
        tma::prefetch_desc(&p.tm_q);
        tma::prefetch_desc(&p.tm_q64);
        tma::prefetch_desc(&p.tm_k);
        tma::prefetch_desc(&p.tm_v);
        tma::prefetch_desc(&p.tm_do);
        tma::prefetch_desc(&p.tm_do64);
    }
    if (warp == kWarpMma) tmem::alloc2<512>(&tmem_slot);
    tmem::fence_before();
    cluster::sync();  // barriers of both CTAs initialised before any remote arrive / complete_tx
    tmem::fence_after();
    const uint32_t tbase = tmem_slot;

    if (warp == kWarpLoad) {
        if (lane == 0) {
            // ------------------------------------------------------------- LOAD (both CTAs)
            const uint64_t pol_stream = tma::policy_evict_first();
            const uint64_t pol_keep = tma::policy_evict_last();
            const uint32_t kv_bar = cluster::map(&kv_full, 0);
            if (leader) mbar_arrive_expect_tx(&kv_full, 4 * C::kTile);
            for (int a = 0; a < 2; ++a) {
                cluster::load_4d(sK + a * kAtomBytes, &p.tm_k, kv_bar, a * 64, kv0, head, batch, pol_stream);
                cluster::load_4d(sV + a * kAtomBytes, &p.tm_v, kv_bar, a * 64, kv0, head, batch, pol_stream);
            }
            const int r64 = 64 * (int)rank;
            // one half tile (16 KB) into this CTA, counted on the leader's barrier
            auto half = [&](mbarrier* full, mbarrier* empty, uint32_t ph, uint8_t* dst, const CUtensorMap* rows64,
                            const CUtensorMap* rows128, bool qhalf, int i, int hq) {
                mbar_wait(empty, ph);
                const uint32_t bar = cluster::map(full, 0);
                if (leader) mbar_arrive_expect_tx(full, 2 * C::kHalf);
                if (qhalf) {  // query rows [64 rank, +64) of the block, all D (two 8 KB atoms)
                    for (int a = 0; a < 2; ++a)
                        cluster::load_4d(dst + a * (kAtomBytes / 2), rows64, bar, a * 64, i * 128 + r64, hq, batch,
                                         pol_keep);
                } else {  // D columns [64 rank, +64), all 128 queries (one atom)
                    cluster::load_4d(dst, rows128, bar, r64, i * 128, hq, batch, pol_keep);
                }
            };
            for (int t = 0; t < T; ++t) {
                const int i = qblock(t), s = t % S, hq = qhead(t);
                const size_t bhq = (size_t)batch * p.heads + hq;
                const uint32_t ph = ((t / S) & 1) ^ 1;
                uint8_t* dos = sDo + s * C::kTile;
                uint8_t* qs = sQ + s * C::kTile;
                half(&qs_full[s], &qs_empty[s], ph, qs, &p.tm_q64, &p.tm_q, true, i, hq);
                half(&dos_full[s], &dos_empty[s], ph, dos, &p.tm_do64, &p.tm_do, true, i, hq);
                half(&qt_full[s], &qt_empty[s], ph, qs + C::kHalf, &p.tm_q64, &p.tm_q, false, i, hq);
                mbar_arrive_expect_tx(&aux_full[s], 1024);  // slot freed with Q_t (dK_{t-S})
                tma::load_1d(sLse + s * 128, p.lse2 + bhq * p.n_pad + i * 128, 512, &aux_full[s]);
                tma::load_1d(sDelta + s * 128, p.delta + bhq * p.n_pad + i * 128, 512, &aux_full[s]);
                half(&dot_full[s], &dot_empty[s], ph, dos + C::kHalf, &p.tm_do64, &p.tm_do, false, i, hq);
            }
        }
    } else if (warp == kWarpMma) {
        if (leader) {
            // ------------------------------------------------------------- MMA (leader, converged)
            const Tile<128> tK{sK}, tV{sV};
            // per ring slot: Q_s / dO_s = this CTA's 64-query half (all D), Q_t / dO_t = its
            // 64-column half of D (all 128 queries)
            auto qs = [&](int t) { return st_bf<64, 128>{sQ + (t % S) * C::kTile}; };
            auto dos = [&](int t) { return st_bf<64, 128>{sDo + (t % S) * C::kTile}; };
            auto qt = [&](int t) { return st_bf<128, 64>{sQ + (t % S) * C::kTile + C::kHalf}; };
            auto dot = [&](int t) { return st_bf<128, 64>{sDo + (t % S) * C::kTile + C::kHalf}; };
            auto ready_of = [&](mbarrier* ready, uint32_t ph) {
                return [=](int g) {
                    cluster::wait(&ready[g], ph);
                    tmem::fence_after();
                };
            };
            auto issue_s = [&](int x) {  // S^T_x = K Q_x^T
                cluster::wait(&qs_full[x % S], (x / S) & 1);
                tmem::fence_after();
                pair::mm_ABt(tt_fl<128>{tbase + C::tmem_s()}, tK, qs(x));
                pair::mma_commit(&s_full);
                pair::mma_commit(&qs_empty[x % S]);
            };
            auto issue_dp = [&](int x) {  // dP^T_x = V dO_x^T
                cluster::wait(&dos_full[x % S], (x / S) & 1);
                tmem::fence_after();
                pair::mm_ABt(tt_fl<128>{tbase + C::tmem_dp()}, tV, dos(x));
                pair::mma_commit(&dp_full);
                pair::mma_commit(&dos_empty[x % S]);
            };
            cluster::wait(&kv_full, 0);
            issue_s(0);
            issue_dp(0);
            // Per step, in issue (= execution) order: dV_t, S^T_{t+1}, dK_t, dP^T_{t+1} — the
            // single-CTA kernel's order. S^T_{t+1} overwrites S^T / P^T_t, which dV_t (issued
            // before) reads first; dP^T_{t+1} overwrites dP^T / dS^T_t after dK_t. The next S^T
            // thus runs under the softmax of this step's dS and the exponentials of step t + 1
            // under dK_t / dP^T_{t+1}.
            for (int t = 0; t < T; ++t) {
                const uint32_t ph = t & 1;
                TKB_TR(0, t, 0);
                // dV += P_t^T dO_t   (P^T in packed columns [32g, 32g + 16) of the S^T region)
                cluster::wait(&dot_full[t % S], (t / S) & 1);
                pair::mma_AB_groups(tt_fl<128>{tbase + C::tmem_dv()}, tt_bf<128>{tbase + C::tmem_s()},
                                    swap_layout(dot(t)), t > 0, ready_of(p_full, ph));
                pair::mma_commit(&dot_empty[t % S]);
                TKB_TR(0, t, 1);
                if (t + 1 < T) issue_s(t + 1);
                TKB_TR(0, t, 2);
                // dK += dS_t^T Q_t   (dS^T in packed columns [32g, 32g + 16) of the dP^T region)
                cluster::wait(&qt_full[t % S], (t / S) & 1);
                pair::mma_AB_groups(tt_fl<128>{tbase + C::tmem_dk()}, tt_bf<128>{tbase + C::tmem_dp()},
                                    swap_layout(qt(t)), t > 0, ready_of(ds_full, ph));
                pair::mma_commit(&qt_empty[t % S]);
                TKB_TR(0, t, 3);
                if (t + 1 < T) issue_dp(t + 1);
                TKB_TR(0, t, 4);
            }
            pair::mma_commit(&dkv_full);
        }
    } else {
        // ----------------------------------------------------------------- COMPUTE (both CTAs)
        const int wq = warp & 3;
        const int g = warp >> 2;       // q group: columns [32g, 32g+32)
        const int r = wq * 32 + lane;  // kv row == TMEM lane
        const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
        const uint32_t tS = tbase + lane_off + C::tmem_s() + 32 * g;
        const uint32_t tDp = tbase + lane_off + C::tmem_dp() + 32 * g;
        const float tau = p.scale_log2;
        const uint32_t p_full_l = cluster::map(&p_full[g], 0);
        const uint32_t ds_full_l = cluster::map(&ds_full[g], 0);
        // all lanes' TMEM accesses retired, then one lane arrives on the leader's barrier
        auto warp_arrive = [&](uint32_t bar) {
            tmem::fence_before();
            __syncwarp();
            if (lane == 0) cluster::arrive_remote(bar);
        };
        for (int t = 0; t < T; ++t) {
            const int i = qblock(t);
            const int s = t % S;
            const bool diag = CAUSAL && (i * 128 < kv0 + 128);
            mbar_wait(&aux_full[s], (t / S) & 1);
            float nlse[8], dlt[8];
            grp_vec_load(smem_u32(sLse + s * 128 + 32 * g), nlse);
            grp_vec_load(smem_u32(sDelta + s * 128 + 32 * g), dlt);
            cluster::wait(&s_full, t & 1);
            if (threadIdx.x == 0) TKB_TR(1, t, 0);
            tmem::fence_after();
            float pf[32];
            grp_load(tS, pf);
            grp_exp(pf, tau, nlse);
            if (diag) {  // key kv0 + row visible to query 128 i + 32 g + col iff col >= row + kv0 - 128 i - 32 g
                const int lim0 = kv0 + wq * 32 + (lane >> 2) - i * 128 - 32 * g - 2 * (lane & 3);
#pragma unroll
                for (int e = 0; e < 32; ++e) pf[e] = (grp_col(e) < lim0 + grp_row(e)) ? 0.f : pf[e];
            }
            uint32_t pk[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) pk[k] = pack_bf16x2(pf[2 * k], pf[2 * k + 1]);
            grp_store_packed(tS, pk);  // P^T over the first 16 of the group's S^T columns
            tmem::wait_st();
            warp_arrive(p_full_l);
            if (threadIdx.x == 0) TKB_TR(1, t, 1);
            cluster::wait(&dp_full, t & 1);
            if (threadIdx.x == 0) TKB_TR(1, t, 2);
            tmem::fence_after();
            uint32_t dpv[32];
            grp_load(tDp, reinterpret_cast<float*>(dpv));
            grp_ds(pf, dpv, dlt, pk);
            grp_store_packed(tDp, pk);
            tmem::wait_st();
            warp_arrive(ds_full_l);
            if (threadIdx.x == 0) TKB_TR(1, t, 3);
        }
        // FINISH: dV, dK (TMEM fp32) -> bf16 -> SMEM (Q and dO rings are free) -> TMA store
        cluster::wait(&dkv_full, 0);
        tmem::fence_after();
        tmem_rows_to_smem_bf16<128>(tbase + lane_off + C::tmem_dv(), Tile<128>{sQ}, r, g);
        tmem_rows_to_smem_bf16<128>(tbase + lane_off + C::tmem_dk(), Tile<128>{sDo}, r, g, p.scale);  // dK = scale dS^T Q
        tma::fence_async_smem();
        named_sync(kBarCompute, kComputeThreads);
        if (threadIdx.x == 0) {
            for (int a = 0; a < 2; ++a) {
                tma::store_4d(&p.tm_dv, sQ + a * kAtomBytes, a * 64, kv0, head, batch);
                tma::store_4d(&p.tm_dk, sDo + a * kAtomBytes, a * 64, kv0, head, batch);
            }
            tma::commit_group();
            tma::wait_group_read<0>();
            TKB_TR(1, kTraceIters - 1, 7);  // CTA finish
        }
    }

    tmem::fence_before();
    cluster::sync();  // the pair's MMAs / remote arrives are all done before TMEM goes away
    if (warp == kWarpMma) tmem::dealloc2<512>(tbase);
}

// ================================================================== bwd_dq (Q-stationary, persistent)
// One CTA per SM walks query-block tasks (b, h, i) — heads in L2-sized groups, heavy causal
// blocks first — with every ring continuing across tasks: the next task's Q / dO are
// TMA-loaded while this one runs, copied into TMEM as soon as this task's last S / dP GEMMs
// retire, so its first S and dP GEMMs overlap this task's dQ finish stage.
template <int D>
struct CfgQ {
    using T = Tiles<D>;
    // K / V ring depths. K_j is released by dQ_j, the last GEMM of step j, and needed again
    // by S_{j+SK}; with SK = 2 only one GEMM (dP_{j+1}) separates them and the L2 -> SMEM
    // latency of the 32 KB reload is exposed (measured: 2650 instead of 1550 clk per step
    // with the compute warps idle). V_j is released by dP_j, early in the step.
    static constexpr int kStagesK = (D == 128) ? 3 : 5;
    static constexpr int kStagesV = (D == 128) ? 2 : 4;
    static constexpr int kOffQ = 0;
    static constexpr int kOffDo = kOffQ + T::kTileBytes;
    static constexpr int kOffK = kOffDo + T::kTileBytes;
    static constexpr int kOffV = kOffK + kStagesK * T::kTileBytes;
    static constexpr int kOffBar = kOffV + kStagesV * T::kTileBytes;
    static constexpr int kSmemBytes = kOffBar + 512 + 1024;
    static_assert(kSmemBytes <= 232448, "smem");
    // S | dP | dQ | Q (A operand) | dO (A operand): 128 + 128 + D + D/2 + D/2 <= 512
    static __device__ __forceinline__ constexpr uint32_t tmem_s() { return 0u; }
    static __device__ __forceinline__ constexpr uint32_t tmem_dp() { return 128u; }
    static __device__ __forceinline__ constexpr uint32_t tmem_dq() { return 256u; }
    static __device__ __forceinline__ constexpr uint32_t tmem_qa() { return 256u + D; }
    static __device__ __forceinline__ constexpr uint32_t tmem_doa() { return 256u + D + D / 2; }
};

struct QTask {
    int i, bh;   // query block, batch * heads + head
    int b;       // batch
    SeqView sv;  // this batch's length and TMA row coordinates (variable-length batches)
};

// task t -> (query block, b*h): heads in groups of p.head_group whose K / V stay in L2,
// inside a group the causal query blocks heavy (late) first, heads innermost
template <bool CAUSAL>
TKB_DEVICE QTask qtask(const BwdParams& p, int t) {
    const int nq = p.n_pad / 128;
    const int G = p.head_group;
    const int sec = p.q_sec.div(t);  // FastDiv: no MUFU.RCP behind the compute warps' exponentials
    const int r = t - sec * G * nq;
    const bool full = p.bh - sec * G >= G;
    const int gs = full ? G : p.bh - sec * G;
    const int mi = full ? p.q_g.div(r) : p.q_grem.div(r);
    QTask w;
    w.bh = sec * G + (r - mi * gs);
    w.i = CAUSAL ? (nq - 1 - mi) : mi;
    w.b = p.q_heads.div(w.bh);
    w.sv = seq_view(p.cu_seqlens, p.vmaps, kBwdMaps, p.n, w.b);
    return w;
}

// The dQ kernel is lcsf::kernel<attn_bwd_dq_template<D, Causal>> (tkb/lcsf.cuh).
template <int D, bool CAUSAL>
struct attn_bwd_dq_template {
    using C = CfgQ<D>;
    using TL = Tiles<D>;
    using globals = BwdParams;
    static constexpr int SK = C::kStagesK;
    static constexpr int SV = C::kStagesV;
    static constexpr int kThreads = bwd::kThreads;
    static constexpr int kTmemCols = 512;
    static constexpr int kProducerWarp = kWarpLoad;
    static constexpr int kMmaWarp = bwd::kWarpMma;
    static constexpr int kConsumerWarps = 16;
    static constexpr int kQueueReaders = 1 + 16;  // the MMA warp and the 16 compute warps
    static constexpr bool kAlignSlack = true;
    static constexpr bool kReleaseEarly = false;
    static constexpr int kAuxWarps = 0, kAuxWarp0 = 0;
    // D = 64 leaves 128 TMEM columns free: dP is double-buffered there (second buffer at
    // column 384), so dP_{j+1} is issued before dQ_j instead of after it and the dS of step
    // j+1 does not wait for the dQ GEMM that reads dS_j. Per-buffer dp_full / ds_full.
    static constexpr bool kDP = (D == 64);

    struct shared {
        uint8_t q[TL::kTileBytes];
        uint8_t dO[TL::kTileBytes];
        uint8_t k[SK][TL::kTileBytes];
        uint8_t v[SV][TL::kTileBytes];
        mbarrier qdo_full;   // Q / dO of a task in SMEM (TMA)
        mbarrier s_full, s_free;
        mbarrier a_ready;    // Q / dO of a task copied into TMEM
        mbarrier qdo_free;   // SMEM Q / dO copied out: the next task's may load
        mbarrier dp_full[2];  // [buffer]
        mbarrier qa_free;    // last S / dP GEMM of a task retired: TMEM Q / dO reusable
        mbarrier dq_full;
        mbarrier k_full[SK], k_empty[SK];
        mbarrier v_full[SV], v_empty[SV];
        mbarrier ds_full[2][kGroups];  // [buffer][column group]
        lcsf::work_queue queue;
        uint32_t tmem_slot;
    };
    static constexpr int kSmemBytes = (int)sizeof(shared) + 1024;  // + alignment slack
    static_assert(kSmemBytes <= 232448, "smem");

    static TKB_DEVICE uint32_t dp_buf(uint32_t it) { return kDP ? ((it & 1) ? 384u : C::tmem_dp()) : C::tmem_dp(); }
    static TKB_DEVICE int buf_of(uint32_t it) { return (kDP && (it & 1)) ? 1 : 0; }
    static TKB_DEVICE uint32_t ph_of(uint32_t it) { return kDP ? ((it >> 1) & 1) : (it & 1); }
    static TKB_DEVICE int num_tasks(const globals& p) { return p.bh * (p.n_pad / 128); }
    static TKB_DEVICE int* counter(const globals& p) { return p.sched; }
    static TKB_DEVICE int nk_of(const globals&, const QTask& w) { return CAUSAL ? (w.i + 1) : (w.sv.n + 127) / 128; }
    // variable-length batches: query blocks past a short sequence have no work
    static TKB_DEVICE bool skip(const globals& p, int t) {
        if (p.cu_seqlens == nullptr) return false;
        const QTask w = qtask<CAUSAL>(p, t);
        return w.i * 128 >= w.sv.n;
    }
    static TKB_DEVICE Tile<D> tK(shared& sh, int x) { return Tile<D>{sh.k[x % SK]}; }
    static TKB_DEVICE Tile<D> tV(shared& sh, int x) { return Tile<D>{sh.v[x % SV]}; }

    static TKB_DEVICE void init(shared& sh, const globals& p) {
        mbar_init(&sh.qdo_full, 1);
        mbar_init(&sh.s_full, 1);
        mbar_init(&sh.s_free, kComputeThreads);
        mbar_init(&sh.a_ready, kComputeThreads);
        mbar_init(&sh.qdo_free, 1);
        mbar_init(&sh.dp_full[0], 1);
        mbar_init(&sh.dp_full[1], 1);
        mbar_init(&sh.qa_free, 1);
        mbar_init(&sh.dq_full, 1);
        for (int g = 0; g < kGroups; ++g) {
            mbar_init(&sh.ds_full[0][g], 128);
            mbar_init(&sh.ds_full[1][g], 128);
        }
        for (int s = 0; s < SK; ++s) {
            mbar_init(&sh.k_full[s], 1);
            mbar_init(&sh.k_empty[s], 1);
        }
        for (int s = 0; s < SV; ++s) {
            mbar_init(&sh.v_full[s], 1);
            mbar_init(&sh.v_empty[s], 1);
        }
        tma::prefetch_desc(&p.tm_q);
        tma::prefetch_desc(&p.tm_k);
        tma::prefetch_desc(&p.tm_v);
        tma::prefetch_desc(&p.tm_do);
    }

    // ------------------------------------------------------------- LOAD
    struct producer {
        struct state {
            int kv = 0;  // K / V ring position, continuous across tasks
        };
        // the skeleton claims the next task once this one's loads are all issued (the atomic
        // counter hands the heavy causal tasks out first and balances them across SMs)
        template <class ClaimNext>
        static TKB_DEVICE void load(const lcsf::args<attn_bwd_dq_template>& a, state& ps, int t, int n, ClaimNext&&) {
            const globals& p = a.g;
            shared& sh = a.sh;
            const uint64_t pol_stream = tma::policy_evict_first();
            const uint64_t pol_keep = tma::policy_evict_last();
            const QTask w = qtask<CAUSAL>(p, t);
            const int b = w.b, h = w.bh - b * p.heads;
            mbar_wait(&sh.qdo_free, (n & 1) ^ 1u);  // the previous task's Q / dO are in TMEM
            mbar_arrive_expect_tx(&sh.qdo_full, 2 * TL::kTileBytes);
            const int bc = w.sv.bcoord;
            if (w.sv.maps != nullptr) {  // this sequence's maps (varlen_maps_kernel)
                for (int m : {kMapQ, kMapK, kMapV, kMapDo}) tma::acquire_map(w.sv.maps + m);
            }
            w.sv.with_map(p.tm_q, kMapQ, [&](const CUtensorMap* m) {
                load_async(Tile<D>{sh.q}, gl{m}, &sh.qdo_full, w.i * 128, h, bc, pol_stream);
            });
            w.sv.with_map(p.tm_do, kMapDo, [&](const CUtensorMap* m) {
                load_async(Tile<D>{sh.dO}, gl{m}, &sh.qdo_full, w.i * 128, h, bc, pol_stream);
            });
            const int nk = nk_of(p, w);
            for (int jj = 0; jj < nk; ++jj, ++ps.kv) {
                const int kv = ps.kv;
                const int sk = kv % SK, sv = kv % SV;
                mbar_wait(&sh.k_empty[sk], ((kv / SK) & 1) ^ 1);
                mbar_arrive_expect_tx(&sh.k_full[sk], TL::kTileBytes);
                w.sv.with_map(p.tm_k, kMapK, [&](const CUtensorMap* m) {
                    load_async(tK(sh, kv), gl{m}, &sh.k_full[sk], jj * 128, h / p.group, bc, pol_keep);
                });
                mbar_wait(&sh.v_empty[sv], ((kv / SV) & 1) ^ 1);
                mbar_arrive_expect_tx(&sh.v_full[sv], TL::kTileBytes);
                w.sv.with_map(p.tm_v, kMapV, [&](const CUtensorMap* m) {
                    load_async(tV(sh, kv), gl{m}, &sh.v_full[sv], jj * 128, h / p.group, bc, pol_keep);
                });
            }
        }
        static TKB_DEVICE void drain(const lcsf::args<attn_bwd_dq_template>&, state&) {}
    };

    // ------------------------------------------------------------- MMA (converged warp)
    struct mma {
        struct state {
            int kv = 0;       // K / V ring position
            uint32_t it = 0;  // global iteration count (s_full / s_free / dp_full / ds_full phases)
            long long t_start = 0;
        };
        static TKB_DEVICE void issue(const lcsf::args<attn_bwd_dq_template>& a, state& ms, int t, int n) {
            const globals& p = a.g;
            shared& sh = a.sh;
            const uint32_t tbase = a.tmem;
            long long* tr = trace_slot(p, (int)blockIdx.x, 1);
            if (n == 0) ms.t_start = clock64();
            const long long t_start = ms.t_start;
            const tt_bf<D / 2> tQa{tbase + C::tmem_qa()}, tDoa{tbase + C::tmem_doa()};  // A operands in TMEM
            auto issue_s = [&](int x) {  // S = Q K^T
                mbar_wait(&sh.k_full[x % SK], (x / SK) & 1);
                tmem::fence_after();
                mm_ABt(tt_fl<128>{tbase + C::tmem_s()}, tQa, tK(sh, x));
                mma_commit(&sh.s_full);
            };
            auto issue_dp = [&](int x, uint32_t itx) {  // dP = dO V^T (iteration itx)
                mbar_wait(&sh.v_full[x % SV], (x / SV) & 1);
                tmem::fence_after();
                mm_ABt(tt_fl<128>{tbase + dp_buf(itx)}, tDoa, tV(sh, x));
                mma_commit(&sh.dp_full[buf_of(itx)]);
                mma_commit(&sh.v_empty[x % SV]);
            };
            int& kv = ms.kv;
            uint32_t& it = ms.it;
            const int nk = nk_of(p, qtask<CAUSAL>(p, t));
            mbar_wait(&sh.a_ready, n & 1);  // this task's Q / dO are in TMEM
            issue_s(kv);
            issue_dp(kv, it);
            if (nk == 1) mma_commit(&sh.qa_free);  // the task's only S and dP are issued
            for (int jj = 0; jj < nk; ++jj, ++kv, ++it) {
                if (jj + 1 < nk) {
                    mbar_wait(&sh.s_free, it & 1);  // S_j read out by the compute warps
                    issue_s(kv + 1);
                    if (kDP) {  // the other dP buffer: its dS_{j-1} went to dQ_{j-1}, issued before
                        issue_dp(kv + 1, it + 1);
                        if (jj + 2 == nk) mma_commit(&sh.qa_free);  // the task's last S and dP are issued
                    }
                }
                TKB_TR(0, (int)it, 0);
                // dQ += dS K (mma_AB: one 32-key chunk per column group as it lands, K read MN-major)
                mma_AB_groups(tt_fl<D>{tbase + C::tmem_dq()}, tt_bf<128>{tbase + dp_buf(it)},
                              swap_layout(tK(sh, kv)), jj > 0, [&](int g) {
                                  mbar_wait(&sh.ds_full[buf_of(it)][g], ph_of(it));
                                  tmem::fence_after();
                              });
                TKB_TR(0, (int)it, 1);
                mma_commit(&sh.k_empty[kv % SK]);
                if (!kDP && jj + 1 < nk) {
                    issue_dp(kv + 1, it + 1);  // overwrites dS_j, read by dQ_j issued before
                    if (jj + 2 == nk) mma_commit(&sh.qa_free);  // the task's last S and dP are issued
                }
                TKB_TR(0, (int)it, 2);
            }
            mma_commit(&sh.dq_full);
        }
    };

    // ------------------------------------------------------------- COMPUTE + FINISH
    struct consumer {
        struct state {
            uint32_t it = 0;
            long long t_start = 0;
        };
        // Q, dO of task nn: SMEM (TMA, swizzled) -> TMEM A operands, once the previous task's
        // last S / dP GEMMs retired (shared -> register -> TMEM)
        static TKB_DEVICE void stage_a(const lcsf::args<attn_bwd_dq_template>& a, int nn) {
            shared& sh = a.sh;
            const int wq = a.warp & 3, g = a.warp >> 2, r = wq * 32 + a.lane;
            const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
            mbar_wait(&sh.qdo_full, nn & 1);
            if (nn > 0) mbar_wait(&sh.qa_free, (nn - 1) & 1);
            tmem::fence_after();
            smem_rows_to_tmem_a<D>(Tile<D>{sh.q}, a.tmem + lane_off + C::tmem_qa(), r, g);
            smem_rows_to_tmem_a<D>(Tile<D>{sh.dO}, a.tmem + lane_off + C::tmem_doa(), r, g);
            tmem::wait_st();
            tmem::fence_before();
            mbar_arrive(&sh.a_ready);
        }
        static TKB_DEVICE void compute(const lcsf::args<attn_bwd_dq_template>& a, state& cs, int t, int n) {
            const globals& p = a.g;
            shared& sh = a.sh;
            const int wq = a.warp & 3;
            const int g = a.warp >> 2;       // kv group: columns [32g, 32g+32)
            const int r = wq * 32 + a.lane;  // q row == TMEM lane
            const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
            const uint32_t tS = a.tmem + lane_off + C::tmem_s() + 32 * g;
            const uint32_t tDp0 = a.tmem + lane_off + 32 * g;  // + dp_buf(it)
            const float tau = p.scale_log2;
            long long* tr = trace_slot(p, (int)blockIdx.x, 1);
            if (n == 0) {
                cs.t_start = clock64();
                // SMEM Q / dO are released (qdo_free) once copied into TMEM AND once the previous
                // task's finish, which stages dQ in sQ for its TMA store, has been read out
                stage_a(a, 0);
                named_sync(kBarCompute, kComputeThreads);
                if (threadIdx.x == 0) mbar_arrive(&sh.qdo_free);
            }
            const long long t_start = cs.t_start;
            const QTask w = qtask<CAUSAL>(p, t);
            const int q0 = w.i * 128;
            const int row = q0 + r;
            const int nk = nk_of(p, w);
            // -lse2 (-inf on padded rows -> P = 0) and Delta, stored group-permuted (perm32)
            const float nlse_r = p.lse2[(size_t)w.bh * p.n_pad + perm32(row)];
            const float dlt_r = p.delta[(size_t)w.bh * p.n_pad + perm32(row)];
            uint32_t& it = cs.it;
            for (int jj = 0; jj < nk; ++jj, ++it) {
                const int kv0 = jj * 128;
                mbar_wait(&sh.s_full, it & 1);
                if (threadIdx.x == 0) TKB_TR(1, (int)it, 0);
                tmem::fence_after();
                float pf[32];
                tmem::ldw_32x32b_x32(tS, reinterpret_cast<uint32_t*>(pf));
                tmem::fence_before();
                mbar_arrive(&sh.s_free);
                exp_chunk<true>(pf, tau, 0u, nlse_r);
                // visible keys: kv < n, and causal kv <= row
                const int lim = (CAUSAL ? min(row, w.sv.n - 1) : (w.sv.n - 1)) - kv0 - 32 * g;  // last visible column
                if (lim < 31) {  // diagonal / ragged tail block only
#pragma unroll
                    for (int c = 0; c < 32; ++c) pf[c] = (c > lim) ? 0.f : pf[c];
                }
                mbar_wait(&sh.dp_full[buf_of(it)], ph_of(it));
                const uint32_t tDp = tDp0 + dp_buf(it);
                if (threadIdx.x == 0) TKB_TR(1, (int)it, 1);
                tmem::fence_after();
                uint32_t dpv[32];
                tmem::ldw_32x32b_x32(tDp, dpv);
                uint32_t pk[16];
#pragma unroll
                for (int c = 0; c < 32; c += 2) {
                    const float2 gg = sub2(make_float2(__uint_as_float(dpv[c]), __uint_as_float(dpv[c + 1])),
                                           make_float2(dlt_r, dlt_r));
                    const float2 d = mul2(make_float2(pf[c], pf[c + 1]), gg);  // dS / scale (scale in the finish)
                    pk[c / 2] = pack_bf16x2(d.x, d.y);
                }
                tmem::st_32x32b_x16(tDp, pk);  // inside the 32 dP columns this thread has read
                tmem::wait_st();
                tmem::fence_before();
                mbar_arrive(&sh.ds_full[buf_of(it)][g]);
                if (threadIdx.x == 0) TKB_TR(1, (int)it, 2);
            }
        }
        // FINISH: the next task's Q / dO into TMEM first (its S / dP GEMMs then overlap this
        // finish), then dQ (TMEM fp32) -> bf16 -> SW128 staging in sQ (its Q is in TMEM by now)
        // -> TMA store; sQ / sDo are released to the load warp once the store has read it.
        // (Per-thread row stores from registers cost ~2,400 clk per task: each store
        // instruction touches 16-32 L2 lines.) The next task's first dQ GEMM waits for its
        // dS, which these warps produce after this.
        static TKB_DEVICE void finish(const lcsf::args<attn_bwd_dq_template>& a, state& cs, int t, int n) {
            const globals& p = a.g;
            shared& sh = a.sh;
            const int wq = a.warp & 3, g = a.warp >> 2, r = wq * 32 + a.lane;
            const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
            const QTask w = qtask<CAUSAL>(p, t);
            const int b = w.b, h = w.bh - b * p.heads;
            long long* tr = trace_slot(p, (int)blockIdx.x, 1);
            const long long t_start = cs.t_start;
            if (threadIdx.x == 0) TKB_TR(1, n, 3);  // finish start (per task n; events 3-7)
            const int t_next = a.queue.get_warp(n + 1);
            if (t_next >= 0) stage_a(a, n + 1);
            if (threadIdx.x == 0) TKB_TR(1, n, 4);  // next task's Q / dO in TMEM
            mbar_wait(&sh.dq_full, n & 1);
            if (threadIdx.x == 0) TKB_TR(1, n, 5);  // last dQ GEMM retired
            tmem::fence_after();
            tmem_rows_to_smem_bf16<D>(a.tmem + lane_off + C::tmem_dq(), Tile<D>{sh.q}, r, g, p.scale);  // dQ = scale dS K
            tma::fence_async_smem();
            named_sync(kBarCompute, kComputeThreads);
            if (threadIdx.x == 0) TKB_TR(1, n, 6);  // dQ staged
            if (threadIdx.x == 0) {
                if (w.sv.maps != nullptr) tma::acquire_map(w.sv.maps + kMapDq);
                w.sv.with_map(p.tm_dq, kMapDq, [&](const CUtensorMap* m) {
                    store_async(gl{m}, Tile<D>{sh.q}, w.i * 128, h, w.sv.bcoord);
                });
                tma::commit_group();
                // (waiting for this read later, after the next task's first step, freed warp 0
                // ~1.2 k clk per boundary but measured neutral: r2c_ab_bwd_dq_defer.txt)
                tma::wait_group_read<0>();
                mbar_arrive(&sh.qdo_free);
                TKB_TR(1, n, 7);  // store read SMEM
            }
        }
        static TKB_DEVICE void drain(const lcsf::args<attn_bwd_dq_template>&, state&) {
            if (threadIdx.x == 0) tma::wait_group<0>();
        }
    };
};
// The backward entry template (attn_bwd_template<D, Causal> beside the
// forward's attn_fwd_template<D, Causal>): dQ / dK / dV from the saved L as three launches on
// one stream — bwd_prep_kernel<D> (Delta = rowsum(dO o O), -L log2 e), then the two LCSF
// kernels lcsf::kernel<dkdv> (KV-stationary) and lcsf::kernel<dq> (Q-stationary).
template <int D, bool CAUSAL>
struct attn_bwd_template {
    using dkdv = attn_bwd_dkdv_template<D, CAUSAL>;
    using dq = attn_bwd_dq_template<D, CAUSAL>;
};

#undef TKB_TR

// Delta = rowsum(dO o O), lse2 = -L log2 e (-inf / 0 on padded rows: P = 0 there), written
// at perm32(row) within each 32-row group (the dK/dV compute threads' column order).
// HBM-bound: each thread owns 16 bytes of kPrepRows rows (rows kPrepRows * 16 / (D / 8) apart
// within the block's row range) and issues all their loads before reducing, so a thread
// keeps 2 * 16 * kPrepRows bytes in flight.
#ifndef TKB_PREP_ROWS
#define TKB_PREP_ROWS 4
#endif
constexpr int kPrepRows = TKB_PREP_ROWS;
// Linear blocks (bh, row block) are walked grid-stride with a 64-bit index: B * H is not
// bounded by gridDim.y's 65535.
template <int D>
__global__ void __launch_bounds__(256) bwd_prep_kernel(const __nv_bfloat16* __restrict__ o,
                                                       const __nv_bfloat16* __restrict__ dout,
                                                       const float* __restrict__ lse, float* __restrict__ lse2,
                                                       float* __restrict__ delta, const int* __restrict__ cu,
                                                       int heads, int n, int n_pad,
                                                       int row_blocks, int64_t total_blocks, int64_t sb, int64_t sh,
                                                       int64_t sn) {
    constexpr int kLanesPerRow = D / 8;
    constexpr int kRowsPerPass = 256 / kLanesPerRow;
    const int c = (threadIdx.x % kLanesPerRow) * 8;
    for (int64_t blk = blockIdx.x; blk < total_blocks; blk += gridDim.x) {
        const int64_t bh = blk / row_blocks;
        const int rb = (int)(blk - bh * row_blocks);
        const int64_t b = bh / heads, hh = bh % heads;
        const SeqView sv = seq_view(cu, nullptr, 0, n, (int)b);  // varlen: rows [cu[b], cu[b+1]), sb = 0
        const int row_base = rb * kRowsPerPass * kPrepRows + threadIdx.x / kLanesPerRow;
        uint4 ov[kPrepRows], dv[kPrepRows];
#pragma unroll
        for (int k = 0; k < kPrepRows; ++k) {
            const int row = row_base + k * kRowsPerPass;
            ov[k] = make_uint4(0, 0, 0, 0);
            dv[k] = make_uint4(0, 0, 0, 0);
            if (row < sv.n) {
                const int64_t off = b * sb + hh * sh + (int64_t)(sv.off + row) * sn + c;
                ov[k] = __ldg(reinterpret_cast<const uint4*>(o + off));
                dv[k] = __ldg(reinterpret_cast<const uint4*>(dout + off));
            }
        }
#pragma unroll
        for (int k = 0; k < kPrepRows; ++k) {
            const int row = row_base + k * kRowsPerPass;
            const __nv_bfloat162* o2 = reinterpret_cast<const __nv_bfloat162*>(&ov[k]);
            const __nv_bfloat162* d2 = reinterpret_cast<const __nv_bfloat162*>(&dv[k]);
            float acc = 0.f;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float2 a = __bfloat1622float2(o2[q]);
                const float2 g = __bfloat1622float2(d2[q]);
                acc = fmaf(a.x, g.x, acc);
                acc = fmaf(a.y, g.y, acc);
            }
#pragma unroll
            for (int s = kLanesPerRow / 2; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
            if (row < n_pad && (threadIdx.x % kLanesPerRow) == 0) {
                const size_t idx = (size_t)bh * n_pad + perm32(row);  // group-permuted (perm32)
                delta[idx] = row < sv.n ? acc : 0.f;
                lse2[idx] = row < sv.n ? -lse[(size_t)bh * n + row] * 1.44269504088896340736f : -INFINITY;
            }
        }
    }
}

// Grouped-query split (kv_split > 1): dV = sum_c dV_c, dK = scale * sum_c dK_c over the chunks in
// chunk order (deterministic), bf16 into dv / dk with their strides. HBM-bound; 8 columns per
// thread, grid-stride over (unit, row, column block).
template <int D>
__global__ void __launch_bounds__(256) dkv_reduce_kernel(const float* __restrict__ part, int split, int units, int n,
                                                         int n_pad, int hkv, __nv_bfloat16* dv, __nv_bfloat16* dk,
                                                         int64_t sb, int64_t sh, int64_t sn, float scale) {
    constexpr int kCb = D / 8;
    const int64_t total = (int64_t)units * n * kCb;
    const size_t plane = (size_t)units * n_pad * D;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int cb = (int)(i % kCb);
        const int64_t ur = i / kCb;
        const int row = (int)(ur % n);
        const int u = (int)(ur / n);
        const size_t src = ((size_t)u * n_pad + row) * D + cb * 8;
        const int64_t dst = (int64_t)(u / hkv) * sb + (int64_t)(u % hkv) * sh + (int64_t)row * sn + cb * 8;
#pragma unroll
        for (int which = 0; which < 2; ++which) {
            const float* pp = part + (size_t)which * split * plane + src;
            float acc[8];
            {
                const float4 a = *reinterpret_cast<const float4*>(pp), b = *reinterpret_cast<const float4*>(pp + 4);
                acc[0] = a.x, acc[1] = a.y, acc[2] = a.z, acc[3] = a.w, acc[4] = b.x, acc[5] = b.y, acc[6] = b.z, acc[7] = b.w;
            }
            for (int c = 1; c < split; ++c) {
                const float4 a = *reinterpret_cast<const float4*>(pp + c * plane);
                const float4 b = *reinterpret_cast<const float4*>(pp + c * plane + 4);
                acc[0] += a.x, acc[1] += a.y, acc[2] += a.z, acc[3] += a.w;
                acc[4] += b.x, acc[5] += b.y, acc[6] += b.z, acc[7] += b.w;
            }
            const float m = which ? scale : 1.f;  // dK = scale dS^T Q
            uint4 o;
            o.x = pack_bf16x2(acc[0] * m, acc[1] * m), o.y = pack_bf16x2(acc[2] * m, acc[3] * m);
            o.z = pack_bf16x2(acc[4] * m, acc[5] * m), o.w = pack_bf16x2(acc[6] * m, acc[7] * m);
            *reinterpret_cast<uint4*>((which ? dk : dv) + dst) = o;
        }
    }
}

template <int D, bool CAUSAL>
int launch_main(const BwdParams& p, int batches, cudaStream_t stream, int phases, int* launches) {
    static std::atomic<unsigned long long> set_dq{0}, set_kv2{0}, set_kvp{0};  // per device
    using DQ = typename attn_bwd_template<D, CAUSAL>::dq;
    if (int e = ensure_smem(lcsf::kernel<DQ>, DQ::kSmemBytes, set_dq)) return e;
    using KV = typename attn_bwd_template<D, CAUSAL>::dkdv;
    if (int e = ensure_smem(lcsf::kernel<KV>, KV::kSmemBytes, set_kvp)) return e;
    if (D == 128)
        if (int e = ensure_smem(attn_bwd_dkdv2_kernel<CAUSAL>, CfgKV2::kSmemBytes, set_kv2)) return e;
    if (phases & 2) {
        if (D == 128 && p.pairs && p.cu_seqlens == nullptr && p.kv_split == 1) {  // CTA pairs: kv blocks rounded up to even
            dim3 grid2((p.n_pad / 128 + 1) & ~1, p.heads / p.group, batches);
            attn_bwd_dkdv2_kernel<CAUSAL><<<grid2, kThreads, CfgKV2::kSmemBytes, stream>>>(p);
        } else {
            const int64_t tasks_kv = (int64_t)(p.n_pad / 128) * p.kv_units;
            lcsf::kernel<KV><<<(unsigned)(tasks_kv < p.num_sms ? tasks_kv : p.num_sms), KV::kThreads,
                               KV::kSmemBytes, stream>>>(p);
        }
        int e = (int)cudaGetLastError();
        if (e) return e;
        ++*launches;
        if (p.kv_split > 1) {
            const int hkv = p.heads / p.group;
            const int units = hkv * batches;
            const int64_t work = (int64_t)units * p.n * (D / 8);
            const int64_t cap = (int64_t)p.num_sms * 8;
            dkv_reduce_kernel<D><<<(unsigned)((work + 255) / 256 < cap ? (work + 255) / 256 : cap), 256, 0, stream>>>(
                p.dkv_part, p.kv_split, units, p.n, p.n_pad, hkv, reinterpret_cast<__nv_bfloat16*>(p.dv),
                reinterpret_cast<__nv_bfloat16*>(p.dk), p.kv_sb, p.kv_sh, p.kv_sn, p.scale);
            if ((e = (int)cudaGetLastError())) return e;
            ++*launches;
        }
    }
    if (phases & 4) {
        const int64_t tasks = (int64_t)p.bh * (p.n_pad / 128);
        lcsf::kernel<DQ><<<(unsigned)(tasks < p.num_sms ? tasks : p.num_sms), DQ::kThreads, DQ::kSmemBytes,
                           stream>>>(p);
        int e = (int)cudaGetLastError();
        if (e) return e;
        ++*launches;
    }
    return 0;
}

template <int D>
int launch_all(bool causal, const BwdParams& p, int batches, const void* o, const void* dout, const float* lse,
               float* lse2, float* delta, int64_t sb, int64_t sh, int64_t sn, cudaStream_t stream, int phases,
               int* launches) {
    *launches = 0;
    if (phases & 1) {
        constexpr int kRowsPerBlock = 256 / (D / 8) * kPrepRows;
        const int row_blocks = (p.n_pad + kRowsPerBlock - 1) / kRowsPerBlock;
        const int64_t total = (int64_t)row_blocks * batches * p.heads;
        const int64_t cap = (int64_t)p.num_sms * 16;  // 16 x 256 threads per SM in flight
        bwd_prep_kernel<D><<<(unsigned)(total < cap ? total : cap), 256, 0, stream>>>(
            reinterpret_cast<const __nv_bfloat16*>(o), reinterpret_cast<const __nv_bfloat16*>(dout), lse, lse2, delta,
            p.cu_seqlens, p.heads, p.n, p.n_pad, row_blocks, total, sb, sh, sn);
        int e = (int)cudaGetLastError();
        if (e) return e;
        ++*launches;
    }
    return causal ? launch_main<D, true>(p, batches, stream, phases, launches)
                  : launch_main<D, false>(p, batches, stream, phases, launches);
}

}  // namespace bwd

int launch_attn_bwd(int head_dim, bool causal, const BwdParams& p, int batches, const void* o, const void* dout,
                    const float* lse, float* lse2, float* delta, int64_t sb, int64_t sh, int64_t sn,
                    cudaStream_t stream, int phases, int* launches) {
    if (head_dim == 128)
        return bwd::launch_all<128>(causal, p, batches, o, dout, lse, lse2, delta, sb, sh, sn, stream, phases,
                                    launches);
    return bwd::launch_all<64>(causal, p, batches, o, dout, lse, lse2, delta, sb, sh, sn, stream, phases,
                               launches);
}

}  // namespace tkb
