// cluster.cuh — CTA pairs (cta_group::2): two SMs of one TPC run one tcgen05.mma with
// M = 256, each CTA holding half of A (its 128 rows, also its half of the accumulator in
// its own TMEM) and half of B (N / 2 rows). Per SM the tensor core then reads 4 KB of A and
// 2 KB of B per K = 16 step instead of 4 + 4 KB: the shared-memory port (128 B/clk, also
// fed by the TMA writes) stops being the bound of SS GEMMs with N = 128.
//
// Protocol used by the kernels (leader = cluster rank 0 issues every tcgen05.mma):
//   operand loads   both CTAs TMA into their own SMEM and complete_tx on the LEADER's
//                   full barrier (cp.async.bulk.tensor .cta_group::2); the leader alone
//                   arrives with expect_tx of both halves
//   MMA -> CTAs     tcgen05.commit .multicast::cluster arrives on both CTAs' barrier
//   CTAs -> MMA     one lane per warp arrives on the leader's barrier through the cluster
//                   window (mapa + mbarrier.arrive.release.cluster)
#pragma once
#include "mbarrier.cuh"

namespace tkb {
namespace cluster {

TKB_DEVICE uint32_t ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// All threads of every CTA of the cluster.
TKB_DEVICE void sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Shared::cluster address of `local` in CTA `rank`.
TKB_DEVICE uint32_t map(const void* local, uint32_t rank) {
    uint32_t a;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(local)), "r"(rank));
    return a;
}

TKB_DEVICE void arrive_remote(uint32_t bar_cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster_addr) : "memory");
}

TKB_DEVICE bool try_wait(mbarrier* b, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}

// mbar_wait with cluster-scope acquire (arrivals from the peer CTA / multicast commits);
// same 20 s deadlock trap.
TKB_DEVICE void wait(mbarrier* b, uint32_t parity) {
#ifndef TKB_NO_DEADLOCK_TRAP
    if (try_wait(b, parity)) return;
    uint32_t spins = 0;
    uint64_t t0 = 0;
    while (!try_wait(b, parity)) {
        if ((++spins & 4095u) == 0) {
            const uint64_t now = globaltimer_ns();
            if (t0 == 0)
                t0 = now;
            else if (now - t0 > 20000000000ull)
                __trap();
        }
    }
#else
    while (!try_wait(b, parity)) {
    }
#endif
}

// 4-D tiled load into this CTA's SMEM whose completion is counted on a barrier of either
// CTA of the pair (bar = shared::cluster address).
TKB_DEVICE void load_4d(void* smem_dst, const void* tmap, uint32_t bar, int c0, int c1, int c2, int c3,
                        uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        ".L2::cache_hint [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "l"(policy)
        : "memory");
}

// 2-D variant (GEMM panels)
TKB_DEVICE void load_2d(void* smem_dst, const void* tmap, uint32_t bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
}

}  // namespace cluster

namespace tmem {
// Pair allocation: one warp of EACH CTA executes it; both get the same column base.
template <int kCols>
TKB_DEVICE void alloc2(uint32_t* smem_dst) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <int kCols>
TKB_DEVICE void dealloc2(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}
}  // namespace tmem

namespace umma {

// kind::f16 instruction descriptor for the pair MMA (M = 256; N = the full N of both halves)
template <int N, bool AMajorMN, bool BMajorMN>
TKB_DEVICE constexpr uint32_t idesc_bf16_m256() {
    static_assert(N % 16 == 0 && N >= 32 && N <= 256, "cta_group::2 N");
    return (1u << 4) | (1u << 7) | (1u << 10) | ((AMajorMN ? 1u : 0u) << 15) | ((BMajorMN ? 1u : 0u) << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}

// Warp-converged pair MMAs (leader CTA only; operand addresses are CTA-local and valid in
// both CTAs because their SMEM / TMEM layouts are identical).
TKB_DEVICE void mma2_ss_e(uint32_t d_tmem, uint32_t a_lo, uint32_t a_hi, uint32_t b_lo, uint32_t b_hi,
                          uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 da, db;\n\t"
        "mov.b64 da, {%1, %2};\n\t"
        "mov.b64 db, {%3, %4};\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], da, db, %5, p;\n\t}" ::"r"(d_tmem),
        "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accumulate)
        : "memory");
}
TKB_DEVICE void mma2_ts_e(uint32_t d_tmem, uint32_t a_tmem, uint32_t b_lo, uint32_t b_hi, uint32_t idesc,
                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 db;\n\t"
        "mov.b64 db, {%2, %3};\n\t"
        "setp.ne.b32 p, %5, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], db, %4, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Arrive on `bar` (same CTA-local offset) in both CTAs once the prior pair MMAs finish.
TKB_DEVICE void commit2_e(mbarrier* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::
            "r"(smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}

}  // namespace umma
}  // namespace tkb
