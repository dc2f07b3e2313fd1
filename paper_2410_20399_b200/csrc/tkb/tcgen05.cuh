// tcgen05.cuh — TMEM tiles (tt) and the 5th-generation tensor-core MMA.
//
// Reference mapping (kittensim, /root/reference/proj/include/kittensim):
//   mm_ABt / mma_ABt (tiles.hpp:348-355)  -> umma_ss with both operands K-major
//   mma_AB with V viewed ColMajor          -> umma_ss / umma_ts with B MN-major
//     (swap_layout, tiles.hpp:358-362, becomes the b_major bit of the
//      instruction descriptor: no data movement)
//   fp32 accumulator register tile (Tile, tiles.hpp:50-70) -> TMEM columns
//
// TMEM address: bits [31:16] lane, [15:0] column. A warp can only touch the
// 32-lane quarter (warp_id % 4) of TMEM.
#pragma once
#include "mbarrier.cuh"
#include "tmem_ops_gen.cuh"

namespace tkb {
namespace tmem {

// Warp-collective. Writes the base TMEM address to *smem_dst.
template <int kCols>
TKB_DEVICE void alloc(uint32_t* smem_dst) {
    static_assert(kCols == 32 || kCols == 64 || kCols == 128 || kCols == 256 || kCols == 512, "pow2 >= 32");
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

template <int kCols>
TKB_DEVICE void dealloc(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}

TKB_DEVICE void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
TKB_DEVICE void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
TKB_DEVICE void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
TKB_DEVICE void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

TKB_DEVICE constexpr uint32_t addr(uint32_t base, uint32_t lane, uint32_t col) {
    return base + (lane << 16) + col;
}

}  // namespace tmem

namespace umma {

// Shared-memory matrix descriptor (tcgen05 "version 1" format).
//   [0,14)  start address >> 4       [16,30) leading byte offset >> 4
//   [32,46) stride byte offset >> 4  [46,48) version = 1
//   [49,52) base offset              [52]    lbo mode
//   [61,64) layout: 0 none, 2 SW128, 4 SW64, 6 SW32
TKB_DEVICE uint64_t smem_desc_sw128(uint32_t smem_addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// K-major SW128 tile: rows of 64 bf16 (128 B), 8-row core groups 1024 B apart.
// Column blocks of 64 elements are separate atoms (advance start address).
TKB_DEVICE uint64_t desc_kmajor(uint32_t smem_addr) { return smem_desc_sw128(smem_addr, 16, 1024); }

// MN-major SW128 tile stored [K rows][64 MN elements] per atom; atoms of 64 MN
// elements are `atom_bytes` apart (LBO); 8-row K groups 1024 B apart (SBO).
TKB_DEVICE uint64_t desc_mnmajor(uint32_t smem_addr, uint32_t atom_bytes) {
    return smem_desc_sw128(smem_addr, atom_bytes, 1024);
}

// Instruction descriptor, kind::f16 with bf16 inputs and fp32 accumulation.
//   [4,6) c fmt (1=f32)  [7,10) a fmt (1=bf16)  [10,13) b fmt (1=bf16)
//   [15] a major (1=MN)  [16] b major (1=MN)  [17,23) N>>3  [24,29) M>>4
template <int M, int N, bool AMajorMN, bool BMajorMN>
TKB_DEVICE constexpr uint32_t idesc_bf16() {
    static_assert(M == 64 || M == 128, "cta_group::1 M");
    static_assert(N % 16 == 0 && N >= 16 && N <= 256, "N");
    return (1u << 4) | (1u << 7) | (1u << 10) | ((AMajorMN ? 1u : 0u) << 15) | ((BMajorMN ? 1u : 0u) << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// Split-descriptor forms: lo = start/LBO word (varies per k-step), hi = SBO/version/layout
// word (constant per operand). Keeping the halves apart stops the compiler from hoisting
// dozens of 64-bit descriptors into registers of the (register-starved) MMA warp.
TKB_DEVICE constexpr uint32_t desc_hi_sw128(uint32_t sbo_bytes) {
    return ((sbo_bytes >> 4) & 0x3FFFu) | (1u << 14) | (2u << 29);
}
TKB_DEVICE uint32_t desc_lo(uint32_t smem_addr, uint32_t lbo_bytes) {
    return ((smem_addr >> 4) & 0x3FFFu) | (((lbo_bytes >> 4) & 0x3FFFu) << 16);
}
TKB_DEVICE void mma_ss_split(uint32_t d_tmem, uint32_t a_lo, uint32_t a_hi, uint32_t b_lo, uint32_t b_hi,
                             uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b64 da, db;\n\t"
        "mov.b64 da, {%1, %2};\n\t"
        "mov.b64 db, {%3, %4};\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, p;\n\t}" ::"r"(d_tmem),
        "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accumulate)
        : "memory");
}
TKB_DEVICE void mma_ts_split(uint32_t d_tmem, uint32_t a_tmem, uint32_t b_lo, uint32_t b_hi, uint32_t idesc,
                             uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b64 db;\n\t"
        "mov.b64 db, {%2, %3};\n\t"
        "setp.ne.b32 p, %5, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], db, %4, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accumulate)
        : "memory");
}

// Warp-converged forms: every lane of the MMA warp executes the call with the same
// (warp-uniform) operands and elect.sync picks the one lane that issues. Keeping the
// warp converged lets ptxas hold descriptors in uniform registers: no per-MMA
// R2UR/elect loop, which otherwise costs ~15 issue slots per tcgen05.mma.
TKB_DEVICE void mma_ss_e(uint32_t d_tmem, uint32_t a_lo, uint32_t a_hi, uint32_t b_lo, uint32_t b_hi,
                         uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 da, db;\n\t"
        "mov.b64 da, {%1, %2};\n\t"
        "mov.b64 db, {%3, %4};\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, p;\n\t}" ::"r"(d_tmem),
        "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accumulate)
        : "memory");
}
TKB_DEVICE void mma_ts_e(uint32_t d_tmem, uint32_t a_tmem, uint32_t b_lo, uint32_t b_hi, uint32_t idesc,
                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 db;\n\t"
        "mov.b64 db, {%2, %3};\n\t"
        "setp.ne.b32 p, %5, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], db, %4, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accumulate)
        : "memory");
}

// Make a value opaque to the optimiser (blocks loop-invariant hoisting).
TKB_DEVICE uint32_t opaque(uint32_t x) {
    asm volatile("" : "+r"(x));
    return x;
}

// D[tmem] (+)= A[smem] * B[smem]
TKB_DEVICE void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// D[tmem] (+)= A[tmem] * B[smem]   (A K-major in TMEM: lane = row, 2 bf16 per column)
TKB_DEVICE void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// Arrive on `bar` once all previously issued tcgen05 ops of this thread finish.
TKB_DEVICE void commit(mbarrier* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// Warp-converged commit: one elected lane arrives on `bar` when the prior MMAs finish.
TKB_DEVICE void commit_e(mbarrier* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
        : "memory");
}

}  // namespace umma
}  // namespace tkb
