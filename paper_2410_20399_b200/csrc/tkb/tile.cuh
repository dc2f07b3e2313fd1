// tile.cuh — the ThunderKittens tile vocabulary (rt / st / tt / gl and the tile ops),
// re-based on Blackwell.
//
// Reference (kittensim, /root/reference/proj/include/kittensim/tiles.hpp) models the
// paper's tiles on the CPU:
//   Tile (register tile, rt)          tiles.hpp:50-70   -> rt_fl<N> / rt_bf<N>: the row
//        fragment one thread owns after tcgen05.ld (thread = TMEM lane = tile row)
//   SharedTileHandle (st)             tiles.hpp:119-160 -> st_bf<R, C>: SW128-swizzled SMEM
//        tile, stored as C/64 column atoms of R x 128 B (layouts.hpp:111-132 at a 128-B pitch)
//   GlobalTensor (gl)                 tiles.hpp:93-114  -> gl: a 4-D TMA descriptor over
//        [B, H, N, D] with a {64, 128, 1, 1} box
//   (new) tt<T, C>                    the TMEM accumulator tile: 128 lanes x C 32-bit columns
//   TileVector (col_vec)              tiles.hpp:74-89   -> one float per thread (its row)
// and the ops of tiles.hpp:188-362 keep their names:
//   mma_ABt / mm_ABt  (tiles.hpp:348-349) -> tcgen05.mma, A and B both K-major in SMEM
//   mma_AB  / mm_AB   (tiles.hpp:350-352) -> tcgen05.mma, A from TMEM, B MN-major in SMEM
//                                            (swap_layout, tiles.hpp:358-362, is the B-major bit)
//   row_max / row_sum (tiles.hpp:290-309) -> accumulating per-thread reductions
//   exp2 / sub_row / mul_row / div_row    -> packed f32x2 FMA-pipe + MUFU element ops
//   load / store      (tiles.hpp:392-459) -> TMA (gl <-> st), tcgen05.ld/st (tt <-> rt)
#pragma once
#include <cuda.h>

#include "tcgen05.cuh"
#include "tma.cuh"

namespace tkb {

// ------------------------------------------------------------------------------ gl
// A [B, H, N, D] bf16 tensor in HBM seen through a 4-D CUtensorMap {D, N, H, B}
// with a {64, 128, 1, 1} box and SWIZZLE_128B (host/tmap.hpp builds it).
struct gl {
    const CUtensorMap* tm;
    TKB_DEVICE void prefetch() const { tma::prefetch_desc(tm); }
};

// ------------------------------------------------------------------------------ st
// R x C bf16 shared tile, SW128: C/64 atoms of R rows x 128 B; 16-byte chunk c of row r
// sits at chunk c ^ (r % 8) (layouts.hpp:111-132 at a 128-B row pitch).
template <int R, int C>
struct st_bf {
    static_assert(C % 64 == 0 && R % 8 == 0, "st_bf: 64-column atoms, 8-row swizzle groups");
    static constexpr int kRows = R;
    static constexpr int kCols = C;
    static constexpr int kAtoms = C / 64;
    static constexpr int kAtomBytes = R * 128;
    static constexpr int kBytes = R * C * 2;
    uint8_t* ptr;
    TKB_DEVICE uint8_t* atom(int a) const { return ptr + a * kAtomBytes; }
    TKB_DEVICE uint32_t addr() const { return smem_u32(ptr); }
    // address of 16-byte chunk `c` (0 .. C/8-1) of row `r`
    TKB_DEVICE uint8_t* chunk(int r, int c) const {
        return ptr + (c >> 3) * kAtomBytes + r * 128 + (((c & 7) ^ (r & 7)) << 4);
    }
};

// ------------------------------------------------------------------------------ tt
// TMEM tile: 128 lanes x C 32-bit columns starting at column `col` of the CTA's allocation.
// A warp addresses only its lane quarter (warp % 4); `quarter()` folds that in.
template <typename T, int C>
struct tt {
    uint32_t addr;  // lane 0, first column
    TKB_DEVICE uint32_t quarter(int wq) const { return addr + ((uint32_t)(wq * 32) << 16); }
    template <int C2>
    TKB_DEVICE tt<T, C2> sub(int col) const { return tt<T, C2>{addr + (uint32_t)col}; }
};
template <int C>
using tt_fl = tt<float, C>;  // fp32 accumulators
template <int C>
using tt_bf = tt<uint32_t, C>;  // bf16 pairs: C columns hold 2C bf16 (a TS-MMA A operand)

// ------------------------------------------------------------------------------ rt
// The row fragment one thread holds (thread = TMEM lane = tile row).
template <int N>
struct rt_fl {
    float v[N];
};
template <int N>
struct rt_bf {
    static_assert(N % 2 == 0, "bf16 pairs");
    uint32_t v[N / 2];
};

// ============================================================================== ops

// ---- load / store: gl <-> st (TMA), the LCSF load/store stages (tiles.hpp:416-459)
template <int R, int C>
TKB_DEVICE void load_async(const st_bf<R, C>& dst, const gl& src, mbarrier* bar, int row, int head, int batch,
                           uint64_t policy) {
    static_assert(R == 128, "TMA box is 128 rows");
#pragma unroll
    for (int a = 0; a < st_bf<R, C>::kAtoms; ++a) tma::load_4d(dst.atom(a), src.tm, bar, a * 64, row, head, batch, policy);
}
template <int R, int C>
TKB_DEVICE void store_async(const gl& dst, const st_bf<R, C>& src, int row, int head, int batch) {
    static_assert(R == 128, "TMA box is 128 rows");
#pragma unroll
    for (int a = 0; a < st_bf<R, C>::kAtoms; ++a) tma::store_4d(dst.tm, src.atom(a), a * 64, row, head, batch);
}

// ---- load / store: tt <-> rt (tcgen05.ld / st, warp-collective over the lane quarter)
template <int N>
TKB_DEVICE void load(rt_fl<N>& dst, uint32_t taddr) {
    static_assert(N == 32 || N == 64 || N == 128, "x32/x64/x128");
    if constexpr (N == 128) {  // two x64 loads: no single instruction needs > 128 registers
        tmem::ld_32x32b_x64(taddr, reinterpret_cast<uint32_t*>(dst.v));
        tmem::ld_32x32b_x64(taddr + 64, reinterpret_cast<uint32_t*>(dst.v) + 64);
    }
    if constexpr (N == 64) tmem::ld_32x32b_x64(taddr, reinterpret_cast<uint32_t*>(dst.v));
    if constexpr (N == 32) tmem::ld_32x32b_x32(taddr, reinterpret_cast<uint32_t*>(dst.v));
}
template <int N>
TKB_DEVICE void load_wait(rt_fl<N>& dst) {
    if constexpr (N == 128) {
        tmem::wait_ld_x64(reinterpret_cast<uint32_t*>(dst.v));
        tmem::wait_ld_x64(reinterpret_cast<uint32_t*>(dst.v) + 64);
    }
    if constexpr (N == 64) tmem::wait_ld_x64(reinterpret_cast<uint32_t*>(dst.v));
    if constexpr (N == 32) tmem::wait_ld_x32(reinterpret_cast<uint32_t*>(dst.v));
}
template <int N>
TKB_DEVICE void store(uint32_t taddr, const rt_bf<N>& src) {
    static_assert(N == 128 || N == 64, "x64/x32 pairs");
    if constexpr (N == 128) tmem::st_32x32b_x64(taddr, src.v);
    if constexpr (N == 64) tmem::st_32x32b_x32(taddr, src.v);
}

// ---- MMA (tcgen05; called by the whole converged MMA warp, one elected lane issues;
//      D accumulates in TMEM)
// D[M x N] (+)= A[M x K] B[N x K]^T, A and B K-major SW128 SMEM tiles (mma_ABt, tiles.hpp:348-349)
template <int M, int N, int K>
TKB_DEVICE void mma_ABt(const tt_fl<N>& d, const st_bf<M, K>& a, const st_bf<N, K>& b, bool accumulate) {
    constexpr uint32_t idesc = umma::idesc_bf16<M, N, false, false>();
    constexpr uint32_t hi = umma::desc_hi_sw128(1024);
    const uint32_t aa = a.addr(), bb = b.addr();
#pragma unroll
    for (int k = 0; k < K / 16; ++k) {
        const uint32_t off = (k / 4) * st_bf<M, K>::kAtomBytes + (k % 4) * 32;
        const uint32_t offb = (k / 4) * st_bf<N, K>::kAtomBytes + (k % 4) * 32;
        umma::mma_ss_e(d.addr, umma::desc_lo(aa + off, 16), hi, umma::desc_lo(bb + offb, 16), hi, idesc,
                       (accumulate || k > 0) ? 1u : 0u);
    }
}
template <int M, int N, int K>
TKB_DEVICE void mm_ABt(const tt_fl<N>& d, const st_bf<M, K>& a, const st_bf<N, K>& b) {
    mma_ABt(d, a, b, false);
}

// D[128 x N] (+)= A[128 x K] B[K x N]: A bf16 pairs in TMEM (K/2 columns), B [K rows][N]
// row-major SW128 SMEM tile read MN-major (mma_AB with B viewed ColMajor, tiles.hpp:350-352)
template <int N, int K>
TKB_DEVICE void mma_AB(const tt_fl<N>& d, const tt_bf<K / 2>& a, const st_bf<K, N>& b, bool accumulate) {
    constexpr uint32_t idesc = umma::idesc_bf16<128, N, false, true>();
    constexpr uint32_t hi = umma::desc_hi_sw128(1024);
    const uint32_t bb = b.addr();
#pragma unroll
    for (int k = 0; k < K / 16; ++k)
        umma::mma_ts_e(d.addr, a.addr + k * 8, umma::desc_lo(bb + k * 16 * 128, st_bf<K, N>::kAtomBytes), hi,
                       idesc, (accumulate || k > 0) ? 1u : 0u);
}
// Partial-K form: D (+)= A[:, k0 : k0+KC] B[k0 : k0+KC, :] with A's KC/2 columns in TMEM
// (a chunk of a larger P) and B the full [K rows][N] tile (rows k0 .. k0+KC-1 used).
template <int N, int KC, int K>
TKB_DEVICE void mma_AB_k(const tt_fl<N>& d, const tt_bf<KC / 2>& a, const st_bf<K, N>& b, int k0, bool accumulate) {
    constexpr uint32_t idesc = umma::idesc_bf16<128, N, false, true>();
    constexpr uint32_t hi = umma::desc_hi_sw128(1024);
    const uint32_t bb = b.addr() + k0 * 128;
#pragma unroll
    for (int k = 0; k < KC / 16; ++k)
        umma::mma_ts_e(d.addr, a.addr + k * 8, umma::desc_lo(bb + k * 16 * 128, st_bf<K, N>::kAtomBytes), hi, idesc,
                       (accumulate || k > 0) ? 1u : 0u);
}
template <int N, int K>
TKB_DEVICE void mm_AB(const tt_fl<N>& d, const tt_bf<K / 2>& a, const st_bf<K, N>& b) {
    mma_AB(d, a, b, false);
}

// ---- row reductions over a thread's row fragment (accumulating forms, tiles.hpp:290-309)
template <int N>
TKB_DEVICE void row_max(float& m, const rt_fl<N>& x) {
    // three-input FMNMX3 (sm_100): two elements per instruction, four independent chains
    float acc[4] = {x.v[0], x.v[1], x.v[2], x.v[3]};
    int j = 4;
#pragma unroll
    for (; j + 8 <= N; j += 8) {
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[k] = fmax3(acc[k], x.v[j + 2 * k], x.v[j + 2 * k + 1]);
    }
#pragma unroll
    for (; j < N; ++j) acc[j & 3] = fmaxf(acc[j & 3], x.v[j]);
    m = fmax3(m, fmax3(acc[0], acc[1], acc[2]), acc[3]);
}
template <int N>
TKB_DEVICE void row_sum(float& l, const rt_fl<N>& x) {
    float2 acc[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
#pragma unroll
    for (int j = 0; j < N; j += 8) {
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] = add2(acc[q], make_float2(x.v[j + 2 * q], x.v[j + 2 * q + 1]));
    }
    l += ((acc[0].x + acc[0].y) + (acc[1].x + acc[1].y)) + ((acc[2].x + acc[2].y) + (acc[3].x + acc[3].y));
}

// ---- element ops on row fragments (tiles.hpp:217-287)
template <int N>
TKB_DEVICE void mul(rt_fl<N>& x, float s) {  // x *= s  (tiles.hpp:220-227)
#pragma unroll
    for (int j = 0; j < N; j += 2) {
        const float2 r = mul2(make_float2(x.v[j], x.v[j + 1]), make_float2(s, s));
        x.v[j] = r.x;
        x.v[j + 1] = r.y;
    }
}
template <int N>
TKB_DEVICE void sub_row(rt_fl<N>& x, float m) {  // x -= m (row broadcast, tiles.hpp:270-275)
#pragma unroll
    for (int j = 0; j < N; j += 2) {
        const float2 r = sub2(make_float2(x.v[j], x.v[j + 1]), make_float2(m, m));
        x.v[j] = r.x;
        x.v[j + 1] = r.y;
    }
}
template <int N>
TKB_DEVICE void mul_row(rt_fl<N>& x, float s) {  // tiles.hpp:282-287
    mul(x, s);
}
template <int N>
TKB_DEVICE void div_row(rt_fl<N>& x, float l) {  // tiles.hpp:276-281
    mul(x, 1.f / l);
}
template <int N>
TKB_DEVICE void exp2(rt_fl<N>& x) {  // tiles.hpp:217-219 (MUFU ex2)
#pragma unroll
    for (int j = 0; j < N; ++j) x.v[j] = ex2_approx(x.v[j]);
}
// bf16 RNE copy (copy(att_mma, att), tiles.hpp:195-200; round_to_bf16 tiles.hpp:40-46)
template <int N>
TKB_DEVICE void copy(rt_bf<N>& dst, const rt_fl<N>& src) {
#pragma unroll
    for (int j = 0; j < N; j += 2) dst.v[j / 2] = pack_bf16x2(src.v[j], src.v[j + 1]);
}
template <int N>
TKB_DEVICE void zero(rt_fl<N>& x) {
#pragma unroll
    for (int j = 0; j < N; ++j) x.v[j] = 0.f;
}
template <int N>
TKB_DEVICE void neg_infty(rt_fl<N>& x) {
#pragma unroll
    for (int j = 0; j < N; ++j) x.v[j] = -INFINITY;
}

}  // namespace tkb
