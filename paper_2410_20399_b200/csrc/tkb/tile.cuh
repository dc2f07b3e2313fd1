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
//   mma_AB  / mm_AB   (tiles.hpp:350-352) -> tcgen05.mma, A K-major in SMEM or in TMEM, B MN-major
//                                            in SMEM: B = swap_layout(st) (tiles.hpp:358-362), the
//                                            same SMEM read through the B-major bit (st_mn view)
//   row_max / row_sum (tiles.hpp:290-309) -> accumulating per-thread reductions
//   exp2 / sub_row / mul_row / div_row    -> packed f32x2 FMA-pipe + MUFU element ops
//   load / store      (tiles.hpp:392-459) -> every flavour of the reference:
//        global <-> shared    load_async / store_async (TMA, gl)
//        global <-> register  load / store on a gv (plain pointer view), 16-byte accesses
//        shared <-> register  load / store of a thread's row fragment of an st_bf (swizzled)
//        TMEM   <-> register  load / store (tcgen05.ld / st of the thread's TMEM lane)
//   mma_commit                            -> tcgen05.commit: an mbarrier arrives when the MMAs
//                                            issued so far have retired (the LCSF hand-off)
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "cluster.cuh"
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

// ------------------------------------------------------------------------------ gv
// The same [B, H, N, D] tensor seen through a plain pointer and element strides, for the
// register <-> global transfers (GlobalTensor::index, tiles.hpp:106-108).
template <typename T>
struct gv {
    T* ptr;
    int64_t sb, sh, sn;
    TKB_DEVICE T* row(int64_t b, int64_t h, int64_t n) const { return ptr + b * sb + h * sh + n * sn; }
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

// The same SMEM tile read MN-major — what the reference calls a ColMajor tile: a B operand
// [K rows][N] stored row-major (N contiguous) is consumed as B^T's K-major transpose through
// the instruction descriptor's B-major bit, with no data movement.
template <int R, int C>
struct st_mn {
    st_bf<R, C> t;
    TKB_DEVICE uint32_t addr() const { return t.addr(); }
};
// swap_layout (tiles.hpp:358-362): same logical matrix, opposite major flag; an involution
template <int R, int C>
TKB_DEVICE st_mn<R, C> swap_layout(const st_bf<R, C>& t) {
    return st_mn<R, C>{t};
}
template <int R, int C>
TKB_DEVICE st_bf<R, C> swap_layout(const st_mn<R, C>& t) {
    return t.t;
}

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
// col0: first column of the tile in the tensor (a multiple of 64) when the tile is narrower
template <int R, int C>
TKB_DEVICE void store_async(const gl& dst, const st_bf<R, C>& src, int row, int head, int batch, int col0 = 0) {
    static_assert(R == 128, "TMA box is 128 rows");
#pragma unroll
    for (int a = 0; a < st_bf<R, C>::kAtoms; ++a)
        tma::store_4d(dst.tm, src.atom(a), col0 + a * 64, row, head, batch);
}

// ---- load / store: tt <-> rt (tcgen05.ld / st, warp-collective over the lane quarter)
template <int N>
TKB_DEVICE void load(rt_fl<N>& dst, uint32_t taddr) {
    static_assert(N == 16 || N == 32 || N == 64 || N == 128, "x16/x32/x64/x128");
    if constexpr (N == 128) {  // two x64 loads: no single instruction needs > 128 registers
        tmem::ld_32x32b_x64(taddr, reinterpret_cast<uint32_t*>(dst.v));
        tmem::ld_32x32b_x64(taddr + 64, reinterpret_cast<uint32_t*>(dst.v) + 64);
    }
    if constexpr (N == 64) tmem::ld_32x32b_x64(taddr, reinterpret_cast<uint32_t*>(dst.v));
    if constexpr (N == 32) tmem::ld_32x32b_x32(taddr, reinterpret_cast<uint32_t*>(dst.v));
    if constexpr (N == 16) tmem::ld_32x32b_x16(taddr, reinterpret_cast<uint32_t*>(dst.v));
}
template <int N>
TKB_DEVICE void load_wait(rt_fl<N>& dst) {
    if constexpr (N == 128) {
        tmem::wait_ld_x64(reinterpret_cast<uint32_t*>(dst.v));
        tmem::wait_ld_x64(reinterpret_cast<uint32_t*>(dst.v) + 64);
    }
    if constexpr (N == 64) tmem::wait_ld_x64(reinterpret_cast<uint32_t*>(dst.v));
    if constexpr (N == 32) tmem::wait_ld_x32(reinterpret_cast<uint32_t*>(dst.v));
    if constexpr (N == 16) tmem::wait_ld_x16(reinterpret_cast<uint32_t*>(dst.v));
}
// fp32 -> TMEM (N columns), e.g. a rescaled accumulator
template <int N>
TKB_DEVICE void store(uint32_t taddr, const rt_fl<N>& src) {
    static_assert(N == 32 || N == 16, "x32/x16");
    if constexpr (N == 32) tmem::st_32x32b_x32(taddr, reinterpret_cast<const uint32_t*>(src.v));
    if constexpr (N == 16) tmem::st_32x32b_x16(taddr, reinterpret_cast<const uint32_t*>(src.v));
}
// bf16 pairs -> TMEM (N/2 columns), e.g. a TS-MMA A operand or P over S
template <int N>
TKB_DEVICE void store(uint32_t taddr, const rt_bf<N>& src) {
    static_assert(N == 128 || N == 64 || N == 32 || N == 16, "x64/x32/x16/x8 pairs");
    if constexpr (N == 128) tmem::st_32x32b_x64(taddr, src.v);
    if constexpr (N == 64) tmem::st_32x32b_x32(taddr, src.v);
    if constexpr (N == 32) tmem::st_32x32b_x16(taddr, src.v);
    if constexpr (N == 16) tmem::st_32x32b_x8(taddr, src.v);
}

// ---- shared <-> register: a thread's row fragment (tiles.hpp:441-459). N bf16 of row `row`
//      starting at column col0 (a multiple of 8), one 16-byte swizzled chunk per 8 values.
template <int N, int R, int C>
TKB_DEVICE void load(rt_bf<N>& dst, const st_bf<R, C>& src, int row, int col0) {
    static_assert(N % 8 == 0, "16-byte chunks");
#pragma unroll
    for (int q = 0; q < N / 8; ++q) {
        const uint4 u = *reinterpret_cast<const uint4*>(src.chunk(row, col0 / 8 + q));
        dst.v[4 * q] = u.x, dst.v[4 * q + 1] = u.y, dst.v[4 * q + 2] = u.z, dst.v[4 * q + 3] = u.w;
    }
}
template <int N, int R, int C>
TKB_DEVICE void store(const st_bf<R, C>& dst, const rt_bf<N>& src, int row, int col0) {
    static_assert(N % 8 == 0, "16-byte chunks");
#pragma unroll
    for (int q = 0; q < N / 8; ++q)
        *reinterpret_cast<uint4*>(dst.chunk(row, col0 / 8 + q)) =
            make_uint4(src.v[4 * q], src.v[4 * q + 1], src.v[4 * q + 2], src.v[4 * q + 3]);
}

// ---- global <-> register: a row fragment of a gv (tiles.hpp:392-413), 16-byte accesses
template <int N>
TKB_DEVICE void load(rt_bf<N>& dst, const gv<const __nv_bfloat16>& src, int64_t b, int64_t h, int64_t n, int col0) {
    const uint4* p = reinterpret_cast<const uint4*>(src.row(b, h, n) + col0);
#pragma unroll
    for (int q = 0; q < N / 8; ++q) {
        const uint4 u = __ldg(p + q);
        dst.v[4 * q] = u.x, dst.v[4 * q + 1] = u.y, dst.v[4 * q + 2] = u.z, dst.v[4 * q + 3] = u.w;
    }
}
template <int N>
TKB_DEVICE void store(const gv<__nv_bfloat16>& dst, const rt_bf<N>& src, int64_t b, int64_t h, int64_t n, int col0) {
    uint4* p = reinterpret_cast<uint4*>(dst.row(b, h, n) + col0);
#pragma unroll
    for (int q = 0; q < N / 8; ++q) p[q] = make_uint4(src.v[4 * q], src.v[4 * q + 1], src.v[4 * q + 2], src.v[4 * q + 3]);
}

// Warp-collective register -> global store of 32 rows: lane l holds N bf16 of row row0 + l
// (columns col0 ..). Stored as is, every 16-byte store instruction of the warp would touch
// 32 rows = 32 L2 lines; the fragments are first transposed through shuffles so that one
// instruction writes N * 2 contiguous bytes of 32 / (N / 8) rows (4x fewer lines at N = 32).
// Rows >= rows_valid are skipped.
template <int N>
TKB_DEVICE void store_rows(const gv<__nv_bfloat16>& dst, const rt_bf<N>& src, int64_t b, int64_t h, int row0,
                           int col0, int rows_valid) {
    constexpr int kCh = N / 8;      // 16-byte chunks per row segment
    constexpr int kRpi = 32 / kCh;  // rows per store instruction
    const int lane = laneid();
    const int c = lane % kCh;
#pragma unroll
    for (int k = 0; k < kCh; ++k) {
        const int srow = k * kRpi + lane / kCh;  // the row this lane writes now
        uint32_t out[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            out[j] = 0;
#pragma unroll
            for (int cc = 0; cc < kCh; ++cc) {
                const uint32_t t = __shfl_sync(0xffffffffu, src.v[4 * cc + j], srow);
                out[j] = (cc == c) ? t : out[j];
            }
        }
        if (srow < rows_valid)
            st_global_v4(dst.row(b, h, row0 + srow) + col0 + 8 * c, make_uint4(out[0], out[1], out[2], out[3]));
    }
}

// ---- MMA (tcgen05; called by the whole converged MMA warp, one elected lane issues;
//      D accumulates in TMEM). K-steps of 16; an SW128 atom holds 64 K-columns (4 steps).
namespace detail {
template <int R, int C>
TKB_DEVICE uint32_t kmajor_step(const st_bf<R, C>& t, int k) {  // K-major operand, K-step k
    return t.addr() + (k / 4) * st_bf<R, C>::kAtomBytes + (k % 4) * 32;
}
template <int R, int C>
TKB_DEVICE uint32_t mnmajor_step(const st_mn<R, C>& t, int k) {  // MN-major operand, rows k*16 ..
    return t.addr() + k * 16 * 128;
}
}  // namespace detail

// D[M x N] (+)= A[M x K] B[N x K]^T, A and B K-major SW128 SMEM tiles (mma_ABt, tiles.hpp:348-349)
template <int M, int N, int K>
TKB_DEVICE void mma_ABt(const tt_fl<N>& d, const st_bf<M, K>& a, const st_bf<N, K>& b, bool accumulate) {
    constexpr uint32_t idesc = umma::idesc_bf16<M, N, false, false>();
    constexpr uint32_t hi = umma::desc_hi_sw128(1024);
#pragma unroll
    for (int k = 0; k < K / 16; ++k)
        umma::mma_ss_e(d.addr, umma::desc_lo(detail::kmajor_step(a, k), 16), hi,
                       umma::desc_lo(detail::kmajor_step(b, k), 16), hi, idesc, (accumulate || k > 0) ? 1u : 0u);
}
template <int M, int N, int K>
TKB_DEVICE void mm_ABt(const tt_fl<N>& d, const st_bf<M, K>& a, const st_bf<N, K>& b) {
    mma_ABt(d, a, b, false);
}
// D[128 x N] (+)= A[128 x K] B[N x K]^T with A = bf16 pairs in TMEM (K/2 columns), B K-major SMEM
template <int N, int K>
TKB_DEVICE void mma_ABt(const tt_fl<N>& d, const tt_bf<K / 2>& a, const st_bf<N, K>& b, bool accumulate) {
    constexpr uint32_t idesc = umma::idesc_bf16<128, N, false, false>();
    constexpr uint32_t hi = umma::desc_hi_sw128(1024);
#pragma unroll
    for (int k = 0; k < K / 16; ++k)
        umma::mma_ts_e(d.addr, a.addr + k * 8, umma::desc_lo(detail::kmajor_step(b, k), 16), hi, idesc,
                       (accumulate || k > 0) ? 1u : 0u);
}
template <int N, int K>
TKB_DEVICE void mm_ABt(const tt_fl<N>& d, const tt_bf<K / 2>& a, const st_bf<N, K>& b) {
    mma_ABt(d, a, b, false);
}

// D[128 x N] (+)= A[128 x K] B[K x N]: A K-major SMEM, B = swap_layout of a [K rows][N] tile
// (mma_AB with B viewed ColMajor, tiles.hpp:350-352)
template <int N, int K>
TKB_DEVICE void mma_AB(const tt_fl<N>& d, const st_bf<128, K>& a, const st_mn<K, N>& b, bool accumulate) {
    constexpr uint32_t idesc = umma::idesc_bf16<128, N, false, true>();
    constexpr uint32_t hi = umma::desc_hi_sw128(1024);
#pragma unroll
    for (int k = 0; k < K / 16; ++k)
        umma::mma_ss_e(d.addr, umma::desc_lo(detail::kmajor_step(a, k), 16), hi,
                       umma::desc_lo(detail::mnmajor_step(b, k), st_bf<K, N>::kAtomBytes), hi, idesc,
                       (accumulate || k > 0) ? 1u : 0u);
}
// ... with A = bf16 pairs in TMEM (K/2 columns)
template <int N, int K>
TKB_DEVICE void mma_AB(const tt_fl<N>& d, const tt_bf<K / 2>& a, const st_mn<K, N>& b, bool accumulate) {
    constexpr uint32_t idesc = umma::idesc_bf16<128, N, false, true>();
    constexpr uint32_t hi = umma::desc_hi_sw128(1024);
#pragma unroll
    for (int k = 0; k < K / 16; ++k)
        umma::mma_ts_e(d.addr, a.addr + k * 8, umma::desc_lo(detail::mnmajor_step(b, k), st_bf<K, N>::kAtomBytes), hi,
                       idesc, (accumulate || k > 0) ? 1u : 0u);
}
template <int N, int K>
TKB_DEVICE void mm_AB(const tt_fl<N>& d, const st_bf<128, K>& a, const st_mn<K, N>& b) {
    mma_AB(d, a, b, false);
}
template <int N, int K>
TKB_DEVICE void mm_AB(const tt_fl<N>& d, const tt_bf<K / 2>& a, const st_mn<K, N>& b) {
    mma_AB(d, a, b, false);
}
// Partial-K form: D (+)= A[:, k0 : k0+KC] B[k0 : k0+KC, :] with A's KC/2 columns in TMEM
// (a chunk of a larger P) and B the full [K rows][N] tile (rows k0 .. k0+KC-1 used).
template <int N, int KC, int K>
TKB_DEVICE void mma_AB_k(const tt_fl<N>& d, const tt_bf<KC / 2>& a, const st_mn<K, N>& b, int k0, bool accumulate) {
    constexpr uint32_t idesc = umma::idesc_bf16<128, N, false, true>();
    constexpr uint32_t hi = umma::desc_hi_sw128(1024);
#pragma unroll
    for (int k = 0; k < KC / 16; ++k)
        umma::mma_ts_e(d.addr, a.addr + k * 8,
                       umma::desc_lo(detail::mnmajor_step(b, k0 / 16 + k), st_bf<K, N>::kAtomBytes), hi, idesc,
                       (accumulate || k > 0) ? 1u : 0u);
}
// Grouped-A form for K = 128: A is bf16 in TMEM as 4 chunks of 32 K-values, chunk g in the
// 16 packed columns [32 g, 32 g + 16) of a (each written by compute column group g); chunk g
// is issued as soon as wait_chunk(g) returns, so the GEMM starts while later chunks are
// still being produced.
template <int N, class WaitChunk>
TKB_DEVICE void mma_AB_groups(const tt_fl<N>& d, const tt_bf<128>& a, const st_mn<128, N>& b, bool accumulate,
                              WaitChunk&& wait_chunk) {
    constexpr uint32_t idesc = umma::idesc_bf16<128, N, false, true>();
    constexpr uint32_t hi = umma::desc_hi_sw128(1024);
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        wait_chunk(g);
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
            const int k = 2 * g + kk;
            umma::mma_ts_e(d.addr, a.addr + 32 * g + 8 * kk,
                           umma::desc_lo(detail::mnmajor_step(b, k), st_bf<128, N>::kAtomBytes), hi, idesc,
                           (accumulate || k > 0) ? 1u : 0u);
        }
    }
}

// tcgen05.commit: `bar` gets one arrival when every MMA this thread issued so far retired
// (warp-converged; the elected lane commits)
TKB_DEVICE void mma_commit(mbarrier* bar) { umma::commit_e(bar); }

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

// ---- CTA-pair MMAs (tcgen05 cta_group::2, M = 256 over a 2-CTA cluster; the leader's
//      MMA warp issues for both CTAs, each CTA holding its 128 rows of A and half of B)
namespace pair {
// D[256 x N] (+)= A[256 x K] B[N x K]^T: this CTA's A rows and its N/2 rows of B, both K-major
template <int N, int K>
TKB_DEVICE void mma_ABt(const tt_fl<N>& d, const st_bf<128, K>& a, const st_bf<N / 2, K>& b_half, bool accumulate) {
    constexpr uint32_t idesc = umma::idesc_bf16_m256<N, false, false>();
    constexpr uint32_t hi = umma::desc_hi_sw128(1024);
#pragma unroll
    for (int k = 0; k < K / 16; ++k)
        umma::mma2_ss_e(d.addr, umma::desc_lo(detail::kmajor_step(a, k), 16), hi,
                        umma::desc_lo(detail::kmajor_step(b_half, k), 16), hi, idesc, (accumulate || k > 0) ? 1u : 0u);
}
template <int N, int K>
TKB_DEVICE void mm_ABt(const tt_fl<N>& d, const st_bf<128, K>& a, const st_bf<N / 2, K>& b_half) {
    mma_ABt(d, a, b_half, false);
}
// the grouped-A mma_AB over the pair: B = this CTA's N/2 columns of a [128 K rows][N] operand
template <int N, class WaitChunk>
TKB_DEVICE void mma_AB_groups(const tt_fl<N>& d, const tt_bf<128>& a, const st_mn<128, N / 2>& b_half,
                              bool accumulate, WaitChunk&& wait_chunk) {
    constexpr uint32_t idesc = umma::idesc_bf16_m256<N, false, true>();
    constexpr uint32_t hi = umma::desc_hi_sw128(1024);
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        wait_chunk(g);
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
            const int k = 2 * g + kk;
            umma::mma2_ts_e(d.addr, a.addr + 32 * g + 8 * kk,
                            umma::desc_lo(detail::mnmajor_step(b_half, k), st_bf<128, N / 2>::kAtomBytes), hi, idesc,
                            (accumulate || k > 0) ? 1u : 0u);
        }
    }
}
// commit to the same-offset barrier in both CTAs (multicast)
TKB_DEVICE void mma_commit(mbarrier* bar) { umma::commit2_e(bar); }
}  // namespace pair

}  // namespace tkb
