// selftest_sm100.cu — unit kernels for the tile primitives (TMA SW128 load,
// tcgen05.mma SS/TS with K- and MN-major operands, TMEM ld/st). Each variant
// computes one 128 x N fp32 tile that the tests compare with torch.
//
// These pin the descriptor encodings that fail silently:
//   0: C = A  * B^T  A[128][K] K-major, B[N][K] K-major        (S = Q K^T)
//   1: C = A  * B    A[128][K] K-major, B[K][N] MN-major       (O += P V, SS)
//   2: C = A  * B    A in TMEM (bf16 pairs), B[K][N] MN-major   (O += P V, TS)
//   3: C = A  * B    A stored transposed [K][128] (MN-major), B[K][N] MN-major (dQ = dS K)
//   4: C = A^T * B^T-free check of TMEM st/ld round trip (C = A as fp32)
//   5: C = A  * B^T  A in TMEM (bf16 pairs), B[N][K] K-major        (S = Q K^T, Q in TMEM)
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <string>

#include "host/tmap.hpp"
#include "tkb/tcgen05.cuh"
#include "tkb/lcsf.cuh"
#include "tkb/tile.cuh"
#include "tkb/tma.cuh"

using namespace tkb;

namespace {

constexpr int M = 128;

template <int N, int K, int VARIANT>
__global__ void __launch_bounds__(128, 1)
    selftest_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __nv_bfloat16* __restrict__ A_gmem, float* __restrict__ C, int reps,
                    long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;                 // up to 32 KB
    uint8_t* sB = smem + 32768;         // up to 32 KB
    __shared__ mbarrier bar_load, bar_mma;
    __shared__ uint32_t tmem_base_slot;

    const int warp = warpid();
    const int lane = laneid();
    if (threadIdx.x == 0) {
        mbar_init(&bar_load, 1);
        mbar_init(&bar_mma, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem::alloc<256>(&tmem_base_slot);
    tmem::fence_before();
    __syncthreads();
    tmem::fence_after();
    const uint32_t tbase = tmem_base_slot;
    const uint32_t t_c = tbase;          // C: cols [0, N)
    const uint32_t t_a = tbase + 128;    // A (TS variant): cols [128, 128 + K/2)

    // A rows/cols as loaded: variant 3 stores A^T [K][128]
    constexpr int A_ROWS = (VARIANT == 3) ? K : M;
    constexpr int A_COLS = (VARIANT == 3) ? M : K;
    constexpr int B_ROWS = (VARIANT == 0 || VARIANT == 5) ? N : K;
    constexpr int B_COLS = (VARIANT == 0 || VARIANT == 5) ? K : N;

    if (threadIdx.x == 0) {
        uint32_t bytes = B_ROWS * B_COLS * 2;
        if (VARIANT != 2 && VARIANT != 5) bytes += A_ROWS * A_COLS * 2;
        mbar_arrive_expect_tx(&bar_load, bytes);
        if (VARIANT != 2 && VARIANT != 5)
            for (int a = 0; a < A_COLS / 64; ++a) tma::load_2d(sA + a * A_ROWS * 128, &tmA, &bar_load, a * 64, 0);
        for (int a = 0; a < B_COLS / 64; ++a) tma::load_2d(sB + a * B_ROWS * 128, &tmB, &bar_load, a * 64, 0);
    }
    if (VARIANT == 2 || VARIANT == 4 || VARIANT == 5) {
        // stage A (row = TMEM lane) into TMEM as bf16 pairs
        const int row = warp * 32 + lane;
        uint32_t r[64];
#pragma unroll
        for (int c = 0; c < K / 2; ++c) {
            const uint32_t* src = reinterpret_cast<const uint32_t*>(A_gmem + (size_t)row * K);
            r[c] = src[c];
        }
        if constexpr (K == 128) {
            tmem::st_32x32b_x64(tmem::addr(t_a, warp * 32, 0), r);
        } else {
            tmem::st_32x32b_x32(tmem::addr(t_a, warp * 32, 0), r);
        }
        tmem::wait_st();
        tmem::fence_before();
    }
    __syncthreads();
    tmem::fence_after();

    if (VARIANT != 4 && warp == 0) {
        mbar_wait(&bar_load, 0);
        tmem::fence_after();
        if (elect_one()) {
            constexpr uint32_t idesc = umma::idesc_bf16<M, N, VARIANT == 3, VARIANT != 0 && VARIANT != 5>();
            const long long c0 = clock64();
            for (int rep = 0; rep < reps; ++rep)
#pragma unroll
            for (int s = 0; s < K / 16; ++s) {
                uint64_t bdesc;
                if constexpr (VARIANT == 0 || VARIANT == 5) {
                    bdesc = umma::desc_kmajor(smem_u32(sB + (s / 4) * (N * 128) + (s % 4) * 32));
                } else {
                    bdesc = umma::desc_mnmajor(smem_u32(sB + s * 16 * 128), K * 128);
                }
                if constexpr (VARIANT == 2 || VARIANT == 5) {
                    umma::mma_ts(t_c, t_a + s * 8, bdesc, idesc, s > 0);
                } else {
                    uint64_t adesc;
                    if constexpr (VARIANT == 3) {
                        adesc = umma::desc_mnmajor(smem_u32(sA + s * 16 * 128), K * 128);
                    } else {
                        adesc = umma::desc_kmajor(smem_u32(sA + (s / 4) * (M * 128) + (s % 4) * 32));
                    }
                    umma::mma_ss(t_c, adesc, bdesc, idesc, s > 0);
                }
            }
            umma::commit(&bar_mma);
            if (cycles != nullptr) {
                mbar_wait(&bar_mma, 0);
                cycles[0] = clock64() - c0;
            }
        }
        __syncwarp();
    }
    if (VARIANT != 4) mbar_wait(&bar_mma, 0);
    tmem::fence_after();
    {
        const int row = warp * 32 + lane;
        uint32_t r[32];
        if (VARIANT == 4) {
            // read back the bf16-pair staging area and widen
            for (int c0 = 0; c0 < K / 2; c0 += 32) {
                tmem::ldw_32x32b_x32(tmem::addr(t_a, warp * 32, c0), r);
                for (int j = 0; j < 32; ++j) {
                    __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&r[j]);
                    C[(size_t)row * K + 2 * (c0 + j)] = __bfloat162float(h.x);
                    C[(size_t)row * K + 2 * (c0 + j) + 1] = __bfloat162float(h.y);
                }
            }
        } else {
            for (int c0 = 0; c0 < N; c0 += 32) {
                tmem::ldw_32x32b_x32(tmem::addr(t_c, warp * 32, c0), r);
                for (int j = 0; j < 32; ++j) C[(size_t)row * N + c0 + j] = __uint_as_float(r[j]);
            }
        }
    }
    tmem::fence_before();
    __syncthreads();
    if (warp == 0) tmem::dealloc<256>(tbase);
}

bool make_2d(CUtensorMap* tm, const void* p, int rows, int cols, std::string* err) {
    uint64_t dims[2] = {(uint64_t)cols, (uint64_t)rows};
    uint64_t strides[2] = {1, (uint64_t)cols};
    uint32_t box[2] = {64, (uint32_t)rows};
    return host::make_tmap(tm, p, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, 2, dims, strides, box,
                           CU_TENSOR_MAP_SWIZZLE_128B, err);
}

template <int N, int K, int V>
int launch(const void* A, const void* B, float* C, cudaStream_t st, int reps, long long* cycles) {
    CUtensorMap ta, tb;
    std::string err;
    const int a_rows = (V == 3) ? K : M, a_cols = (V == 3) ? M : K;
    const int b_rows = (V == 0 || V == 5) ? N : K, b_cols = (V == 0 || V == 5) ? K : N;
    if (!make_2d(&ta, A, a_rows, a_cols, &err) || !make_2d(&tb, B, b_rows, b_cols, &err)) {
        fprintf(stderr, "selftest tmap: %s\n", err.c_str());
        return -1;
    }
    auto k = selftest_kernel<N, K, V>;
    const int smem = 65536 + 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<1, 128, smem, st>>>(ta, tb, reinterpret_cast<const __nv_bfloat16*>(A), C, reps, cycles);
    return (int)cudaGetLastError();
}

}  // namespace

extern "C" __attribute__((visibility("default"))) int tkb_selftest_umma(int variant, int n, int k, const void* A,
                                                                       const void* B, float* C, cudaStream_t stream,
                                                                       int reps, long long* cycles) {
#define TKB_ST(V, NN, KK) \
    if (variant == V && n == NN && k == KK) return launch<NN, KK, V>(A, B, C, stream, reps, cycles);
    TKB_ST(0, 128, 128) TKB_ST(0, 128, 64) TKB_ST(1, 128, 128) TKB_ST(1, 64, 128) TKB_ST(2, 128, 128)
    TKB_ST(2, 64, 128) TKB_ST(3, 128, 128) TKB_ST(3, 64, 128) TKB_ST(4, 128, 128)
    TKB_ST(5, 128, 128) TKB_ST(5, 128, 64)
#undef TKB_ST
    return -2;
}

// ---------------------------------------------------------------------------------------------
// Tile-API selftest (tkb/tile.cuh): one 128 x 128 attention tile written only with the
// ThunderKittens vocabulary, checked against torch on the host (tests/test_tile_api_gpu.py):
//   load_async(st_bf, gl)  Q, K, V (TMA, SW128)                 tiles.hpp:416-426
//   mm_ABt(tt_fl, st_bf, st_bf)  S = Q K^T                     tiles.hpp:349
//   load(rt_fl, tt) / row_max / sub_row / exp2 / row_sum       tiles.hpp:217-309
//   copy(rt_bf, rt_fl)  P -> bf16 (RNE); store(tt_bf, rt_bf)   tiles.hpp:195-200
//   mma_AB(tt_fl, tt_bf, st_bf)  O = P V (V MN-major)          tiles.hpp:350-352
//   div_row  O / l                                             tiles.hpp:276-281
// plus st_bf::chunk addressing against the TMA placement (the SW128 element_offset rule,
// layouts.hpp:111-132): out_q = Q read back through chunk(r, c).
// Outputs: O [128][128] fp32, m [128] (row max of S), l [128] (row sum of exp2(S - m)),
// p_bf [128][128] (the bf16 P bits as float), q_back [128][128] (bf16 as float).
__global__ void __launch_bounds__(128, 1)
    tile_api_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, float* O, float* m_out, float* l_out, float* p_out,
                    float* q_back) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    using T = st_bf<128, 128>;
    const T sQ{smem}, sK{smem + T::kBytes}, sV{smem + 2 * T::kBytes};
    const gl gQ{&tmQ}, gK{&tmK}, gV{&tmV};
    __shared__ mbarrier bar_load, bar_s, bar_o;
    __shared__ uint32_t tslot;
    const int warp = warpid(), lane = laneid();
    if (threadIdx.x == 0) {
        mbar_init(&bar_load, 1);
        mbar_init(&bar_s, 1);
        mbar_init(&bar_o, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem::alloc<512>(&tslot);
    tmem::fence_before();
    __syncthreads();
    tmem::fence_after();
    const tt_fl<128> tS{tslot}, tO{tslot + 128};
    const tt_bf<64> tP{tslot + 256};
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bar_load, 3 * T::kBytes);
        load_async(sQ, gQ, &bar_load, 0, 0, 0, tma::policy_evict_first());  // 2-D maps: head = batch = 0
        load_async(sK, gK, &bar_load, 0, 0, 0, tma::policy_evict_first());
        load_async(sV, gV, &bar_load, 0, 0, 0, tma::policy_evict_first());
    }
    mbar_wait(&bar_load, 0);
    if (warp == 0) {  // converged MMA warp
        tmem::fence_after();
        mm_ABt(tS, sQ, sK);
        mma_commit(&bar_s);
    }
    mbar_wait(&bar_s, 0);
    tmem::fence_after();
    const int r = warp * 32 + lane;
    rt_fl<128> x;
    load(x, tS.quarter(warp));
    load_wait(x);
    float mx = -INFINITY;
    row_max(mx, x);
    sub_row(x, mx);
    exp2(x);
    float l = 0.f;
    row_sum(l, x);
    rt_bf<128> pb;
    copy(pb, x);
    store(tP.quarter(warp), pb);
    tmem::wait_st();
    for (int c = 0; c < 128; c += 2) {
        p_out[(size_t)r * 128 + c] = __uint_as_float(pb.v[c / 2] << 16);
        p_out[(size_t)r * 128 + c + 1] = __uint_as_float(pb.v[c / 2] & 0xFFFF0000u);
    }
    m_out[r] = mx;
    l_out[r] = l;
    tmem::fence_before();
    __syncthreads();
    if (warp == 0) {
        tmem::fence_after();
        mma_AB(tO, tP, swap_layout(sV), false);
        mma_commit(&bar_o);
    }
    mbar_wait(&bar_o, 0);
    tmem::fence_after();
    rt_fl<128> o;
    load(o, tO.quarter(warp));
    load_wait(o);
    div_row(o, l);
    for (int c = 0; c < 128; ++c) O[(size_t)r * 128 + c] = o.v[c];
    for (int c = 0; c < 16; ++c) {  // SW128 addressing: 16-byte chunk c of row r
        const uint4 u = *reinterpret_cast<const uint4*>(sQ.chunk(r, c));
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
        for (int e = 0; e < 4; ++e) {
            q_back[(size_t)r * 128 + 8 * c + 2 * e] = __uint_as_float(w[e] << 16);
            q_back[(size_t)r * 128 + 8 * c + 2 * e + 1] = __uint_as_float(w[e] & 0xFFFF0000u);
        }
    }
    tmem::fence_before();
    __syncthreads();
    if (warp == 0) tmem::dealloc<512>(tslot);
}

// Tile-API selftest 2: the operand / transfer flavours the backward uses, on one 128 x 128 x
// 128 product (tests/test_tile_api_gpu.py checks each against torch):
//   load(rt_bf, gv) / store(st_bf, rt_bf)   A: global -> register -> shared (SW128)
//   mm_AB(tt_fl, st_bf, swap_layout(st_bf)) C1 = A B   (SS, B read MN-major)
//   load(rt_bf, st_bf) / store(tt, rt_bf)   A: shared -> register -> TMEM
//   mm_ABt(tt_fl, tt_bf, st_bf)             C2 = A B^T (TS, A in TMEM)
//   mma_AB_groups(tt_fl, tt_bf, st_mn)      C3 = A B   (TS, A as four 32-column chunks)
//   store_rows(gv, rt_bf)                   C3 -> bf16 rows in global (warp-transposed)
__global__ void __launch_bounds__(128, 1)
    tile_api2_kernel(const __nv_bfloat16* A, const __grid_constant__ CUtensorMap tmB, float* C1, float* C2,
                     float* C3, __nv_bfloat16* C3b) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    using T = st_bf<128, 128>;
    const T sA{smem}, sB{smem + T::kBytes};
    __shared__ mbarrier bar_load, bar_mma;
    __shared__ uint32_t tslot;
    const int warp = warpid(), lane = laneid();
    const int r = warp * 32 + lane;
    if (threadIdx.x == 0) {
        mbar_init(&bar_load, 1);
        mbar_init(&bar_mma, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem::alloc<512>(&tslot);
    tmem::fence_before();
    __syncthreads();
    tmem::fence_after();
    const tt_fl<128> tC1{tslot}, tC2{tslot + 384};
    const tt_bf<64> tA{tslot + 128};
    const tt_bf<128> tAg{tslot + 256};
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bar_load, T::kBytes);
        load_async(sB, gl{&tmB}, &bar_load, 0, 0, 0, tma::policy_evict_first());
    }
    {  // A: global -> register -> shared
        const gv<const __nv_bfloat16> gA{A, 0, 0, 128};
        rt_bf<128> a;
        load(a, gA, 0, 0, r, 0);
        store(sA, a, r, 0);
    }
    tma::fence_async_smem();  // generic-proxy SMEM writes -> visible to the tensor core (async proxy)
    __syncthreads();
    {  // A: shared -> register -> TMEM (dense K = 128, and the grouped 4 x 32 layout)
        rt_bf<128> a;
        load(a, sA, r, 0);
        store(tA.quarter(warp), a);
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            rt_bf<32> c;
#pragma unroll
            for (int j = 0; j < 16; ++j) c.v[j] = a.v[16 * g + j];
            store(tAg.quarter(warp) + 32 * g, c);
        }
        tmem::wait_st();
    }
    mbar_wait(&bar_load, 0);
    tmem::fence_before();
    __syncthreads();
    auto read_out = [&](const tt_fl<128>& t, float* out) {
        rt_fl<128> c;
        load(c, t.quarter(warp));
        load_wait(c);
        for (int j = 0; j < 128; ++j) out[(size_t)r * 128 + j] = c.v[j];
    };
    uint32_t ph = 0;
    // C1 = A B (SS)
    if (warp == 0) {
        tmem::fence_after();
        mm_AB(tC1, sA, swap_layout(sB));
        mma_commit(&bar_mma);
    }
    mbar_wait(&bar_mma, ph);
    ph ^= 1;
    tmem::fence_after();
    read_out(tC1, C1);
    // C2 = A B^T (A in TMEM)
    tmem::fence_before();
    __syncthreads();
    if (warp == 0) {
        tmem::fence_after();
        mm_ABt(tC2, tA, sB);
        mma_commit(&bar_mma);
    }
    mbar_wait(&bar_mma, ph);
    ph ^= 1;
    tmem::fence_after();
    read_out(tC2, C2);
    // C3 = A B (grouped A in TMEM), into tC1
    tmem::fence_before();
    __syncthreads();
    if (warp == 0) {
        tmem::fence_after();
        mma_AB_groups(tC1, tAg, swap_layout(sB), false, [](int) {});
        mma_commit(&bar_mma);
    }
    mbar_wait(&bar_mma, ph);
    tmem::fence_after();
    read_out(tC1, C3);
    {  // C3 -> bf16 -> global rows (register -> global, warp-collective), 32 columns per pass
        const gv<__nv_bfloat16> gC{C3b, 0, 0, 128};
        for (int c0 = 0; c0 < 128; c0 += 32) {
            rt_fl<32> f;
            load(f, tC1.quarter(warp) + c0);
            load_wait(f);
            rt_bf<32> h;
            copy(h, f);
            store_rows(gC, h, 0, 0, warp * 32, c0, 32);
        }
    }
    tmem::fence_before();
    __syncthreads();
    if (warp == 0) tmem::dealloc<512>(tslot);
}

extern "C" __attribute__((visibility("default"))) int tkb_selftest_tile_api2(const void* A, const void* B, float* C1,
                                                                            float* C2, float* C3, void* C3b,
                                                                            cudaStream_t stream) {
    CUtensorMap tb;
    std::string err;
    uint64_t dims[4] = {128, 128, 1, 1}, strides[4] = {1, 128, 128 * 128, 128 * 128};
    uint32_t box[4] = {64, 128, 1, 1};
    if (!host::make_tmap(&tb, B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, 4, dims, strides, box,
                         CU_TENSOR_MAP_SWIZZLE_128B, &err))
        return -1;
    const int smem = 2 * 32768 + 1024;
    cudaFuncSetAttribute(tile_api2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    tile_api2_kernel<<<1, 128, smem, stream>>>(reinterpret_cast<const __nv_bfloat16*>(A), tb, C1, C2, C3,
                                                reinterpret_cast<__nv_bfloat16*>(C3b));
    return (int)cudaGetLastError();
}

// bf16 RNE of `n` floats through copy(rt_bf, rt_fl) = cvt.rn.bf16x2.f32 (tiles.hpp:40-46, 195-200)
__global__ void rne_kernel(const float* in, float* out, int n) {
    const int i = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (i + 1 < n) {
        rt_fl<2> a;
        a.v[0] = in[i];
        a.v[1] = in[i + 1];
        rt_bf<2> b;
        copy(b, a);
        out[i] = __uint_as_float(b.v[0] << 16);
        out[i + 1] = __uint_as_float(b.v[0] & 0xFFFF0000u);
    }
}

extern "C" __attribute__((visibility("default"))) int tkb_selftest_tile_api(const void* Q, const void* K,
                                                                           const void* V, float* O, float* m,
                                                                           float* l, float* p, float* q_back,
                                                                           cudaStream_t stream) {
    CUtensorMap tq, tk, tv;
    std::string err;
    auto mk = [&](CUtensorMap* tm, const void* ptr) {  // 4-D {128, 128, 1, 1} view, box {64, 128, 1, 1}
        uint64_t dims[4] = {128, 128, 1, 1}, strides[4] = {1, 128, 128 * 128, 128 * 128};
        uint32_t box[4] = {64, 128, 1, 1};
        return host::make_tmap(tm, ptr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, 4, dims, strides, box,
                               CU_TENSOR_MAP_SWIZZLE_128B, &err);
    };
    if (!mk(&tq, Q) || !mk(&tk, K) || !mk(&tv, V)) return -1;
    const int smem = 3 * 32768 + 1024;
    cudaFuncSetAttribute(tile_api_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    tile_api_kernel<<<1, 128, smem, stream>>>(tq, tk, tv, O, m, l, p, q_back);
    return (int)cudaGetLastError();
}

extern "C" __attribute__((visibility("default"))) int tkb_selftest_rne(const float* in, float* out, int n,
                                                                      cudaStream_t stream) {
    rne_kernel<<<(n / 2 + 127) / 128, 128, 0, stream>>>(in, out, n);
    return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Reduce-throughput microbenchmark: every CTA repeatedly adds 16 KB fp32 chunks from SMEM into
// a global fp32 region (L2-resident), via (mode 0) the tensor TMA reduce {32 x 128 box, SW128},
// (mode 1) the 1-D bulk reduce of a contiguous 16 KB, (mode 2) red.global.add.v4.f32 from
// registers. `inflight` bulk groups may be outstanding. Returns nothing; time it with events.
namespace {
__global__ void __launch_bounds__(128, 1)
    reduce_bench_kernel(const __grid_constant__ CUtensorMap tm, float* __restrict__ g, int mode, int iters,
                        int inflight, int region_chunks) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    for (int i = threadIdx.x; i < 4 * 4096; i += 128) reinterpret_cast<float*>(smem)[i] = 1.0f;
    tma::fence_async_smem();
    __syncthreads();
    if (mode == 2) {
        for (int it = 0; it < iters; ++it) {
            const int chunk = (blockIdx.x * 7 + it) % region_chunks;
            float* dst = g + (size_t)chunk * 4096 + threadIdx.x * 32;
#pragma unroll
            for (int c = 0; c < 32; c += 4)
                asm volatile("red.global.add.v4.f32 [%0], {%1, %1, %1, %1};" ::"l"(dst + c), "f"(1.0f) : "memory");
        }
        return;
    }
    if (threadIdx.x == 0) {
        for (int it = 0; it < iters; ++it) {
            const int chunk = (blockIdx.x * 7 + it) % region_chunks;
            const uint8_t* src = smem + (it & 3) * 16384;
            if (mode == 0) {
                tma::reduce_add_3d(&tm, src, 0, (chunk % 64) * 128, chunk / 64);
            } else {
                asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 16384;" ::"l"(
                                 g + (size_t)chunk * 4096),
                             "r"(smem_u32(src))
                             : "memory");
            }
            tma::commit_group();
            if (inflight <= 1) tma::wait_group_read<0>();
            else if (inflight == 2) tma::wait_group_read<1>();
            else tma::wait_group_read<3>();
        }
        tma::wait_group<0>();
    }
}
}  // namespace

extern "C" __attribute__((visibility("default"))) int tkb_selftest_reduce_bench(float* g, int mode, int ctas,
                                                                               int iters, int inflight,
                                                                               int region_chunks, cudaStream_t st) {
    CUtensorMap tm;
    std::string err;
    // region viewed as {32 cols, 64*128 rows, region_chunks/64 planes}: chunk = 128 x 32 fp32 (row pitch 128 B)
    uint64_t dims[3] = {32, 64 * 128, (uint64_t)(region_chunks / 64)};
    uint64_t strides[3] = {1, 32, (uint64_t)64 * 128 * 32};
    uint32_t box[3] = {32, 128, 1};
    if (!host::make_tmap(&tm, g, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, 3, dims, strides, box,
                         CU_TENSOR_MAP_SWIZZLE_128B, &err))
        return -1;
    const int smem = 4 * 16384 + 1024;
    cudaFuncSetAttribute(reduce_bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    reduce_bench_kernel<<<ctas, 128, smem, st>>>(tm, g, mode, iters, inflight, region_chunks);
    return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Pipe-throughput microbenchmark for the softmax inner loop (one CTA of 256 threads):
//   mode 0: ex2.approx (MUFU)       mode 1: cvt.rn.bf16x2.f32     mode 2: ex2 + cvt
//   mode 3: ffma                    mode 4: fma.rn.f32x2 (packed)  mode 5: poly-3 exp2 emulation (f32x2)
namespace {
__global__ void __launch_bounds__(256, 1) pipe_bench_kernel(float* out, int mode, int iters, long long* cycles) {
    float a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = -0.01f * (threadIdx.x + i);
    uint32_t acc = 0;
    __syncthreads();
    const long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (mode == 0) {
#pragma unroll
            for (int i = 0; i < 16; ++i) a[i] = ex2_approx(a[i]);
        } else if (mode == 1) {
#pragma unroll
            for (int i = 0; i < 16; i += 2) acc += pack_bf16x2(a[i], a[i + 1]), a[i] += 1e-7f;
        } else if (mode == 2) {
#pragma unroll
            for (int i = 0; i < 16; i += 2) {
                a[i] = ex2_approx(a[i]);
                a[i + 1] = ex2_approx(a[i + 1]);
                acc += pack_bf16x2(a[i], a[i + 1]);
            }
        } else if (mode == 3) {
#pragma unroll
            for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], 0.999f, 1e-7f);
        } else if (mode == 4) {
#pragma unroll
            for (int i = 0; i < 16; i += 2) {
                asm volatile("{.reg .b64 x, y, z; mov.b64 x, {%0, %1}; mov.b64 y, {%2, %2}; mov.b64 z, {%3, %3};"
                             "fma.rn.f32x2 x, x, y, z; mov.b64 {%0, %1}, x;}"
                             : "+f"(a[i]), "+f"(a[i + 1]) : "f"(0.999f), "f"(1e-7f));
            }
        } else {
#pragma unroll
            for (int i = 0; i < 16; i += 2) {
                float x0 = fmaxf(a[i], -127.f), x1 = fmaxf(a[i + 1], -127.f);
                float r0, r1, f0, f1, p0, p1;
                asm("{.reg .b64 x, rr, big, bk, fr, c3, c2, c1, c0, p;\n\t"
                    "mov.b64 x, {%6, %7};\n\t"
                    "mov.b64 big, {%8, %8};\n\t"
                    "add.rm.ftz.f32x2 rr, x, big;\n\t"
                    "sub.rn.ftz.f32x2 bk, rr, big;\n\t"
                    "sub.rn.ftz.f32x2 fr, x, bk;\n\t"
                    "mov.b64 c3, {%9, %9}; mov.b64 c2, {%10, %10}; mov.b64 c1, {%11, %11}; mov.b64 c0, {%12, %12};\n\t"
                    "fma.rn.ftz.f32x2 p, fr, c3, c2;\n\t"
                    "fma.rn.ftz.f32x2 p, p, fr, c1;\n\t"
                    "fma.rn.ftz.f32x2 p, p, fr, c0;\n\t"
                    "mov.b64 {%0, %1}, rr; mov.b64 {%2, %3}, fr; mov.b64 {%4, %5}, p;}"
                    : "=f"(r0), "=f"(r1), "=f"(f0), "=f"(f1), "=f"(p0), "=f"(p1)
                    : "f"(x0), "f"(x1), "f"(12582912.0f), "f"(0.0770954f), "f"(0.2275836f), "f"(0.6944390f),
                      "f"(1.0f));
                a[i] = __int_as_float((__float_as_int(r0) << 23) + __float_as_int(p0)) - 1e-3f;
                a[i + 1] = __int_as_float((__float_as_int(r1) << 23) + __float_as_int(p1)) - 1e-3f;
            }
        }
    }
    const long long c1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += a[i];
    out[threadIdx.x] = s + (float)acc;
    if (threadIdx.x == 0) cycles[0] = c1 - c0;
}
}  // namespace

extern "C" __attribute__((visibility("default"))) int tkb_selftest_pipe_bench(float* out, int mode, int iters,
                                                                             long long* cycles, cudaStream_t st) {
    pipe_bench_kernel<<<1, 256, 0, st>>>(out, mode, iters, cycles);
    return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------- deadlock
// The LCSF contract violation the reference detects as DeadlockError (lcsf.hpp:486-489,
// tests/test_lcsf.cpp:204-233): a consumer waits on a ring slot whose producer never
// arrives. mbar_wait's bound (TKB_DEADLOCK_NS; this library is built with 0.2 s) traps.
// mode 0: the producer is missing (deadlock); mode 1: the producer arrives (completes).
namespace {
__global__ void deadlock_kernel(int mode, int* done) {
    __shared__ lcsf::ring<2> r;
    if (threadIdx.x == 0) r.init(1, 1);
    __syncthreads();
    lcsf::ring_state<2> st;
    if (mode == 1 && threadIdx.x == 32) mbar_arrive(&r.full[0]);
    if (threadIdx.x == 0) {
        r.wait_full(st);
        *done = 1;
    }
}
}  // namespace

extern "C" __attribute__((visibility("default"))) int tkb_selftest_deadlock(int mode, int* done_dev) {
    deadlock_kernel<<<1, 64>>>(mode, done_dev);
    cudaError_t e = cudaDeviceSynchronize();
    return (int)e;
}

// ---------------------------------------------------------------------------- TMEM shapes
// Pins the 16-lane tcgen05 data-movement maps the backward's dK/dV compute relies on
// (attn_bwd_sm100.cu, grp_load / grp_store_packed):
//   ld.16x256b.x4 at lane block L: register 4 r + 2 h + b <- lane L + lane/4 + 8 h, column
//                                  2 (lane % 4) + 8 r + b
//   st.16x128b.x4 at lane block L: register 2 r + h -> lane L + lane/4 + 8 h, column lane % 4 + 4 r
// Returns the number of mismatching elements in *bad.
namespace {
__global__ void __launch_bounds__(128, 1) tmem_shape_kernel(int* bad) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0) tmem::alloc<64>(&slot);
    tmem::fence_before();
    __syncthreads();
    tmem::fence_after();
    const uint32_t base = slot + ((uint32_t)(warp * 32) << 16);
    const int row = warp * 32 + lane;
    uint32_t v[32];
    for (int c = 0; c < 32; ++c) v[c] = (uint32_t)(row * 64 + c);
    tmem::st_32x32b_x32(base, v);
    tmem::wait_st();
    int errs = 0;
    for (int blk = 0; blk < 2; ++blk) {
        uint32_t w[16];
        tmem::ld_16x256b_x4(base + ((uint32_t)(16 * blk) << 16), w);
        tmem::wait_ld_x16(w);
        for (int rr = 0; rr < 4; ++rr)
            for (int h = 0; h < 2; ++h)
                for (int b = 0; b < 2; ++b) {
                    const int R = warp * 32 + 16 * blk + lane / 4 + 8 * h;
                    const int C = 2 * (lane % 4) + 8 * rr + b;
                    errs += w[4 * rr + 2 * h + b] != (uint32_t)(R * 64 + C);
                }
    }
    for (int blk = 0; blk < 2; ++blk) {
        uint32_t pk[8];
        for (int k = 0; k < 8; ++k) pk[k] = (uint32_t)(100000 * (blk + 1) + 1000 * k + threadIdx.x);
        tmem::st_16x128b_x4(base + 32 + ((uint32_t)(16 * blk) << 16), pk);
    }
    tmem::wait_st();
    uint32_t got[16];
    tmem::ld_32x32b_x16(base + 32, got);
    tmem::wait_ld_x16(got);
    for (int m = 0; m < 16; ++m) {  // this thread holds lane `lane` of the quarter: its row
        const int R16 = lane % 16, blk = lane / 16;
        const int h = R16 / 8, writer = 4 * (R16 % 8) + m % 4, rr = m / 4;
        const uint32_t want = (uint32_t)(100000 * (blk + 1) + 1000 * (2 * rr + h) + warp * 32 + writer);
        errs += got[m] != want;
    }
    atomicAdd(bad, errs);
    tmem::fence_before();
    __syncthreads();
    if (warp == 0) tmem::dealloc<64>(slot);
}
}  // namespace

extern "C" __attribute__((visibility("default"))) int tkb_selftest_tmem_shapes(int* bad_dev) {
    tmem_shape_kernel<<<1, 128>>>(bad_dev);
    return (int)cudaDeviceSynchronize();
}
