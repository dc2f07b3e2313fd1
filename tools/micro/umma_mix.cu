// Microbenchmark: cycles per step of the dK/dV kernel's MMA sequence on one SM, alone and
// with the traffic the other roles add. One CTA per SM (148), operands resident in SMEM /
// TMEM (contents irrelevant). A step = S^T = K Q^T (SS), dV += P^T dO (TS), dP^T = V dO^T
// (SS), dK += dS^T Q (TS): 4 GEMMs of 128 x 128 x 128 = 32 MMAs of 128x128x16 (2048 clk at
// the tensor peak).
//   mode 0: the four GEMMs              mode 1: SS GEMMs only (x2 per step)
//   mode 2: TS GEMMs only (x2 per step) mode 3: mode 0 + 16 warps doing the compute warps'
//           TMEM traffic (ld 32 cols, st 16 cols, ld 32 cols, st 16 cols per step)
//   mode 4: mode 0 + a TMA-like 64 KB SMEM write stream (cp.async.bulk global->shared)
#include <cstdio>
#include <cstdint>
#include "tkb/tcgen05.cuh"
#include "tkb/tma.cuh"
using namespace tkb;

constexpr int kAtom = 128 * 128;
constexpr uint32_t kHi = umma::desc_hi_sw128(1024);

__device__ void mm_abt(uint32_t dst, uint32_t a, uint32_t b, uint32_t idesc) {
    for (int k = 0; k < 8; ++k) {
        const uint32_t off = (k / 4) * kAtom + (k % 4) * 32;
        umma::mma_ss_e(dst, umma::desc_lo(a + off, 16), kHi, umma::desc_lo(b + off, 16), kHi, idesc, k > 0);
    }
}
__device__ void mma_ts(uint32_t dst, uint32_t a_tmem, uint32_t b, uint32_t idesc) {
    for (int k = 0; k < 8; ++k)
        umma::mma_ts_e(dst, a_tmem + k * 8, umma::desc_lo(b + k * 2048, kAtom), kHi, idesc, 1);
}

__global__ void __launch_bounds__(576, 1) k(int mode, int steps, long long* cyc, const uint8_t* gsrc) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tslot;
    __shared__ mbarrier done, ld_bar;
    __shared__ int stop;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        mbar_init(&done, 1);
        mbar_init(&ld_bar, 1);
        fence_barrier_init();
        stop = 0;
    }
    if (warp == 16) tmem::alloc<512>(&tslot);
    tmem::fence_before();
    __syncthreads();
    tmem::fence_after();
    const uint32_t tb = tslot;
    const uint32_t sK = smem_u32(smem), sV = sK + 32768, sQ = sK + 65536, sDo = sK + 98304;
    constexpr uint32_t id_s = umma::idesc_bf16<128, 128, false, false>();
    constexpr uint32_t id_kv = umma::idesc_bf16<128, 128, false, true>();
    if (warp == 16) {
        long long t0 = clock64();
        for (int s = 0; s < steps; ++s) {
            if (mode != 2) mm_abt(tb + 0, sK, sQ, id_s);
            if (mode != 1) mma_ts(tb + 128, tb + 32, sDo, id_kv);
            if (mode != 2) mm_abt(tb + 256, sV, sDo, id_s);
            if (mode != 1) mma_ts(tb + 384, tb + 288, sQ, id_kv);
        }
        umma::commit_e(&done);
        mbar_wait(&done, 0);
        long long t1 = clock64();
        if (lane == 0) {
            if (blockIdx.x == 0) *cyc = t1 - t0;
            stop = 1;
        }
    } else if (warp < 16 && mode == 3) {
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const int g = warp >> 2;
        uint32_t v[32], acc = 0;
        while (*reinterpret_cast<volatile int*>(&stop) == 0) {
            tmem::ldw_32x32b_x32(tb + lane_off + 32 * g, v);
            for (int i = 0; i < 32; ++i) acc += v[i];
            tmem::st_32x32b_x16(tb + lane_off + 32 * g, v);
            tmem::wait_st();
            tmem::ldw_32x32b_x32(tb + lane_off + 256 + 32 * g, v);
            for (int i = 0; i < 32; ++i) acc += v[i];
            tmem::st_32x32b_x16(tb + lane_off + 256 + 32 * g, v);
            tmem::wait_st();
            __nanosleep(400);  // ~the compute warps' duty cycle
        }
        if (acc == 12345) printf("x");
    } else if (warp == 17 && mode == 4 && lane == 0) {
        uint32_t ph = 0;
        uint8_t* dst = smem + 131072;  // 64 KB landing zone (not an MMA operand)
        while (*reinterpret_cast<volatile int*>(&stop) == 0) {
            mbar_arrive_expect_tx(&ld_bar, 65536);
            for (int c = 0; c < 4; ++c) tma::load_1d(dst + c * 16384, gsrc + (blockIdx.x * 4 + c) * 16384, 16384, &ld_bar);
            mbar_wait(&ld_bar, ph);
            ph ^= 1;
        }
    }
    tmem::fence_before();
    __syncthreads();
    if (warp == 16) tmem::dealloc<512>(tb);
}

int main() {
    long long* cyc;
    uint8_t* g;
    cudaMallocManaged(&cyc, 8);
    cudaMalloc(&g, 148 * 4 * 16384 + 4096);
    const int smem = 196608 + 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const char* names[] = {"4 GEMMs (SS,TS,SS,TS)", "SS only", "TS only", "4 GEMMs + TMEM ld/st by 16 warps",
                           "4 GEMMs + 64 KB/step-ish TMA writes"};
    for (int mode = 0; mode < 5; ++mode) {
        const int steps = 200;
        k<<<148, 576, smem>>>(mode, steps, cyc, g);
        cudaDeviceSynchronize();
        k<<<148, 576, smem>>>(mode, steps, cyc, g);
        cudaDeviceSynchronize();
        const int mmas = (mode == 1 || mode == 2) ? 16 : 32;
        printf("%-40s: %7.1f clk/step  %5.1f clk per 128x128x16 MMA  (%s)\n", names[mode], (double)*cyc / steps,
               (double)*cyc / steps / mmas, cudaGetErrorString(cudaGetLastError()));
    }
}
