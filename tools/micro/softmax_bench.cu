// Microbenchmark: cost (cycles) of the forward softmax exp pass over one 128-column row per
// thread (FFMA2 scale, MUFU ex2 + polynomial share, FADD2 row sum, bf16 pack), for
// 1 or 2 warps per SM sub-partition and poly shares 0..4 of 8.
#include <cstdio>
#include <cstdint>
#include "tkb/common.cuh"
using namespace tkb;

template <int POLY>
__global__ void k(const float* in, uint32_t* out, int iters, long long* cyc) {
    float x[128];
    for (int i = 0; i < 128; ++i) x[i] = in[(threadIdx.x * 7 + i) & 1023];
    const float tau = 0.12f;
    float m = 1.5f, l = 0.f;
    uint32_t sink = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const float2 tau2 = make_float2(tau, tau), nm2 = make_float2(-m, -m);
        float2 acc[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
        uint32_t pk[64];
#pragma unroll
        for (int c = 0; c < 128; c += 2) {
            const float2 xv = fma2(make_float2(x[c], x[c + 1]), tau2, nm2);
            float2 pv;
            if (((c / 2) % 8) < POLY) {
                pv = ex2_poly2(xv);
            } else {
                pv.x = ex2_approx(xv.x);
                pv.y = ex2_approx(xv.y);
            }
            acc[(c / 2) % 4] = add2(acc[(c / 2) % 4], pv);
            pk[c / 2] = pack_bf16x2(pv.x, pv.y);
        }
        l += ((acc[0].x + acc[0].y) + (acc[1].x + acc[1].y)) + ((acc[2].x + acc[2].y) + (acc[3].x + acc[3].y));
#pragma unroll
        for (int i = 0; i < 64; ++i) sink ^= pk[i];
        m += 1e-7f * (float)(sink & 1);
    }
    __syncthreads();
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = sink + __float_as_uint(l);
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    float* in;
    uint32_t* out;
    long long* cyc;
    cudaMalloc(&in, 4096);
    cudaMemset(in, 0, 4096);
    cudaMalloc(&out, 148 * 256 * 4);
    cudaMallocManaged(&cyc, 8);
    const int iters = 200;
    for (int threads : {128, 256}) {
        for (int poly = 0; poly <= 4; ++poly) {
            auto fn = poly == 0 ? k<0> : poly == 1 ? k<1> : poly == 2 ? k<2> : poly == 3 ? k<3> : k<4>;
            fn<<<148, threads>>>(in, out, iters, cyc);
            cudaDeviceSynchronize();
            fn<<<148, threads>>>(in, out, iters, cyc);
            cudaDeviceSynchronize();
            printf("warps/SMSP %d poly %d/8: %6.0f clk per 128-col row pass (per warp)\n", threads / 128, poly,
                   (double)*cyc / iters);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
