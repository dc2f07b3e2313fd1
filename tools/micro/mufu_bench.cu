// Microbenchmark: MUFU ex2 throughput per SM for f32 / bf16x2 / f16x2 (elements per clk per SM).
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

template <int KIND>
__global__ void k(float* out, int iters, long long* cyc) {
    uint32_t r[16];
    for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(-0.001f * (threadIdx.x + i));
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (KIND == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(r[i]));
            if (KIND == 1) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(r[i]));
            if (KIND == 2) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(r[i]));
        }
    }
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 16; ++i) s += __uint_as_float(r[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    float* out; long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 4 * 8);
    cudaMallocManaged(&cyc, 8);
    const int iters = 4096;
    const char* names[3] = {"f32", "bf16x2", "f16x2"};
    for (int threads : {128, 256, 512, 1024}) {
        for (int kind = 0; kind < 3; ++kind) {
            auto fn = kind == 0 ? k<0> : kind == 1 ? k<1> : k<2>;
            fn<<<148, threads>>>(out, iters, cyc);
            cudaDeviceSynchronize();
            fn<<<148, threads>>>(out, iters, cyc);
            cudaDeviceSynchronize();
            double insts = (double)threads * iters * 16;  // thread-instructions per SM
            double elems = insts * (kind == 0 ? 1 : 2);
            printf("threads %4d %-7s : %6.2f thread-inst/clk/SM  %6.2f elem/clk/SM  (%lld clk)\n", threads, names[kind],
                   insts / *cyc, elems / *cyc, *cyc);
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
