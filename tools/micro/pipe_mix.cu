// Microbenchmark: per-SMSP throughput of the softmax instruction mix pieces
// (cycles per warp-instruction, 1 and 2 warps per SM sub-partition).
#include <cstdio>
#include <cstdint>
#include "tkb/common.cuh"
using namespace tkb;

template <int MODE>
__global__ void k(uint32_t* out, int iters, long long* cyc) {
    float x[32];
    uint32_t u[32];
    for (int i = 0; i < 32; ++i) {
        x[i] = 0.001f * (threadIdx.x + i);
        u[i] = threadIdx.x * 3 + i;
    }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
            if (MODE == 0) {  // F2FP pack
                u[i] ^= pack_bf16x2(x[i], x[i + 1]);
                x[i] = __uint_as_float(u[i + 1] & 0x3f800000u) + x[i];
            }
            if (MODE == 1) {  // FFMA2
                float2 r = fma2(make_float2(x[i], x[i + 1]), make_float2(1.0001f, 1.0001f), make_float2(0.5f, 0.5f));
                x[i] = r.x;
                x[i + 1] = r.y;
            }
            if (MODE == 2) {  // FFMA scalar
                x[i] = fmaf(x[i], 1.0001f, 0.5f);
                x[i + 1] = fmaf(x[i + 1], 1.0001f, 0.5f);
            }
            if (MODE == 3) {  // FADD2
                float2 r = add2(make_float2(x[i], x[i + 1]), make_float2(0.5f, 0.5f));
                x[i] = r.x;
                x[i + 1] = r.y;
            }
            if (MODE == 4) {  // FMNMX
                x[i] = fmaxf(x[i], x[(i + 5) & 31]);
                x[i + 1] = fmaxf(x[i + 1], x[(i + 7) & 31]);
            }
            if (MODE == 5) {  // IMAD
                u[i] = u[i] * 0x800000u + u[i + 1];
                u[i + 1] = u[i + 1] * 0x800000u + u[i];
            }
            if (MODE == 6) {  // pack only (independent)
                u[i] = pack_bf16x2(x[i], x[i + 1]);
                u[i + 1] = pack_bf16x2(x[i + 1], x[i]);
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    uint32_t s = 0;
    for (int i = 0; i < 32; ++i) s += u[i] + __float_as_uint(x[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    uint32_t* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMallocManaged(&cyc, 8);
    const int iters = 1000;
    const char* names[] = {"F2FP+FADD(dep)", "FFMA2", "FFMA", "FADD2", "FMNMX", "IMAD", "F2FP pack"};
    const int per_iter[] = {32, 16, 32, 16, 32, 32, 32};  // warp-instructions of the named kind per iteration
    for (int threads : {128, 256, 512}) {
        for (int mode = 0; mode < 7; ++mode) {
            auto fn = mode == 0 ? k<0> : mode == 1 ? k<1> : mode == 2 ? k<2> : mode == 3 ? k<3> : mode == 4 ? k<4> : mode == 5 ? k<5> : k<6>;
            fn<<<148, threads>>>(out, iters, cyc);
            cudaDeviceSynchronize();
            fn<<<148, threads>>>(out, iters, cyc);
            cudaDeviceSynchronize();
            const double warps_per_smsp = threads / 128.0;
            printf("warps/SMSP %.0f %-16s: %5.2f clk per warp-instr per SMSP\n", warps_per_smsp, names[mode],
                   (double)*cyc / (iters * per_iter[mode] * warps_per_smsp));
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
