// Microbenchmark: tcgen05.ld (TMEM -> registers) throughput per SM, 32x32b.x32 / x64 / x128 shapes,
// 4 / 8 / 16 warps per CTA (one CTA per SM).
#include <cstdio>
#include <cstdint>

template <int X>
__device__ __forceinline__ void ld(uint32_t taddr, uint32_t* r);
template <>
__device__ __forceinline__ void ld<32>(uint32_t t, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(t));
}

__global__ void __launch_bounds__(512, 1) k(uint32_t* out, int iters, long long* cyc, int nwarps) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp / 4) * 128);
    uint32_t acc = 0;
    long long t0 = clock64();
    if (warp < nwarps) {
        for (int it = 0; it < iters; ++it) {
            uint32_t r[128];
#pragma unroll
            for (int c = 0; c < 4; ++c) ld<32>(base + c * 32, r + 32 * c);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int i = 0; i < 128; ++i) acc ^= r[i];
        }
    }
    __syncthreads();
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

int main() {
    uint32_t* out;
    long long* cyc;
    cudaMalloc(&out, 148 * 512 * 4);
    cudaMallocManaged(&cyc, 8);
    const int iters = 2000;
    for (int nw : {1, 2, 4, 8, 16}) {
        k<<<148, 512>>>(out, iters, cyc, nw);
        cudaDeviceSynchronize();
        k<<<148, 512>>>(out, iters, cyc, nw);
        cudaDeviceSynchronize();
        double bytes = (double)nw * 32 * 128 * 4 * iters;
        printf("warps %2d: %7.1f B/clk/SM TMEM->reg (%lld clk)  %s\n", nw, bytes / *cyc, *cyc,
               cudaGetErrorString(cudaGetLastError()));
    }
}
