// Prints the dynamic shared-memory base alignment seen by a kernel with no static smem.
#include <cstdio>
#include <cstdint>
__global__ void k(unsigned* out) {
    extern __shared__ uint8_t smem[];
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned)__cvta_generic_to_shared(smem);
}
int main() {
    unsigned* out;
    cudaMallocManaged(&out, 4 * 148);
    for (int bytes : {1024, 100000, 232448}) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        k<<<148, 32, bytes>>>(out);
        cudaDeviceSynchronize();
        unsigned mx = 0;
        for (int i = 0; i < 148; ++i) mx |= out[i] & 1023u;
        printf("dyn smem %d: base %u (low bits OR over CTAs: %u) %s\n", bytes, out[0], mx,
               cudaGetErrorString(cudaGetLastError()));
    }
}
