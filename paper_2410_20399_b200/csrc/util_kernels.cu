// util_kernels.cu — small helper kernels of the hot path's boundary.
//   check_finite: the reference's "task 0 scans all inputs for non-finite"
//   (kernels.hpp:277-284), as an opt-in device scan (tkb_attn_desc.check_finite).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace tkb {
namespace {

struct FinitePtrs {
    const __nv_bfloat16* p[5];
};

// Linear (bh, row block) index walked grid-stride in 64 bits: B * H may exceed gridDim.y's 65535.
__global__ void check_finite_kernel(FinitePtrs ptrs, int nptrs, int heads, int n, int d, int64_t sb, int64_t sh,
                                    int64_t sn, int64_t total_blocks, int row_blocks, int* flag) {
    const int rows_per_block = blockDim.x * 8 / d;  // 8 bf16 per thread per row chunk
    for (int64_t blk = blockIdx.x; blk < total_blocks; blk += gridDim.x) {
        const int64_t bh = blk / row_blocks;
        const int64_t b = bh / heads, h = bh % heads;
        const int r = (int)(blk - bh * row_blocks) * rows_per_block + (int)(threadIdx.x * 8) / d;
        const int c = (threadIdx.x * 8) % d;
        if (r >= n) continue;
        for (int t = 0; t < nptrs; ++t) {
            const uint4 v = *reinterpret_cast<const uint4*>(ptrs.p[t] + b * sb + h * sh + (int64_t)r * sn + c);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
            bool bad = false;
#pragma unroll
            for (int j = 0; j < 4; ++j)  // bf16 exponent all-ones = inf / nan
                bad |= ((w[j] & 0x7F80u) == 0x7F80u) | ((w[j] & 0x7F800000u) == 0x7F800000u);
            if (bad) atomicOr(flag, 1);
        }
    }
}

}  // namespace

int launch_check_finite(const void* const* ptrs, int nptrs, int batches, int heads, int n, int d, int64_t sb,
                        int64_t sh, int64_t sn, int* flag_dev, cudaStream_t stream) {
    FinitePtrs fp{};
    for (int i = 0; i < nptrs && i < 5; ++i) fp.p[i] = reinterpret_cast<const __nv_bfloat16*>(ptrs[i]);
    const int rows_per_block = 256 * 8 / d;
    const int row_blocks = (n + rows_per_block - 1) / rows_per_block;
    const int64_t total = (int64_t)row_blocks * batches * heads;
    const int64_t cap = 148 * 16;
    check_finite_kernel<<<(unsigned)(total < cap ? total : cap), 256, 0, stream>>>(fp, nptrs, heads, n, d, sb, sh, sn,
                                                                                 total, row_blocks, flag_dev);
    return (int)cudaGetLastError();
}

}  // namespace tkb
