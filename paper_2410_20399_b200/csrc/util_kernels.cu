// util_kernels.cu — small helper kernels of the hot path's boundary.
//   check_finite: the reference's "task 0 scans all inputs for non-finite"
//   (kernels.hpp:277-284), as an opt-in device scan (tkb_attn_desc.check_finite).
//   varlen_maps: the per-sequence TMA maps of a variable-length batch (tensormap.replace).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "attn_common.cuh"

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

// One thread per (sequence b, tensor m): copy the host-encoded template of tensor m (rows =
// the maximum length over the packed tensor's base) into out[b][m], then point it at the
// sequence — base += cu[b] * row_bytes, rows = n_b (>= 1; an empty sequence's map is never
// used) — and release it to the tensor-map proxy. The kernels acquire each map before use.
__global__ void varlen_maps_kernel(const __grid_constant__ VarlenMapTemplates t, const int* __restrict__ cu,
                                   int batches, CUtensorMap* __restrict__ out) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= batches * t.nmaps) return;
    const int b = idx / t.nmaps, m = idx - b * t.nmaps;
    CUtensorMap* dst = out + idx;
    const uint4* src = reinterpret_cast<const uint4*>(&t.tmpl[m]);
    uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int i = 0; i < (int)(sizeof(CUtensorMap) / sizeof(uint4)); ++i) d[i] = src[i];
    const int s0 = cu[b], s1 = cu[b + 1];
    const unsigned rows = (unsigned)max(s1 - s0, 1);
    const unsigned long long addr = t.base[m] + (unsigned long long)s0 * (unsigned long long)t.row_bytes[m];
    asm volatile("tensormap.replace.tile.global_address.global.b1024.b64 [%0], %1;" ::"l"(dst), "l"(addr) : "memory");
    asm volatile("tensormap.replace.tile.global_dim.global.b1024.b32 [%0], 1, %1;" ::"l"(dst), "r"(rows) : "memory");
    asm volatile("fence.proxy.tensormap::generic.release.gpu;" ::: "memory");
}

}  // namespace

int launch_varlen_maps(const VarlenMapTemplates& t, const int* cu, int batches, CUtensorMap* out, cudaStream_t stream) {
    const int total = batches * t.nmaps;
    if (total == 0) return 0;
    varlen_maps_kernel<<<(total + 127) / 128, 128, 0, stream>>>(t, cu, batches, out);
    return (int)cudaGetLastError();
}

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
