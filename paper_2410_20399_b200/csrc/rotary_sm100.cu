// rotary_sm100.cu — rotary position embedding, the Q/K prologue of attention.
//
// Reference: kittensim rotary_kernel (kernels.hpp:357-513) and oracle_rotary
// (oracles.hpp:66-90): for position p and pair index i < hd/2 the pair
// (x[p][i], x[p][i + hd/2]) is rotated by the table angle,
//   o[p][i] = x1 cos - x2 sin,   o[p][i + hd/2] = x2 cos + x1 sin,
// with fp32 [N, hd/2] sin / cos tables shared by every (batch, head).
//
// HBM-bound elementwise work: one thread rotates 8 pairs —
// two 16-byte bf16 vectors and two float4 pairs of the tables — in fp32 and writes
// bf16 (RNE). One launch covers Q ([B, H, N, hd]) and K ([B, Hkv, N, hd]) so the
// rotation before attention is a single pass over both tensors; the grid is a
// multiple of the SM count and grid-strides over 16-pair work items.
// Algorithmic bytes: 2 x 2 B per element of Q and K (read + write) + the tables.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "attn_common.cuh"
#include "tkb/common.cuh"

namespace tkb {
namespace rope {

TKB_DEVICE float2 bf2f(uint32_t u) {
    return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xFFFF0000u));
}

__global__ void __launch_bounds__(256) rotary_kernel(const __grid_constant__ Params p) {
    const int half = p.hd / 2;
    const int chunks = p.hd / 16;  // 8-pair chunks per row
    const int64_t total = p.t[0].items + p.t[1].items;
    for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < total;
         it += (int64_t)gridDim.x * blockDim.x) {
        const bool second = it >= p.t[0].items;
        const Tensor& t = p.t[second ? 1 : 0];
        const int64_t item = second ? it - p.t[0].items : it;
        const int c = (int)(item % chunks);
        const int64_t row = item / chunks;
        const int pos = (int)(row % p.n);
        const int64_t bh = row / p.n;
        const int64_t b = bh / t.heads, h = bh % t.heads;
        const __nv_bfloat16* xr =
            reinterpret_cast<const __nv_bfloat16*>(t.x) + b * t.xb + h * t.xh + pos * t.xn + 8 * c;
        __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(t.o) + b * t.ob + h * t.oh + pos * t.on + 8 * c;
        const uint4 a = *reinterpret_cast<const uint4*>(xr);
        const uint4 bb = *reinterpret_cast<const uint4*>(xr + half);
        const float4* sp = reinterpret_cast<const float4*>(p.sin_tab + (size_t)pos * half + 8 * c);
        const float4* cp = reinterpret_cast<const float4*>(p.cos_tab + (size_t)pos * half + 8 * c);
        const float4 s0 = __ldg(sp), s1 = __ldg(sp + 1), c0 = __ldg(cp), c1 = __ldg(cp + 1);
        const float sn[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
        const float cs[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
        const uint32_t av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {bb.x, bb.y, bb.z, bb.w};
        uint32_t o1[4], o2[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float2 x1 = bf2f(av[q]), x2 = bf2f(bv[q]);
            const float s_lo = sn[2 * q], s_hi = sn[2 * q + 1], c_lo = cs[2 * q], c_hi = cs[2 * q + 1];
            o1[q] = pack_bf16x2(fmaf(x1.x, c_lo, -x2.x * s_lo), fmaf(x1.y, c_hi, -x2.y * s_hi));
            o2[q] = pack_bf16x2(fmaf(x2.x, c_lo, x1.x * s_lo), fmaf(x2.y, c_hi, x1.y * s_hi));
        }
        *reinterpret_cast<uint4*>(orow) = make_uint4(o1[0], o1[1], o1[2], o1[3]);
        *reinterpret_cast<uint4*>(orow + half) = make_uint4(o2[0], o2[1], o2[2], o2[3]);
    }
}

}  // namespace rope

// Launch over one or two tensors; num_sms sizes the grid (resident blocks x SMs).
int launch_rotary(const rope::Params& p, int num_sms, cudaStream_t stream) {
    const int64_t total = p.t[0].items + p.t[1].items;
    if (total == 0) return 0;
    int64_t blocks = (total + 255) / 256;
    const int64_t cap = (int64_t)num_sms * 8;  // 8 x 256 threads per SM in flight
    if (blocks > cap) blocks = cap;
    rope::rotary_kernel<<<(unsigned)blocks, 256, 0, stream>>>(p);
    return (int)cudaGetLastError();
}

}  // namespace tkb
