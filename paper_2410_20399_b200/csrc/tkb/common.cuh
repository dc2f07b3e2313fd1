// tkb — ThunderKittens-style tile vocabulary re-based on Blackwell (sm_100a).
//
// common.cuh: warp/lane helpers, elect-one, named barriers, bf16 packing.
// The reference models these abstractions on the CPU (kittensim,
// /root/reference/proj/include/kittensim/tiles.hpp:27-160); here they are the
// real hardware objects.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>

#if !defined(__CUDA_ARCH__) || (__CUDA_ARCH__ >= 1000)
#else
#error "tkb kernels target sm_100a only"
#endif

#define TKB_DEVICE __device__ __forceinline__

namespace tkb {

constexpr int WARP_THREADS = 32;
constexpr int WARPGROUP_THREADS = 128;

TKB_DEVICE int warpid() { return __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0); }
TKB_DEVICE int laneid() { return (int)(threadIdx.x & 31); }

// One lane of the (fully converged) warp returns true.
TKB_DEVICE bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .b32 %%rx;\n\t.reg .pred %%px;\n\t"
        "elect.sync %%rx|%%px, %1;\n\t"
        "@%%px mov.s32 %0, 1;\n\t}"
        : "+r"(pred)
        : "r"(0xffffffffu));
    return pred != 0;
}

TKB_DEVICE uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Explicit shared-space accesses (a generic pointer into dynamic SMEM can make the
// compiler fall back to 64-bit generic loads/stores).
TKB_DEVICE void sts_f32(uint32_t addr, float v) { asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory"); }
TKB_DEVICE void sts_u32(uint32_t addr, uint32_t v) { asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory"); }
TKB_DEVICE float lds_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
    return v;
}
TKB_DEVICE uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
TKB_DEVICE void sts_v4(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// Named barriers (ids 1..15; id 0 is __syncthreads).
TKB_DEVICE void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
TKB_DEVICE void named_arrive(int id, int nthreads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Pack two fp32 into bf16x2 with RNE (lo -> bits 0..15, hi -> bits 16..31).
// Matches round_to_bf16 (tiles.hpp:40-46) for finite inputs.
TKB_DEVICE void st_global_v4(void* ptr, uint4 v) {
    asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(ptr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// max(a, b, c) in one FMNMX3 (sm_100); NaN handling as fmaxf
TKB_DEVICE float fmax3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

TKB_DEVICE uint32_t pack_bf16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

TKB_DEVICE float ex2_approx(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// Blackwell packed fp32 pair ops (one FMA-pipe instruction for two lanes of work).
// d = a * b + c, elementwise on (x, y) pairs.
TKB_DEVICE float2 fma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %3}; mov.b64 rb, {%4, %5}; mov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\t"
        "mov.b64 {%0, %1}, rd;}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}
TKB_DEVICE float2 mul2(float2 a, float2 b) {
    float2 d;
    asm("{.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3}; mov.b64 rb, {%4, %5};\n\t"
        "mul.rn.f32x2 rd, ra, rb;\n\t"
        "mov.b64 {%0, %1}, rd;}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
TKB_DEVICE float2 add2(float2 a, float2 b) {
    float2 d;
    asm("{.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3}; mov.b64 rb, {%4, %5};\n\t"
        "add.rn.f32x2 rd, ra, rb;\n\t"
        "mov.b64 {%0, %1}, rd;}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
TKB_DEVICE float2 sub2(float2 a, float2 b) {
    float2 d;
    asm("{.reg .b64 ra, rb, rd;\n\t"
        "mov.b64 ra, {%2, %3}; mov.b64 rb, {%4, %5};\n\t"
        "sub.rn.f32x2 rd, ra, rb;\n\t"
        "mov.b64 {%0, %1}, rd;}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}

// 2^x for a pair on the FMA pipe (no MUFU): 2^floor(x) * p(frac(x)) with a degree-3
// minimax polynomial (max rel. error ~9e-5, below bf16 resolution). x <= 127; x = -inf -> 0.
TKB_DEVICE float2 ex2_poly2(float2 x) {
    x.x = fmaxf(x.x, -127.f);
    x.y = fmaxf(x.y, -127.f);
    float2 r, p;
    asm("{.reg .b64 x, rr, big, bk, fr, c3, c2, c1, c0, p;\n\t"
        "mov.b64 x, {%4, %5};\n\t"
        "mov.b64 big, {%6, %6};\n\t"
        "add.rm.ftz.f32x2 rr, x, big;\n\t"  // integer part in the low mantissa bits
        "sub.rn.ftz.f32x2 bk, rr, big;\n\t"
        "sub.rn.ftz.f32x2 fr, x, bk;\n\t"   // fraction in [0, 1)
        "mov.b64 c3, {%7, %7}; mov.b64 c2, {%8, %8}; mov.b64 c1, {%9, %9}; mov.b64 c0, {%10, %10};\n\t"
        "fma.rn.ftz.f32x2 p, fr, c3, c2;\n\t"
        "fma.rn.ftz.f32x2 p, p, fr, c1;\n\t"
        "fma.rn.ftz.f32x2 p, p, fr, c0;\n\t"
        "mov.b64 {%0, %1}, rr; mov.b64 {%2, %3}, p;}"
        : "=f"(r.x), "=f"(r.y), "=f"(p.x), "=f"(p.y)
        : "f"(x.x), "f"(x.y), "f"(12582912.0f), "f"(0.07711909f), "f"(0.22756439f), "f"(0.69514614f), "f"(1.0f));
    float2 out;
    out.x = __int_as_float((__float_as_int(r.x) << 23) + __float_as_int(p.x));
    out.y = __int_as_float((__float_as_int(r.y) << 23) + __float_as_int(p.y));
    return out;
}

template <int kRegs>
TKB_DEVICE void setmaxnreg_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegs)); }
template <int kRegs>
TKB_DEVICE void setmaxnreg_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegs)); }

}  // namespace tkb
