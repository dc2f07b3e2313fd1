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

// Named barriers (ids 1..15; id 0 is __syncthreads).
TKB_DEVICE void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
TKB_DEVICE void named_arrive(int id, int nthreads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Pack two fp32 into bf16x2 with RNE (lo -> bits 0..15, hi -> bits 16..31).
// Matches round_to_bf16 (tiles.hpp:40-46) for finite inputs.
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

template <int kRegs>
TKB_DEVICE void setmaxnreg_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegs)); }
template <int kRegs>
TKB_DEVICE void setmaxnreg_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegs)); }

}  // namespace tkb
