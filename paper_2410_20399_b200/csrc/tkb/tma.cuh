// tma.cuh — global <-> shared tile movement (the `load`/`store` of gl/st).
//
// Reference: kittensim's global->shared `load` places every element through
// element_offset() with the SW128 XOR rule (tiles.hpp:416-426,
// layouts.hpp:111-132). Here the Tensor Memory Accelerator does the same
// placement in hardware (CU_TENSOR_MAP_SWIZZLE_128B): 16-byte chunk c of row r
// lands at chunk c ^ (r % 8) of a 128-byte row, which equals the reference rule
// at a 128-B row pitch. Tiles wider than 128 B are stored as several 128-B-wide
// column blocks ("atoms").
#pragma once
#include "mbarrier.cuh"

namespace tkb {
namespace tma {

TKB_DEVICE void prefetch_desc(const void* tmap) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}

// A tensor map written in global memory by an earlier kernel (tensormap.replace, the
// per-sequence maps of variable-length batches): invalidate this SM's cached copy of the
// descriptor at that address before the calling thread's next TMA through it.
TKB_DEVICE void acquire_map(const void* tmap) {
    asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(reinterpret_cast<uint64_t>(tmap))
                 : "memory");
}

// L2 cache policies (createpolicy.fractional.L2::evict_*).
TKB_DEVICE uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
TKB_DEVICE uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// 4-D tiled load {c0 innermost .. c3}; completes `bytes` on mbarrier `bar`.
TKB_DEVICE void load_4d(void* smem_dst, const void* tmap, mbarrier* bar, int c0, int c1, int c2, int c3,
                        uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
        "l"(policy)
        : "memory");
}

TKB_DEVICE void load_2d(void* smem_dst, const void* tmap, mbarrier* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// Non-tensor bulk copy global -> shared (16-byte aligned, size multiple of 16).
TKB_DEVICE void load_1d(void* smem_dst, const void* gsrc, uint32_t bytes, mbarrier* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(gsrc)), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

TKB_DEVICE void store_2d(const void* tmap, const void* smem_src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(tmap)),
                 "r"(smem_u32(smem_src)), "r"(c0), "r"(c1)
                 : "memory");
}

TKB_DEVICE void store_3d(const void* tmap, const void* smem_src, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
            reinterpret_cast<uint64_t>(tmap)),
        "r"(smem_u32(smem_src)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

TKB_DEVICE void reduce_add_3d(const void* tmap, const void* smem_src, int c0, int c1, int c2) {
    asm volatile(
        "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
            reinterpret_cast<uint64_t>(tmap)),
        "r"(smem_u32(smem_src)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

// L2 prefetch of a 4-D tile (no SMEM destination, no barrier).
TKB_DEVICE void prefetch_4d(const void* tmap, int c0, int c1, int c2, int c3) {
    asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(
                     reinterpret_cast<uint64_t>(tmap)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(c3)
                 : "memory");
}

// Order generic-proxy global accesses with async-proxy (TMA) ones.
TKB_DEVICE void fence_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

TKB_DEVICE void store_4d(const void* tmap, const void* smem_src, int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
            reinterpret_cast<uint64_t>(tmap)),
        "r"(smem_u32(smem_src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}

// Element-wise add-reduce of an smem tile into global (fp32): used for dQ.
TKB_DEVICE void reduce_add_4d(const void* tmap, const void* smem_src, int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.reduce.async.bulk.tensor.4d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, %4, %5}], "
        "[%1];" ::"l"(reinterpret_cast<uint64_t>(tmap)),
        "r"(smem_u32(smem_src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}

TKB_DEVICE void commit_group() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

template <int N>
TKB_DEVICE void wait_group_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
TKB_DEVICE void wait_group() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// Generic-proxy smem writes -> visible to TMA (async proxy) reads.
TKB_DEVICE void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

}  // namespace tma
}  // namespace tkb
