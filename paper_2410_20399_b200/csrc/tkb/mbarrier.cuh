// mbarrier.cuh — the hardware form of the LCSF counter barrier.
//
// Reference semantics: kittensim::Barrier (lcsf.hpp:40-54) counts arrivals per
// generation; a slot s of the N-stage ring is used by iteration i with
// generation i / stages (lcsf.hpp:302-379). On Blackwell the same contract is
// an mbarrier whose phase parity is generation & 1: a consumer waits on
// full[s] with parity (i / stages) & 1, a producer waits on empty[s] with the
// opposite parity before overwriting the slot.
#pragma once
#include "common.cuh"

namespace tkb {

struct alignas(8) mbarrier {
    uint64_t word;
};

TKB_DEVICE void mbar_init(mbarrier* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}

// Make barrier inits visible to the async proxy (TMA, tcgen05.commit).
TKB_DEVICE void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

TKB_DEVICE void mbar_arrive(mbarrier* b) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}

// Arrive without release semantics: for hand-offs of TMEM data (ordered by the tcgen05
// fences) where no generic-proxy memory written before the arrive is read by the waiter.
// A release arrive would first wait for the thread's outstanding global stores.
TKB_DEVICE void mbar_arrive_relaxed(mbarrier* b) {
    asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}

TKB_DEVICE void mbar_arrive_cnt(mbarrier* b, uint32_t cnt) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt)
                 : "memory");
}

// Arrive once and announce `bytes` of TMA transactions for this phase.
TKB_DEVICE void mbar_arrive_expect_tx(mbarrier* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}

TKB_DEVICE bool mbar_try_wait(mbarrier* b, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}

// Non-blocking: has the phase with this parity completed?
TKB_DEVICE bool mbar_test_wait(mbarrier* b, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}

TKB_DEVICE uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Blocking wait for the phase with the given parity to complete. A wait that has spun
// for TKB_DEADLOCK_NS (20 s) traps instead of hanging the GPU: the DeadlockError analogue
// of the reference (lcsf.hpp:486-489); the launch then fails with a CUDA error that the
// C ABI reports as TKB_ERR_CUDA. -DTKB_NO_DEADLOCK_TRAP removes the bound.
#ifndef TKB_DEADLOCK_NS
#define TKB_DEADLOCK_NS 20000000000ull
#endif
TKB_DEVICE void mbar_wait(mbarrier* b, uint32_t parity) {
#ifndef TKB_NO_DEADLOCK_TRAP
    if (mbar_try_wait(b, parity)) return;
    uint32_t spins = 0;
    uint64_t t0 = 0;
    while (!mbar_try_wait(b, parity)) {
        if ((++spins & 4095u) == 0) {
            const uint64_t now = globaltimer_ns();
            if (t0 == 0)
                t0 = now;
            else if (now - t0 > (uint64_t)(TKB_DEADLOCK_NS))
                __trap();
        }
    }
#else
    while (!mbar_try_wait(b, parity)) {
    }
#endif
}

}  // namespace tkb
