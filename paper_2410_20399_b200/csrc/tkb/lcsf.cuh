// lcsf.cuh — the load-compute-store-finish (LCSF) template on Blackwell.
//
// Reference: kittensim's LCSF executor (lcsf.hpp:38-819): a producer worker fills an
// N-slot input ring, consumer workers compute on it, each slot guarded by a counter
// barrier with generations (Barrier lcsf.hpp:40-54; TaskRun lcsf.hpp:302-379: slot
// = i % stages, generation = i / stages, inputs_arrived expects 1 arrival,
// inputs_finished expects one per consumer), tasks enumerated with the sequence
// block innermost (make_common, kernels.hpp:267-275).
//
// On B200 the workers are warp roles of one persistent CTA:
//   ring<S>        the N-slot ring; full[s] completes on TMA transaction bytes (the
//                  producer's arrive + expect_tx), empty[s] on the consumers' release
//                  (a tcgen05.commit when the consumer is the tensor core);
//                  phase parity = generation & 1
//   ring_state     (slot, phase) cursor that every role advances in lockstep
//   work_queue     the persistent task scheduler: one producer lane claims task ids
//                  from a global atomic counter (dynamic, so heavy causal tasks first
//                  balance across SMs) and broadcasts them through a 2-slot SMEM ring
//                  to the other roles; the counter resets itself at grid exit.
//
// kernel<T>: the LCSF kernel skeleton (the reference's KernelSpec callbacks,
// lcsf.hpp:112-161, and the paper's lcf::kernel<attn_fwd_template<D>>),
// persistent and warp-specialised. A template T supplies the layout and the hooks; the
// skeleton owns the SMEM carve-up, barrier / queue initialisation, the TMEM allocation, the
// task queue (claims, broadcast, release), the role dispatch and the grid exit:
//   using globals; struct shared { ... work_queue queue; uint32_t tmem_slot; }
//   kThreads, kTmemCols, kProducerWarp, kMmaWarp, kConsumerWarps (warps [0, kConsumerWarps)),
//   kQueueReaders (MMA warp + consumer warps), kAlignSlack (1024-align the dynamic window
//   vs. require it aligned), kReleaseEarly (consumers release a task id on reading it, or
//   after their finish)
//   static void init(shared&, const globals&)          barrier init, descriptor prefetch
//   static int num_tasks(const globals&); static int* counter(const globals&)
//   static bool skip(const globals&, int task)         optional: the task is empty (never dispatched)
//   producer::state, producer::load(args, state&, task, n, claim_next), producer::drain
//       (the LCSF load stage; claim_next() claims task n + 1 when the hook wants it —
//        e.g. to warm its inputs in L2 — otherwise the skeleton claims after load returns)
//   mma::state, mma::issue(args, state&, task, n)       the tensor-core half of compute
//   consumer::state, consumer::compute(args, state&, task, n), consumer::finish(...),
//   consumer::drain(args, state&)                        compute (softmax etc.) + finish
//   kAuxWarps, kAuxWarp0, aux::run(args, index)         optional warps outside the task queue
//                                                        (e.g. a prologue producing inputs)
#pragma once
#include "mbarrier.cuh"
#include "tcgen05.cuh"

namespace tkb {
namespace lcsf {

// (slot, phase) cursor over an S-slot ring
template <int S>
struct ring_state {
    int slot = 0;
    uint32_t phase = 0;
    TKB_DEVICE void advance() {
        if (++slot == S) {
            slot = 0;
            phase ^= 1u;
        }
    }
};

template <int S>
struct ring {
    mbarrier full[S];
    mbarrier empty[S];
    TKB_DEVICE void init(uint32_t full_count, uint32_t empty_count) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], full_count);
            mbar_init(&empty[s], empty_count);
        }
    }
    // producer side: wait until the consumers released generation (phase ^ 1) of this slot
    TKB_DEVICE void wait_empty(const ring_state<S>& st) { mbar_wait(&empty[st.slot], st.phase ^ 1u); }
    // consumer side: wait until the producer filled the current generation
    TKB_DEVICE void wait_full(const ring_state<S>& st) { mbar_wait(&full[st.slot], st.phase); }
};

// Persistent task queue (ids in [0, total)); -1 terminates.
struct work_queue {
    static constexpr int kSlots = 2;
    int id[kSlots];
    mbarrier full[kSlots];
    mbarrier empty[kSlots];
    TKB_DEVICE void init(uint32_t consumers) {
        for (int s = 0; s < kSlots; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], consumers);
        }
    }
    // producer lane: claim the n-th task of this CTA (n = 0 is blockIdx.x) and publish it;
    // ids for which skip(id) holds (empty tasks, e.g. query blocks past a short sequence of a
    // variable-length batch) are passed over here, so no other role ever sees them
    template <class Skip>
    TKB_DEVICE int claim(int n, int* counter, int total, Skip&& skip) {
        int t = (n == 0) ? (int)blockIdx.x : (int)gridDim.x + atomicAdd(counter, 1);
        while (t < total && skip(t)) t = (int)gridDim.x + atomicAdd(counter, 1);
        if (t >= total) t = -1;
        const int s = n % kSlots;
        mbar_wait(&empty[s], ((n / kSlots) & 1) ^ 1u);
        id[s] = t;
        mbar_arrive(&full[s]);  // release: the id store is visible to acquirers
        return t;
    }
    // consumer: read the n-th task (one lane per warp calls release() after use)
    TKB_DEVICE int get(int n) {
        const int s = n % kSlots;
        mbar_wait(&full[s], (n / kSlots) & 1);
        return *reinterpret_cast<volatile int*>(&id[s]);
    }
    // warp-collective get(): the id comes back warp-uniform (a shuffle from lane 0), so the
    // task-derived loop bounds and addresses stay in uniform registers — an MMA warp whose
    // descriptors depend on a per-thread id would pay R2UR / VOTEU per tcgen05.mma
    TKB_DEVICE int get_warp(int n) { return __shfl_sync(0xffffffffu, get(n), 0); }
    TKB_DEVICE void release(int n) { mbar_arrive(&empty[n % kSlots]); }
};

// Grid exit: the last CTA resets the task counter so the next launch starts at zero.
// counter[0] = claims beyond the grid, counter[1] = CTAs finished, counter[3] = a second
// (auxiliary) work counter some kernels use (the fused rotary prologue's block claims).
TKB_DEVICE void queue_exit(int* counter) {
    __threadfence();
    if (atomicAdd(&counter[1], 1) == (int)gridDim.x - 1) {
        counter[0] = 0;
        counter[1] = 0;
        counter[3] = 0;
        __threadfence();
    }
}

// Cross-CTA block flags (a producer publishes a global-memory block for other CTAs' TMA
// loads): the writer's generic-proxy stores are made visible to the async proxy and the
// flag is a gpu-scope release; the reader acquires the flag, then fences the async proxy
// before its TMA reads the block. The wait is bounded like mbar_wait (TKB_DEADLOCK_NS).
// writer: every thread that wrote part of the block calls flag_writer_fence(), then the warp
// syncs, then one thread publishes (the release is cumulative over the synced writes)
TKB_DEVICE void flag_writer_fence() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
TKB_DEVICE void flag_publish(unsigned* f, unsigned v) {
    __threadfence();
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}
TKB_DEVICE unsigned flag_load(const unsigned* f) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    return v;
}
TKB_DEVICE void flag_wait(const unsigned* f, unsigned v) {
    if (flag_load(f) != v) {
        uint64_t t0 = globaltimer_ns();
        while (flag_load(f) != v) {
#ifndef TKB_NO_DEADLOCK_TRAP
            if (globaltimer_ns() - t0 > (uint64_t)(TKB_DEADLOCK_NS)) __trap();
#endif
            __nanosleep(64);
        }
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Wait for a run of flags [f, f + n) to all carry v: relaxed polls (up to 16 in flight per
// round), then one acquire fence for the lot — one L2 round trip per round instead of one
// per flag.
TKB_DEVICE void flags_wait_all(const unsigned* f, int n, unsigned v) {
    uint64_t t0 = 0;
    for (int i0 = 0; i0 < n;) {
        unsigned x[16];
        const int m = min(16, n - i0);
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (j < m) asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(x[j]) : "l"(f + i0 + j) : "memory");
        int ok = 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) ok += (j < m && x[j] == v) ? 1 : 0;
        if (ok == m) {
            i0 += m;
            continue;
        }
        if (t0 == 0) t0 = globaltimer_ns();
#ifndef TKB_NO_DEADLOCK_TRAP
        else if (globaltimer_ns() - t0 > (uint64_t)(TKB_DEADLOCK_NS)) __trap();
#endif
        __nanosleep(64);
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Everything a hook sees: the kernel parameters, the SMEM layout, the task queue (to peek at
// the next task), the TMEM base, and the calling thread's warp / lane.
template <class T>
struct args {
    const typename T::globals& g;
    typename T::shared& sh;
    work_queue& queue;
    uint32_t tmem;
    int warp, lane;
};

// optional hook: static bool T::skip(const globals&, int task) — the task has no work
template <class T, class = void>
struct has_skip {
    static constexpr bool value = false;
};
template <class T>
struct has_skip<T, decltype((void)T::skip(*(const typename T::globals*)nullptr, 0))> {
    static constexpr bool value = true;
};

template <class T>
__global__ void __launch_bounds__(T::kThreads, 1) kernel(const __grid_constant__ typename T::globals g) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = smem_raw;
    if constexpr (T::kAlignSlack) {
        base += (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;  // SW128 tiles need 1024-byte alignment
    } else if ((smem_u32(smem_raw) & 1023u) != 0) {
        __trap();  // no slack budgeted: the dynamic window must start aligned (no static SMEM)
    }
    typename T::shared& sh = *reinterpret_cast<typename T::shared*>(base);
    const int warp = warpid();
    const int lane = laneid();
    if (warp == T::kProducerWarp && lane == 0) {
        sh.queue.init(T::kQueueReaders);
        T::init(sh, g);
        fence_barrier_init();
    }
    if (warp == T::kMmaWarp) tmem::alloc<T::kTmemCols>(&sh.tmem_slot);
    tmem::fence_before();
    __syncthreads();
    tmem::fence_after();
    const args<T> a{g, sh, sh.queue, sh.tmem_slot, warp, lane};
    int* const counter = T::counter(g);
    const int total = T::num_tasks(g);

    if (warp == T::kProducerWarp) {
        // ------------------------------------------------------------- LOAD (producer)
        if (lane == 0) {
            typename T::producer::state st{};
            int n = 0;
            auto skip = [&](int id) {
                if constexpr (has_skip<T>::value) return T::skip(g, id);
                return false;
            };
            int t = sh.queue.claim(0, counter, total, skip);
            while (t >= 0) {
                int next = -2;
                auto claim_next = [&]() {
                    if (next == -2) next = sh.queue.claim(n + 1, counter, total, skip);
                    return next;
                };
                T::producer::load(a, st, t, n, claim_next);
                t = claim_next();
                ++n;
            }
            T::producer::drain(a, st);
        }
    } else if (warp == T::kMmaWarp) {
        // ------------------------------------------------------------- MMA (converged warp)
        typename T::mma::state st{};
        for (int n = 0;; ++n) {
            const int t = sh.queue.get_warp(n);
            if (lane == 0) sh.queue.release(n);
            if (t < 0) break;
            T::mma::issue(a, st, t, n);
        }
    } else if (warp < T::kConsumerWarps) {
        // ------------------------------------------------------------- COMPUTE + FINISH
        typename T::consumer::state st{};
        for (int n = 0;; ++n) {
            const int t = sh.queue.get_warp(n);
            if (T::kReleaseEarly) {
                __syncwarp();
                if (lane == 0) sh.queue.release(n);
            }
            if (t < 0) break;
            T::consumer::compute(a, st, t, n);
            T::consumer::finish(a, st, t, n);
            if (!T::kReleaseEarly) {
                __syncwarp();
                if (lane == 0) sh.queue.release(n);
            }
        }
        T::consumer::drain(a, st);
    }
    if constexpr (T::kAuxWarps > 0) {
        if (warp >= T::kAuxWarp0 && warp < T::kAuxWarp0 + T::kAuxWarps) T::aux::run(a, warp - T::kAuxWarp0);
    }

    tmem::fence_before();
    __syncthreads();
    if (warp == T::kMmaWarp) tmem::dealloc<T::kTmemCols>(sh.tmem_slot);
    if (threadIdx.x == 0) queue_exit(counter);
}

}  // namespace lcsf
}  // namespace tkb
