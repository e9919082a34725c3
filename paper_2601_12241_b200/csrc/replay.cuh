// replay.cuh — shared pieces of the replay kernels: trace/scratch views, the
// per-replay result, and the TMA (cp.async.bulk + mbarrier) staging helpers.
//
// History: the first (v0) joint replay kernel lived here — per-thread worker
// state in local memory, one instant per loop, member scans for decode
// batches.  It was replaced by static_path.cuh (factorized static path) and
// dynamic_path.cuh (joint kernel, N ≤ 8 and N ≤ 64); see DESIGN.md §5 and
// profiles/r1_v0_*.txt for why.
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"
#include "controller.cuh"

namespace padsim {

#define PAD_INF __longlong_as_double(0x7ff0000000000000ULL)

enum : unsigned char { F_DRAIN = 1, F_DIRTY = 2, F_BND = 4, F_CHG = 8 };

struct TraceView {
    const double* s_unit;
    const double* kv;
    const int* in_tok;
    const int* out_tok;
    const unsigned char* phase;
    int R;
};

// lane-interleaved scratch accessors
struct Scratch {
    int* link;             // [i*32]
    double* pe;            // [i*32]
    int2* mem;             // [(g*max_db + k)*32]  {fin, id}
    int* ordt;             // [k*32] TTFT window: request ids in prefill-end order
    double* tst;           // [k] per lane (lane·Rmax + k) TPOT window: completion stamps
    unsigned char* tfl;    // [k] per lane, TPOT window: flags (le0, lt0, le1, lt1)
};

struct ReplayResult {
    int met, near;
    double duration, goodput;
    long long events;
    double watts;                  // time-weighted mean of Σ effective caps
};

// ---------------------------------------------------------------------------
// TMA (cp.async.bulk) trace staging helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
    unsigned done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    }
}

}  // namespace padsim
