// spk_smallk.cuh — device helpers shared by the small-k engine's kernels
// (spk_smallk.cu, spk_smallk_solve.cu): the cooperative grid barrier and the
// TMA bulk-copy / mbarrier primitives.
#pragma once

#include <cuda_runtime.h>

#include "spk_launch.h"

namespace spk {
namespace {

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Grid barrier of a cooperative launch: one monotonic arrival counter (*bar,
// zeroed before the launch); barrier number b of the kernel waits until every
// CTA has arrived b times.  One atomic per CTA, no reset.
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& target) {
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        while (ld_acquire_u32(bar) < target) __nanosleep(32);
    }
    __syncthreads();
}

__device__ __forceinline__ void mbar_init1(unsigned long long* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                     (unsigned)__cvta_generic_to_shared(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait0(unsigned long long* bar) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n"
        " .reg .pred p;\n"
        "SKW_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
        " @!p bra SKW_%=;\n"
        "}\n" ::"r"(a)
        : "memory");
}
// TMA 1-D bulk copy global -> shared, completion on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            (unsigned)__cvta_generic_to_shared(dst)),
        "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
        : "memory");
}

// cp.async (LDGSTS) 8-byte copy global -> shared, no register round trip;
// sk_cp_wait_all waits for all of the thread's copies
__device__ __forceinline__ void sk_cp8(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void sk_cp_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

__device__ __forceinline__ void sk_stamp(unsigned long long* trace, int ph, int mark) {
    if (trace && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        trace[((long long)ph * gridDim.x + blockIdx.x) * 4 + mark] = t;
    }
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

}  // namespace

// CTAs of a cooperative launch: all resident at once
inline int sk_coop_grid(const void* fn, int threads, size_t smem) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem);
    (void)per_sm;  // one CTA per SM: fewer barrier arrivals, no oversubscription
    return device_sms();
}

}  // namespace spk
