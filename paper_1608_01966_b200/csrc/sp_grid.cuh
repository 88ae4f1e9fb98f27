// sp_grid.cuh -- building blocks of the grid-resident (cooperative, one CTA per SM) learning
// kernels (sp_learn_grid.cu, sp_learn_grid_full.cu).
#pragma once

#include <cstdint>

namespace sp {

// Grid-wide barrier number m (0, 1, ..) over G co-resident CTAs: a monotonic arrival counter
// in global memory (zeroed before the launch); the CTA barrier makes the CTA's writes part of
// thread 0's causality order, its red.release publishes them at gpu scope, the ld.acquire spin
// observes every CTA's arrival.
__device__ __forceinline__ void grid_barrier(uint32_t* gbar, uint32_t target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(gbar) : "memory");
        uint32_t v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gbar) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

// one thread: bulk copy of bytes [src, src + bytes) into smem dst, completion on bar
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    constexpr uint32_t kChunk = 32768u;
    for (uint32_t off = 0; off < bytes; off += kChunk) {
        const uint32_t n = min(kChunk, bytes - off);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                static_cast<uint32_t>(__cvta_generic_to_shared(static_cast<uint8_t*>(dst) + off))),
            "l"(static_cast<const uint8_t*>(src) + off), "r"(n), "r"(b)
            : "memory");
    }
}

}  // namespace sp
