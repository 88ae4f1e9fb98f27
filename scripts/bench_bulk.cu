// Microbenchmark (development aid, not part of libsp): per-SM streaming rate of
// cp.async.bulk rings vs plain LDG.128, to size the batched kernel's staging.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bench_bulk scripts/bench_bulk.cu
// Each CTA streams its own contiguous slice of a 2 GiB buffer; rows of `sz` bytes
// are taken `rows` at a time from `rows` sub-streams (like 32 frames of a group).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(1024, 1) k_bulk(const uint8_t* buf, size_t slice, int sz, int rows,
                                                  int nst, int iters, unsigned long long* sink) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* bars = (uint64_t*)(smem + (size_t)nst * rows * sz);
    const uint8_t* base = buf + (size_t)blockIdx.x * slice;
    const size_t sub = slice / rows / 16 * 16;  // each row-stream gets slice/rows bytes
    if (threadIdx.x < nst) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bars[threadIdx.x])));
    __syncthreads();
    auto issue = [&](int j) {
        int st = j % nst;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bars[st])), "r"(sz * rows));
        for (int r = 0; r < rows; ++r)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(sa(smem + (size_t)(st * rows + r) * sz)), "l"(base + r * sub + (size_t)j * sz),
                         "r"(sz), "r"(sa(&bars[st])) : "memory");
    };
    unsigned long long acc = 0;
    if (threadIdx.x == 0) {
        for (int j = 0; j < nst && j < iters; ++j) issue(j);
        for (int j = 0; j < iters; ++j) {
            int st = j % nst;
            uint32_t par = (j / nst) & 1;
            asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n"
                         ::"r"(sa(&bars[st])), "r"(par) : "memory");
            acc += smem[(size_t)st * rows * sz];
            if (j + nst < iters) issue(j + nst);
        }
        sink[blockIdx.x] = acc;
    }
}

__global__ void __launch_bounds__(1024, 1) k_ldg(const uint4* buf, size_t slice16, unsigned long long* sink) {
    const uint4* base = buf + (size_t)blockIdx.x * slice16;
    uint32_t acc = 0;
    for (size_t i = threadIdx.x; i < slice16; i += 1024 * 8) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = (i + u * 1024 < slice16) ? __ldg(base + i + u * 1024) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
    }
    if (acc == 0x12345678u) sink[blockIdx.x] = acc;
}

int main() {
    const int sms = 148;
    const size_t total = (size_t)2 << 30;
    const size_t slice = total / sms / 65536 * 65536;
    uint8_t* buf;
    unsigned long long* sink;
    cudaMalloc(&buf, total);
    cudaMalloc(&sink, sms * 8);
    cudaMemset(buf, 1, total);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    // LDG baseline
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        k_ldg<<<sms, 1024>>>((const uint4*)buf, slice / 16, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("LDG.128 x8 unroll: %.1f GB/s\n", slice * sms / ms / 1e6);
    int szs[] = {512, 1024, 2048, 4096, 8192, 16384};
    int rowss[] = {1, 4, 8, 16, 28, 32};
    int nsts[] = {2, 3, 4, 6, 8};
    for (int sz : szs)
        for (int rows : rowss)
            for (int nst : nsts) {
                size_t smem = (size_t)nst * rows * sz + 64;
                if (smem > 227 * 1024) continue;
                if ((size_t)sz * rows * nst < 32768) continue;
                int iters = (int)(slice / rows / 16 * 16 / sz);
                cudaEventRecord(a);
                k_bulk<<<sms, 32, smem>>>(buf, slice, sz, rows, nst, iters, sink);
                cudaEventRecord(b);
                cudaError_t e = cudaEventSynchronize(b);
                if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
                cudaEventElapsedTime(&ms, a, b);
                double bytes = (double)iters * rows * sz * sms;
                printf("bulk sz=%5d rows=%2d nst=%d inflight=%6zu B: %7.1f GB/s (%.1f GB/s/SM)\n", sz, rows,
                       nst, (size_t)sz * rows * nst, bytes / ms / 1e6, bytes / ms / 1e6 / sms);
            }
    return 0;
}
