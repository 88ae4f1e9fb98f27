// Microbenchmark (development aid, not part of libsp): streaming rate of 2D tensor TMA
// (cp.async.bulk.tensor.2d) boxes of {bx bytes, by rows} vs the row-wise bulk copies.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bench_tma scripts/bench_tma.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Each CTA streams rows [blockIdx.x*32, +32) of a [R][X] uint8 tensor, columns in steps of bx
// per box; `per_stage` boxes (consecutive column steps) make one stage.
__global__ void __launch_bounds__(32, 1) k_tma(const __grid_constant__ CUtensorMap map, int X, int bx,
                                               int by, int per_stage, int nst, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int stage_bytes = bx * by * per_stage;
    uint64_t* bars = (uint64_t*)(smem + (size_t)nst * stage_bytes);
    if (threadIdx.x < nst) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bars[threadIdx.x])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    __syncthreads();
    const int iters = X / (bx * per_stage);
    const int row0 = blockIdx.x * by;
    auto issue = [&](int j) {
        int st = j % nst;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bars[st])), "r"(stage_bytes));
        for (int b = 0; b < per_stage; ++b) {
            int x = (j * per_stage + b) * bx;
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                ::"r"(sa(smem + (size_t)st * stage_bytes + (size_t)b * bx * by)), "l"(&map), "r"(x), "r"(row0),
                "r"(sa(&bars[st])) : "memory");
        }
    };
    unsigned long long acc = 0;
    if (threadIdx.x == 0) {
        for (int j = 0; j < nst && j < iters; ++j) issue(j);
        for (int j = 0; j < iters; ++j) {
            int st = j % nst;
            uint32_t par = (j / nst) & 1;
            asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n"
                         ::"r"(sa(&bars[st])), "r"(par) : "memory");
            acc += smem[(size_t)st * stage_bytes];
            if (j + nst < iters) issue(j + nst);
        }
        sink[blockIdx.x] = acc;
    }
}

int main() {
    const int sms = 148, rows_per_cta = 32;
    const int R = sms * rows_per_cta;
    const int X = 518400 / 2048 * 2048 - 2048 * 4;  // ~ one frame per row
    uint8_t* buf;
    unsigned long long* sink;
    cudaMalloc(&buf, (size_t)R * 518400);
    cudaMalloc(&sink, sms * 8);
    cudaMemset(buf, 1, (size_t)R * 518400);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    int bxs[] = {64, 128, 256};
    int bys[] = {28, 32};
    int pss[] = {1, 2, 4, 8, 16};
    int nsts[] = {2, 3, 4};
    int swz[] = {0, 1};
    for (int sw : swz)
        for (int bx : bxs)
            for (int by : bys)
                for (int ps : pss)
                    for (int nst : nsts) {
                        if (sw && bx > 128) continue;
                        size_t sb = (size_t)bx * by * ps;
                        if (sb * nst + 64 > 227 * 1024 || sb * nst < 16384) continue;
                        CUtensorMap map;
                        cuuint64_t dims[2] = {(cuuint64_t)518400, (cuuint64_t)R};
                        cuuint64_t strides[1] = {518400};
                        cuuint32_t box[2] = {(cuuint32_t)bx, (cuuint32_t)by};
                        cuuint32_t es[2] = {1, 1};
                        CUresult r = cuTensorMapEncodeTiled(
                            &map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE,
                            sw ? (bx == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B)
                               : CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                        if (r != CUDA_SUCCESS) { printf("encode failed %d bx=%d by=%d sw=%d\n", r, bx, by, sw); continue; }
                        cudaEventRecord(a);
                        k_tma<<<sms, 32, sb * nst + 64>>>(map, X, bx, by, ps, nst, sink);
                        cudaEventRecord(b);
                        cudaError_t e = cudaEventSynchronize(b);
                        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
                        float ms;
                        cudaEventElapsedTime(&ms, a, b);
                        int iters = X / (bx * ps);
                        double bytes = (double)iters * sb * sms;
                        printf("tma2d sw=%d box=%3dx%2d per_stage=%2d nst=%d stage=%6zu B: %7.1f GB/s (%.1f GB/s/SM)\n", sw,
                               bx, by, ps, nst, sb, bytes / ms / 1e6, bytes / ms / 1e6 / sms);
                    }
    return 0;
}
