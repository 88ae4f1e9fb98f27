// sp_hist.cu — per-video SDR histograms ("histograms of
// consecutive frames are built from SP output on a per-video basis"; DESIGN R22).
//
//   counts[v][c] = #{i in [off[v], off[v+1]) : bit c of sdr[i] set}
//   hist[v][c]   = fp32(counts) / fp32(n_v)   (one IEEE RN division; 0 for an empty video)
//
// k_hist_count: block = 8 warps = 8 consecutive SDR words; lane = column inside the word, so
// a warp's 32 lanes read the same word (one broadcast load per input) and each lane counts its
// bit.  Inputs of a video are split over gridDim.z slices (enough CTAs for the SMs at any
// video count); partial counts meet in global memory with one atomicAdd per (lane, slice).
// k_hist_norm: one thread per (video, column), only when a video was split (else k_hist_count
// writes the final counts and the histogram itself: one launch).
#include <algorithm>

#include "sp_internal.h"

namespace sp {

namespace {

__global__ void __launch_bounds__(256) k_hist_count(const uint32_t* __restrict__ sdr, uint32_t ncw, uint32_t C,
                                                    const uint32_t* __restrict__ off, uint32_t* __restrict__ counts,
                                                    float* __restrict__ hist, uint32_t v0) {
    const uint32_t v = v0 + blockIdx.y;  // videos beyond gridDim.y's 65535 go to further launches
    const uint32_t cw = blockIdx.x * 8u + (threadIdx.x >> 5);
    const uint32_t lane = threadIdx.x & 31u;
    if (cw >= ncw) return;
    const uint32_t lo = off[v], hi = off[v + 1];
    const uint32_t n = hi - lo, nz = gridDim.z;
    const uint32_t b = lo + static_cast<uint32_t>(static_cast<uint64_t>(n) * blockIdx.z / nz);
    const uint32_t e = lo + static_cast<uint32_t>(static_cast<uint64_t>(n) * (blockIdx.z + 1u) / nz);
    const uint32_t* p = sdr + cw;
    uint32_t c0 = 0, c1 = 0, c2 = 0, c3 = 0;
    uint32_t i = b;
    for (; i + 8u <= e; i += 8u) {  // eight independent loads in flight
        uint32_t w[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) w[u] = __ldg(p + static_cast<size_t>(i + u) * ncw);
        c0 += ((w[0] >> lane) & 1u) + ((w[4] >> lane) & 1u);
        c1 += ((w[1] >> lane) & 1u) + ((w[5] >> lane) & 1u);
        c2 += ((w[2] >> lane) & 1u) + ((w[6] >> lane) & 1u);
        c3 += ((w[3] >> lane) & 1u) + ((w[7] >> lane) & 1u);
    }
    for (; i < e; ++i) c0 += (__ldg(p + static_cast<size_t>(i) * ncw) >> lane) & 1u;
    const uint32_t cnt = (c0 + c1) + (c2 + c3);
    const uint32_t c = cw * 32u + lane;
    if (c >= C) return;
    const size_t k = static_cast<size_t>(v) * C + c;
    if (nz > 1u) {  // slices meet in memory (zeroed before the launch)
        if (cnt) atomicAdd(counts + k, cnt);
        return;
    }
    // one slice per video: final counts and the normalised histogram directly
    counts[k] = cnt;
    if (hist) hist[k] = n ? __fdiv_rn(static_cast<float>(cnt), static_cast<float>(n)) : 0.0f;
}

__global__ void k_hist_norm(const uint32_t* __restrict__ counts, const uint32_t* __restrict__ off, uint32_t C,
                            uint32_t V, float* __restrict__ hist) {
    const size_t k = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= static_cast<size_t>(V) * C) return;
    const uint32_t v = static_cast<uint32_t>(k / C);
    const uint32_t n = off[v + 1] - off[v];
    // counts and n are exact in fp32 (< 2^24: n <= max_inputs); the quotient is rounded once
    hist[k] = n ? __fdiv_rn(static_cast<float>(counts[k]), static_cast<float>(n)) : 0.0f;
}

}  // namespace

cudaError_t launch_histograms(const uint32_t* sdr, uint32_t ncw, uint32_t C, const uint32_t* off_dev,
                              uint32_t V, uint32_t max_video_inputs, int sm_count, uint32_t* counts,
                              float* hist, cudaStream_t s, uint32_t* launches) {
    const uint32_t bx = (ncw + 7u) / 8u;
    // slices per video: ~2 CTAs per SM overall, >= 64 inputs per slice
    const uint64_t base = static_cast<uint64_t>(bx) * V;
    uint32_t nz = static_cast<uint32_t>(std::max<uint64_t>(1, (2ull * sm_count + base - 1) / base));
    nz = std::min<uint32_t>(nz, std::max<uint32_t>(1u, (max_video_inputs + 63u) / 64u));
    nz = std::min<uint32_t>(nz, 65535u);
    cudaError_t e = cudaSuccess;
    if (nz > 1u && (e = cudaMemsetAsync(counts, 0, static_cast<size_t>(V) * C * 4u, s)) != cudaSuccess) return e;
    *launches = 0;
    for (uint32_t v0 = 0; v0 < V && e == cudaSuccess; v0 += 65535u) {  // gridDim.y <= 65535
        k_hist_count<<<dim3(bx, std::min(V - v0, 65535u), nz), 256, 0, s>>>(sdr, ncw, C, off_dev, counts, hist,
                                                                           v0);
        ++*launches;
        e = cudaGetLastError();
    }
    if (nz > 1u && hist) ++*launches;
    if (e != cudaSuccess || !hist || nz == 1u) return e;
    const size_t n = static_cast<size_t>(V) * C;
    k_hist_norm<<<static_cast<uint32_t>((n + 255u) / 256u), 256, 0, s>>>(counts, off_dev, C, V, hist);
    return cudaGetLastError();
}

}  // namespace sp
