// sp_synth.cu — seeded synthetic frames on the device (bench/test utility, never timed).
// Recipe of include/sp_synth.h / sp_inputs/__init__.py.
#include "sp_internal.h"
#include "../../include/sp_synth.h"

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// 16 pixels per thread, one uint4 store when the row of 16 is in range and aligned.
__global__ void k_synth(uint8_t* out, uint64_t first, uint32_t npix, uint64_t seed, uint32_t thr,
                        uint32_t mode) {
    const uint32_t f = blockIdx.y;
    const uint64_t hf = splitmix64(seed ^ ((first + f) * 0xD1B54A32D192ED03ull));
    uint8_t* fr = out + static_cast<size_t>(f) * npix;
    const uint32_t i0 = (blockIdx.x * blockDim.x + threadIdx.x) * 16u;
    if (i0 >= npix) return;
    uint8_t v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const uint64_t h = splitmix64(hf ^ static_cast<uint64_t>(i0 + j));
        const bool on = (h >> 40) < thr;
        const uint8_t val = mode == 0 ? 255u : (mode == 1 ? 1u : static_cast<uint8_t>((h & 0xFFu) | 1u));
        v[j] = on ? val : 0u;
    }
    const bool aligned = ((reinterpret_cast<uintptr_t>(fr + i0)) & 15u) == 0;
    if (i0 + 16u <= npix && aligned) {
        uint4 w;
        w.x = v[0] | (v[1] << 8) | (v[2] << 16) | (static_cast<uint32_t>(v[3]) << 24);
        w.y = v[4] | (v[5] << 8) | (v[6] << 16) | (static_cast<uint32_t>(v[7]) << 24);
        w.z = v[8] | (v[9] << 8) | (v[10] << 16) | (static_cast<uint32_t>(v[11]) << 24);
        w.w = v[12] | (v[13] << 8) | (v[14] << 16) | (static_cast<uint32_t>(v[15]) << 24);
        *reinterpret_cast<uint4*>(fr + i0) = w;
    } else {
        for (uint32_t j = 0; j < 16u && i0 + j < npix; ++j) fr[i0 + j] = v[j];
    }
}

// Colour frames for the encoder (recipe in include/sp_synth.h), one thread per pixel.
__global__ void k_synth_bgr(uint8_t* out, uint64_t first, uint32_t H, uint32_t W, uint64_t seed) {
    const uint32_t f = blockIdx.y;
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;  // pixel
    if (i >= H * W) return;
    const int64_t fi = static_cast<int64_t>(first + f);
    const int64_t y = i / W, x = i % W;
    const uint64_t hf = splitmix64(seed ^ ((first + f) * 0xD1B54A32D192ED03ull));
    const int64_t cx = (17 * fi + 200) % W, cy = (11 * fi + 150) % H, r = min(H, W) / 7;
    const bool disc = (x - cx) * (x - cx) + (y - cy) * (y - cy) < r * r;
    uint8_t* px = out + (static_cast<size_t>(f) * H * W + i) * 3u;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const int64_t base = ((x * (c + 1)) >> 2) + (y >> 1) + 5 * fi + (disc ? 128 : 0);
        const uint64_t noise = splitmix64(hf ^ (static_cast<uint64_t>(i) * 3u + c)) >> 59;
        px[c] = static_cast<uint8_t>((base + static_cast<int64_t>(noise)) & 255);
    }
}

}  // namespace

extern "C" sp_status sp_synth_bgr_frames(uint8_t* frames_dev, uint64_t first_frame, uint32_t num_frames,
                                         uint32_t height, uint32_t width, uint64_t seed, void* cuda_stream) {
    if (num_frames == 0) return SP_OK;
    if (!frames_dev || height == 0 || width == 0) return SP_E_ARG;
    dim3 grid((height * width + 255u) / 256u, num_frames);
    k_synth_bgr<<<grid, 256, 0, static_cast<cudaStream_t>(cuda_stream)>>>(frames_dev, first_frame, height, width,
                                                                           seed);
    return cudaGetLastError() == cudaSuccess ? SP_OK : SP_E_CUDA;
}

extern "C" sp_status sp_synth_frames(uint8_t* frames_dev, uint64_t first_frame, uint32_t num_frames,
                                     uint32_t height, uint32_t width, uint64_t seed, uint32_t rho_q24,
                                     uint32_t nonzero_mode, void* cuda_stream) {
    if (num_frames == 0) return SP_OK;
    if (!frames_dev || height == 0 || width == 0 || rho_q24 > (1u << 24) || nonzero_mode > 2)
        return SP_E_ARG;
    const uint32_t npix = height * width;
    dim3 grid((npix + 16u * 256u - 1u) / (16u * 256u), num_frames);
    k_synth<<<grid, 256, 0, static_cast<cudaStream_t>(cuda_stream)>>>(frames_dev, first_frame, npix,
                                                                       seed, rho_q24, nonzero_mode);
    return cudaGetLastError() == cudaSuccess ? SP_OK : SP_E_CUDA;
}
