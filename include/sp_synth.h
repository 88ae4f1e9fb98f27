/*
 * sp_synth.h — seeded synthetic frame generator on the device (bench/test
 * utility; NOT part of the SP hot path, never timed).
 *
 * Same recipe as sp_inputs/__init__.py:
 *   h_f   = splitmix64(seed ^ (f * 0xD1B54A32D192ED03))
 *   u     = splitmix64(h_f ^ i) >> 40                (i = y*W + x)
 *   pixel = u < rho_q24 ? value : 0
 * with splitmix64(x) = mix64(x + 0x9E3779B97F4A7C15) (Vigna's constants).
 * value: nonzero_mode 0 -> 255, 1 -> 1, 2 -> (u64 hash & 0xFF) | 1.
 * The Python generator and this kernel are cross-checked byte for byte by
 * tests/test_gpu_parity.py.
 */
#ifndef HTM_SP_SYNTH_H
#define HTM_SP_SYNTH_H

#include <stdint.h>
#include "sp.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Writes frames first_frame .. first_frame+num_frames-1 of the stream into
 * frames_dev: uint8[num_frames][height][width] (device memory, caller-owned).
 * rho_q24 in [0, 2^24].  Errors: SP_E_ARG, SP_E_CUDA.  Asynchronous. */
sp_status sp_synth_frames(uint8_t* frames_dev, uint64_t first_frame, uint32_t num_frames,
                          uint32_t height, uint32_t width, uint64_t seed, uint32_t rho_q24,
                          uint32_t nonzero_mode, void* cuda_stream);

/* Colour frames for the encoder, uint8[num_frames][height][width][3]
 * BGR, same recipe as sp_inputs.bgr_frames (integer-only):
 *   base  = ((x*(c+1)) >> 2) + (y >> 1) + 5f + (128 inside the disc (x-cx)^2+(y-cy)^2 < r^2,
 *           cx = (17f+200) % W, cy = (11f+150) % H, r = min(H,W)/7)
 *   value = (base + (splitmix64(h_f ^ ((y*W+x)*3 + c)) >> 59)) & 255
 * Errors: SP_E_ARG, SP_E_CUDA.  Asynchronous. */
sp_status sp_synth_bgr_frames(uint8_t* frames_dev, uint64_t first_frame, uint32_t num_frames,
                              uint32_t height, uint32_t width, uint64_t seed, void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* HTM_SP_SYNTH_H */
