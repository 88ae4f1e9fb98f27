/*
 * sp_encoder.h — C ABI of the on-device adaptive video encoder, the
 * step before the SP hot path: "an original video frame is converted to a binary image ...
 * first reduced in size ... converted to a grayscale one, which is later binarized using
 * adaptive thresholding ... 'ADAPTIVE_THRESH_GAUSSIAN_C' algorithm from OpenCV" (PAPER.md
 * P:164-168).  Its output frames are sp_compute's input.
 *
 * Per frame (DESIGN R23-R25):
 *   R23 downscale src -> dst by OpenCV INTER_AREA (fp32 area weights, OpenCV's order of
 *       operations, round half to even), channels independent;
 *   R24 gray: Y = (3735 B + 19235 G + 9798 R + 2^14) >> 15 (OpenCV 8-bit BGR2GRAY);
 *   R25 mean = cv2.adaptiveThreshold's Gaussian mean: float32 blur of the block_size window
 *       (replicated borders; OpenCV's float32 kernel; row then symmetric column pass, one fp32
 *       FMA per tap in OpenCV's order), rounded half to even; output byte = 255 if
 *       Y - mean > -ceil(bias) else 0.
 * Conventions as in sp.h: sp_status results, device pointers owned by the caller,
 * stream-ordered asynchronous calls, no CPU fallback.
 */
#ifndef HTM_SP_ENCODER_H
#define HTM_SP_ENCODER_H

#include <stdint.h>
#include "sp.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sp_encoder_config {
    uint32_t src_width, src_height;  /* input BGR frame W0 x H0 (960 x 540) */
    uint32_t dst_width, dst_height;  /* output W1 x H1 <= input (240 x 134) */
    uint32_t block_size;             /* Gaussian window, odd in [3, 15] (11) */
    float bias;                      /* C of T = mean - C, |C| <= 255 (2.0) */
    int32_t device;
} sp_encoder_config;

typedef struct sp_encoder sp_encoder;

typedef struct sp_encoder_info {
    uint32_t band_rows;      /* output rows per streamed band */
    uint32_t bands;          /* bands per frame */
    uint32_t stages;         /* shared-memory ring depth (bulk copies in flight per CTA) */
    uint32_t stage_bytes;
    uint32_t smem_bytes;     /* dynamic shared memory per CTA */
    uint32_t ctas_per_sm;
    uint32_t xfast;          /* 1 if the x table is an exact 4:1 average (vectorised path) */
    uint64_t kernel_launches;
    float kernel[16];        /* the float32 Gaussian kernel (block_size weights) */
    uint32_t chunk_frames;   /* sp_encode_compute: frames per chunk */
    uint32_t l2_window_set;  /* 1 if the chunk buffer is a persisting-L2 access-policy window */
    uint64_t l2_window_bytes; /* persisting-L2 set-aside granted for it (0 before the first call) */
} sp_encoder_info;

/* Defaults: 960x540 -> 240x134, block 11, bias 2, device 0.  SP_E_ARG for NULL. */
sp_status sp_encoder_config_default(sp_encoder_config* cfg);

/* Validates *cfg (SP_E_CONFIG: zero or upscaling dims, even / out-of-range block_size,
 * bias), builds the area tables and the Gaussian kernel, uploads them to cfg->device.
 * Errors: SP_E_ARG, SP_E_CONFIG, SP_E_CUDA. */
sp_status sp_encoder_create(const sp_encoder_config* cfg, sp_encoder** out);

/* Frees the encoder (NULL is a no-op). */
sp_status sp_encoder_destroy(sp_encoder* enc);

/* Encodes num_frames frames:
 *   bgr_dev: uint8[num_frames][src_height][src_width][3] (B, G, R), device memory;
 *   out_dev: uint8[num_frames][dst_height][dst_width] = 255 / 0, device memory.
 * Rows are streamed with bulk copies when bgr_dev is 16-byte aligned and 3*src_width is a
 * multiple of 16, else with plain loads.  Asynchronous on cuda_stream.
 * Errors: SP_E_ARG (NULL), SP_E_CUDA.  num_frames == 0 is a no-op. */
sp_status sp_encode(sp_encoder* enc, const uint8_t* bgr_dev, uint32_t num_frames, uint8_t* out_dev,
                    void* cuda_stream);

/* Raw video to SDRs in one call: the encoder (R23-R25) and the SP's inference (sp_compute_into,
 * learn = 0) over chunks of frames, the chunk's binarised frames held in an encoder-owned
 * buffer that is the stream's persisting-L2 access-policy window for the call (the binarised
 * frames go from the encoder's stores to the SP's TMA loads through L2, not HBM: the
 * "encoder fused into staging" of SURVEY §8(f) NEXT-3 at the memory level; the device-wide
 * persisting-L2 limit is raised to the buffer size for the call and restored at its end, which
 * makes the call wait for its last chunk; the encoder's BGR reads are marked L2 evict-first and
 * its binarised writes evict-last).  Chunk: 1024 frames (env SP_ENC_CHUNK).
 *   sp:        an SP handle whose input frame is dst_width x dst_height, on the same device;
 *   bgr_dev:   uint8[num_frames][src_height][src_width][3], device memory;
 *   sdr_dev:   uint32[num_frames * P][sdr_words], count_dev: uint32[num_frames * P], device
 *              memory (P = the SP's inputs per frame); they become the SP's last results.
 * Errors: SP_E_ARG (NULL, device mismatch), SP_E_CONFIG (frame size mismatch), SP_E_OOM,
 * the SP's errors (e.g. chunk * P > max_inputs: SP_E_ARG).  Ordered on cuda_stream; returns after
 * the last chunk completed when the persisting set-aside was raised. */
sp_status sp_encode_compute(sp_encoder* enc, sp_handle* sp, const uint8_t* bgr_dev, uint32_t num_frames,
                            uint32_t* sdr_dev, uint32_t* count_dev, void* cuda_stream);

/* Launch plan and kernel of the encoder.  Errors: SP_E_ARG. */
sp_status sp_encoder_get_info(sp_encoder* enc, sp_encoder_info* out);

/* Thread-local message of the last failing encoder call. */
const char* sp_encoder_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* HTM_SP_ENCODER_H */
