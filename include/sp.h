/*
 * sp.h — C ABI of the B200-native HTM Spatial Pooler hot path
 *         (Wielgosz & Pietron, arxiv 1608.01966).
 *
 * Citations: PAPER.md = P:n (/root/reference/PAPER.md line n, read-only copy
 * of the paper), SPEC.md = S:n, readings Rn.
 *
 * The hot path:
 *   a1 staging   uint8 frame -> input bits, bit = byte != 0, row-major
 *                (DESIGN R12/R13)
 *   a2 overlap   raw[c] = #{s : perm[c,s] >= tau and bit(idx[c,s])}   (Alg. 1 l.1-5)
 *   a3 boost     raw < min_overlap -> 0, else raw * boost[c]           (Alg. 1 l.6-10)
 *   a4 inhibit   k-winners, global or radius-r 1-D window, ties to the lower index
 *                (Alg. 2; DESIGN R5-R7, R9)
 *   a5 learn     winners' potential synapses: perm +inc if the input bit is set,
 *                -dec otherwise, clamped to [0,1], fp32 (P:92 -> whitepaper; S:119(a); R3, R10)
 *   full learning (SP_FLAG_FULL_LEARNING; S:119(b-e), S:149-151;
 *                DESIGN R17-R21), after a5 for every input: duty cycles, boost update,
 *                weak-column bump and (configured radius > 0) inhibition-radius adaptation
 *
 * Conventions shared by every entry point:
 *  - Every function returns sp_status; on failure sp_last_error() returns a
 *    thread-local message naming the violated invariant.
 *  - "dev" pointers are CUDA device pointers on the handle's device, owned by
 *    the caller (torch allocates them); "host" pointers are host memory owned
 *    by the caller.  The handle owns all SP state and scratch (allocated in
 *    sp_create, freed in sp_destroy).
 *  - cuda_stream is a cudaStream_t (NULL = legacy default stream).  Device
 *    calls are asynchronous and stream-ordered; results are valid after the
 *    stream reaches them.  A handle is single-caller; distinct handles
 *    are independent.
 *  - No CPU fallback: without a usable CUDA device every device call fails
 *    with SP_E_CUDA.
 */
#ifndef HTM_SP_H
#define HTM_SP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum sp_status {
    SP_OK = 0,
    SP_E_CONFIG = 1,   /* configuration violates an invariant      */
    SP_E_ARG = 2,      /* bad argument: NULL, out of range, state out of domain    */
    SP_E_SHAPE = 3,    /* buffer shape/dtype/device mismatch (raised by bindings)  */
    SP_E_CUDA = 4,     /* CUDA runtime error / no device                           */
    SP_E_OOM = 5,      /* device or host allocation failed                         */
    SP_E_STATE = 6     /* call out of sequence (e.g. sp_winners before compute)    */
} sp_status;

/* Kernel path selection (sp_config.force_path).  AUTO picks BATCHED whenever
 * it is eligible (see sp_plan), PER_INPUT otherwise.  Both are CUDA paths;
 * forcing exists so the parity tests can cover both. */
enum { SP_PATH_AUTO = 0, SP_PATH_PER_INPUT = 1, SP_PATH_BATCHED = 2 };

/* sp_config.flags */
enum {
    SP_FLAG_RECORD_OVERLAPS = 1u, /* keep raw/boosted overlaps of the last call for sp_overlaps */
    SP_FLAG_LEARN_GRID = 2u,      /* learn=1: prefer the grid-resident kernel (one CTA per SM) over
                                     the cluster-resident one (default: cluster when it fits) */
    SP_FLAG_FULL_LEARNING = 4u,   /* learn=1 also runs S:119(b-e) after each input's permanence
                                     update (DESIGN R17-R21): active/overlap duty cycles (EMA of
                                     period duty_cycle_period), boost = linear rule up to
                                     max_boost, weak-column bump by 0.1*tau, and, when
                                     inhibition_radius > 0, the radius recomputed from the
                                     connected spans.  The radius in force governs inhibition
                                     of every later call (learn or not). */
    SP_FLAG_PATCH_GATHER = 8u,    /* patch mode inference: the bit-sliced gather kernel (the
                                     default since round 2: measured faster) */
    SP_FLAG_PATCH_TENSOR = 16u    /* patch mode inference: the tcgen05 kind::i8 GEMM kernel where
                                     eligible (NEXT-2; identical results; opt-in, A/B tests) */
};

/*
 * SP configuration (Tab. 2).  Invariants checked by
 * sp_create (SP_E_CONFIG, message names the invariant):
 *   input_width, input_height >= 1; patch_width/patch_height both 0 (the
 *     whole frame is one SP input) or both >= 1 and dividing the frame dims;
 *   nbits = input bits per SP input = pw*ph (whole frame: W*H) <= 1,800,000;
 *   1 <= num_columns <= 20480 (the per-input inhibition holds 10 bytes per column in one
 *     CTA's shared memory); 1 <= synapses_per_column <= min(nbits, 4095);
 *   min_overlap <= synapses_per_column; 1 <= winners_set_size <= num_columns;
 *   perm_increment, perm_decrement, initial_permanence, connected_threshold in [0,1];
 *   ceil(log2(S+1)) + 27 + ceil(log2(C32)) <= 64 (the exact rank key fits 64 bits, R4);
 *   max_inputs >= 1 (capacity of one sp_compute call, in SP inputs);
 *   with SP_FLAG_FULL_LEARNING: duty_cycle_period >= 1 and 1 <= max_boost < 16 (boosts
 *     stay in the exact-key domain, R4).
 */
typedef struct sp_config {
    uint32_t input_width, input_height;   /* frame W x H in pixels; bit = y*W + x */
    uint32_t patch_width, patch_height;   /* 0,0 = whole frame; else tiles in raster order (R13) */
    uint32_t num_columns;                 /* C  (Tab. 2: 2048) */
    uint32_t synapses_per_column;         /* S  (Tab. 2: 128) */
    uint32_t min_overlap;                 /* theta (Tab. 2: 8) */
    uint32_t winners_set_size;            /* k = n of Alg. 2 (Tab. 2: 40) */
    uint32_t inhibition_radius;           /* r; 0 = global k-winners (R9) */
    float perm_increment;                 /* Tab. 2: 0.1 */
    float perm_decrement;                 /* Tab. 2: 0.1 */
    float initial_permanence;             /* Tab. 2: 0.21 */
    float connected_threshold;            /* tau = 0.2 (R2; not in the paper) */
    uint64_t seed;                        /* potential-pool sampling seed (R8) */
    int32_t device;                       /* CUDA device ordinal */
    uint32_t max_inputs;                  /* per-call capacity in SP inputs */
    uint32_t flags;                       /* SP_FLAG_* */
    uint32_t force_path;                  /* SP_PATH_* */
    uint32_t duty_cycle_period;           /* full learning: EMA period P (default 1000) */
    float max_boost;                      /* full learning: boost ceiling (default 2.0) */
} sp_config;

typedef struct sp_handle sp_handle;

/* Derived launch plan (host-only computation, no GPU needed). */
typedef struct sp_plan_info {
    uint32_t path;               /* SP_PATH_PER_INPUT or SP_PATH_BATCHED */
    uint32_t input_bits;         /* nbits */
    uint32_t inputs_per_frame;   /* P (1 in whole-frame mode) */
    uint32_t num_inputs;         /* frames * P for the planned call */
    uint32_t columns_padded;     /* C32 = C rounded up to 32 */
    uint32_t sdr_words;          /* C32 / 32 words per SP input */
    /* batched path only (0 otherwise) */
    uint32_t groups;             /* groups of <= 32 inputs, bit-sliced together */
    uint32_t cluster;            /* K CTAs per group (pixel windows split, DSMEM reduce) */
    uint32_t ctas;               /* groups * cluster */
    uint32_t window_bits;        /* Lw pixels per resident bit-sliced window */
    uint32_t num_windows;
    uint32_t chunk_bits;         /* Lc pixels per pipeline stage */
    uint32_t stages;             /* pipeline depth of the bulk-copy ring */
    uint32_t smem_bytes;         /* dynamic shared memory per CTA */
    uint32_t reason;             /* why not batched: 0 eligible, else bitmask */
    uint32_t tensor_cores;       /* patch mode: 1 if the overlap runs as a tcgen05 kind::i8 GEMM
                                    (NEXT-2; groups = blocks of 4 tile-rows, cluster = C32/128) */
    uint32_t group_inputs;       /* whole frames: inputs per group (the TMA box rows, <= 32);
                                    group g = inputs [g*group_inputs, min(n, (g+1)*group_inputs)) */
    uint32_t global_split;       /* 1: the `cluster` CTAs of a group are no thread-block cluster but
                                    members of one cooperative launch, partial counts summed through
                                    global memory (small batches) */
} sp_plan_info;

/* Run-time information about a handle. */
typedef struct sp_info {
    sp_plan_info plan;           /* plan of the last sp_compute call (or of max_inputs) */
    uint64_t kernel_launches;    /* kernels launched by this handle since creation */
    uint32_t last_num_inputs;    /* inputs processed by the last sp_compute call */
    uint32_t ell_slots;          /* batched layout size in uint16 slots (0 if none) */
    int32_t sm_count;            /* device SMs */
    int32_t max_smem_optin;      /* device max dynamic smem per block */
    uint32_t learn_cluster;      /* CTAs per cluster of the resident learning kernel (0: learning
                                    uses the per-input kernels) */
    uint32_t last_learn_cluster; /* 1 if the last learn=1 call used the cluster kernel */
    uint32_t learn_grid_ctas;    /* CTAs of the grid-resident learning kernel (0: not eligible) */
    uint32_t last_learn_path;    /* path of the last learn=1 call: SP_LEARN_PER_INPUT,
                                    SP_LEARN_CLUSTER or SP_LEARN_GRID */
} sp_info;

/* learning paths (sp_info.last_learn_path) */
#define SP_LEARN_PER_INPUT 0u /* per-input kernels, one launch per step per input */
#define SP_LEARN_CLUSTER 1u   /* one launch, cluster of <= 16 CTAs, synapse table in smem */
#define SP_LEARN_GRID 2u      /* one cooperative launch, one CTA per SM, table streamed from L2 */

/* Fills *cfg with Tab. 2 defaults on a 240x134 frame (Tab. 1),
 * tau 0.2, seed 42, device 0, max_inputs 4096, duty_cycle_period 1000, max_boost 2.0.
 * Never fails for non-NULL cfg. */
sp_status sp_config_default(sp_config* cfg);

/* Validates *cfg, samples the potential pools (R8: per column c a splitmix64
 * stream from splitmix64(seed ^ (c+1)*0x9E3779B97F4A7C15); idx = ((u>>32)*nbits)>>32,
 * duplicates rejected, sorted ascending), sets perm = initial_permanence and
 * boost = 1, allocates all device state on cfg->device and
 * writes the new handle to *out.  Errors: SP_E_ARG (NULL), SP_E_CONFIG,
 * SP_E_CUDA, SP_E_OOM (nothing leaks on failure). */
sp_status sp_create(const sp_config* cfg, sp_handle** out);

/* Frees the handle and all its device memory.  NULL is a no-op. */
sp_status sp_destroy(sp_handle* h);

/* One pass of the hot path over num_frames frames.
 *   frames_dev: uint8[num_frames][input_height][input_width], C-contiguous,
 *               device memory (any byte != 0 is an active bit, R12).
 *   learn = 0: inference; a pure function of the state.
 *   learn = 1: the SP inputs (frames x patches, in order) are processed
 *              SEQUENTIALLY: input t+1 sees input t's permanence update
 *              (SURVEY §8(a) a5).
 * The winners of every input are kept for sp_winners (and the overlaps, with
 * SP_FLAG_RECORD_OVERLAPS, for sp_overlaps) until the next call.
 * Errors: SP_E_ARG (NULL handle/frames with num_frames>0, num_frames*P >
 * max_inputs), SP_E_CUDA.  num_frames == 0 is a no-op. */
sp_status sp_compute(sp_handle* h, const uint8_t* frames_dev, uint32_t num_frames,
                     int learn, void* cuda_stream);

/* sp_compute writing the winners straight into caller buffers (no copy afterwards):
 *   sdr_dev:   uint32[num_frames * P][sdr_words], count_dev: uint32[num_frames * P], device
 *              memory on the handle's device.  They stay the "last call's results" for
 *              sp_winners / sp_histograms until the next compute call, so the caller keeps them
 *              alive until then.  Errors: as sp_compute; SP_E_ARG for NULL buffers. */
sp_status sp_compute_into(sp_handle* h, const uint8_t* frames_dev, uint32_t num_frames, int learn,
                          uint32_t* sdr_dev, uint32_t* count_dev, void* cuda_stream);

/* Copies the winners of the last sp_compute call:
 *   sdr_dev:   uint32[num_inputs][sdr_words]; bit c of word c/32 (LSB first)
 *              set iff column c is active (the SDR).
 *   count_dev: uint32[num_inputs] number of active columns, or NULL.
 * Errors: SP_E_ARG (NULL handle or sdr_dev), SP_E_STATE (no compute yet). */
sp_status sp_winners(sp_handle* h, uint32_t* sdr_dev, uint32_t* count_dev, void* cuda_stream);

/* Copies the overlaps of the last call (needs SP_FLAG_RECORD_OVERLAPS):
 *   raw_dev:     uint16[num_inputs][num_columns] raw counts (Alg. 1 l.1-5), or NULL;
 *   boosted_dev: float[num_inputs][num_columns]: 0 if raw < min_overlap, else
 *                the fp32 product raw*boost correctly rounded (Alg. 1 l.6-10, R4), or NULL.
 * With learn=1 each input's overlaps are those seen before its own update.
 * Errors: SP_E_ARG, SP_E_STATE (flag not set or no compute yet). */
sp_status sp_overlaps(sp_handle* h, uint16_t* raw_dev, float* boosted_dev, void* cuda_stream);

/* Exports the state in canonical order (host pointers, synchronous):
 *   idx:   uint32[C][S] potential-pool input indices, ascending per column (or NULL)
 *   perm:  float[C][S] permanences (or NULL)
 *   boost: float[C] (or NULL).
 * Errors: SP_E_ARG, SP_E_CUDA. */
sp_status sp_get_state(sp_handle* h, uint32_t* idx, float* perm, float* boost);

/* Imports a state (host pointers, synchronous; checkpoint / oracle injection).
 * Domain (SP_E_ARG, message names it): idx entries < nbits and strictly
 * ascending within a column (distinct); perm in [0,1]; boost in
 * [1,16) (the exact-key domain, R4).  NULL keeps the current array. */
sp_status sp_set_state(sp_handle* h, const uint32_t* idx, const float* perm, const float* boost);

/* Per-video SDR histograms of the last sp_compute call (P:118-120
 * "histograms of consecutive frames are built from SP output on a per-video basis";
 * S:422-430; DESIGN R22).  Video v is the range [offsets[v], offsets[v+1]) of SP inputs of that
 * call (frames x patches, in order):
 *   video_offsets_host: uint32[num_videos + 1], host memory, non-decreasing, last <= the
 *                       number of inputs of the last call (SP_E_ARG otherwise);
 *   counts_dev: uint32[num_videos][C] number of inputs with column c active (or NULL);
 *   hist_dev:   float[num_videos][C] = fp32(count) / fp32(inputs of the video), one IEEE RN
 *               division; 0 for an empty video (or NULL).
 * Stream-ordered like sp_winners (the offsets are copied before the call returns).
 * Errors: SP_E_ARG, SP_E_STATE (no compute yet), SP_E_OOM, SP_E_CUDA. */
sp_status sp_histograms(sp_handle* h, const uint32_t* video_offsets_host, uint32_t num_videos,
                        uint32_t* counts_dev, float* hist_dev, void* cuda_stream);

/* Full-learning state (S:88, S:119(b-e)); host pointers, synchronous.
 *   active_duty, overlap_duty: float[C] duty cycles (or NULL);
 *   radius: the inhibition radius in force (0 = global) (or NULL);
 *   iteration: number of SP inputs learned since creation (or NULL).
 * Errors: SP_E_ARG (NULL handle), SP_E_CUDA. */
sp_status sp_get_learning_state(sp_handle* h, float* active_duty, float* overlap_duty, uint32_t* radius,
                                uint64_t* iteration);

/* Imports the full-learning state (checkpoint / oracle injection; synchronous).
 *   active_duty, overlap_duty: float[C] in [0,1] (SP_E_ARG otherwise), NULL keeps the current;
 *   radius: new radius in force; must be 0 iff the configured inhibition_radius is 0, else in
 *   [1, C] (SP_E_ARG). */
sp_status sp_set_learning_state(sp_handle* h, const float* active_duty, const float* overlap_duty,
                                uint32_t radius);

/* End-to-end variant ("OCL" accounting of P:316): frames in HOST memory,
 * winners returned to HOST memory.  The library pipelines host->device copies,
 * compute and device->host copies in chunks on cuda_stream (plus an internal
 * copy stream); pinned host memory makes the copies asynchronous.  Returns
 * after the results are in sdr_host / count_host (synchronous).
 *   frames_host: uint8[num_frames][H][W]; sdr_host: uint32[num_inputs][sdr_words];
 *   count_host: uint32[num_inputs] or NULL.  learn as in sp_compute. */
sp_status sp_compute_host(sp_handle* h, const uint8_t* frames_host, uint32_t num_frames,
                          int learn, uint32_t* sdr_host, uint32_t* count_host,
                          void* cuda_stream);

/* ---- bit-plane input ------------------------------------------------------------
 * "Changing from integer to boolean data type will result in approximately 32-fold reduction of
 * the amount of data to be transferred to the accelerator".  Frames may be given as
 * bit-planes: uint32[num_frames][Wp], Wp = ceil(W*H / 32) rounded up to a multiple of 4 (16-byte
 * rows); bit i of word w is pixel 32w + i in row-major order (R12's bit, LSB first), words and
 * bits past W*H are ignored.  8x fewer bytes than uint8 frames cross PCIe and HBM.  Whole-frame
 * configurations (no patches) that the batched kernel serves (sp_plan path BATCHED); inference
 * only (the state is not changed).  The results are the same as sp_compute on the uint8 frames
 * whose nonzero bytes are the set bits. */

/* Packs uint8 frames (device, uint8[num_frames][H][W]) into bit-planes (device,
 * uint32[num_frames][Wp], caller-owned), stream-ordered.  Errors: SP_E_ARG (NULL buffers),
 * SP_E_CONFIG (patch configuration), SP_E_CUDA. */
sp_status sp_pack_frames(sp_handle* h, const uint8_t* frames_dev, uint32_t num_frames, uint32_t* planes_dev,
                         void* cuda_stream);

/* Inference on bit-planes (device, 16-byte aligned): the winners go to sdr_dev / count_dev
 * (uint32[num_frames][sdr_words] / uint32[num_frames], device) or, both NULL, to the handle's
 * buffers (read with sp_winners).  Async, stream-ordered.  Errors: SP_E_ARG (NULL planes,
 * misalignment, one of sdr_dev / count_dev NULL, num_frames > max_inputs), SP_E_CONFIG (patch
 * configuration or not eligible for the batched kernel), SP_E_CUDA. */
sp_status sp_compute_packed(sp_handle* h, const uint32_t* planes_dev, uint32_t num_frames, uint32_t* sdr_dev,
                            uint32_t* count_dev, void* cuda_stream);

/* End-to-end variant of sp_compute_packed with HOST bit-planes and HOST results (as
 * sp_compute_host; synchronous). */
sp_status sp_compute_packed_host(sp_handle* h, const uint32_t* planes_host, uint32_t num_frames,
                                 uint32_t* sdr_host, uint32_t* count_host, void* cuda_stream);

/* Host-only planning (no GPU): the launch plan sp_compute would use for
 * num_frames frames with learn=0, assuming a B200 (148 SMs, 232448 B smem)
 * when sm_count <= 0.  Errors: SP_E_ARG, SP_E_CONFIG. */
sp_status sp_plan(const sp_config* cfg, uint32_t num_frames, int32_t sm_count,
                  sp_plan_info* out);

/* Host-only: the potential pools sp_create would sample (R8), uint32[C][S].
 * Lets CPU tests compare the library's initialisation with the oracle's. */
sp_status sp_init_pools_host(const sp_config* cfg, uint32_t* idx_out);

/* Handle information (plan of the last call, kernel-launch counter). */
sp_status sp_get_info(sp_handle* h, sp_info* out);

/* Thread-local message of the last failing call on this thread ("" if none). */
const char* sp_last_error(void);

/* Library version string. */
const char* sp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HTM_SP_H */
