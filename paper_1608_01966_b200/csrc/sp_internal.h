// sp_internal.h — shared declarations of the libsp CUDA sources (not part of the ABI).
#pragma once

#include <cstdint>
#include <cuda.h>  // CUtensorMap (types only; the encoder is fetched via cudaGetDriverEntryPoint)
#include <cuda_runtime.h>

#include "../../include/sp.h"

namespace sp {

constexpr uint32_t kChunkBits = 1024;      // Lc: pixels per input per pipeline stage
constexpr uint32_t kBoxBytes = 128;        // TMA box: 128 B (pixels) x 32 rows (inputs), swizzle 128B
constexpr uint32_t kStageBytes = 32u * kChunkBits;  // 8 boxes = 32 KiB per stage
constexpr uint32_t kPackedStagesPer = 8;  // packed input: 4 KiB stages (one box) per 32 KiB stage
constexpr uint32_t kMaxBatchedColumns = 2048;
constexpr uint32_t kMaxBatchedSynapses = 1023;  // 10 vertical-counter planes
constexpr uint32_t kHiPlanes = 7;          // planes of weight 8..512 (ones/twos/fours separate)
constexpr uint32_t kPerInputChunk = 256;   // inputs per sub-batch of the per-input path

// Reasons the batched path is not eligible (sp_plan_info.reason bits).
enum : uint32_t {
    kNotBatchedLearn = 1u,      // learn=1 is sequential -> per-input path
    kNotBatchedPatch = 2u,      // patch mode (NEXT-2)
    kNotBatchedAlign = 4u,      // nbits % 16 != 0 (bulk copies need 16-byte rows)
    kNotBatchedColumns = 8u,    // C32 > 2048 (vertical counters exceed registers)
    kNotBatchedSynapses = 16u,  // S > 1023
    kNotBatchedForced = 32u,    // force_path = PER_INPUT
    kNotBatchedSmem = 64u,      // no (stages, window) fits shared memory
    kNotBatchedTensorMap = 128u, // the TMA descriptor could not be encoded
    kNotPatchGeometry = 256u,   // patch mode: pw % 32, pw*ph <= 1536, C32 <= 1024 needed
};

struct Geometry {
    uint32_t W, H, pw, ph;   // frame and patch (pw = W, ph = H in whole-frame mode)
    uint32_t P;              // inputs per frame
    uint32_t nbits;          // bits per SP input
    uint32_t C, C32, ncw;    // columns, padded, column-warps (= sdr words)
    uint32_t S;
    uint32_t keyL;           // ceil(log2(C32)) index bits of the rank key
    uint32_t keyBits;        // total significant key bits
    bool whole;              // whole-frame mode
};

// Layout of the batched (bit-sliced) path, fixed at create time (depends on C, S, nbits).
struct BatchedLayout {
    bool ok = false;
    uint32_t stages = 0, xbufs = 0, Lw = 0, nwin = 0;
    uint32_t ring_bytes = 0;   // TMA ring; `stages` = the 32-row (32 KiB) stages it holds
    static constexpr uint32_t kMaxStages = 8;  // barriers reserved for uint8 stages of fewer rows
    uint32_t region_bytes = 0, smem_bytes = 0;
};

struct alignas(64) BatchedParams {
    CUtensorMap tmap;          // 2-D uint8 view of the frames: {nbits, num_inputs}, box {128, rows}
    uint32_t num_inputs, nbits;
    uint32_t bdbg;             // development (SP_BATCHED_DBG; honoured only by -DSP_BATCHED_DBG_ON=1
                               // builds, timing experiments): 1 skip the gathers, 2 skip the
                               // transposes, 8 no loads (consumer-only), 32 no release (results wrong)
    uint32_t ring_bytes;       // TMA ring (stages * rows KiB <= ring_bytes; the window region follows)
    uint32_t gsplit;           // K CTAs per group WITHOUT a cluster (cooperative launch, all resident):
                               // partial counts through global memory (part), group barrier (gbar)
    uint4* part;               // gsplit: [groups][K][32][C32] u16 partial counts (L2)
    uint32_t* gbar;            // gsplit: [2][groups] arrivals, departures (zero between launches)
    uint32_t rows;             // whole frames: inputs per group = TMA box rows (<= 32); group g holds
                               // inputs [g*rows, min(n, (g+1)*rows)), so no box reads another group's rows
    uint32_t C, C32, ncw;
    uint32_t min_overlap, k, radius;
    uint32_t keyL, keyBits;
    uint32_t Lw, nwin, stages, region_bytes, xbufs;
    uint32_t one;              // always 1 (opaque to the compiler; see nz_flags)
    uint32_t S;                // synapses per column (histogram range of the fast top-k)
    uint32_t uniform_bc;       // all boosts equal: key order = (raw desc, index asc)
    uint32_t threads;          // 1024 or 512 threads per CTA
    // patch kernel
    uint32_t patch_w, patch_h, tiles_x, patch_stage_bytes;
    uint64_t* trace;           // nullable [ctas][4] phase timestamps (development aid)
    uint32_t groups, K;
    const uint32_t* ell_off;   // [nwin][ncw] offset in uint4 units
    const uint16_t* ell_nb;    // [nwin][ncw] number of 8-slot blocks
    const uint4* ell;          // [.. blocks][32 lanes] x 8 uint16 slots
    const uint32_t* bc;        // [C32] boost * 2^23 (0 on pad columns)
    const float* boost;        // [C32]
    uint32_t* sdr;             // [num_inputs][ncw]
    uint32_t* counts;          // [num_inputs]
    uint16_t* raw_out;         // nullable [num_inputs][C]
    float* boosted_out;        // nullable [num_inputs][C]
    const uint32_t* radius_dev;  // nullable: radius in force (full learning adapts it), else `radius`
    uint32_t wm_min_radius;    // per-column boosts: wavelet top-k from this radius on (else comparator)
    uint32_t packed;           // frames are bit-planes uint32[inputs][Wn4] (sp_compute_packed)
    uint32_t wm_umax;          // per-column-boost wavelet: largest coarse key - 1 (levels = its bits)
    uint32_t cand_min_radius;  // local inhibition, per-column boosts: candidate pruning from this radius on
    uint32_t cand_min_radius_u;  // the same with a uniform boost (sp_select.cuh local_candidates)
    uint32_t cand_dbg;           // development (SP_CAND_DBG, timing experiments only): 1 skip the beats step,
                                 // 2 skip the patch kernel's selection, 4 its gathers
};

// Tensor-core patch kernel (NEXT-2, sp_patch_mma.cu): raw counts of 128 tile slots per block
// as a kind::i8 GEMM conn[C32 x nbits] . tiles[nbits x 128], one cluster of Q = C32/128 CTAs.
struct alignas(64) PatchMmaParams {
    CUtensorMap tmap_b;        // frames {W/k, k, ph, tile_rows}, box {W/k, k, sps, 4}: whole rows
    BatchedParams bp;          // selection parameters and outputs (sp_topk.cuh)
    uint32_t Q;                // CTAs per cluster (128 columns each)
    uint32_t W;                // frame width (bytes per frame row)
    uint32_t nbits;            // pw * ph = K
    uint32_t patch_w, patch_h; // pw (a power of two, multiple of 32), ph
    uint32_t xchunks;          // pw / 32 slabs per tile row
    uint32_t sps;              // frame rows y per stage: 2 when ph is even, else 1
    uint32_t tile_rows;        // frames * (H / ph)
    uint32_t tiles_x;          // W / pw (<= 32)
    uint32_t nblocks;          // ceil(tile_rows / 4)
    uint32_t raw_stages, conv_stages, raw_stage_bytes;
    uint32_t multicast;        // one CTA fetches each raw stage for the whole cluster (TMA multicast)
    uint32_t region_bytes;     // top-k scratch
    const uint8_t* conn;       // conn u8 [C32][nbits], loaded into TMEM with tcgen05.st
    uint32_t dbg;              // development (SP_MMA_DBG): 1 skip the selection, 2 the exchange,
                               // 4 the MMAs, 8 the conversion, 16 the exchange handshakes
    uint64_t* trace;           // nullable (SP_MMA_TRACE): [ctas][trace_blocks][6] %globaltimer stamps
    uint32_t trace_blocks;
};
uint32_t patch_mma_smem(uint32_t W, uint32_t sps, uint32_t xchunks, uint32_t raw_stages, uint32_t conv_stages,
                        uint32_t Q, uint32_t C32, uint32_t region_bytes);
cudaError_t configure_patch_mma(int max_smem);
cudaError_t launch_patch_mma(const PatchMmaParams& p, uint32_t smem_bytes, uint32_t clusters, cudaStream_t s);
cudaError_t patch_mma_max_clusters(uint32_t smem_bytes, uint32_t Q, int* n);
cudaError_t launch_build_conn(const uint32_t* idx, const float* perm, float tau, uint32_t C, uint32_t C32, uint32_t S,
                              uint32_t nbits, uint8_t* conn, cudaStream_t s);

// Full learning (NEXT-1; S:119(b-e); DESIGN R17-R21): device state and constants.
struct FullLearn {
    uint32_t on;               // SP_FLAG_FULL_LEARNING
    uint32_t adapt;            // radius adaptation (configured radius > 0, R21)
    float pm1, P;              // duty_cycle_period - 1, duty_cycle_period (fp32)
    float mb1;                 // fp32(max_boost - 1)
    float bump;                // fp32(0.1f * tau)
    float* adc;                // [C32] active duty cycles
    float* odc;                // [C32] overlap duty cycles
    float* boost;              // [C32] boosts (written)
    uint32_t* bc;              // [C32] boost * 2^23 (written)
    uint32_t* radius;          // device scalar: radius in force
    uint32_t* span;            // [C32] connected spans (R21)
    float* scratch;            // window-maximum tables: pre, suf [C32] + table [levels][C32/32]
};

struct PerInputParams {
    const uint8_t* frames;     // frames of this sub-batch
    uint32_t uniform_bc;       // all boosts equal (bit-sliced local inhibition)
    uint32_t first_input;      // global index (within the call) of the sub-batch's first input
    uint32_t num_inputs;       // inputs in this sub-batch
    Geometry g;
    uint32_t min_overlap, k, radius;
    float inc, dec, tau;
    uint32_t* bits;            // [num_inputs][bits_stride] packed input bits (scratch)
    uint32_t Wn;
    uint32_t bits_stride;      // words between planes (0: Wn)
    const uint32_t* syn;       // [S][C32] idx | connected << 31
    uint32_t* syn_rw;          // same, writable (learning)
    const uint32_t* idx;       // [C][S]
    float* perm;               // [C][S]
    const uint32_t* bc;        // [C32]
    const float* boost;        // [C32]
    uint32_t* raw;             // [num_inputs][C32] scratch
    uint32_t* sdr;             // [call inputs][ncw]
    uint32_t* counts;          // [call inputs]
    uint16_t* raw_out;         // nullable [call inputs][C]
    float* boosted_out;        // nullable [call inputs][C]
    const uint32_t* radius_dev;  // nullable: radius in force, else `radius`
    FullLearn fl;              // full learning (k_learn keeps spans; k_full runs (b)-(e))
    uint32_t wm_ok;            // k_inhibit may use the CTA wavelet (smem sized for it)
    uint32_t wm_min_radius;    // ... from this radius on (per-column boosts)
};
uint32_t inhibit_wavelet_smem(const Geometry& g);

struct LearnParams {
    const uint8_t* frames;     // frames of the call
    uint32_t first_input;      // row of the first input in the result buffers
    uint32_t num_inputs;       // inputs (frames x patches), processed in order
    Geometry g;
    uint32_t Q, cols_per_cta, Wn;
    uint32_t syn_stride;       // padded column-major stride of the resident synapse slice
    uint32_t tpc;              // threads per column in the overlap
    uint32_t min_overlap, k, radius, uniform_bc;
    float inc, dec, tau;
    const uint32_t* idx;       // [C][S]
    float* perm;               // [C][S]
    uint32_t* syn;             // [S][C32] idx | connected << 31 (loaded, written back)
    const uint32_t* bc;        // [C32]
    const float* boost;        // [C32]
    uint32_t* bits_g;          // [2][Wn rounded to 4] scratch bit-planes (L2), by input parity, or
                               // [num_inputs][Wn rounded to 4] planes prepacked by k_pack
    uint32_t prepacked;        // bits_g holds every input's plane (no packing in the kernel)
    uint32_t dbl_bits;         // two smem bit-plane buffers (load of t+1 overlaps learning of t)
    uint32_t dbg;              // development switches (SP_LEARN_DBG, timing experiments only): 1 no proxy
                               // fence, 2 no prefetch, 4 no pack, 8 no selection, 16 load the next plane
                               // late, 32 packing loads via L2 (.cg), 64 warp-level global selection,
                               // 128 no window split of the local selection
    uint64_t* trace;           // nullable [6] summed phase times of CTA 0 (development aid)
    uint32_t* sdr;             // [rows][ncw]
    uint32_t* counts;          // [rows]
    uint16_t* raw_out;         // nullable
    float* boosted_out;        // nullable
    FullLearn fl;              // full learning, steps (b)-(e) after each input
};

struct LearnGridParams {
    const uint8_t* frames;     // frames of the call
    uint32_t first_input;      // row of the first input in the result buffers
    uint32_t num_inputs;       // inputs (frames x patches), processed in order
    Geometry g;
    uint32_t G;                // co-resident CTAs (cooperative launch, one per SM)
    uint32_t Wn;
    uint32_t own_words, win_words, ccols, stages;  // smem sizing (learn_grid_smem)
    uint32_t dbl_bits;         // two smem bit-plane buffers
    uint32_t min_overlap, k, radius, uniform_bc;
    float inc, dec, tau;
    uint32_t* synT;            // [C32][S] idx | connected << 31, column-major (updated)
    float* perm;               // [C][S]
    const uint32_t* bc;        // [C32]
    const float* boost;        // [C32]
    uint32_t* bits_g;          // [2][Wn rounded to 4] bit-planes, by input parity, or
                               // [num_inputs][Wn rounded to 4] planes prepacked by k_pack
    uint32_t prepacked;        // bits_g holds every input's plane
    uint16_t* raw_g;           // [2][C32] raw counts, by input parity
    uint32_t* gbar;            // grid barrier counter (zeroed before the launch)
    uint32_t* sdr;             // [rows][ncw]
    uint32_t* counts;          // [rows]
    uint16_t* raw_out;         // nullable
    float* boosted_out;        // nullable
    uint32_t dbg;              // development switches (see LearnParams)
    uint64_t* trace;           // nullable [6] summed phase times of CTA 0 (development aid)
    // full-learning grid kernel (sp_learn_grid_full.cu)
    FullLearn fl;              // duty cycles, boosts, spans, radius, window-maximum scratch
    unsigned long long* span_part;  // [2][G] per-CTA connected-span sums, by input parity
    uint32_t cand_cap;         // candidate list capacity (shared memory)
    uint32_t vsh;              // selection value v = N >> vsh (< 2^16)
};

// grid learning (sp_learn_grid.cu)
uint32_t learn_grid_smem(const Geometry& g, uint32_t radius, uint32_t G, bool dbl_bits, uint32_t* own_words,
                         uint32_t* win_words, uint32_t* ccols, uint32_t* stages);
cudaError_t configure_learn_grid(int max_smem);
cudaError_t learn_grid_max_ctas(uint32_t smem, int* n);
cudaError_t launch_learn_grid(const LearnGridParams& p, uint32_t smem, cudaStream_t s);
// grid learning with the full learning step (sp_learn_grid_full.cu)
uint32_t learn_grid_full_smem(const Geometry& g, uint32_t G, uint32_t stages, uint32_t cap, uint32_t* own_words,
                              uint32_t* ccols);
cudaError_t configure_learn_grid_full(int max_smem);
cudaError_t learn_grid_full_max_ctas(uint32_t smem, int* n);
cudaError_t launch_learn_grid_full(const LearnGridParams& p, uint32_t smem, cudaStream_t s);
uint32_t learn_grid_chunk_cols(uint32_t S);
cudaError_t launch_build_synT(const uint32_t* idx, const float* perm, float tau, uint32_t C, uint32_t C32,
                              uint32_t S, uint32_t* synT, cudaStream_t s);

// cluster learning (sp_learn.cu)
uint32_t learn_cluster_smem(const Geometry& g, uint32_t Q, uint32_t* cols_per_cta, bool dbl_bits, bool full);
uint32_t learn_syn_stride(uint32_t S);
uint32_t learn_threads_per_column(uint32_t cpc);
cudaError_t configure_learn(int max_smem);
cudaError_t learn_max_clusters(uint32_t Q, uint32_t smem, int* n);
cudaError_t launch_learn_cluster(const LearnParams& p, uint32_t smem, cudaStream_t s);

// host planning (sp_host.cu)
Geometry make_geometry(const sp_config& cfg);
BatchedLayout plan_batched_layout(const Geometry& g, int max_smem);
BatchedLayout plan_patch_layout(const Geometry& g, int max_smem);
void plan_batched_grid(const Geometry& g, uint32_t nwin, uint32_t num_inputs, int sm_count,
                       const int* max_clusters /* [9] by K, or nullptr */,
                       uint32_t* groups, uint32_t* K, uint32_t* R, uint32_t* gsplit);

// TMA descriptor of the frames for the batched kernel (sp_host.cu); false on failure
bool encode_frames_tmap(CUtensorMap* map, const uint8_t* frames, uint32_t nbits, uint32_t rows, uint32_t box_rows);
bool encode_patches_tmap(CUtensorMap* map, const uint8_t* frames, const Geometry& g, uint32_t frames_n);

// one-time kernel attributes (max dynamic smem)
cudaError_t configure_batched(int max_smem);
cudaError_t configure_per_input(int max_smem);

// launchers (return cudaError_t of the launch)
cudaError_t launch_batched(const BatchedParams& p, uint32_t smem_bytes, cudaStream_t s);
bool encode_packed_tmap(CUtensorMap* map, const uint32_t* planes, uint32_t words, uint32_t rows, uint32_t box_rows);
cudaError_t launch_patch(const BatchedParams& p, uint32_t smem_bytes, uint32_t ctas, cudaStream_t s);
cudaError_t batched_max_clusters(uint32_t smem_bytes, int max_clusters[9]);
cudaError_t launch_pack(const PerInputParams& p, cudaStream_t s);
cudaError_t launch_overlap(const PerInputParams& p, cudaStream_t s);
cudaError_t launch_inhibit(const PerInputParams& p, cudaStream_t s, uint32_t parts = 1);
cudaError_t launch_learn(const PerInputParams& p, uint32_t input, cudaStream_t s);
cudaError_t launch_full(const PerInputParams& p, uint32_t input, cudaStream_t s, uint32_t* launches);
cudaError_t launch_span(const uint32_t* idx, const float* perm, float tau, uint32_t C, uint32_t S,
                        uint32_t* span, cudaStream_t s);
size_t full_scratch_floats(uint32_t C32);
// per-video SDR histograms (sp_hist.cu); returns the number of kernels launched in *launches
cudaError_t launch_histograms(const uint32_t* sdr, uint32_t ncw, uint32_t C, const uint32_t* off_dev,
                              uint32_t V, uint32_t max_video_inputs, int sm_count, uint32_t* counts,
                              float* hist, cudaStream_t s, uint32_t* launches);
cudaError_t launch_build_syn(const uint32_t* idx, const float* perm, float tau, uint32_t C,
                             uint32_t C32, uint32_t S, uint32_t* syn, cudaStream_t s);
cudaError_t launch_refresh_ell(const uint32_t* idx, const float* perm, const uint32_t* pos,
                               float tau, uint32_t C, uint32_t S, uint32_t Lw, uint16_t* ell,
                               cudaStream_t s);

// handle accessors for the encoder's fused call (sp_encode_compute, sp_encoder.cu)
sp_status handle_frame_dims(const sp_handle* h, uint32_t* W, uint32_t* H, uint32_t* P, uint32_t* words,
                            int* device);
void handle_set_result(sp_handle* h, uint32_t* sdr, uint32_t* counts, uint32_t inputs);

inline uint32_t ceil_log2(uint32_t v) {
    uint32_t l = 0;
    while ((1ull << l) < v) ++l;
    return l;
}
inline uint32_t bits_for(uint32_t v) {  // number of bits to represent 0..v
    uint32_t l = 0;
    while ((1ull << l) <= v) ++l;
    return l;
}

}  // namespace sp
