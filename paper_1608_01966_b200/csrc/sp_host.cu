// sp_host.cu — host side of libsp: the C ABI of include/sp.h.
//
// Owns: configuration validation, seeded potential-pool
// initialisation (DESIGN R8), the derived device layouts
// (synapse-major idx|flag words; the bit-sliced path's windowed ELL), the
// launch planner and the stream-ordered dispatch of the CUDA kernels.
// There is no CPU compute path: every SP step runs in the kernels.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cudaTypedefs.h>

#include "sp_internal.h"
#include "../../include/sp_synth.h"

#define SP_VERSION "htm-sp-b200 0.1.0 (sm_100a)"

namespace {

thread_local std::string g_err;

sp_status fail(sp_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

sp_status cuda_fail(cudaError_t e, const char* what) {
    return fail(SP_E_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
constexpr int kDefaultSms = 148;
constexpr int kDefaultSmem = 232448;   // B200 max dynamic smem per block (opt-in)
constexpr uint32_t kMaxInputBits = 1800000u;
constexpr uint32_t kPrepackInputs = 1024u;  // inputs per prepacked learning chunk

inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Potential pools (DESIGN R8): column c's splitmix64 state starts at
// splitmix64(seed ^ (c+1)*gamma); each draw advances the state by gamma and
// outputs mix64(state); idx = ((u >> 32) * nbits) >> 32; duplicates are
// rejected; the accepted S indices are sorted ascending.
void init_pools(const sp_config& cfg, const sp::Geometry& g, uint32_t* idx) {
    std::vector<uint8_t> seen(g.nbits, 0);
    std::vector<uint32_t> chosen;
    chosen.reserve(g.S);
    for (uint32_t c = 0; c < g.C; ++c) {
        uint64_t state = mix64((cfg.seed ^ (static_cast<uint64_t>(c + 1) * kGamma)) + kGamma);
        chosen.clear();
        while (chosen.size() < g.S) {
            state += kGamma;
            const uint64_t u = mix64(state);
            const uint32_t i = static_cast<uint32_t>(((u >> 32) * g.nbits) >> 32);
            if (!seen[i]) {
                seen[i] = 1;
                chosen.push_back(i);
            }
        }
        for (uint32_t i : chosen) seen[i] = 0;
        std::sort(chosen.begin(), chosen.end());
        std::memcpy(idx + static_cast<size_t>(c) * g.S, chosen.data(), g.S * sizeof(uint32_t));
    }
}

sp_status validate(const sp_config* c) {
    if (!c) return fail(SP_E_ARG, "config is NULL");
    if (c->input_width == 0 || c->input_height == 0)
        return fail(SP_E_CONFIG, "input_width and input_height must be >= 1");
    const bool whole = c->patch_width == 0 && c->patch_height == 0;
    if (!whole) {
        if (c->patch_width == 0 || c->patch_height == 0)
            return fail(SP_E_CONFIG, "patch_width and patch_height must both be 0 or both >= 1");
        if (c->input_width % c->patch_width || c->input_height % c->patch_height)
            return fail(SP_E_CONFIG, "patch dims must divide the frame dims (%ux%u vs %ux%u)",
                        c->patch_width, c->patch_height, c->input_width, c->input_height);
    }
    const uint64_t nbits = whole ? static_cast<uint64_t>(c->input_width) * c->input_height
                                 : static_cast<uint64_t>(c->patch_width) * c->patch_height;
    if (nbits > kMaxInputBits)
        return fail(SP_E_CONFIG, "input bits per SP input (%llu) exceed %u",
                    static_cast<unsigned long long>(nbits), kMaxInputBits);
    // the per-input inhibition keeps raw counts, Bc and key bit-planes of every column in one
    // CTA's shared memory (10 bytes per column)
    if (c->num_columns == 0 || c->num_columns > 20480)
        return fail(SP_E_CONFIG, "num_columns must be in [1, 20480]");
    if (c->synapses_per_column == 0 || c->synapses_per_column > 4095)
        return fail(SP_E_CONFIG, "synapses_per_column must be in [1, 4095]");
    if (c->synapses_per_column > nbits)
        return fail(SP_E_CONFIG, "synapses_per_column <= input_size violated (S:50): %u > %llu",
                    c->synapses_per_column, static_cast<unsigned long long>(nbits));
    if (c->min_overlap > c->synapses_per_column)
        return fail(SP_E_CONFIG, "min_overlap <= synapses_per_column violated (S:49)");
    if (c->winners_set_size == 0 || c->winners_set_size > c->num_columns)
        return fail(SP_E_CONFIG, "1 <= winners_set_size <= num_columns violated (S:49)");
    const float fr[4] = {c->perm_increment, c->perm_decrement, c->initial_permanence,
                         c->connected_threshold};
    const char* names[4] = {"perm_increment", "perm_decrement", "initial_permanence",
                            "connected_threshold"};
    for (int i = 0; i < 4; ++i)
        if (!(fr[i] >= 0.0f && fr[i] <= 1.0f))
            return fail(SP_E_CONFIG, "%s must be in [0,1] (S:48)", names[i]);
    const uint32_t C32 = (c->num_columns + 31u) & ~31u;
    if (sp::bits_for(c->synapses_per_column) + 27u + sp::ceil_log2(C32) > 64u)
        return fail(SP_E_CONFIG, "rank key exceeds 64 bits: ceil(log2(S+1))+27+ceil(log2(C32)) > 64");
    if (c->max_inputs == 0) return fail(SP_E_CONFIG, "max_inputs must be >= 1");
    if (c->force_path > SP_PATH_BATCHED)
        return fail(SP_E_CONFIG, "force_path must be SP_PATH_AUTO/PER_INPUT/BATCHED");
    if (c->flags & SP_FLAG_FULL_LEARNING) {
        if (c->duty_cycle_period == 0 || c->duty_cycle_period > (1u << 24))
            return fail(SP_E_CONFIG, "full learning: duty_cycle_period must be in [1, 2^24] (S:150)");
        if (!(c->max_boost >= 1.0f && c->max_boost < 16.0f))
            return fail(SP_E_CONFIG, "full learning: max_boost must be in [1,16) (S:149, R4)");
    }
    return SP_OK;
}

}  // namespace

namespace sp {

Geometry make_geometry(const sp_config& cfg) {
    Geometry g{};
    g.W = cfg.input_width;
    g.H = cfg.input_height;
    g.whole = cfg.patch_width == 0 && cfg.patch_height == 0;
    g.pw = g.whole ? g.W : cfg.patch_width;
    g.ph = g.whole ? g.H : cfg.patch_height;
    g.P = (g.W / g.pw) * (g.H / g.ph);
    g.nbits = g.pw * g.ph;
    g.C = cfg.num_columns;
    g.C32 = (g.C + 31u) & ~31u;
    g.ncw = g.C32 / 32u;
    g.S = cfg.synapses_per_column;
    g.keyL = ceil_log2(g.C32);
    g.keyBits = bits_for(g.S) + 27u + g.keyL;
    return g;
}

// Shared-memory plan of the batched kernel.
BatchedLayout plan_batched_layout(const Geometry& g, int max_smem) {
    // Ring of `stages` x 32 KiB stages filled by 2-D TMA boxes of 128 B x 32 inputs (8 per
    // stage), then the window of Lw bit-sliced words (+ zero slot), Bc, barriers.  The raw
    // counts uint16[32][C32] reuse the ring once streaming is over, so the ring must hold
    // them.  scripts/bench_tma.cu: 4 x 32 KiB in flight streams at ~7 TB/s.
    BatchedLayout L;
    if (g.C32 > kMaxBatchedColumns || g.S > kMaxBatchedSynapses) return L;
    const uint32_t counts_bytes = 32u * g.C32 * 2u;
    const uint32_t fixed = g.C32 * 4u + 128u;  // Bc + barriers + release counters
    const uint32_t nbits_r = (g.nbits + kChunkBits - 1) / kChunkBits * kChunkBits;
    const char* es = std::getenv("SP_STAGES");  // development overrides (experiments only)
    const char* eb = std::getenv("SP_XBUFS");
    const char* er = std::getenv("SP_RING_KB");
    const uint32_t want_stages = es ? static_cast<uint32_t>(std::atoi(es)) : 0u;
    const uint32_t want_xbufs = eb ? static_cast<uint32_t>(std::atoi(eb)) : 0u;
    const uint32_t want_ring = er ? static_cast<uint32_t>(std::atoi(er)) * 1024u : 0u;
    // preference (measured on B200, 4096 x 960x540, C=1024, 512 threads, ELL prefetch):
    // 4 stages + double-buffered X 0.376 ms; 4 stages, one X 0.380; 3 stages + 2 X 0.383;
    // 3 stages, one X 0.384.  (The 1024-thread kernel without prefetch preferred one X.)
    // C32 > 1024 (4 column-warps per warp, no ELL prefetch registers): one X window wins
    // (C=2048, S=256: 0.458 vs 0.494 ms).  Round 2: a stage is `rows` KiB, so a 140 KiB ring
    // holds 5 stages of 28-input groups (the headline's) where 4 x 32 KiB held 4.
    const uint32_t K32 = kStageBytes;
    const uint32_t pref2[9][2] = {{5 * 28672u, 2}, {4 * K32, 2}, {4 * K32, 1}, {3 * K32, 2}, {3 * K32, 1},
                                  {2 * K32, 1},    {2 * K32, 2}, {5 * K32, 1}, {5 * K32, 2}};
    const uint32_t pref1[9][2] = {{4 * K32, 1}, {3 * K32, 1}, {2 * K32, 1}, {4 * K32, 2}, {3 * K32, 2},
                                  {2 * K32, 2}, {5 * K32, 1}, {5 * K32, 2}, {5 * 28672u, 1}};
    const auto& options = g.C32 > 1024u ? pref1 : pref2;
    for (const auto& o : options) {
        const uint32_t ring = o[0], xbufs = o[1], stages = ring / K32;
        if ((want_stages && (stages != want_stages || ring % K32)) || (want_xbufs && xbufs != want_xbufs) ||
            (want_ring && ring != want_ring))
            continue;
        if (ring < counts_bytes) continue;
        const int64_t avail = static_cast<int64_t>(max_smem) - ring - fixed;
        if (avail < 8 * static_cast<int64_t>(kChunkBits + 1)) continue;
        // largest Lw (multiple of the chunk, local idx < 65536) with xbufs*(Lw+1)*4 <= avail
        uint32_t Lw = static_cast<uint32_t>((avail / 4 / xbufs - 1) / kChunkBits * kChunkBits);
        Lw = std::min<uint32_t>(Lw, 64512u);
        Lw = std::min<uint32_t>(Lw, nbits_r);
        if (Lw == 0) continue;
        // one buffer is pointless when a single window covers the input
        if (xbufs == 2 && Lw >= g.nbits && !want_xbufs) continue;
        // large inputs need windows of >= 8 chunks or the per-window barriers dominate
        if (Lw < 8 * kChunkBits && nbits_r > Lw) continue;
        // balance the windows: same count, smallest Lw (multiple of the chunk) covering nbits
        const uint32_t nwin = (g.nbits + Lw - 1) / Lw;
        const uint32_t per = (g.nbits + nwin - 1) / nwin;
        Lw = (per + kChunkBits - 1) / kChunkBits * kChunkBits;
        L.ok = true;
        L.stages = stages;
        L.ring_bytes = ring;
        L.xbufs = xbufs;
        L.Lw = Lw;
        L.nwin = (g.nbits + Lw - 1) / Lw;
        // the window(s) double as the per-warp scratch of the top-k: tie lists (64 keys),
        // histograms ((S+2)/2 words) or raw bit-planes (ncw x nb <= 640 words), 32 warps;
        // coarse-key bit-planes (ncw x 16 <= 1024 words), 16 warps
        const uint32_t topk_bytes = std::max(32u * 64u * 8u, std::max(32u * 640u * 4u, 16u * 1024u * 4u));
        L.region_bytes = (std::max(xbufs * (Lw + 1u) * 4u, topk_bytes) + 127u) & ~127u;
        L.smem_bytes = ring + L.region_bytes + g.C32 * 4u + BatchedLayout::kMaxStages * 12u;
        if (static_cast<int64_t>(L.smem_bytes) > max_smem) {
            L.ok = false;
            continue;
        }
        return L;
    }
    return L;
}

// Patch mode (NEXT-2): one X window = one tile; groups of <= 32 tiles of a tile-row.
BatchedLayout plan_patch_layout(const Geometry& g, int max_smem) {
    BatchedLayout L;
    if (g.whole || g.pw % 32u || 32u * g.nbits > 49152u || g.C32 > 1024u || g.S > kMaxBatchedSynapses) return L;
    const uint32_t stage_bytes = (32u * g.nbits + 1023u) / 1024u * 1024u;
    const uint32_t Lw = (g.nbits + 31u) / 32u * 32u;
    const uint32_t topk_bytes = 16u * 1024u * 4u;  // 16 warps: coarse bit-planes <= 1024 words
    for (uint32_t stages = 4; stages >= 2; --stages) {
        const uint32_t smem = stages * stage_bytes + ((Lw + 4u) & ~3u) * 4u + 32u * g.C32 * 2u + topk_bytes +
                              g.C32 * 4u + stages * 12u;
        if (static_cast<int>(smem) > max_smem) continue;
        L.ok = true;
        L.stages = stages;
        L.xbufs = 1;
        L.Lw = Lw;
        L.nwin = 1;
        L.region_bytes = topk_bytes;
        L.smem_bytes = smem;
        return L;
    }
    return L;
}

bool encode_patches_tmap(CUtensorMap* map, const uint8_t* frames, const Geometry& g, uint32_t frames_n) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q{};
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return false;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    // view of the frames as {x in tile, tile, y in tile, tile-row}: tile t of tile-row r is
    // frame r / ty, tile-row r % ty, column t (R13); box {pw, 32 tiles, ph, 1}
    const uint32_t tx = g.W / g.pw, ty = g.H / g.ph;
    const cuuint64_t dims[4] = {g.pw, tx, g.ph, static_cast<cuuint64_t>(ty) * frames_n};
    const cuuint64_t strides[3] = {g.pw, g.W, static_cast<cuuint64_t>(g.W) * g.ph};
    const cuuint32_t box[4] = {g.pw, 32u, g.ph, 1u};
    const cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<uint8_t*>(frames), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Tensor-core patch kernel (sp_patch_mma.cu): whole frame rows of 4 tile-rows, as a view
// {W/k, k, y in tile, tile-row} with W/k <= 256 (TMA box dimension limit); box {W/k, k, sps, 4}.
uint32_t mma_row_split(uint32_t W) {
    for (uint32_t k = 1; k <= W; ++k)
        if (W % k == 0 && W / k <= 256u && (W / k) % 16u == 0) return k;
    return 0;
}

bool encode_mma_tmap(CUtensorMap* b, const uint8_t* frames, const Geometry& g, uint32_t frames_n, uint32_t sps) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q{};
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return false;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const uint32_t k = mma_row_split(g.W), ty = g.H / g.ph;
    if (!k) return false;
    const cuuint64_t dims[4] = {g.W / k, k, g.ph, static_cast<cuuint64_t>(ty) * frames_n};
    const cuuint64_t str[3] = {g.W / k, g.W, static_cast<cuuint64_t>(g.W) * g.ph};
    const cuuint32_t box[4] = {g.W / k, k, sps, 4u};
    const cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
    return encode(b, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<uint8_t*>(frames), dims, str, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool encode_frames_tmap(CUtensorMap* map, const uint8_t* frames, uint32_t nbits, uint32_t rows, uint32_t box_rows) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q{};
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return false;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[2] = {nbits, rows};
    const cuuint64_t strides[1] = {nbits};
    const cuuint32_t box[2] = {kBoxBytes, box_rows};
    const cuuint32_t estr[2] = {1u, 1u};
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(frames), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Bit-planes uint32[rows][words] (words % 4 == 0: 16-byte row stride), box {32 words, 32 rows}.
bool encode_packed_tmap(CUtensorMap* map, const uint32_t* planes, uint32_t words, uint32_t rows, uint32_t box_rows) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q{};
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return false;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[2] = {words, rows};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(words) * 4u};
    const cuuint32_t box[2] = {kChunkBits / 32u, box_rows};
    const cuuint32_t estr[2] = {1u, 1u};
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<uint32_t*>(planes), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Groups of R <= 32 inputs and cluster size K: estimated time of each (K, R)
// from an HBM term, a per-CTA streaming term and the cluster tail.
void plan_batched_grid(const Geometry& g, uint32_t nwin, uint32_t n, int sm_count,
                       const int* max_clusters, uint32_t* groups, uint32_t* Kout, uint32_t* Rout,
                       uint32_t* gsplit_out) {
    // Time model, fitted to measurements (960x540, C 1024, S 256): a CTA's time is
    // its ceil(nwin / K) windows at ~0.7 us per 1024-pixel chunk whatever its rows R (16..32:
    // the per-SM transpose/flag/release work, not HBM, sets the pace: 4096 frames on one CTA per
    // SM and 512 frames on 6-CTA clusters both spend ~7 us per 10-chunk window); R only decides
    // how many groups (clusters) there are, so one wave needs G = ceil(n / R) <= cap; the chip's
    // HBM (~7 TB/s) bounds the whole batch; the cluster tail (DSMEM sum of the partial counts,
    // one warp per input's selection) is ~17 us for K > 1, ~9 us for K = 1.
    const double hbm_bpc = 3600.0;   // chip HBM read bytes per SM-cycle (~7 TB/s @ 1.95 GHz)
    const double chunk_cyc = 0.70 * 1950.0;
    const double cyc_us = 1950.0;
    const uint32_t gmin = (n + 31u) / 32u;
    double best = 1e300;
    uint32_t bestG = gmin, bestK = 1, bestR = (n + gmin - 1u) / gmin;
    const char* fk = std::getenv("SP_FORCE_K");  // development: cluster size K (timing experiments)
    const uint32_t force_k = fk ? static_cast<uint32_t>(std::atoi(fk)) : 0u;
    const char* fr = std::getenv("SP_FORCE_R");  // development: inputs per group
    const uint32_t force_r = fr ? static_cast<uint32_t>(std::atoi(fr)) : 0u;
    // a group's K CTAs split its chunks evenly (sp_batched.cu); a split CTA may gather up to two
    // partial windows in full (their ELL cells), ~1.5 chunks' time
    const uint32_t nct = (g.nbits + kChunkBits - 1u) / kChunkBits;
    auto cta_chunks = [&](uint32_t K) { return (nct + K - 1u) / K + (K > 1u ? 1.5 : 0.0); };
    (void)nwin;
    for (uint32_t K = 1; K <= 8u; ++K) {
        if (K > nwin) break;
        if (force_k && K != force_k) continue;
        int cap = max_clusters ? max_clusters[K] : sm_count / static_cast<int>(K);
        if (cap <= 0) continue;
        const uint32_t rlo = std::max<uint32_t>(1u, (n + cap - 1u) / static_cast<uint32_t>(cap));
        for (uint32_t R = force_r ? std::min(force_r, 32u) : std::min<uint32_t>(rlo, 32u); R <= 32u; ++R) {
            if (force_r && R != std::min(force_r, 32u)) continue;
            const uint32_t G = (n + R - 1u) / R;
            const uint32_t waves = (G + cap - 1) / cap;
            const double stream_cta = cta_chunks(K) * chunk_cyc;
            const double t = std::max(static_cast<double>(n) * g.nbits / hbm_bpc, waves * stream_cta) +
                             (K > 1 ? 17.0 : 9.0) * cyc_us;
            if (std::getenv("SP_PLAN_DEBUG"))
                std::fprintf(stderr, "plan n %u K %u cap %d R %u G %u waves %u t_us %.1f\n", n, K, cap, R, G, waves,
                             t / cyc_us);
            if (t < best * 0.98) {
                best = t;
                bestG = G;
                bestK = K;
                bestR = R;
            }
            if (R >= n) break;
        }
    }
    // global split (K CTAs per group in one cooperative launch, partial counts through L2): any
    // K, all SMs usable (clusters of 6+ pack into GPCs badly: 22 of 6, 15 of 8 or 9), one wave
    // only; its tail (partial counts to L2, the group barrier, the K-row sums) measured ~22 us
    // (512 frames: K 9 on 144 SMs 0.064 ms vs clusters of 6 on 132 SMs 0.069; 1024 and 2048
    // frames stay on clusters: 0.103 vs 0.106, 0.182 vs 0.187)
    uint32_t bestS = 0;
    const char* fs = std::getenv("SP_FORCE_GSPLIT");  // development / tests: 1 force, 0 forbid
    const int force_s = fs ? std::atoi(fs) : -1;
    if (force_s == 1) best = 1e300;
    for (uint32_t K = 2; force_s != 0 && K <= 16u && K <= nwin; ++K) {
        if (force_k && K != force_k) continue;
        const uint32_t cap = static_cast<uint32_t>(sm_count) / K;
        if (cap == 0) continue;
        uint32_t R = std::max<uint32_t>(1u, (n + cap - 1u) / cap);
        if (force_r) R = std::min(force_r, 32u);
        if (R > 32u) continue;
        const uint32_t G = (n + R - 1u) / R;
        if (G > cap) continue;
        const double stream_cta = cta_chunks(K) * chunk_cyc;
        const double t = std::max(static_cast<double>(n) * g.nbits / hbm_bpc, stream_cta) + 22.0 * cyc_us;
        if (std::getenv("SP_PLAN_DEBUG"))
            std::fprintf(stderr, "plan gsplit n %u K %u cap %u R %u G %u t_us %.1f\n", n, K, cap, R, G, t / cyc_us);
        if (t < best * 0.98) {
            best = t;
            bestG = G;
            bestK = K;
            bestR = R;
            bestS = 1;
        }
    }
    *groups = bestG;
    *Kout = bestK;
    *Rout = bestR;
    *gsplit_out = bestS;
}

}  // namespace sp

struct sp_handle {
    sp_config cfg{};
    sp::Geometry g{};
    sp::BatchedLayout lay{};
    int device = 0, sm_count = kDefaultSms, max_smem = kDefaultSmem;
    int max_clusters[9] = {0};
    // device state (canonical order) and derived layouts
    uint32_t* d_idx = nullptr;
    float* d_perm = nullptr;
    float* d_boost = nullptr;
    uint32_t* d_bc = nullptr;
    uint32_t* d_syn = nullptr;
    uint4* d_ell = nullptr;
    uint32_t* d_ell_off = nullptr;
    uint16_t* d_ell_nb = nullptr;
    uint32_t* d_ell_pos = nullptr;
    uint32_t ell_slots = 0;
    bool ell_dirty = false;
    uint64_t* d_trace = nullptr;  // SP_TRACE=1: per-CTA phase timestamps of the batched kernel
    uint4* d_part = nullptr;      // global split: partial counts [SMs][32][C32] u16
    uint32_t* d_gsbar = nullptr;  // global split: [2][SMs] group barrier counters (zero at rest)
    bool uniform_bc = true;       // all boosts equal (enables the histogram top-k)
    uint32_t batched_threads = 512;  // threads per CTA of the batched kernel
    // per-column boosts: wavelet local top-k from this radius on, the bit-sliced comparator below
    // (crossover measured at r ~ 80-100 for C = 1024: scripts/local_general_timing.py)
    uint32_t wm_min_radius = 96;
    uint32_t wm_min_radius_pi = 256;  // the same for the per-input k_inhibit (CTA wavelet)
    // local inhibition (batched kernels): candidate pruning from this radius on, when the
    // candidates fit the warp's scratch (else the wavelet / comparator).  Set at create from the
    // expected candidate count ~ k*C/(2r) (scripts/local_topk_timing.py): it beats
    // the 15-level per-column-boost wavelet / comparator and (uniform boost, level sweep) the
    // <= 8-level uniform wavelet below ~350 candidates.
    uint32_t cand_min_radius = 0, cand_min_radius_u = 0;
    uint32_t force_groups = 0;        // SP_GROUPS (tests): batched groups per call, cluster size 1
    // tensor-core patch kernel (NEXT-2, sp_patch_mma.cu): 0 clusters = not eligible
    uint8_t* d_conn = nullptr;        // conn u8 [C32][nbits]: 1 where a connected synapse sits
    bool conn_dirty = true;
    uint32_t mma_Q = 0, mma_smem = 0, mma_region = 0, mma_raw_stages = 0, mma_conv_stages = 0, mma_sps = 1,
             mma_clusters = 0;
    uint32_t wm_umax = 32766u;        // per-warp wavelet coarse keys: u - 1 <= wm_umax (15 levels;
                                      // 12 bits: 0.603 vs 0.614 ms with seeded boosts in [1, 2] but
                                      // 0.697 vs 0.665 ms with full-learning boosts near 1)
    uint32_t learn_Q = 0, learn_smem = 0;  // cluster learning: CTAs per cluster (0 = not eligible)
    bool learn_dbl = false;                 // cluster learning: double-buffered bit-planes
    bool last_learn_cluster = false;
    // grid-resident learning (one CTA per SM; column-major synapse table streamed from L2)
    uint32_t* d_synT = nullptr;  // [C32][S] idx | connected << 31
    uint32_t* d_gbar = nullptr;  // grid barrier counter
    uint32_t grid_G = 0, grid_smem = 0, grid_own = 0, grid_win = 0, grid_ccols = 0, grid_stages = 0;
    // grid-resident learning with the full learning step (sp_learn_grid_full.cu)
    uint32_t gridf_G = 0, gridf_smem = 0, gridf_own = 0, gridf_ccols = 0, gridf_stages = 0, gridf_cap = 0;
    unsigned long long* d_span_part = nullptr;  // [2][gridf_G]
    bool grid_dbl = false;
    bool synT_dirty = true;      // d_synT must be rebuilt from idx/perm before grid learning
    // full learning (NEXT-1; DESIGN R17-R21)
    float* d_adc = nullptr;      // [C32] active duty cycles
    float* d_odc = nullptr;      // [C32] overlap duty cycles
    uint32_t* d_span = nullptr;  // [C32] connected spans
    uint32_t* d_radius = nullptr;  // radius in force (device scalar)
    float* d_fscratch = nullptr;   // window-maximum tables of k_full
    uint32_t* d_bits_all = nullptr;  // prepacked bit-planes of a learning chunk [inputs][Wn4]
    uint32_t bits_all_cap = 0;       // capacity in inputs
    bool span_dirty = true;      // d_span must be recomputed before full learning
    uint64_t iteration = 0;      // SP inputs learned
    // per-video histograms (NEXT-4): offsets and count scratch, grown on demand
    uint32_t* d_hist_off = nullptr;
    uint32_t* d_hist_counts = nullptr;
    size_t hist_off_cap = 0, hist_counts_cap = 0;
    std::vector<uint32_t> h_hist_off;  // offsets last uploaded (skip the upload when unchanged)
    bool syn_dirty = false;      // d_syn must be rebuilt from idx/perm before the per-input path
    uint32_t last_learn_path = SP_LEARN_PER_INPUT;
    // scratch and results
    uint32_t Wn = 0, sub_inputs = 0;
    uint32_t* d_bits = nullptr;
    uint32_t* d_raw = nullptr;
    uint32_t* d_sdr = nullptr;
    uint32_t* d_counts = nullptr;
    // where the last call's results live: the handle's buffers, or the caller's (sp_compute_into)
    uint32_t* res_sdr = nullptr;
    uint32_t* res_counts = nullptr;
    uint16_t* d_raw_rec = nullptr;
    float* d_boosted_rec = nullptr;
    // end-to-end staging
    uint8_t* d_stage[2] = {nullptr, nullptr};
    uint32_t stage_frames = 0;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr};
    // bookkeeping
    std::vector<uint32_t> h_idx;
    uint32_t last_inputs = 0;
    bool has_result = false;
    std::atomic<uint64_t> launches{0};
    sp_plan_info last_plan{};
};

namespace {

template <typename T>
cudaError_t dalloc(T** p, size_t count) {
    if (count == 0) count = 1;
    return cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T));
}

void release(sp_handle* h) {
    if (!h) return;
    cudaSetDevice(h->device);
    void* ptrs[] = {h->d_part, h->d_gsbar, h->d_trace, h->d_idx,  h->d_perm,    h->d_boost,   h->d_bc,      h->d_syn,
                    h->d_ell,  h->d_ell_off, h->d_ell_nb,  h->d_ell_pos, h->d_bits,
                    h->d_raw,  h->d_sdr,     h->d_counts,  h->d_raw_rec, h->d_boosted_rec,
                    h->d_stage[0], h->d_stage[1], h->d_synT,  h->d_gbar, h->d_adc, h->d_odc,
                    h->d_span, h->d_radius, h->d_fscratch, h->d_hist_off, h->d_hist_counts,
                    h->d_bits_all, h->d_conn, h->d_span_part};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
    for (int i = 0; i < 2; ++i) {
        if (h->ev_h2d[i]) cudaEventDestroy(h->ev_h2d[i]);
        if (h->ev_free[i]) cudaEventDestroy(h->ev_free[i]);
    }
    delete h;
}

sp_plan_info make_plan(const sp_handle* h, uint32_t n, bool learn, const uint8_t* frames) {
    sp_plan_info pl{};
    const sp::Geometry& g = h->g;
    pl.input_bits = g.nbits;
    pl.inputs_per_frame = g.P;
    pl.num_inputs = n;
    pl.columns_padded = g.C32;
    pl.sdr_words = g.ncw;
    uint32_t reason = 0;
    if (learn) reason |= sp::kNotBatchedLearn;
    if (!g.whole && !h->lay.ok) reason |= sp::kNotBatchedPatch | sp::kNotPatchGeometry;
    if (g.nbits % 16u) reason |= sp::kNotBatchedAlign;
    if (frames && (reinterpret_cast<uintptr_t>(frames) & 15u)) reason |= sp::kNotBatchedAlign;
    if (g.C32 > sp::kMaxBatchedColumns) reason |= sp::kNotBatchedColumns;
    if (g.S > sp::kMaxBatchedSynapses) reason |= sp::kNotBatchedSynapses;
    if (h->cfg.force_path == SP_PATH_PER_INPUT) reason |= sp::kNotBatchedForced;
    if (!h->lay.ok) reason |= sp::kNotBatchedSmem;
    pl.reason = reason;
    const bool mma = !g.whole && !learn && h->mma_clusters && (h->cfg.flags & SP_FLAG_PATCH_TENSOR) &&
                     !(h->cfg.flags & SP_FLAG_PATCH_GATHER) &&
                     h->cfg.force_path != SP_PATH_PER_INPUT && !(frames && (reinterpret_cast<uintptr_t>(frames) & 15u));
    if (mma && n > 0) {
        // tensor-core patch kernel: blocks of 4 tile-rows x 32 slots, clusters of C32/128 CTAs
        const uint32_t tile_rows = n / (g.W / g.pw);
        pl.path = SP_PATH_BATCHED;
        pl.reason = 0;
        pl.tensor_cores = 1;
        pl.groups = (tile_rows + 3u) / 4u;
        pl.cluster = h->mma_Q;
        pl.ctas = std::min(pl.groups, h->mma_clusters) * h->mma_Q;
        pl.window_bits = g.nbits;
        pl.num_windows = 1;
        pl.chunk_bits = 32;
        pl.stages = h->mma_raw_stages;
        pl.smem_bytes = h->mma_smem;
        return pl;
    }
    if (reason == 0 && n > 0 && !g.whole) {
        // patch kernel: groups of <= 32 tiles of one tile-row, persistent CTAs
        const uint32_t tx = g.W / g.pw;
        pl.path = SP_PATH_BATCHED;
        pl.groups = (n / tx) * ((tx + 31u) / 32u);
        pl.cluster = 1;
        pl.ctas = std::min<uint32_t>(pl.groups, static_cast<uint32_t>(h->sm_count));
        pl.window_bits = h->lay.Lw;
        pl.num_windows = 1;
        pl.chunk_bits = g.nbits;
        pl.stages = h->lay.stages;
        pl.smem_bytes = h->lay.smem_bytes;
    } else if (reason == 0 && n > 0) {
        pl.path = SP_PATH_BATCHED;
        uint32_t G = 0, K = 1, R = 32, S = 0;
        sp::plan_batched_grid(g, h->lay.nwin, n, h->sm_count, h->max_clusters[1] ? h->max_clusters : nullptr, &G,
                              &K, &R, &S);
        if (h->force_groups) {  // test override: fewer, fuller groups (the paired top-k branches
            G = std::max<uint32_t>((n + 31u) / 32u, std::min<uint32_t>(n, h->force_groups));  // need > NW
            K = 1;                                                                 // inputs per group)
            R = (n + G - 1u) / G;
            G = (n + R - 1u) / R;
            S = 0;
        }
        pl.global_split = S;
        // groups of exactly R inputs (the last one shorter): a box of R rows reads only its own
        // group's frames (with balanced groups of 27/28 in 32-row boxes, 13% of the bytes a CTA
        // ingested were its neighbour's rows, L2 hits that still cost the SM's TMA ingest)
        pl.group_inputs = R;
        pl.groups = G;
        pl.cluster = K;
        pl.ctas = G * K;
        pl.window_bits = h->lay.Lw;
        pl.num_windows = h->lay.nwin;
        pl.chunk_bits = sp::kChunkBits;
        // stages of R KiB (8 boxes of R rows x 128 B) in the ring
        pl.stages = std::min<uint32_t>(sp::BatchedLayout::kMaxStages, h->lay.ring_bytes / (R * 1024u));
        pl.smem_bytes = h->lay.smem_bytes;
    } else {
        pl.path = SP_PATH_PER_INPUT;
    }
    return pl;
}

// Windowed ELL of the batched path.  Cell (w, cw) holds, for the 32
// columns of column-warp cw, their synapses falling in window w as uint16 window-local
// indices, 8 slots per lane per block, blocks laid out [block][lane] (coalesced uint4
// per lane).  Disconnected synapses and padding point to the zero slot Lw.
// Slot schedule of one ELL cell (window w, column-word cw): slot t of lane l gathers X[i] for one
// of column 32 cw + l's synapses i in the window.  The 32 lanes of a slot are one shared-memory
// load, so lanes whose indices share a bank (i mod 32) serialise.  The sum is order-invariant, so
// the slots are scheduled greedily to be conflict-free: per slot, lanes in order of remaining
// synapses take one from a bank not yet used in the slot (the bank of most remaining synapses),
// a bipartite edge colouring that needs ~max(lane degree, bank degree) slots (random synapses:
// 16 slots at 2.1x fewer bank-cycles per window cell of the whole-frame kernel, 288-296 instead
// of 256 slots at 2x fewer bank-cycles for a 32x30 patch).  Development: SP_ELL_SCHED=0 keeps
// the synapses in index order.
void schedule_cell(const std::vector<std::pair<uint32_t, uint32_t>>* lanes, uint32_t nl,
                   std::vector<uint32_t>* slot_of) {
    static const bool sched = [] {
        const char* e = std::getenv("SP_ELL_SCHED");
        return !(e && std::atoi(e) == 0);
    }();
    for (uint32_t l = 0; l < nl; ++l) slot_of[l].assign(lanes[l].size(), 0u);
    if (!sched) {
        for (uint32_t l = 0; l < nl; ++l)
            for (uint32_t j = 0; j < lanes[l].size(); ++j) slot_of[l][j] = j;
        return;
    }
    std::vector<uint32_t> bucket[32][32];  // [lane][bank] -> entries j of lanes[l]
    uint32_t cnt[32] = {0};
    for (uint32_t l = 0; l < nl; ++l) {
        for (uint32_t j = 0; j < lanes[l].size(); ++j) bucket[l][lanes[l][j].second & 31u].push_back(j);
        cnt[l] = static_cast<uint32_t>(lanes[l].size());
    }
    uint32_t order[32];
    for (uint32_t t = 0;; ++t) {
        uint32_t left = 0;
        for (uint32_t l = 0; l < nl; ++l) left += cnt[l], order[l] = l;
        if (!left) break;
        std::sort(order, order + nl, [&](uint32_t a, uint32_t b) { return cnt[a] > cnt[b]; });
        uint32_t used = 0;
        for (uint32_t q = 0; q < nl; ++q) {
            const uint32_t l = order[q];
            if (!cnt[l]) break;
            int best = -1;
            for (uint32_t bk = 0; bk < 32u; ++bk)
                if (!(used >> bk & 1u) && !bucket[l][bk].empty() &&
                    (best < 0 || bucket[l][bk].size() > bucket[l][best].size()))
                    best = static_cast<int>(bk);
            if (best < 0) continue;  // every bank of this lane is taken in this slot: wait
            slot_of[l][bucket[l][best].back()] = t;
            bucket[l][best].pop_back();
            used |= 1u << best;
            --cnt[l];
        }
    }
}

sp_status build_ell(sp_handle* h, const float* perm_host) {
    const sp::Geometry& g = h->g;
    const uint32_t Lw = h->lay.Lw, nwin = h->lay.nwin;
    // per cell and lane: (synapse s, window-local index) in index order, then the slot schedule
    std::vector<uint32_t> slot_of_syn(static_cast<size_t>(g.C) * g.S, 0u);
    std::vector<uint32_t> off(static_cast<size_t>(nwin) * g.ncw), nb(off.size());
    {
        std::vector<std::pair<uint32_t, uint32_t>> lanes[32];
        std::vector<uint32_t> slot_of[32];
        for (uint32_t cw = 0; cw < g.ncw; ++cw) {
            for (uint32_t w = 0; w < nwin; ++w) {
                for (uint32_t l = 0; l < 32u; ++l) {
                    lanes[l].clear();
                    const uint32_t c = cw * 32u + l;
                    if (c >= g.C) continue;
                    for (uint32_t s2 = 0; s2 < g.S; ++s2) {  // the column's synapses in window w
                        const uint32_t i = h->h_idx[c * g.S + s2];
                        if (i / Lw == w) lanes[l].emplace_back(s2, i % Lw);
                    }
                }
                schedule_cell(lanes, 32u, slot_of);
                uint32_t mx = 0;
                for (uint32_t l = 0; l < 32u; ++l)
                    for (uint32_t j = 0; j < lanes[l].size(); ++j) {
                        mx = std::max(mx, slot_of[l][j] + 1u);
                        slot_of_syn[static_cast<size_t>(cw * 32u + l) * g.S + lanes[l][j].first] = slot_of[l][j];
                    }
                nb[static_cast<size_t>(w) * g.ncw + cw] = (mx + 7u) / 8u;
            }
        }
    }
    uint64_t total = 0;
    for (uint32_t w = 0; w < nwin; ++w)
        for (uint32_t cw = 0; cw < g.ncw; ++cw) {
            const size_t cell = static_cast<size_t>(w) * g.ncw + cw;
            off[cell] = static_cast<uint32_t>(total);
            total += static_cast<uint64_t>(nb[cell]) * 32u;
            if (nb[cell] > 65535u) return fail(SP_E_CONFIG, "ELL cell too large");
        }
    if (total * 8u >= (1ull << 32)) return fail(SP_E_CONFIG, "ELL exceeds 2^32 slots");
    std::vector<uint16_t> ell(static_cast<size_t>(total) * 8u, static_cast<uint16_t>(Lw));
    std::vector<uint32_t> pos(static_cast<size_t>(g.C) * g.S);
    const float tau = h->cfg.connected_threshold;
    for (uint32_t c = 0; c < g.C; ++c) {
        const uint32_t cw = c / 32u, lane = c % 32u;
        for (uint32_t s = 0; s < g.S; ++s) {
            const uint32_t i = h->h_idx[c * g.S + s];
            const uint32_t w = i / Lw;
            const uint32_t slot = slot_of_syn[static_cast<size_t>(c) * g.S + s];
            const size_t cell = static_cast<size_t>(w) * g.ncw + cw;
            const size_t p = (static_cast<size_t>(off[cell]) + (slot / 8u) * 32u + lane) * 8u + slot % 8u;
            ell[p] = static_cast<uint16_t>(perm_host[c * g.S + s] >= tau ? i % Lw : Lw);
            pos[static_cast<size_t>(c) * g.S + s] = static_cast<uint32_t>(p);
        }
    }
    std::vector<uint16_t> nb16(nb.begin(), nb.end());
    if (h->d_ell) cudaFree(h->d_ell), h->d_ell = nullptr;
    if (h->d_ell_off) cudaFree(h->d_ell_off), h->d_ell_off = nullptr;
    if (h->d_ell_nb) cudaFree(h->d_ell_nb), h->d_ell_nb = nullptr;
    if (h->d_ell_pos) cudaFree(h->d_ell_pos), h->d_ell_pos = nullptr;
    cudaError_t e = dalloc(&h->d_ell, total);
    if (e == cudaSuccess) e = dalloc(&h->d_ell_off, off.size());
    if (e == cudaSuccess) e = dalloc(&h->d_ell_nb, nb16.size());
    if (e == cudaSuccess) e = dalloc(&h->d_ell_pos, pos.size());
    if (e != cudaSuccess) return fail(SP_E_OOM, "ELL allocation failed: %s", cudaGetErrorString(e));
    e = cudaMemcpy(h->d_ell, ell.data(), ell.size() * 2u, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(h->d_ell_off, off.data(), off.size() * 4u, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(h->d_ell_nb, nb16.data(), nb16.size() * 2u, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(h->d_ell_pos, pos.data(), pos.size() * 4u, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "ELL upload");
    h->ell_slots = static_cast<uint32_t>(total * 8u);
    h->ell_dirty = false;
    return SP_OK;
}

// Uploads a full canonical state and rebuilds every derived layout (synchronous).
sp_status upload_state(sp_handle* h, const uint32_t* idx, const float* perm, const float* boost) {
    const sp::Geometry& g = h->g;
    const size_t cs = static_cast<size_t>(g.C) * g.S;
    h->h_idx.assign(idx, idx + cs);
    std::vector<float> boost32(g.C32, 1.0f);
    std::vector<uint32_t> bc(g.C32, 0u);
    for (uint32_t c = 0; c < g.C; ++c) {
        boost32[c] = boost[c];
        bc[c] = static_cast<uint32_t>(boost[c] * 8388608.0f);  // exact: boost in [1,16) (R4)
    }
    h->uniform_bc = std::all_of(bc.begin(), bc.begin() + g.C, [&](uint32_t v) { return v == bc[0]; });
    if (std::getenv("SP_NO_UNIFORM_TOPK")) h->uniform_bc = false;  // development override
    cudaError_t e = cudaMemcpy(h->d_idx, idx, cs * 4u, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(h->d_perm, perm, cs * 4u, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(h->d_boost, boost32.data(), g.C32 * 4u, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(h->d_bc, bc.data(), g.C32 * 4u, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "state upload");
    e = sp::launch_build_syn(h->d_idx, h->d_perm, h->cfg.connected_threshold, g.C, g.C32, g.S,
                             h->d_syn, nullptr);
    h->launches++;
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(e, "synapse layout build");
    h->syn_dirty = false;
    h->synT_dirty = true;
    h->span_dirty = true;
    h->conn_dirty = true;
    if (h->lay.ok) return build_ell(h, perm);
    return SP_OK;
}

sp_status check_handle(sp_handle* h) {
    if (!h) return fail(SP_E_ARG, "handle is NULL");
    cudaError_t e = cudaSetDevice(h->device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    return SP_OK;
}

// CTAs per input of k_inhibit: local inhibition over many columns is O(C * r) per input, so
// the SDR words of one input are split over CTAs (each builds the key planes it needs) until
// the SMs are busy; global inhibition and small C keep one CTA per input.
uint32_t inhibit_parts(const sp_handle* h, uint32_t inputs) {
    const sp::Geometry& g = h->g;
    if (h->cfg.inhibition_radius == 0 || g.C32 < 2048u || std::getenv("SP_NO_SPLIT_INHIBIT")) return 1u;
    const uint32_t want = (2u * static_cast<uint32_t>(h->sm_count) + inputs - 1u) / std::max(inputs, 1u);
    return std::max(1u, std::min(want, g.ncw / 4u));
}

// Scratch for the bit-planes a learning chunk prepacks: sized once for the largest chunk a call
// can have (the allocation synchronises).
sp_status ensure_prepack_scratch(sp_handle* h, uint32_t fpc, uint32_t n_frames, uint32_t Wn4) {
    const sp::Geometry& g = h->g;
    if (h->bits_all_cap >= std::min(fpc, n_frames) * g.P) return SP_OK;
    const uint32_t cap = std::min(fpc * g.P, std::max(h->cfg.max_inputs / g.P, 1u) * g.P);
    if (h->d_bits_all) cudaFree(h->d_bits_all), h->d_bits_all = nullptr;
    const cudaError_t e = dalloc(&h->d_bits_all, static_cast<size_t>(cap) * Wn4);
    if (e != cudaSuccess) return fail(SP_E_OOM, "prepacked bit-planes: %s", cudaGetErrorString(e));
    h->bits_all_cap = cap;
    return SP_OK;
}

// k_pack of a chunk's inputs into the prepacked planes (stride Wn4 words)
cudaError_t launch_prepack(sp_handle* h, const uint8_t* frames, uint32_t inputs, uint32_t Wn4, cudaStream_t s) {
    sp::PerInputParams pk{};
    pk.frames = frames;
    pk.num_inputs = inputs;
    pk.g = h->g;
    pk.bits = h->d_bits_all;
    pk.Wn = h->Wn;
    pk.bits_stride = Wn4;
    h->launches++;
    return sp::launch_pack(pk, s);
}

// Full-learning constants and device state (R17-R21) for the learning kernels.
sp::FullLearn full_learn_params(const sp_handle* h) {
    sp::FullLearn f{};
    f.on = (h->cfg.flags & SP_FLAG_FULL_LEARNING) ? 1u : 0u;
    f.adapt = f.on && h->cfg.inhibition_radius > 0 ? 1u : 0u;
    f.pm1 = static_cast<float>(h->cfg.duty_cycle_period) - 1.0f;  // exact: P <= 2^24
    f.P = static_cast<float>(h->cfg.duty_cycle_period);
    f.mb1 = h->cfg.max_boost - 1.0f;           // one fp32 RN subtraction (R19)
    f.bump = 0.1f * h->cfg.connected_threshold;  // one fp32 RN product (R20)
    f.adc = h->d_adc;
    f.odc = h->d_odc;
    f.boost = h->d_boost;
    f.bc = h->d_bc;
    f.radius = h->d_radius;
    f.span = f.on ? h->d_span : nullptr;
    f.scratch = h->d_fscratch;
    return f;
}

// Shared memory of the packed-input batched kernel: the same ring bytes cut into 8x as many
// 4 KiB stages (one mbarrier + release counter each).
uint32_t packed_smem_bytes(const sp::BatchedLayout& L) {
    return L.smem_bytes + L.stages * (sp::kPackedStagesPer - 1u) * 12u;
}

// The batched path (rows a1-a4) for n inputs of uint8 frames or (planes != NULL) bit-planes.
sp_status launch_batched_path(sp_handle* h, const uint8_t* frames, const uint32_t* planes, uint32_t n_frames,
                              uint32_t n, const sp_plan_info& pl, cudaStream_t s, uint32_t row0) {
    const sp::Geometry& g = h->g;
    const bool rec = (h->cfg.flags & SP_FLAG_RECORD_OVERLAPS) != 0;
    cudaError_t e = cudaSuccess;
    if (h->ell_dirty) {
        e = sp::launch_refresh_ell(h->d_idx, h->d_perm, h->d_ell_pos, h->cfg.connected_threshold,
                                   g.C, g.S, h->lay.Lw, reinterpret_cast<uint16_t*>(h->d_ell), s);
        h->launches++;
        if (e != cudaSuccess) return cuda_fail(e, "ELL refresh launch");
        h->ell_dirty = false;
    }
    sp::BatchedParams p{};
    if (planes) {
        if (!sp::encode_packed_tmap(&p.tmap, planes, ((h->Wn + 3u) / 4u * 4u), n, pl.group_inputs))
            return fail(SP_E_CUDA, "cuTensorMapEncodeTiled failed for the bit-planes (words %u, rows %u)",
                        ((h->Wn + 3u) / 4u * 4u), n);
    } else if (!g.whole) {
        if (!sp::encode_patches_tmap(&p.tmap, frames, g, n_frames))
            return fail(SP_E_CUDA, "cuTensorMapEncodeTiled failed for the tiles");
    } else if (!sp::encode_frames_tmap(&p.tmap, frames, g.nbits, n, pl.group_inputs))
        return fail(SP_E_CUDA, "cuTensorMapEncodeTiled failed for the frames (nbits %u, rows %u)",
                    g.nbits, n);
    p.num_inputs = n;
    p.rows = pl.group_inputs;
    p.nbits = g.nbits;
    p.C = g.C;
    p.C32 = g.C32;
    p.ncw = g.ncw;
    p.min_overlap = h->cfg.min_overlap;
    p.k = h->cfg.winners_set_size;
    p.radius = h->cfg.inhibition_radius;
    p.keyL = g.keyL;
    p.keyBits = g.keyBits;
    p.Lw = h->lay.Lw;
    p.nwin = h->lay.nwin;
    p.stages = planes ? h->lay.stages * sp::kPackedStagesPer : pl.stages;
    p.ring_bytes = h->lay.ring_bytes;
    p.gsplit = pl.global_split;
    p.part = h->d_part;
    p.gbar = h->d_gsbar;
    if (p.gsplit && (!p.part || !p.gbar || pl.ctas > static_cast<uint32_t>(h->sm_count)))
        return fail(SP_E_STATE, "global split without its scratch or with more CTAs than SMs");
    p.packed = planes ? 1u : 0u;
    p.region_bytes = h->lay.region_bytes;
    p.xbufs = h->lay.xbufs;
    p.one = 1u;
    p.S = g.S;
    p.uniform_bc = h->uniform_bc ? 1u : 0u;
    p.threads = h->batched_threads;
    p.trace = h->d_trace;
    p.groups = pl.groups;
    p.K = pl.cluster;
    p.ell_off = h->d_ell_off;
    p.ell_nb = h->d_ell_nb;
    p.ell = h->d_ell;
    p.bc = h->d_bc;
    p.boost = h->d_boost;
    p.sdr = h->res_sdr + static_cast<size_t>(row0) * g.ncw;
    p.counts = h->res_counts + row0;
    p.raw_out = rec ? h->d_raw_rec + static_cast<size_t>(row0) * g.C : nullptr;
    p.boosted_out = rec ? h->d_boosted_rec + static_cast<size_t>(row0) * g.C : nullptr;
    p.radius_dev = h->d_radius;
    p.wm_min_radius = h->wm_min_radius;
    p.wm_umax = h->wm_umax;
    p.cand_min_radius = h->cand_min_radius;
    p.cand_min_radius_u = h->cand_min_radius_u;
    if (const char* ecd = std::getenv("SP_CAND_DBG")) p.cand_dbg = static_cast<uint32_t>(std::atoi(ecd));
    if (const char* ebd = std::getenv("SP_BATCHED_DBG")) p.bdbg = static_cast<uint32_t>(std::atoi(ebd));
    if (pl.tensor_cores) {
        if (h->conn_dirty) {
            e = sp::launch_build_conn(h->d_idx, h->d_perm, h->cfg.connected_threshold, g.C, g.C32, g.S, g.nbits,
                                      h->d_conn, s);
            h->launches++;
            if (e != cudaSuccess) return cuda_fail(e, "connectivity build launch");
            h->conn_dirty = false;
        }
        sp::PatchMmaParams q{};
        if (!sp::encode_mma_tmap(&q.tmap_b, frames, g, n_frames, h->mma_sps))
            return fail(SP_E_CUDA, "cuTensorMapEncodeTiled failed for the tensor-core patch kernel");
        q.bp = p;
        q.bp.region_bytes = h->mma_region;
        q.Q = h->mma_Q;
        q.W = g.W;
        q.nbits = g.nbits;
        q.patch_w = g.pw;
        q.patch_h = g.ph;
        q.xchunks = g.pw / 32u;
        q.sps = h->mma_sps;
        q.tiles_x = g.W / g.pw;
        q.tile_rows = n_frames * (g.H / g.ph);
        q.nblocks = (q.tile_rows + 3u) / 4u;
        q.raw_stages = h->mma_raw_stages;
        q.conv_stages = h->mma_conv_stages;
        q.raw_stage_bytes = g.W * h->mma_sps * 4u;
        q.region_bytes = h->mma_region;
        q.conn = h->d_conn;
        q.multicast = 0u;  // per-CTA TMA (L2 hits) measured faster than the cluster multicast: 0.876 vs 0.964 ms
        if (const char* em = std::getenv("SP_MMA_MULTICAST")) q.multicast = q.Q > 1 && std::atoi(em) ? 1u : 0u;
        if (const char* ed = std::getenv("SP_MMA_DBG")) q.dbg = static_cast<uint32_t>(std::atoi(ed));
        const uint32_t clusters = std::min(q.nblocks, h->mma_clusters);
        static uint64_t* d_mtrace = nullptr;  // development aid: phase stamps of the tensor-core kernel
        const bool mtrace = std::getenv("SP_MMA_TRACE") != nullptr;
        if (mtrace) {
            q.trace_blocks = 256;
            if (!d_mtrace) cudaMalloc(&d_mtrace, 148u * 256u * 8u * 8u);
            cudaMemsetAsync(d_mtrace, 0, 148u * 256u * 8u * 8u, s);
            q.trace = d_mtrace;
        }
        e = sp::launch_patch_mma(q, h->mma_smem, clusters, s);
        if (mtrace && e == cudaSuccess) {
            std::vector<uint64_t> t(148u * 256u * 8u);
            cudaStreamSynchronize(s);
            cudaMemcpy(t.data(), d_mtrace, t.size() * 8u, cudaMemcpyDeviceToHost);
            double acc[8] = {0};
            uint64_t n = 0, t0 = ~0ull, t1 = 0;
            for (uint32_t c = 0; c < clusters * q.Q; ++c)
                for (uint32_t j = 0; j + 1u < 256u; ++j) {
                    const uint64_t* a = &t[(static_cast<size_t>(c) * 256u + j) * 8u];
                    const uint64_t* b = a + 8;
                    if (!a[0] || !a[5] || !b[0]) continue;
                    acc[0] += double(a[1] - a[0]);   // MMA issue span of a block
                    acc[1] += double(a[3] - a[2]);   // drain
                    acc[2] += double(a[5] - a[4]);   // top-k
                    acc[3] += double(a[2] - a[1]);   // last MMA issued -> drain start
                    acc[4] += double(a[4] - a[3]);   // drain end -> top-k start (this CTA's view)
                    acc[5] += double(b[0] - a[0]);   // block period
                    acc[6] += double(a[6]);          // converters waiting for raw data
                    acc[7] += double(a[7]);          // converters waiting for a free converted slot
                    t0 = std::min(t0, a[0]);
                    t1 = std::max(t1, a[5]);
                    ++n;
                }
            if (n)
                std::fprintf(stderr,
                             "[SP_MMA_TRACE] blocks %llu: mma span %.0f ns, drain %.0f, topk %.0f, mma->drain %.0f, "
                             "period %.0f ns, converters wait raw %.0f / slot %.0f ns\n",
                             (unsigned long long)n, acc[0] / n, acc[1] / n, acc[2] / n, acc[3] / n,
                             acc[5] / n, acc[6] / n, acc[7] / n);
        }
    } else if (!g.whole) {
        p.patch_w = g.pw;
        p.patch_h = g.ph;
        p.tiles_x = g.W / g.pw;
        p.patch_stage_bytes = (32u * g.nbits + 1023u) / 1024u * 1024u;
        e = sp::launch_patch(p, h->lay.smem_bytes, pl.ctas, s);
    } else {
        e = sp::launch_batched(p, planes ? packed_smem_bytes(h->lay) : h->lay.smem_bytes, s);
    }
    h->launches++;
    if (e != cudaSuccess) return cuda_fail(e, "batched kernel launch");
    return SP_OK;
}

// Launches the hot path for n_frames frames; results go to rows [row0, row0 + n) of the
// handle's result buffers.
sp_status compute_impl(sp_handle* h, const uint8_t* frames, uint32_t n_frames, int learn,
                       cudaStream_t s, uint32_t row0) {
    const sp::Geometry& g = h->g;
    const uint32_t n = n_frames * g.P;
    sp_plan_info pl = make_plan(h, n, learn != 0, frames);
    if (h->cfg.force_path == SP_PATH_BATCHED && pl.path != SP_PATH_BATCHED)
        return fail(SP_E_ARG, "force_path=BATCHED but the batched path is not eligible (reason 0x%x)",
                    pl.reason);
    h->last_plan = pl;
    const bool rec = (h->cfg.flags & SP_FLAG_RECORD_OVERLAPS) != 0;
    const bool full = learn && (h->cfg.flags & SP_FLAG_FULL_LEARNING) != 0;
    cudaError_t e = cudaSuccess;
    if (pl.path == SP_PATH_BATCHED) return launch_batched_path(h, frames, nullptr, n_frames, n, pl, s, row0);
    const char* lp = std::getenv("SP_LEARN_PATH");  // development override: cluster | grid | input
    if (full && h->span_dirty) {  // connected spans for the radius adaptation (R21)
        e = sp::launch_span(h->d_idx, h->d_perm, h->cfg.connected_threshold, g.C, g.S, h->d_span, s);
        h->launches++;
        if (e != cudaSuccess) return cuda_fail(e, "span launch");
        h->span_dirty = false;
    }
    if (learn) {
        h->iteration += n;
        if (full) h->uniform_bc = false;  // boosts now change on the device
        else h->span_dirty = true;
    }
    // the grid kernel plans its shared memory for a fixed radius: no full learning there
    const bool want_grid = learn && !full && h->grid_G && h->cfg.force_path != SP_PATH_PER_INPUT &&
                           (lp ? std::strcmp(lp, "grid") == 0
                               : ((h->cfg.flags & SP_FLAG_LEARN_GRID) != 0 || h->learn_Q == 0));
    // full learning on the grid: when the cluster kernel cannot hold the table (config 5), or asked
    const bool want_grid_full = learn && full && h->gridf_G && h->cfg.force_path != SP_PATH_PER_INPUT &&
                                (lp ? std::strcmp(lp, "grid") == 0
                                    : ((h->cfg.flags & SP_FLAG_LEARN_GRID) != 0 || h->learn_Q == 0));
    const bool want_cluster = learn && h->learn_Q && h->cfg.force_path != SP_PATH_PER_INPUT && !want_grid &&
                              !want_grid_full && !(lp && std::strcmp(lp, "input") == 0);
    if (want_grid || want_grid_full) {
        // the whole sequential stream in one cooperative launch over the SMs
        if (h->synT_dirty) {
            e = sp::launch_build_synT(h->d_idx, h->d_perm, h->cfg.connected_threshold, g.C, g.C32, g.S,
                                      h->d_synT, s);
            h->launches++;
            if (e != cudaSuccess) return cuda_fail(e, "column-major synapse table build");
            h->synT_dirty = false;
        }
        sp::LearnGridParams q{};
        q.frames = frames;
        q.first_input = row0;
        q.num_inputs = n;
        q.g = g;
        q.G = want_grid_full ? h->gridf_G : h->grid_G;
        q.Wn = h->Wn;
        q.own_words = want_grid_full ? h->gridf_own : h->grid_own;
        q.win_words = h->grid_win;
        q.ccols = want_grid_full ? h->gridf_ccols : h->grid_ccols;
        q.stages = want_grid_full ? h->gridf_stages : h->grid_stages;
        q.dbl_bits = h->grid_dbl && !want_grid_full ? 1u : 0u;
        if (want_grid_full) {
            q.fl = full_learn_params(h);
            q.span_part = h->d_span_part;
            q.cand_cap = h->gridf_cap;
            q.vsh = sp::bits_for(g.S) + 27u > 16u ? sp::bits_for(g.S) + 27u - 16u : 0u;  // N < 2^(bits(S)+27)
        }
        q.min_overlap = h->cfg.min_overlap;
        q.k = h->cfg.winners_set_size;
        q.radius = h->cfg.inhibition_radius;
        q.uniform_bc = h->uniform_bc ? 1u : 0u;
        q.inc = h->cfg.perm_increment;
        q.dec = h->cfg.perm_decrement;
        q.tau = h->cfg.connected_threshold;
        q.synT = h->d_synT;
        q.perm = h->d_perm;
        q.bc = h->d_bc;
        q.boost = h->d_boost;
        q.bits_g = h->d_bits;
        q.raw_g = reinterpret_cast<uint16_t*>(h->d_raw);
        q.gbar = h->d_gbar;
        q.sdr = h->res_sdr;
        q.counts = h->res_counts;
        q.raw_out = rec ? h->d_raw_rec : nullptr;
        q.boosted_out = rec ? h->d_boosted_rec : nullptr;
        if (const char* d = std::getenv("SP_LEARN_DBG")) q.dbg = static_cast<uint32_t>(std::atoi(d));
        q.trace = h->d_trace;
        // bit-planes prepacked per chunk by k_pack (as for the cluster kernel)
        const uint32_t Wn4 = (h->Wn + 3u) / 4u * 4u;
        const bool prepack = want_grid_full || !std::getenv("SP_NO_PREPACK");
        const uint32_t fpc = prepack ? std::max<uint32_t>(1u, kPrepackInputs / g.P) : n_frames;
        if (prepack) {
            sp_status st = ensure_prepack_scratch(h, fpc, n_frames, Wn4);
            if (st != SP_OK) return st;
        }
        for (uint32_t f0 = 0; f0 < n_frames; f0 += fpc) {
            const uint32_t nf = std::min(fpc, n_frames - f0);
            sp::LearnGridParams qc = q;
            qc.frames = frames + static_cast<size_t>(f0) * g.W * g.H;
            qc.first_input = row0 + f0 * g.P;
            qc.num_inputs = nf * g.P;
            if (prepack) {
                e = launch_prepack(h, qc.frames, qc.num_inputs, Wn4, s);
                if (e != cudaSuccess) return cuda_fail(e, "prepack launch");
                qc.bits_g = h->d_bits_all;
                qc.prepacked = 1u;
            }
            e = want_grid_full ? sp::launch_learn_grid_full(qc, h->gridf_smem, s)
                               : sp::launch_learn_grid(qc, h->grid_smem, s);
            h->launches++;
            if (e != cudaSuccess) return cuda_fail(e, "grid learning launch");
        }
        h->ell_dirty = true;
        h->conn_dirty = true;
        h->syn_dirty = true;
        h->last_plan.path = SP_PATH_PER_INPUT;
        h->last_learn_cluster = false;
        h->last_learn_path = SP_LEARN_GRID;
        return SP_OK;
    }
    if (h->syn_dirty && (learn || pl.path != SP_PATH_BATCHED)) {
        e = sp::launch_build_syn(h->d_idx, h->d_perm, h->cfg.connected_threshold, g.C, g.C32, g.S, h->d_syn, s);
        h->launches++;
        if (e != cudaSuccess) return cuda_fail(e, "synapse layout build");
        h->syn_dirty = false;
    }
    if (want_cluster) {
        // the whole sequential stream in one launch of the cluster-resident kernel
        sp::LearnParams q{};
        q.frames = frames;
        q.first_input = row0;
        q.num_inputs = n;
        q.g = g;
        q.Q = h->learn_Q;
        sp::learn_cluster_smem(g, q.Q, &q.cols_per_cta, h->learn_dbl, full);
        q.dbl_bits = h->learn_dbl ? 1u : 0u;
        if (const char* d = std::getenv("SP_LEARN_DBG")) q.dbg = static_cast<uint32_t>(std::atoi(d));
        q.syn_stride = sp::learn_syn_stride(g.S);
        q.tpc = sp::learn_threads_per_column(q.cols_per_cta);
        q.Wn = h->Wn;
        q.min_overlap = h->cfg.min_overlap;
        q.k = h->cfg.winners_set_size;
        q.radius = h->cfg.inhibition_radius;
        q.uniform_bc = h->uniform_bc ? 1u : 0u;
        q.inc = h->cfg.perm_increment;
        q.dec = h->cfg.perm_decrement;
        q.tau = h->cfg.connected_threshold;
        q.idx = h->d_idx;
        q.perm = h->d_perm;
        q.syn = h->d_syn;
        q.bc = h->d_bc;
        q.boost = h->d_boost;
        q.bits_g = h->d_bits;
        q.trace = h->d_trace;
        q.sdr = h->res_sdr;
        q.counts = h->res_counts;
        q.raw_out = rec ? h->d_raw_rec : nullptr;
        q.boosted_out = rec ? h->d_boosted_rec : nullptr;
        q.fl = full_learn_params(h);
        // the bit-planes do not depend on learning: k_pack packs a chunk of inputs ahead (an
        // HBM-bound pass), and the cluster kernel only bulk-loads them (no packing on the
        // sequential critical path).  Chunks bound the scratch; the state carries over.
        const uint32_t Wn4 = (h->Wn + 3u) / 4u * 4u;
        const bool prepack = want_grid_full || !std::getenv("SP_NO_PREPACK");
        const uint32_t fpc = prepack ? std::max<uint32_t>(1u, kPrepackInputs / g.P) : n_frames;
        if (prepack) {
            sp_status st = ensure_prepack_scratch(h, fpc, n_frames, Wn4);
            if (st != SP_OK) return st;
        }
        for (uint32_t f0 = 0; f0 < n_frames; f0 += fpc) {
            const uint32_t nf = std::min(fpc, n_frames - f0);
            sp::LearnParams qc = q;
            qc.frames = frames + static_cast<size_t>(f0) * g.W * g.H;
            qc.first_input = row0 + f0 * g.P;
            qc.num_inputs = nf * g.P;
            if (prepack) {
                e = launch_prepack(h, qc.frames, qc.num_inputs, Wn4, s);
                if (e != cudaSuccess) return cuda_fail(e, "prepack launch");
                qc.bits_g = h->d_bits_all;
                qc.prepacked = 1u;
            }
            e = sp::launch_learn_cluster(qc, h->learn_smem, s);
            h->launches++;
            if (e != cudaSuccess) return cuda_fail(e, "cluster learning launch");
        }
        h->ell_dirty = true;
        h->conn_dirty = true;
        h->last_plan.path = SP_PATH_PER_INPUT;
        h->last_learn_cluster = true;
        h->last_learn_path = SP_LEARN_CLUSTER;
        h->synT_dirty = true;
        return SP_OK;
    }
    if (learn) {
        h->last_learn_cluster = false;
        h->last_learn_path = SP_LEARN_PER_INPUT;
        h->synT_dirty = true;
    }
    // per-input path, sub-batches of whole frames
    const uint32_t fpb = std::max<uint32_t>(1u, h->sub_inputs / g.P);
    for (uint32_t f0 = 0; f0 < n_frames; f0 += fpb) {
        const uint32_t nf = std::min(fpb, n_frames - f0);
        sp::PerInputParams p{};
        p.frames = frames + static_cast<size_t>(f0) * g.W * g.H;
        p.uniform_bc = h->uniform_bc ? 1u : 0u;
        p.first_input = row0 + f0 * g.P;
        p.num_inputs = nf * g.P;
        p.g = g;
        p.min_overlap = h->cfg.min_overlap;
        p.k = h->cfg.winners_set_size;
        p.radius = h->cfg.inhibition_radius;
        p.inc = h->cfg.perm_increment;
        p.dec = h->cfg.perm_decrement;
        p.tau = h->cfg.connected_threshold;
        p.bits = h->d_bits;
        p.Wn = h->Wn;
        p.syn = h->d_syn;
        p.syn_rw = h->d_syn;
        p.idx = h->d_idx;
        p.perm = h->d_perm;
        p.bc = h->d_bc;
        p.boost = h->d_boost;
        p.raw = h->d_raw;
        p.sdr = h->res_sdr;
        p.counts = h->res_counts;
        p.raw_out = rec ? h->d_raw_rec : nullptr;
        p.boosted_out = rec ? h->d_boosted_rec : nullptr;
        p.radius_dev = h->d_radius;
        p.fl = full_learn_params(h);
        // CTA wavelet for local inhibition with per-column boosts (k_inhibit), when its scratch fits
        p.wm_ok = static_cast<int>(sp::inhibit_wavelet_smem(g)) <= h->max_smem ? 1u : 0u;
        p.wm_min_radius = h->wm_min_radius_pi;
        if (full) p.uniform_bc = 0u;
        e = sp::launch_pack(p, s);
        h->launches++;
        if (e != cudaSuccess) return cuda_fail(e, "pack launch");
        if (!learn) {
            e = sp::launch_overlap(p, s);
            h->launches++;
            if (e == cudaSuccess) e = sp::launch_inhibit(p, s, inhibit_parts(h, p.num_inputs));
            h->launches++;
            if (e != cudaSuccess) return cuda_fail(e, "overlap/inhibit launch");
            continue;
        }
        // learning: the recurrence over inputs, in order
        for (uint32_t t = 0; t < p.num_inputs; ++t) {
            sp::PerInputParams q = p;
            q.bits = h->d_bits + static_cast<size_t>(t) * h->Wn;
            q.raw = h->d_raw + static_cast<size_t>(t) * g.C32;
            q.first_input = p.first_input + t;
            q.num_inputs = 1;
            e = sp::launch_overlap(q, s);
            h->launches++;
            if (e == cudaSuccess) e = sp::launch_inhibit(q, s, inhibit_parts(h, 1u));
            h->launches++;
            if (e == cudaSuccess) e = sp::launch_learn(q, 0, s);
            h->launches++;
            if (full && e == cudaSuccess) {
                uint32_t nl = 0;
                e = sp::launch_full(q, 0, s, &nl);
                h->launches += nl;
            }
            if (e != cudaSuccess) return cuda_fail(e, "learning step launch");
        }
        h->ell_dirty = true;
        h->conn_dirty = true;
    }
    return SP_OK;
}

}  // namespace

namespace sp {
sp_status handle_frame_dims(const sp_handle* h, uint32_t* W, uint32_t* H, uint32_t* P, uint32_t* words,
                            int* device) {
    if (!h) return SP_E_ARG;
    *W = h->cfg.input_width, *H = h->cfg.input_height, *P = h->g.P, *words = h->g.ncw, *device = h->device;
    return SP_OK;
}
void handle_set_result(sp_handle* h, uint32_t* sdr, uint32_t* counts, uint32_t inputs) {
    h->res_sdr = sdr, h->res_counts = counts, h->last_inputs = inputs, h->has_result = true;
}
}  // namespace sp

extern "C" {


const char* sp_last_error(void) { return g_err.c_str(); }

const char* sp_version(void) { return SP_VERSION; }

sp_status sp_config_default(sp_config* cfg) {
    if (!cfg) return fail(SP_E_ARG, "config is NULL");
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->input_width = 240;   // Tab. 1
    cfg->input_height = 134;
    cfg->num_columns = 2048;  // Tab. 2
    cfg->synapses_per_column = 128;
    cfg->min_overlap = 8;
    cfg->winners_set_size = 40;
    cfg->inhibition_radius = 0;
    cfg->perm_increment = 0.1f;
    cfg->perm_decrement = 0.1f;
    cfg->initial_permanence = 0.21f;
    cfg->connected_threshold = 0.2f;
    cfg->seed = 42;
    cfg->device = 0;
    cfg->max_inputs = 4096;
    cfg->duty_cycle_period = 1000;  // S:150, SURVEY §8(f) NEXT-1
    cfg->max_boost = 2.0f;
    return SP_OK;
}

sp_status sp_init_pools_host(const sp_config* cfg, uint32_t* idx_out) {
    sp_status st = validate(cfg);
    if (st != SP_OK) return st;
    if (!idx_out) return fail(SP_E_ARG, "idx_out is NULL");
    init_pools(*cfg, sp::make_geometry(*cfg), idx_out);
    return SP_OK;
}

sp_status sp_plan(const sp_config* cfg, uint32_t num_frames, int32_t sm_count, sp_plan_info* out) {
    sp_status st = validate(cfg);
    if (st != SP_OK) return st;
    if (!out) return fail(SP_E_ARG, "out is NULL");
    sp_handle tmp;
    tmp.cfg = *cfg;
    tmp.g = sp::make_geometry(*cfg);
    tmp.sm_count = sm_count > 0 ? sm_count : kDefaultSms;
    tmp.max_smem = kDefaultSmem;
    tmp.lay = tmp.g.whole ? sp::plan_batched_layout(tmp.g, tmp.max_smem)
                          : sp::plan_patch_layout(tmp.g, tmp.max_smem);
    *out = make_plan(&tmp, num_frames * tmp.g.P, false, nullptr);
    return SP_OK;
}

sp_status sp_create(const sp_config* cfg, sp_handle** out) {
    if (!out) return fail(SP_E_ARG, "out is NULL");
    *out = nullptr;
    sp_status st = validate(cfg);
    if (st != SP_OK) return st;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return fail(SP_E_CUDA, "no CUDA device available (%s)", cudaGetErrorString(e));
    if (cfg->device < 0 || cfg->device >= ndev) return fail(SP_E_ARG, "device %d out of range", cfg->device);
    e = cudaSetDevice(cfg->device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    sp_handle* h = new sp_handle();
    h->cfg = *cfg;
    h->device = cfg->device;
    h->g = sp::make_geometry(*cfg);
    cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, h->device);
    cudaDeviceGetAttribute(&h->max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device);
    h->lay = h->g.whole ? sp::plan_batched_layout(h->g, h->max_smem) : sp::plan_patch_layout(h->g, h->max_smem);
    const sp::Geometry& g = h->g;
    if ((e = sp::configure_batched(h->max_smem)) != cudaSuccess ||
        (e = sp::configure_per_input(h->max_smem)) != cudaSuccess) {
        release(h);
        return cuda_fail(e, "kernel attributes");
    }
    if (h->lay.ok && h->g.whole) {
        sp::batched_max_clusters(h->lay.smem_bytes, h->max_clusters);
        // global-split scratch: one CTA per SM, 32 partial count rows each
        const size_t pb = static_cast<size_t>(h->sm_count) * 32u * h->g.C32 * 2u;
        if (cudaMalloc(&h->d_part, pb) != cudaSuccess ||
            cudaMalloc(&h->d_gsbar, 2u * h->sm_count * sizeof(uint32_t)) != cudaSuccess ||
            cudaMemset(h->d_gsbar, 0, 2u * h->sm_count * sizeof(uint32_t)) != cudaSuccess) {
            release(h);
            return fail(SP_E_OOM, "global-split scratch (%zu bytes)", pb);
        }
    }
    // tensor-core patch kernel (NEXT-2): global inhibition (the selection it feeds is the global
    // top-k; local windows stay on the bit-sliced gather kernel, measured faster there), patch
    // width a power of two >= 32, <= 32 tiles per row, nbits <= 1024 (A in tensor memory beside
    // two accumulators), C32 = 128 Q columns (Q = 1, 2, 4, 8 CTAs per cluster); shared memory:
    // the converted ring (4 stages), two raw-count buffers, the top-k tie lists (8 warps x 512 B)
    // and as many raw frame-row stages as fit (>= 3)
    if (!g.whole && cfg->inhibition_radius == 0 && g.pw % 32u == 0 && (g.pw & (g.pw - 1u)) == 0 &&
        g.W * (g.ph % 2u == 0 ? 2u : 1u) * 4u <= 64u * 8u * 16u &&  // one stage = 64 threads x 8 chunks
        g.W / g.pw <= 32u && g.nbits <= 1024u && g.C32 % 128u == 0 && g.S <= 1023u && sp::mma_row_split(g.W) &&
        !std::getenv("SP_NO_PATCH_MMA")) {
        const uint32_t Q = g.C32 / 128u;
        const uint32_t sps = g.ph % 2u == 0 ? 2u : 1u, region = 4096u, nc = 4u;
        if ((Q == 1 || Q == 2 || Q == 4 || Q == 8) && sp::configure_patch_mma(h->max_smem) == cudaSuccess) {
            uint32_t nr = 0;
            while (sp::patch_mma_smem(g.W, sps, g.pw / 32u, nr + 1u, nc, Q, g.C32, region) + 1024u <=
                       static_cast<uint32_t>(h->max_smem) && nr < 16u)
                ++nr;
            if (const char* es = std::getenv("SP_MMA_STAGES")) nr = std::min<uint32_t>(nr, std::atoi(es));
            if (nr >= 3u) {
                const uint32_t smem = sp::patch_mma_smem(g.W, sps, g.pw / 32u, nr, nc, Q, g.C32, region);
                int ncl = 0;
                if (sp::patch_mma_max_clusters(smem, Q, &ncl) == cudaSuccess && ncl > 0) {
                    h->mma_Q = Q;
                    h->mma_smem = smem;
                    h->mma_region = region;
                    h->mma_raw_stages = nr;
                    h->mma_conv_stages = nc;
                    h->mma_sps = sps;
                    h->mma_clusters = static_cast<uint32_t>(ncl);
                }
            }
        }
        (void)cudaGetLastError();
    }
    // cluster-resident learning: the largest cluster (<= 16 CTAs, >= 32 columns each) whose
    // synapse slice + bit-plane fit in shared memory and that can be co-scheduled
    // (the warp-level global selection holds C32 <= 2048 columns in registers)
    if (h->g.C32 <= 2048u && sp::configure_learn(h->max_smem) == cudaSuccess &&
        !std::getenv("SP_NO_CLUSTER_LEARN")) {
        for (uint32_t Q = 16; Q >= 1; Q /= 2) {
            if (Q > 1 && Q * 32u > h->g.C32) continue;
            for (int dbl = 1; dbl >= 0 && !h->learn_Q; --dbl) {
                const uint32_t smem = sp::learn_cluster_smem(h->g, Q, nullptr, dbl != 0,
                                                             (cfg->flags & SP_FLAG_FULL_LEARNING) != 0);
                if (static_cast<int>(smem) > h->max_smem - 1024) continue;
                int n = 0;
                sp::learn_max_clusters(Q, smem, &n);
                if (n < 1) continue;
                h->learn_Q = Q;
                h->learn_smem = smem;
                h->learn_dbl = dbl != 0;
            }
            if (h->learn_Q) break;
        }
    }
    // grid-resident learning: S % 4 == 0 (16-byte chunk rows), local inhibition or C32 <= 2048
    // (the global selection holds the columns in registers), co-resident CTAs
    int coop = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, h->device);
    if (coop && h->g.S % 4u == 0 && (h->cfg.inhibition_radius > 0 || h->g.C32 <= 2048u) &&
        sp::configure_learn_grid(h->max_smem) == cudaSuccess) {
        const uint32_t G = std::min<uint32_t>(static_cast<uint32_t>(h->sm_count), h->g.ncw);
        // deepest synapse ring that fits (>= 5 stages with two bit-plane buffers, else one)
        for (int pass = 0; pass < 2 && !h->grid_G; ++pass)
            for (uint32_t st = 8; st >= 2 && !h->grid_G; --st) {
                const bool dbl = pass == 0;
                if (dbl && st < 5) break;
                uint32_t stages = st;
                const uint32_t smem = sp::learn_grid_smem(h->g, h->cfg.inhibition_radius, G, dbl, &h->grid_own,
                                                          &h->grid_win, &h->grid_ccols, &stages);
                if (static_cast<int>(smem) > h->max_smem - 2048) continue;
                int cap = 0;
                sp::learn_grid_max_ctas(smem, &cap);
                if (cap < static_cast<int>(G)) continue;
                h->grid_G = G;
                h->grid_smem = smem;
                h->grid_dbl = dbl;
                h->grid_stages = st;
            }
    }
    // the full-learning grid kernel (radius adaptation needs every window size up to C): one
    // bit-plane buffer, the whole raw row and a candidate list in shared memory
    if (coop && (cfg->flags & SP_FLAG_FULL_LEARNING) && h->g.S % 4u == 0 &&
        sp::configure_learn_grid_full(h->max_smem) == cudaSuccess) {
        const uint32_t G = std::min<uint32_t>(static_cast<uint32_t>(h->sm_count), h->g.ncw);
        const uint32_t cap = 2048u;
        for (uint32_t st = 8; st >= 2 && !h->gridf_G; --st) {
            const uint32_t smem = sp::learn_grid_full_smem(h->g, G, st, cap, &h->gridf_own, &h->gridf_ccols);
            if (!smem || static_cast<int>(smem) > h->max_smem - 2048) continue;
            int n = 0;
            sp::learn_grid_full_max_ctas(smem, &n);
            if (n < static_cast<int>(G)) continue;
            h->gridf_G = G, h->gridf_smem = smem, h->gridf_stages = st, h->gridf_cap = cap;
        }
    }
    if (const char* eg = std::getenv("SP_GROUPS"))
        h->force_groups = static_cast<uint32_t>(std::max(0, std::atoi(eg)));
    if (std::getenv("SP_TRACE")) cudaMalloc(&h->d_trace, 4096u * 6u * sizeof(uint64_t));
    if (const char* et = std::getenv("SP_THREADS")) h->batched_threads = std::atoi(et) == 1024 ? 1024u : 512u;
    if (const char* ew = std::getenv("SP_WM_MIN_RADIUS"))
        h->wm_min_radius = h->wm_min_radius_pi = static_cast<uint32_t>(std::atoi(ew));
    {
        const uint64_t kc = static_cast<uint64_t>(cfg->winners_set_size) * g.C;
        h->cand_min_radius = static_cast<uint32_t>((kc + 699u) / 700u);
        h->cand_min_radius_u = static_cast<uint32_t>((kc + 699u) / 700u);
    }
    if (const char* ec = std::getenv("SP_CAND_MIN_RADIUS"))  // experiments / tests (huge = off)
        h->cand_min_radius = h->cand_min_radius_u = static_cast<uint32_t>(std::strtoul(ec, nullptr, 10));
    if (const char* eu = std::getenv("SP_WM_UMAX")) {  // experiments; the per-warp wavelet scratch holds
        const long u = std::atol(eu);                   // at most 15 levels + the lossy plane
        h->wm_umax = static_cast<uint32_t>(std::min<long>(std::max<long>(u, 1), 32766));
    }
    h->Wn = (g.nbits + 31u) / 32u;
    h->sub_inputs = std::max<uint32_t>(sp::kPerInputChunk, g.P);
    const size_t cs = static_cast<size_t>(g.C) * g.S;
    const size_t cap = cfg->max_inputs;
    e = dalloc(&h->d_idx, cs);
    if (e == cudaSuccess && h->mma_clusters) e = dalloc(&h->d_conn, static_cast<size_t>(g.C32) * g.nbits);
    if (e == cudaSuccess) e = dalloc(&h->d_perm, cs);
    if (e == cudaSuccess) e = dalloc(&h->d_boost, g.C32);
    if (e == cudaSuccess) e = dalloc(&h->d_bc, g.C32);
    if (e == cudaSuccess) e = dalloc(&h->d_syn, static_cast<size_t>(g.S) * g.C32);
    if (e == cudaSuccess)
        e = dalloc(&h->d_bits, std::max<size_t>(static_cast<size_t>(h->sub_inputs) * h->Wn,
                                                2u * ((h->Wn + 3u) / 4u * 4u)));
    if (e == cudaSuccess) e = dalloc(&h->d_raw, static_cast<size_t>(h->sub_inputs) * g.C32);
    if (e == cudaSuccess) e = dalloc(&h->d_sdr, cap * g.ncw);
    if (e == cudaSuccess) e = dalloc(&h->d_counts, cap);
    if (e == cudaSuccess && (h->grid_G || h->gridf_G)) {
        e = dalloc(&h->d_synT, static_cast<size_t>(g.C32) * g.S);
        if (e == cudaSuccess) e = dalloc(&h->d_gbar, 1);
    }
    if (e == cudaSuccess && h->gridf_G) e = dalloc(&h->d_span_part, 2u * h->gridf_G);
    if (e == cudaSuccess) e = dalloc(&h->d_adc, g.C32);
    if (e == cudaSuccess) e = dalloc(&h->d_odc, g.C32);
    if (e == cudaSuccess) e = dalloc(&h->d_span, g.C32);
    if (e == cudaSuccess) e = dalloc(&h->d_radius, 1);
    if (e == cudaSuccess) e = dalloc(&h->d_fscratch, sp::full_scratch_floats(g.C32));
    if (e == cudaSuccess) e = cudaMemset(h->d_fscratch, 0, sp::full_scratch_floats(g.C32) * 4u);
    if (e == cudaSuccess) e = cudaMemset(h->d_adc, 0, g.C32 * 4u);
    if (e == cudaSuccess) e = cudaMemset(h->d_odc, 0, g.C32 * 4u);
    if (e == cudaSuccess) e = cudaMemset(h->d_span, 0, g.C32 * 4u);
    if (e == cudaSuccess)
        e = cudaMemcpy(h->d_radius, &cfg->inhibition_radius, 4u, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && (cfg->flags & SP_FLAG_RECORD_OVERLAPS)) {
        e = dalloc(&h->d_raw_rec, cap * g.C);
        if (e == cudaSuccess) e = dalloc(&h->d_boosted_rec, cap * g.C);
    }
    if (e != cudaSuccess) {
        release(h);
        return fail(SP_E_OOM, "device allocation failed: %s", cudaGetErrorString(e));
    }
    std::vector<uint32_t> idx(cs);
    init_pools(*cfg, g, idx.data());
    std::vector<float> perm(cs, cfg->initial_permanence);
    std::vector<float> boost(g.C, 1.0f);
    st = upload_state(h, idx.data(), perm.data(), boost.data());
    if (st != SP_OK) {
        std::string msg = g_err;
        release(h);
        g_err = msg;
        return st;
    }
    h->last_plan = make_plan(h, cfg->max_inputs, false, nullptr);
    h->res_sdr = h->d_sdr;
    h->res_counts = h->d_counts;
    *out = h;
    return SP_OK;
}

sp_status sp_destroy(sp_handle* h) {
    if (!h) return SP_OK;
    cudaSetDevice(h->device);
    cudaDeviceSynchronize();
    release(h);
    return SP_OK;
}

sp_status sp_compute(sp_handle* h, const uint8_t* frames_dev, uint32_t num_frames, int learn,
                     void* cuda_stream) {
    sp_status st = check_handle(h);
    if (st != SP_OK) return st;
    const uint64_t n = static_cast<uint64_t>(num_frames) * h->g.P;
    if (n > h->cfg.max_inputs)
        return fail(SP_E_ARG, "num_frames * inputs_per_frame = %llu exceeds max_inputs %u",
                    static_cast<unsigned long long>(n), h->cfg.max_inputs);
    if (num_frames > 0 && !frames_dev) return fail(SP_E_ARG, "frames_dev is NULL");
    h->last_inputs = static_cast<uint32_t>(n);
    h->has_result = true;
    h->res_sdr = h->d_sdr;
    h->res_counts = h->d_counts;
    if (n == 0) return SP_OK;
    return compute_impl(h, frames_dev, num_frames, learn, static_cast<cudaStream_t>(cuda_stream), 0);
}

sp_status sp_compute_into(sp_handle* h, const uint8_t* frames_dev, uint32_t num_frames, int learn, uint32_t* sdr_dev,
                          uint32_t* count_dev, void* cuda_stream) {
    sp_status st = check_handle(h);
    if (st != SP_OK) return st;
    const uint64_t n = static_cast<uint64_t>(num_frames) * h->g.P;
    if (n > h->cfg.max_inputs)
        return fail(SP_E_ARG, "num_frames * inputs_per_frame = %llu exceeds max_inputs %u",
                    static_cast<unsigned long long>(n), h->cfg.max_inputs);
    if (num_frames > 0 && (!frames_dev || !sdr_dev || !count_dev))
        return fail(SP_E_ARG, "frames_dev, sdr_dev and count_dev must be non-NULL");
    h->last_inputs = static_cast<uint32_t>(n);
    h->has_result = true;
    h->res_sdr = sdr_dev;
    h->res_counts = count_dev;
    if (n == 0) return SP_OK;
    return compute_impl(h, frames_dev, num_frames, learn, static_cast<cudaStream_t>(cuda_stream), 0);
}

sp_status sp_winners(sp_handle* h, uint32_t* sdr_dev, uint32_t* count_dev, void* cuda_stream) {
    sp_status st = check_handle(h);
    if (st != SP_OK) return st;
    if (!h->has_result) return fail(SP_E_STATE, "sp_winners before any sp_compute");
    if (h->last_inputs == 0) return SP_OK;
    if (!sdr_dev) return fail(SP_E_ARG, "sdr_dev is NULL");
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    if (sdr_dev == h->res_sdr && (!count_dev || count_dev == h->res_counts)) return SP_OK;  // already there
    cudaError_t e = cudaMemcpyAsync(sdr_dev, h->res_sdr,
                                    static_cast<size_t>(h->last_inputs) * h->g.ncw * 4u,
                                    cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess && count_dev)
        e = cudaMemcpyAsync(count_dev, h->res_counts, h->last_inputs * 4u, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "sp_winners copy");
    return SP_OK;
}

sp_status sp_overlaps(sp_handle* h, uint16_t* raw_dev, float* boosted_dev, void* cuda_stream) {
    sp_status st = check_handle(h);
    if (st != SP_OK) return st;
    if (!(h->cfg.flags & SP_FLAG_RECORD_OVERLAPS))
        return fail(SP_E_STATE, "sp_overlaps needs SP_FLAG_RECORD_OVERLAPS at create");
    if (!h->has_result) return fail(SP_E_STATE, "sp_overlaps before any sp_compute");
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    const size_t n = static_cast<size_t>(h->last_inputs) * h->g.C;
    cudaError_t e = cudaSuccess;
    if (raw_dev && n) e = cudaMemcpyAsync(raw_dev, h->d_raw_rec, n * 2u, cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess && boosted_dev && n)
        e = cudaMemcpyAsync(boosted_dev, h->d_boosted_rec, n * 4u, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "sp_overlaps copy");
    return SP_OK;
}

sp_status sp_get_state(sp_handle* h, uint32_t* idx, float* perm, float* boost) {
    sp_status st = check_handle(h);
    if (st != SP_OK) return st;
    cudaError_t e = cudaDeviceSynchronize();
    const size_t cs = static_cast<size_t>(h->g.C) * h->g.S;
    if (e == cudaSuccess && idx) e = cudaMemcpy(idx, h->d_idx, cs * 4u, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && perm) e = cudaMemcpy(perm, h->d_perm, cs * 4u, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && boost) e = cudaMemcpy(boost, h->d_boost, h->g.C * 4u, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "sp_get_state");
    return SP_OK;
}

sp_status sp_set_state(sp_handle* h, const uint32_t* idx, const float* perm, const float* boost) {
    sp_status st = check_handle(h);
    if (st != SP_OK) return st;
    const sp::Geometry& g = h->g;
    const size_t cs = static_cast<size_t>(g.C) * g.S;
    if (idx) {
        for (uint32_t c = 0; c < g.C; ++c)
            for (uint32_t s = 0; s < g.S; ++s) {
                const uint32_t v = idx[c * g.S + s];
                if (v >= g.nbits)
                    return fail(SP_E_ARG, "idx[%u][%u] = %u >= input bits %u (S:74)", c, s, v, g.nbits);
                if (s && v <= idx[c * g.S + s - 1])
                    return fail(SP_E_ARG, "idx of column %u not strictly ascending at %u (S:74)", c, s);
            }
    }
    if (perm)
        for (size_t i = 0; i < cs; ++i)
            if (!(perm[i] >= 0.0f && perm[i] <= 1.0f))
                return fail(SP_E_ARG, "perm[%zu] = %g outside [0,1] (S:73)", i, perm[i]);
    if (boost)
        for (uint32_t c = 0; c < g.C; ++c)
            if (!(boost[c] >= 1.0f && boost[c] < 16.0f))
                return fail(SP_E_ARG, "boost[%u] = %g outside [1,16) (R4)", c, boost[c]);
    // merge with the current state for NULL arguments
    std::vector<uint32_t> cur_idx;
    std::vector<float> cur_perm, cur_boost;
    if (!idx || !perm || !boost) {
        cur_idx.resize(cs);
        cur_perm.resize(cs);
        cur_boost.resize(g.C);
        st = sp_get_state(h, cur_idx.data(), cur_perm.data(), cur_boost.data());
        if (st != SP_OK) return st;
    }
    cudaDeviceSynchronize();
    return upload_state(h, idx ? idx : cur_idx.data(), perm ? perm : cur_perm.data(),
                        boost ? boost : cur_boost.data());
}

sp_status sp_histograms(sp_handle* h, const uint32_t* video_offsets_host, uint32_t num_videos,
                        uint32_t* counts_dev, float* hist_dev, void* cuda_stream) {
    sp_status st = check_handle(h);
    if (st != SP_OK) return st;
    if (!h->has_result) return fail(SP_E_STATE, "sp_histograms before any sp_compute");
    if (num_videos == 0 || (!counts_dev && !hist_dev)) return SP_OK;
    if (!video_offsets_host) return fail(SP_E_ARG, "video_offsets_host is NULL");
    uint32_t longest = 0;
    for (uint32_t v = 0; v < num_videos; ++v) {
        if (video_offsets_host[v + 1] < video_offsets_host[v])
            return fail(SP_E_ARG, "video offsets must be non-decreasing (offsets[%u] > offsets[%u])", v, v + 1);
        longest = std::max(longest, video_offsets_host[v + 1] - video_offsets_host[v]);
    }
    if (video_offsets_host[num_videos] > h->last_inputs)
        return fail(SP_E_ARG, "offsets[%u] = %u exceeds the %u inputs of the last call", num_videos,
                    video_offsets_host[num_videos], h->last_inputs);
    const size_t nc = static_cast<size_t>(num_videos) * h->g.C;
    cudaError_t e = cudaSuccess;
    if (h->hist_off_cap < num_videos + 1u) {
        h->h_hist_off.clear();
        if (h->d_hist_off) cudaFree(h->d_hist_off), h->d_hist_off = nullptr;
        e = dalloc(&h->d_hist_off, num_videos + 1u);
        if (e != cudaSuccess) return fail(SP_E_OOM, "histogram offsets: %s", cudaGetErrorString(e));
        h->hist_off_cap = num_videos + 1u;
    }
    uint32_t* counts = counts_dev;
    if (!counts) {
        if (h->hist_counts_cap < nc) {
            if (h->d_hist_counts) cudaFree(h->d_hist_counts), h->d_hist_counts = nullptr;
            e = dalloc(&h->d_hist_counts, nc);
            if (e != cudaSuccess) return fail(SP_E_OOM, "histogram counts: %s", cudaGetErrorString(e));
            h->hist_counts_cap = nc;
        }
        counts = h->d_hist_counts;
    }
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    // the offsets usually repeat from call to call: upload (a staged, host-synchronous copy
    // from pageable memory) only when they change
    if (h->h_hist_off.size() != num_videos + 1u ||
        std::memcmp(h->h_hist_off.data(), video_offsets_host, (num_videos + 1u) * 4u) != 0) {
        e = cudaMemcpyAsync(h->d_hist_off, video_offsets_host, (num_videos + 1u) * 4u, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return cuda_fail(e, "histogram offsets upload");
        h->h_hist_off.assign(video_offsets_host, video_offsets_host + num_videos + 1u);
    }
    uint32_t nl = 0;
    e = sp::launch_histograms(h->res_sdr, h->g.ncw, h->g.C, h->d_hist_off, num_videos, longest, h->sm_count, counts,
                              hist_dev, s, &nl);
    h->launches += nl;
    if (e != cudaSuccess) return cuda_fail(e, "histogram launch");
    return SP_OK;
}

sp_status sp_get_learning_state(sp_handle* h, float* active_duty, float* overlap_duty, uint32_t* radius,
                                uint64_t* iteration) {
    sp_status st = check_handle(h);
    if (st != SP_OK) return st;
    cudaError_t e = cudaDeviceSynchronize();
    const size_t C = h->g.C;
    if (e == cudaSuccess && active_duty) e = cudaMemcpy(active_duty, h->d_adc, C * 4u, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && overlap_duty) e = cudaMemcpy(overlap_duty, h->d_odc, C * 4u, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && radius) e = cudaMemcpy(radius, h->d_radius, 4u, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "sp_get_learning_state");
    if (iteration) *iteration = h->iteration;
    return SP_OK;
}

sp_status sp_set_learning_state(sp_handle* h, const float* active_duty, const float* overlap_duty,
                                uint32_t radius) {
    sp_status st = check_handle(h);
    if (st != SP_OK) return st;
    const uint32_t C = h->g.C;
    for (const float* d : {active_duty, overlap_duty})
        if (d)
            for (uint32_t c = 0; c < C; ++c)
                if (!(d[c] >= 0.0f && d[c] <= 1.0f))
                    return fail(SP_E_ARG, "duty cycle [%u] = %g outside [0,1]", c, d[c]);
    if (h->cfg.inhibition_radius == 0 ? radius != 0 : (radius < 1 || radius > C))
        return fail(SP_E_ARG, "radius %u: must be 0 iff the configured radius is 0, else in [1, C] (R21)",
                    radius);
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess && active_duty) e = cudaMemcpy(h->d_adc, active_duty, C * 4u, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && overlap_duty) e = cudaMemcpy(h->d_odc, overlap_duty, C * 4u, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(h->d_radius, &radius, 4u, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "sp_set_learning_state");
    return SP_OK;
}

namespace {

// Words per frame of the bit-plane input: ceil(nbits / 32) rounded up to 4 (16-byte rows).
uint32_t packed_words(const sp_handle* h) { return (h->Wn + 3u) / 4u * 4u; }

sp_status check_packed(sp_handle* h, uint32_t n, const void* planes) {
    if (!h->g.whole) return fail(SP_E_CONFIG, "bit-plane input needs a whole-frame configuration (no patches)");
    const sp_plan_info pl = make_plan(h, n, false, nullptr);
    if (n > 0 && pl.path != SP_PATH_BATCHED)
        return fail(SP_E_CONFIG, "bit-plane input runs on the batched kernel only (not eligible: reason 0x%x)",
                    pl.reason);
    if (planes && (reinterpret_cast<uintptr_t>(planes) & 15u))
        return fail(SP_E_ARG, "bit-planes must be 16-byte aligned");
    return SP_OK;
}

// End-to-end pipeline shared by sp_compute_host and sp_compute_packed_host: chunks of frames
// (uint8 frames, or bit-planes when packed) copied host->device on the copy stream into two
// staging buffers, computed on s, winners copied back on s.
sp_status compute_host_impl(sp_handle* h, const void* in_host, bool packed, uint32_t num_frames, int learn,
                            uint32_t* sdr_host, uint32_t* count_host, void* cuda_stream) {
    sp_status st = check_handle(h);
    if (st != SP_OK) return st;
    const sp::Geometry& g = h->g;
    const uint64_t n = static_cast<uint64_t>(num_frames) * g.P;
    if (n > h->cfg.max_inputs)
        return fail(SP_E_ARG, "num_frames * inputs_per_frame = %llu exceeds max_inputs %u",
                    static_cast<unsigned long long>(n), h->cfg.max_inputs);
    if (num_frames > 0 && (!in_host || !sdr_host)) return fail(SP_E_ARG, "NULL host buffer");
    if (packed) {
        if (learn) return fail(SP_E_ARG, "bit-plane input is inference only (learn must be 0)");
        st = check_packed(h, static_cast<uint32_t>(n), nullptr);
        if (st != SP_OK) return st;
    }
    h->res_sdr = h->d_sdr;  // results staged in the handle's buffers
    h->res_counts = h->d_counts;
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    const size_t frame_bytes = static_cast<size_t>(g.W) * g.H;
    const size_t in_bytes = packed ? static_cast<size_t>(packed_words(h)) * 4u : frame_bytes;
    cudaError_t e = cudaSuccess;
    if (!h->copy_stream) {
        // chunk of frames per pipeline stage: ~64 MiB, at least 1 frame
        h->stage_frames = static_cast<uint32_t>(std::max<size_t>(1, (64u << 20) / frame_bytes));
        e = cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking);
        for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
            e = cudaEventCreateWithFlags(&h->ev_h2d[i], cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_free[i], cudaEventDisableTiming);
            if (e == cudaSuccess) e = dalloc(&h->d_stage[i], h->stage_frames * frame_bytes);
        }
        if (e != cudaSuccess) return cuda_fail(e, "end-to-end staging setup");
    }
    // frames per chunk: as many as a staging buffer holds (bit-planes: ~8x more per chunk)
    const uint32_t chunk_frames = static_cast<uint32_t>(
        std::max<size_t>(1, std::min<size_t>(h->stage_frames * frame_bytes / in_bytes, 1u << 30)));
    h->last_inputs = static_cast<uint32_t>(n);
    h->has_result = true;
    const uint8_t* src = static_cast<const uint8_t*>(in_host);
    uint32_t chunk = 0;
    for (uint32_t f0 = 0; f0 < num_frames; f0 += chunk_frames, ++chunk) {
        const uint32_t nf = std::min(chunk_frames, num_frames - f0);
        const int b = chunk & 1;
        // H2D on the copy stream once the buffer's previous compute has finished
        if (chunk >= 2) e = cudaStreamWaitEvent(h->copy_stream, h->ev_free[b], 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(h->d_stage[b], src + f0 * in_bytes, nf * in_bytes, cudaMemcpyHostToDevice,
                                h->copy_stream);
        if (e == cudaSuccess) e = cudaEventRecord(h->ev_h2d[b], h->copy_stream);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s, h->ev_h2d[b], 0);
        if (e != cudaSuccess) return cuda_fail(e, "end-to-end H2D");
        if (packed) {
            const uint32_t ni = nf * g.P;
            st = launch_batched_path(h, nullptr, reinterpret_cast<const uint32_t*>(h->d_stage[b]), nf, ni,
                                     make_plan(h, ni, false, nullptr), s, f0 * g.P);
            h->last_plan = make_plan(h, ni, false, nullptr);
        } else {
            st = compute_impl(h, h->d_stage[b], nf, learn, s, f0 * g.P);
        }
        if (st != SP_OK) return st;
        e = cudaEventRecord(h->ev_free[b], s);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(sdr_host + static_cast<size_t>(f0) * g.P * g.ncw,
                                h->d_sdr + static_cast<size_t>(f0) * g.P * g.ncw,
                                static_cast<size_t>(nf) * g.P * g.ncw * 4u, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess && count_host)
            e = cudaMemcpyAsync(count_host + static_cast<size_t>(f0) * g.P, h->d_counts + static_cast<size_t>(f0) * g.P,
                                static_cast<size_t>(nf) * g.P * 4u, cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) return cuda_fail(e, "end-to-end D2H");
    }
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "end-to-end sync");
    return SP_OK;
}

}  // namespace

sp_status sp_compute_host(sp_handle* h, const uint8_t* frames_host, uint32_t num_frames, int learn,
                          uint32_t* sdr_host, uint32_t* count_host, void* cuda_stream) {
    return compute_host_impl(h, frames_host, false, num_frames, learn, sdr_host, count_host, cuda_stream);
}

sp_status sp_compute_packed_host(sp_handle* h, const uint32_t* planes_host, uint32_t num_frames,
                                 uint32_t* sdr_host, uint32_t* count_host, void* cuda_stream) {
    return compute_host_impl(h, planes_host, true, num_frames, 0, sdr_host, count_host, cuda_stream);
}

sp_status sp_compute_packed(sp_handle* h, const uint32_t* planes_dev, uint32_t num_frames, uint32_t* sdr_dev,
                            uint32_t* count_dev, void* cuda_stream) {
    sp_status st = check_handle(h);
    if (st != SP_OK) return st;
    const uint64_t n = static_cast<uint64_t>(num_frames) * h->g.P;
    if (n > h->cfg.max_inputs)
        return fail(SP_E_ARG, "num_frames * inputs_per_frame = %llu exceeds max_inputs %u",
                    static_cast<unsigned long long>(n), h->cfg.max_inputs);
    if (num_frames > 0 && !planes_dev) return fail(SP_E_ARG, "planes_dev is NULL");
    if ((sdr_dev == nullptr) != (count_dev == nullptr))
        return fail(SP_E_ARG, "sdr_dev and count_dev must both be NULL or both be set");
    st = check_packed(h, static_cast<uint32_t>(n), planes_dev);
    if (st != SP_OK) return st;
    h->last_inputs = static_cast<uint32_t>(n);
    h->has_result = true;
    h->res_sdr = sdr_dev ? sdr_dev : h->d_sdr;
    h->res_counts = count_dev ? count_dev : h->d_counts;
    if (n == 0) return SP_OK;
    const sp_plan_info pl = make_plan(h, static_cast<uint32_t>(n), false, nullptr);
    h->last_plan = pl;
    return launch_batched_path(h, nullptr, planes_dev, num_frames, static_cast<uint32_t>(n), pl,
                               static_cast<cudaStream_t>(cuda_stream), 0);
}

sp_status sp_pack_frames(sp_handle* h, const uint8_t* frames_dev, uint32_t num_frames, uint32_t* planes_dev,
                         void* cuda_stream) {
    sp_status st = check_handle(h);
    if (st != SP_OK) return st;
    if (!h->g.whole) return fail(SP_E_CONFIG, "bit-plane input needs a whole-frame configuration (no patches)");
    if (num_frames > 0 && (!frames_dev || !planes_dev)) return fail(SP_E_ARG, "NULL device buffer");
    const uint32_t words = packed_words(h);
    for (uint32_t f0 = 0; f0 < num_frames; f0 += 65535u) {  // grid.y limit
        sp::PerInputParams pk{};
        pk.frames = frames_dev + static_cast<size_t>(f0) * h->g.W * h->g.H;
        pk.num_inputs = std::min(65535u, num_frames - f0);
        pk.g = h->g;
        pk.bits = planes_dev + static_cast<size_t>(f0) * words;
        pk.Wn = h->Wn;
        pk.bits_stride = words;
        h->launches++;
        const cudaError_t e = sp::launch_pack(pk, static_cast<cudaStream_t>(cuda_stream));
        if (e != cudaSuccess) return cuda_fail(e, "pack launch");
    }
    return SP_OK;
}

sp_status sp_get_info(sp_handle* h, sp_info* out) {
    if (!h) return fail(SP_E_ARG, "handle is NULL");
    if (!out) return fail(SP_E_ARG, "out is NULL");
    std::memset(out, 0, sizeof(*out));
    out->plan = h->last_plan;
    out->kernel_launches = h->launches.load();
    out->last_num_inputs = h->last_inputs;
    out->ell_slots = h->ell_slots;
    out->sm_count = h->sm_count;
    out->max_smem_optin = h->max_smem;
    out->learn_cluster = h->learn_Q;
    out->last_learn_cluster = h->last_learn_cluster ? 1u : 0u;
    out->learn_grid_ctas = (h->cfg.flags & SP_FLAG_FULL_LEARNING) ? h->gridf_G : h->grid_G;
    out->last_learn_path = h->last_learn_path;
    return SP_OK;
}

}  // extern "C"

// Development aid (not in include/sp.h): copies the batched kernel's per-CTA phase
// timestamps (SP_TRACE=1 at create) to host memory, uint64[ctas][6].
extern "C" sp_status sp_debug_trace(sp_handle* h, uint64_t* out, uint32_t ctas) {
    if (!h || !h->d_trace || !out) return SP_E_STATE;
    cudaDeviceSynchronize();
    return cudaMemcpy(out, h->d_trace, ctas * 6u * sizeof(uint64_t), cudaMemcpyDeviceToHost) == cudaSuccess
               ? SP_OK
               : SP_E_CUDA;
}
