// sp_encoder.cu — the adaptive video encoder on the device (PAPER.md
// "reduced in size ... converted to a grayscale one, which is later binarized using
// adaptive thresholding ... ADAPTIVE_THRESH_GAUSSIAN_C"; DESIGN R23-R25 and
// §4.9).  BGR uint8 frames -> binarised uint8 frames (255 / 0) that feed sp_compute.
//
// One persistent CTA loop over frames (2 CTAs per SM).  Per frame the source rows are streamed
// band by band (a band = the source rows of `band_rows` output rows: contiguous bytes, one
// cp.async.bulk per band into a ring of shared-memory stages, mbarrier completion), the band
// is area-downscaled (R23: OpenCV INTER_AREA, its fp32 operation order) and converted to gray
// (R24) into a resident gray image; then the Gaussian mean (R25: cv2.adaptiveThreshold's
// float32 blur -- a row pass then a symmetric column pass, one fp32 FMA per tap in OpenCV's
// order -- rounded half to even) and the threshold are computed by a register sliding window
// of row sums down each column pair, while the ring already streams the next frame.
// The path is HBM-bound: 3*W0*H0 bytes read, W1*H1 written per frame.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sp_internal.h"
#include "../../include/sp_encoder.h"

namespace sp {

namespace {

constexpr uint32_t kEncThreads = 256;
constexpr uint32_t kMaxStages = 4;

struct EncParams {
    const uint8_t* src;        // [F][H0][W0][3] BGR
    uint8_t* dst;              // [F][H1][W1]
    uint32_t F;
    uint32_t W0, H0, W1, H1;
    uint32_t row_bytes;        // 3 * W0
    uint32_t bands, band_rows; // output rows per band
    uint32_t stage_bytes, stages;
    uint32_t bulk;             // rows are 16-byte aligned: bulk copies, else cooperative loads
    uint32_t xfast;            // x table = {4dx + j, 0.25}, j < 4 (an exact 4:1 x scale)
    uint32_t l2hint;           // sp_encode_compute: BGR reads evict-first, binarised writes evict-last
                               // in L2 (the binarised chunk stays resident for the SP's loads)
    const uint32_t* band_sy0;  // [bands] first source row of the band
    const uint32_t* band_n;    // [bands] source rows of the band
    const uint32_t* yoff;      // [H1 + 1] y-table range of each output row
    const uint32_t* ysy;       // [.] source row of the entry
    const float* ybeta;        // [.] weight
    const uint32_t* xoff;      // [W1 + 1]
    const uint32_t* xsx;       // [.] source column of the entry
    const float* xalpha;       // [.]
    int32_t K, cbias;          // Gaussian window, ceil(bias)
    float kw[16];              // float32 Gaussian kernel (OpenCV getGaussianKernel, CV_32F)
    uint32_t ny_entries, nx_entries;  // table sizes (staged in shared memory per CTA)
    uint32_t table_bytes;      // shared-memory bytes of the staged tables
};

// the area tables staged in shared memory once per CTA (warp-uniform or conflict-free reads)
struct EncTables {
    const uint32_t* yoff;
    const uint32_t* ysy;
    const float* ybeta;
    const uint32_t* xoff;
    const uint32_t* xsx;
    const float* xalpha;
};

__device__ __forceinline__ void mbar_init_e(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
                 : "memory");
}

__device__ __forceinline__ void mbar_wait_e(uint64_t* bar, uint32_t parity) {
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}

// one thread: the source rows of band `b` of frame `f` into stage buffer `buf` (bulk copy)
__device__ __forceinline__ void issue_band(const EncParams& p, uint32_t f, uint32_t b, uint8_t* buf, uint64_t* bar) {
    const uint32_t bytes = p.band_n[b] * p.row_bytes;
    const uint8_t* g = p.src + (static_cast<size_t>(f) * p.H0 + p.band_sy0[b]) * p.row_bytes;
    const uint32_t ba = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of buf before async writes
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ba), "r"(bytes) : "memory");
    constexpr uint32_t kChunk = 32768u;
    uint64_t pol = 0;
    if (p.l2hint) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    for (uint32_t off = 0; off < bytes; off += kChunk) {
        const uint32_t n = min(kChunk, bytes - off);
        if (p.l2hint)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, "
                "[%3], %4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(buf + off))),
                "l"(g + off), "r"(n), "r"(ba), "l"(pol)
                : "memory");
        else
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    static_cast<uint32_t>(__cvta_generic_to_shared(buf + off))),
                "l"(g + off), "r"(n), "r"(ba)
                : "memory");
    }
}

// R23 + R24 for the output rows of band b: fp32 area sums in OpenCV's order, round half to
// even, saturate, then the 15-bit gray formula.  Thread (ty, tx) handles output pixels
// (dy0 + ty + k*ny, tx + m*sx) of the band.
__device__ __forceinline__ void downscale_band(const EncParams& p, const EncTables& t, uint32_t b, const uint8_t* buf,
                                               uint8_t* gray, uint32_t ty, uint32_t tx, uint32_t ny, uint32_t sx) {
    const uint32_t dy0 = b * p.band_rows, dy1 = min(p.H1, dy0 + p.band_rows);
    const int32_t rb = static_cast<int32_t>(p.row_bytes);
    const uint8_t* buf0 = buf - static_cast<int32_t>(p.band_sy0[b]) * rb;  // row sy of the band at buf0 + sy*rb
    for (uint32_t dy = dy0 + ty; dy < dy1; dy += ny) {
        const uint32_t j0 = t.yoff[dy], j1 = t.yoff[dy + 1];
        for (uint32_t dx = tx; dx < p.W1; dx += sx) {
            float sb, sg, sr;
            if (p.xfast) {
                // 4 BGR pixels = 12 bytes at 12*dx: B0 G0 R0 B1 | G1 R1 B2 G2 | R2 B3 G3 R3.
                // The x partial sums ((0 + S0/4) + S1/4) + ... are multiples of 0.25 below 2^10,
                // so exact: buf = (S0+S1+S2+S3)/4, and beta*buf = RN((beta/4) * (S0+..+S3)) with
                // ybeta holding beta/4 (exact).  Channel sums by byte-masked dot products.
                const uint8_t* col = buf0 + 12u * dx;
                auto sums = [&](uint32_t j, float& b_, float& g_, float& r_) {
                    const uint32_t* w = reinterpret_cast<const uint32_t*>(col + static_cast<int32_t>(t.ysy[j]) * rb);
                    const uint32_t w0 = w[0], w1 = w[1], w2 = w[2];
                    const float be = t.ybeta[j];
                    b_ = __fmul_rn(be, static_cast<float>(__dp4a(w0, 0x01000001u, __dp4a(w1, 0x00010000u, __dp4a(w2, 0x00000100u, 0u)))));
                    g_ = __fmul_rn(be, static_cast<float>(__dp4a(w0, 0x00000100u, __dp4a(w1, 0x01000001u, __dp4a(w2, 0x00010000u, 0u)))));
                    r_ = __fmul_rn(be, static_cast<float>(__dp4a(w0, 0x00010000u, __dp4a(w1, 0x00000100u, __dp4a(w2, 0x01000001u, 0u)))));
                };
                sums(j0, sb, sg, sr);  // the first term is beta*buf itself (OpenCV: sum = beta*buf)
                for (uint32_t j = j0 + 1u; j < j1; ++j) {
                    float tb, tg, tr;
                    sums(j, tb, tg, tr);
                    sb = __fadd_rn(sb, tb), sg = __fadd_rn(sg, tg), sr = __fadd_rn(sr, tr);
                }
            } else {
                sb = sg = sr = 0.0f;
                for (uint32_t j = j0; j < j1; ++j) {
                    const uint8_t* row = buf0 + static_cast<int32_t>(t.ysy[j]) * rb;
                    float bb = 0.0f, bg = 0.0f, br = 0.0f;
                    for (uint32_t k = t.xoff[dx]; k < t.xoff[dx + 1]; ++k) {
                        const uint8_t* s = row + 3u * t.xsx[k];
                        const float a = t.xalpha[k];
                        bb = __fadd_rn(bb, __fmul_rn(static_cast<float>(s[0]), a));
                        bg = __fadd_rn(bg, __fmul_rn(static_cast<float>(s[1]), a));
                        br = __fadd_rn(br, __fmul_rn(static_cast<float>(s[2]), a));
                    }
                    const float beta = t.ybeta[j];
                    const float tb = __fmul_rn(beta, bb), tg = __fmul_rn(beta, bg), tr = __fmul_rn(beta, br);
                    if (j == j0) {
                        sb = tb, sg = tg, sr = tr;
                    } else {
                        sb = __fadd_rn(sb, tb), sg = __fadd_rn(sg, tg), sr = __fadd_rn(sr, tr);
                    }
                }
            }
            const int B = min(255, max(0, __float2int_rn(sb)));  // saturate_cast<uchar>: half to even
            const int G = min(255, max(0, __float2int_rn(sg)));
            const int R = min(255, max(0, __float2int_rn(sr)));
            gray[dy * p.W1 + dx] = static_cast<uint8_t>((3735 * B + 19235 * G + 9798 * R + 16384) >> 15);
        }
    }
}

// R25: Gaussian mean and threshold for columns x and x+1 (one thread, shared loads), rows
// [y0, y1).  A register window holds the K row sums rs(y - R .. y + R) of both columns; row
// sums of the replicated rows outside the image are those of the clamped rows (OpenCV pads the
// source before its row filter).  Row pass: s = fma(g[x + j - R], k_j, s), j = 0..K-1, from
// s = 0; column pass: m = fma(rs(y), k_R, 0), then m = fma(rs(y + j) + rs(y - j), k_{R+j}, m),
// j = 1..R (OpenCV's AVX2/FMA3 RowVec_32f and symmetric SymmColumnVec_32f order).
template <int K>
__device__ __forceinline__ void blur_columns(const EncParams& p, const uint8_t* gray, uint8_t* out, uint32_t x,
                                             uint32_t y0, uint32_t y1, uint64_t pol) {
    constexpr int R = K / 2;
    const int W = static_cast<int>(p.W1), H = static_cast<int>(p.H1);
    const bool two = static_cast<int>(x) + 1 < W;
    int cx[K + 1];
#pragma unroll
    for (int j = 0; j <= K; ++j) cx[j] = min(W - 1, max(0, static_cast<int>(x) + j - R));
    float kw[K];
#pragma unroll
    for (int j = 0; j < K; ++j) kw[j] = p.kw[j];
    auto hsum = [&](int yy, float& a, float& b) {
        const uint8_t* row = gray + min(H - 1, max(0, yy)) * W;
        float v[K + 1];
#pragma unroll
        for (int j = 0; j <= K; ++j) v[j] = static_cast<float>(row[cx[j]]);
        a = 0.0f, b = 0.0f;
#pragma unroll
        for (int j = 0; j < K; ++j) a = __fmaf_rn(v[j], kw[j], a), b = __fmaf_rn(v[j + 1], kw[j], b);
    };
    float ha[K], hb[K];
#pragma unroll
    for (int i = 0; i < K - 1; ++i) hsum(static_cast<int>(y0) - R + i, ha[i], hb[i]);
    // the window is a register ring: row y0 - R + s lives in slot s mod K, so the loop is unrolled
    // K times with compile-time slots instead of shifting K - 1 registers per row
    for (int y = static_cast<int>(y0); y < static_cast<int>(y1); y += K) {
#pragma unroll
        for (int u = 0; u < K; ++u) {
            const int yy = y + u;
            if (yy >= static_cast<int>(y1)) break;
            hsum(yy + R, ha[(u + K - 1) % K], hb[(u + K - 1) % K]);
            float ma = __fmaf_rn(ha[(u + R) % K], kw[R], 0.0f), mb = __fmaf_rn(hb[(u + R) % K], kw[R], 0.0f);
#pragma unroll
            for (int j = 1; j <= R; ++j) {
                ma = __fmaf_rn(__fadd_rn(ha[(u + R + j) % K], ha[(u + R - j) % K]), kw[R + j], ma);
                mb = __fmaf_rn(__fadd_rn(hb[(u + R + j) % K], hb[(u + R - j) % K]), kw[R + j], mb);
            }
            // convertTo(CV_8U): round half to even, saturate
            const int mua = min(255, max(0, __float2int_rn(ma))), mub = min(255, max(0, __float2int_rn(mb)));
            const uint8_t* grow = gray + yy * W + x;
            uint8_t* orow = out + static_cast<size_t>(yy) * W + x;
            const uint32_t o0 = static_cast<int>(grow[0]) - mua > -p.cbias ? 255u : 0u;
            const uint32_t o1 = two && static_cast<int>(grow[1]) - mub > -p.cbias ? 255u : 0u;
            if (p.l2hint) {  // keep the binarised rows in L2 for the SP (sp_encode_compute)
                asm volatile("st.global.L2::cache_hint.u8 [%0], %1, %2;" ::"l"(orow), "r"(o0), "l"(pol) : "memory");
                if (two)
                    asm volatile("st.global.L2::cache_hint.u8 [%0], %1, %2;" ::"l"(orow + 1), "r"(o1), "l"(pol)
                                 : "memory");
            } else {
                orow[0] = static_cast<uint8_t>(o0);
                if (two) orow[1] = static_cast<uint8_t>(o1);
            }
        }
    }
}

__device__ __forceinline__ void blur_frame(const EncParams& p, const uint8_t* gray, uint8_t* out) {
    uint64_t pol = 0;  // L2 evict-last policy of the binarised stores (sp_encode_compute)
    if (p.l2hint) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    // column pairs x0 = 2c; the rows are split into segments so that all threads have work
    // (the K-1 halo rows of a segment are recomputed)
    const uint32_t pairs = (p.W1 + 1u) / 2u;
    const uint32_t segs = max(1u, min(p.H1 / 16u, blockDim.x / pairs));
    for (uint32_t t = threadIdx.x; t < segs * pairs; t += blockDim.x) {
        const uint32_t x = 2u * (t % pairs), sgi = t / pairs;
        const uint32_t y0 = p.H1 * sgi / segs, y1 = p.H1 * (sgi + 1u) / segs;
        switch (p.K) {
            case 3: blur_columns<3>(p, gray, out, x, y0, y1, pol); break;
            case 5: blur_columns<5>(p, gray, out, x, y0, y1, pol); break;
            case 7: blur_columns<7>(p, gray, out, x, y0, y1, pol); break;
            case 9: blur_columns<9>(p, gray, out, x, y0, y1, pol); break;
            case 11: blur_columns<11>(p, gray, out, x, y0, y1, pol); break;
            case 13: blur_columns<13>(p, gray, out, x, y0, y1, pol); break;
            default: blur_columns<15>(p, gray, out, x, y0, y1, pol); break;
        }
    }
}

// R23 + R24 for an exact 4:1 x scale and an even W1: one thread per pair of output pixels
// (dx, dx+1) of a row, whose 8 source pixels are 24 contiguous bytes (three 8-byte loads).
// Same operations and order as downscale_band's fast path (the x sums are exact).
__device__ __forceinline__ uint32_t chan_sums(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t c) {
    // B0 G0 R0 B1 | G1 R1 B2 G2 | R2 B3 G3 R3: byte masks of channel c in the three words
    const uint32_t m0 = c == 0 ? 0x01000001u : (c == 1 ? 0x00000100u : 0x00010000u);
    const uint32_t m1 = c == 0 ? 0x00010000u : (c == 1 ? 0x01000001u : 0x00000100u);
    const uint32_t m2 = c == 0 ? 0x00000100u : (c == 1 ? 0x00010000u : 0x01000001u);
    return __dp4a(w0, m0, __dp4a(w1, m1, __dp4a(w2, m2, 0u)));
}

// (row, pair) of a thread's first item and the per-step increment: the same for every band,
// computed once per kernel (a division per band per thread was 4% of the encoder's samples)
struct PairMap {
    uint32_t r0, q0, rstep, qstep;
};

__device__ __forceinline__ void downscale_band_pairs(const EncParams& p, const EncTables& t, uint32_t b,
                                                     const uint8_t* buf, uint8_t* gray, const PairMap& pm) {
    const uint32_t dy0 = b * p.band_rows, dy1 = min(p.H1, dy0 + p.band_rows);
    const uint32_t pairs = p.W1 / 2u;
    const int32_t rb = static_cast<int32_t>(p.row_bytes);
    const uint8_t* buf0 = buf - static_cast<int32_t>(p.band_sy0[b]) * rb;
    uint32_t r0 = pm.r0, q0 = pm.q0;
    for (uint32_t i = threadIdx.x; i < (dy1 - dy0) * pairs; i += blockDim.x) {
        const uint32_t dy = dy0 + r0, dx = 2u * q0;
        r0 += pm.rstep, q0 += pm.qstep;  // the next item without a division
        if (q0 >= pairs) q0 -= pairs, ++r0;
        const uint8_t* col = buf0 + 12u * dx;
        const uint32_t j0 = t.yoff[dy], j1 = t.yoff[dy + 1];
        float s[6];
        for (uint32_t j = j0; j < j1; ++j) {
            const uint2* w = reinterpret_cast<const uint2*>(col + static_cast<int32_t>(t.ysy[j]) * rb);
            const uint2 a = w[0], bb = w[1], cc = w[2];
            const float be = t.ybeta[j];  // beta / 4
#pragma unroll
            for (uint32_t ch = 0; ch < 3u; ++ch) {
                const float ta = __fmul_rn(be, static_cast<float>(chan_sums(a.x, a.y, bb.x, ch)));
                const float tb = __fmul_rn(be, static_cast<float>(chan_sums(bb.y, cc.x, cc.y, ch)));
                if (j == j0) {
                    s[ch] = ta, s[3 + ch] = tb;
                } else {
                    s[ch] = __fadd_rn(s[ch], ta), s[3 + ch] = __fadd_rn(s[3 + ch], tb);
                }
            }
        }
        int v[6];
#pragma unroll
        for (int q = 0; q < 6; ++q) v[q] = min(255, max(0, __float2int_rn(s[q])));
        const uint8_t g0 = static_cast<uint8_t>((3735 * v[0] + 19235 * v[1] + 9798 * v[2] + 16384) >> 15);
        const uint8_t g1 = static_cast<uint8_t>((3735 * v[3] + 19235 * v[4] + 9798 * v[5] + 16384) >> 15);
        *reinterpret_cast<uint16_t*>(gray + dy * p.W1 + dx) = static_cast<uint16_t>(g0 | (g1 << 8));
    }
}

__global__ void __launch_bounds__(kEncThreads, 2) k_encode(const __grid_constant__ EncParams p) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bars[kMaxStages];
    uint8_t* gray = sm;
    uint8_t* ring = sm + ((p.W1 * p.H1 + 127u) & ~127u);
    // area tables -> shared memory (after the ring)
    EncTables t;
    {
        uint32_t* tu = reinterpret_cast<uint32_t*>(ring + p.stages * p.stage_bytes);
        uint32_t* yoff = tu;
        uint32_t* ysy = yoff + p.H1 + 1u;
        float* ybeta = reinterpret_cast<float*>(ysy + p.ny_entries);
        uint32_t* xoff = reinterpret_cast<uint32_t*>(ybeta + p.ny_entries);
        uint32_t* xsx = xoff + p.W1 + 1u;
        float* xalpha = reinterpret_cast<float*>(xsx + p.nx_entries);
        for (uint32_t i = threadIdx.x; i <= p.H1; i += blockDim.x) yoff[i] = p.yoff[i];
        for (uint32_t i = threadIdx.x; i < p.ny_entries; i += blockDim.x) ysy[i] = p.ysy[i], ybeta[i] = p.ybeta[i];
        if (!p.xfast) {
            for (uint32_t i = threadIdx.x; i <= p.W1; i += blockDim.x) xoff[i] = p.xoff[i];
            for (uint32_t i = threadIdx.x; i < p.nx_entries; i += blockDim.x) xsx[i] = p.xsx[i], xalpha[i] = p.xalpha[i];
        }
        t = EncTables{yoff, ysy, ybeta, xoff, xsx, xalpha};
    }
    // pixel mapping of the downscale: rows of W1 threads (W1 <= blockDim), else one row
    const uint32_t ny = p.W1 <= blockDim.x ? blockDim.x / p.W1 : 1u;
    const uint32_t ty = p.W1 <= blockDim.x ? threadIdx.x / p.W1 : 0u;
    const uint32_t tx = p.W1 <= blockDim.x ? threadIdx.x % p.W1 : threadIdx.x;
    const uint32_t sxs = p.W1 <= blockDim.x ? p.W1 : blockDim.x;
    PairMap pm{};
    if (p.W1 >= 2u) {
        const uint32_t pairs = p.W1 / 2u;
        pm.r0 = threadIdx.x / pairs, pm.q0 = threadIdx.x - pm.r0 * pairs;
        pm.rstep = blockDim.x / pairs, pm.qstep = blockDim.x - pm.rstep * pairs;
    }
    const uint32_t nf = p.F > blockIdx.x ? (p.F - blockIdx.x + gridDim.x - 1u) / gridDim.x : 0u;
    const uint32_t total = nf * p.bands;  // (frame, band) sequence of this CTA
    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < p.stages; ++s) mbar_init_e(&bars[s]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto frame_of = [&](uint32_t seq) { return blockIdx.x + (seq / p.bands) * gridDim.x; };
    if (p.bulk && threadIdx.x == 0)
        for (uint32_t s = 0; s < p.stages && s < total; ++s)
            issue_band(p, frame_of(s), s % p.bands, ring + s * p.stage_bytes, &bars[s]);
    uint32_t seq = 0, st = 0, phase = 0;  // ring position: stage and its mbarrier parity
    for (uint32_t i = 0; i < nf; ++i) {
        const uint32_t f = blockIdx.x + i * gridDim.x;
        for (uint32_t b = 0; b < p.bands; ++b, ++seq) {
            uint8_t* buf = ring + st * p.stage_bytes;
            if (p.bulk) {
                mbar_wait_e(&bars[st], phase);
            } else {  // unaligned rows: cooperative byte copy of the band
                const uint8_t* g = p.src + (static_cast<size_t>(f) * p.H0 + p.band_sy0[b]) * p.row_bytes;
                const uint32_t bytes = p.band_n[b] * p.row_bytes;
                for (uint32_t k = threadIdx.x; k < bytes; k += blockDim.x) buf[k] = g[k];
                __syncthreads();
            }
            if (p.xfast && (p.W1 & 1u) == 0u) downscale_band_pairs(p, t, b, buf, gray, pm);
            else if (ty < ny) downscale_band(p, t, b, buf, gray, ty, tx, ny, sxs);
            __syncthreads();  // the stage is free; the band's gray rows are complete
            if (p.bulk && threadIdx.x == 0 && seq + p.stages < total) {
                const uint32_t nx = seq + p.stages;
                issue_band(p, frame_of(nx), nx % p.bands, buf, &bars[st]);
            }
            if (++st == p.stages) st = 0, phase ^= 1u;
        }
        blur_frame(p, gray, p.dst + static_cast<size_t>(f) * p.W1 * p.H1);
        __syncthreads();  // the gray image is rewritten by the next frame's bands
    }
}

// OpenCV computeResizeAreaTab (R23), implemented from its definition: (dst, src, weight) per
// axis in order, weights computed in double and stored as float
void area_table(uint32_t ssize, uint32_t dsize, std::vector<uint32_t>& off, std::vector<uint32_t>& src,
                std::vector<float>& w) {
    const double scale = static_cast<double>(ssize) / dsize;
    off.assign(dsize + 1u, 0u);
    src.clear();
    w.clear();
    for (uint32_t d = 0; d < dsize; ++d) {
        off[d] = static_cast<uint32_t>(src.size());
        const double f1 = d * scale, f2 = f1 + scale;
        const double cell = std::min(scale, ssize - f1);
        int s1 = static_cast<int>(std::ceil(f1)), s2 = static_cast<int>(std::floor(f2));
        s2 = std::min(s2, static_cast<int>(ssize) - 1);
        s1 = std::min(s1, s2);
        if (s1 - f1 > 1e-3) {
            src.push_back(static_cast<uint32_t>(s1 - 1));
            w.push_back(static_cast<float>((s1 - f1) / cell));
        }
        for (int s = s1; s < s2; ++s) {
            src.push_back(static_cast<uint32_t>(s));
            w.push_back(static_cast<float>(1.0 / cell));
        }
        if (f2 - s2 > 1e-3) {
            src.push_back(static_cast<uint32_t>(s2));
            w.push_back(static_cast<float>(std::min(std::min(f2 - s2, 1.0), cell) / cell));
        }
    }
    off[dsize] = static_cast<uint32_t>(src.size());
}

}  // namespace

}  // namespace sp

struct sp_encoder {
    sp_encoder_config cfg{};
    sp::EncParams p{};
    int device = 0, sm_count = 148;
    uint32_t smem = 0, ctas_per_sm = 1;
    uint32_t* d_u32 = nullptr;  // band_sy0 | band_n | yoff | ysy | xoff | xsx
    float* d_f32 = nullptr;     // ybeta | xalpha
    uint64_t launches = 0;
    // sp_encode_compute: chunk of binarised frames kept in a persisting-L2 window between the
    // encoder and the SP (never written back to HBM while it stays resident).  4096 frames
    // (132 MB): measured 2.30 M frames/s vs 1.98 M at 1024 -- the two kernels' per-chunk tails
    // cost more than the L2 handoff saves
    uint32_t chunk = 4096;
    uint8_t* d_chunk = nullptr;
    size_t l2_window = 0;       // bytes of the window (0: no persisting L2 on this device)
    uint64_t fused_calls = 0;
    cudaStream_t fstream = nullptr;  // internal stream carrying the access-policy window
    cudaEvent_t fev[2] = {nullptr, nullptr};
    bool window_set = false;    // the stream attribute was accepted
};

namespace {

thread_local char g_enc_err[256];

sp_status efail(sp_status st, const char* msg) {
    std::snprintf(g_enc_err, sizeof(g_enc_err), "%s", msg);
    return st;
}

// float32 Gaussian kernel (R25), OpenCV getGaussianKernel(k, 0, CV_32F): fixed tables for
// k <= 9, else exp(-x^2 / (2 sigma^2)) with sigma = fma(k, 0.15, 0.35), normalised in double
// (outer weights summed in order, doubled, plus the centre's 1), rounded to float
void gaussian_f32(int k, float* kw) {
    static const double small3[] = {0.25, 0.5, 0.25};
    static const double small5[] = {0.0625, 0.25, 0.375, 0.25, 0.0625};
    static const double small7[] = {0.03125, 0.109375, 0.21875, 0.28125, 0.21875, 0.109375, 0.03125};
    static const double small9[] = {4 / 256., 13 / 256., 30 / 256., 51 / 256., 60 / 256.,
                                    51 / 256., 30 / 256., 13 / 256., 4 / 256.};
    if (k <= 9) {
        const double* t = k == 3 ? small3 : (k == 5 ? small5 : (k == 7 ? small7 : small9));
        for (int i = 0; i < k; ++i) kw[i] = static_cast<float>(t[i]);
        return;
    }
    const int n2 = k / 2;
    std::vector<double> w(n2);
    const double sigma = std::fma(static_cast<double>(k), 0.15, 0.35);
    const double s2 = -0.125 / (sigma * sigma);
    double total = 0.0;
    for (int i = 0; i < n2; ++i) {
        const double x = 2.0 * i - (k - 1);
        w[i] = std::exp(x * x * s2);
        total += w[i];
    }
    total = total * 2.0 + 1.0;
    const double mul = 1.0 / total;
    for (int i = 0; i < n2; ++i) kw[i] = kw[k - 1 - i] = static_cast<float>(w[i] * mul);
    kw[n2] = static_cast<float>(1.0 * mul);
}

sp_status encode_impl(sp_encoder* e, const uint8_t* bgr_dev, uint32_t num_frames, uint8_t* out_dev, void* cuda_stream,
                      uint32_t l2hint) {
    if (!e) return efail(SP_E_ARG, "encoder is NULL");
    if (num_frames == 0) return SP_OK;
    if (!bgr_dev || !out_dev) return efail(SP_E_ARG, "NULL frame buffer");
    cudaSetDevice(e->device);
    sp::EncParams p = e->p;
    p.src = bgr_dev;
    p.dst = out_dev;
    p.F = num_frames;
    p.bulk = ((reinterpret_cast<uintptr_t>(bgr_dev) & 15u) == 0 && (p.row_bytes & 15u) == 0) ? 1u : 0u;
    p.l2hint = l2hint;
    const uint32_t grid = std::min<uint32_t>(num_frames, e->ctas_per_sm * static_cast<uint32_t>(e->sm_count));
    sp::k_encode<<<grid, sp::kEncThreads, e->smem, static_cast<cudaStream_t>(cuda_stream)>>>(p);
    e->launches++;
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return efail(SP_E_CUDA, cudaGetErrorString(err));
    return SP_OK;
}

}  // namespace

extern "C" {

sp_status sp_encoder_config_default(sp_encoder_config* cfg) {
    if (!cfg) return efail(SP_E_ARG, "config is NULL");
    cfg->src_width = 960;   // rendered frames
    cfg->src_height = 540;
    cfg->dst_width = 240;   // resized to 240x134
    cfg->dst_height = 134;
    cfg->block_size = 11;
    cfg->bias = 2.0f;
    cfg->device = 0;
    return SP_OK;
}

const char* sp_encoder_last_error(void) { return g_enc_err; }

sp_status sp_encoder_create(const sp_encoder_config* cfg, sp_encoder** out) {
    if (!cfg || !out) return efail(SP_E_ARG, "NULL argument");
    *out = nullptr;
    if (!cfg->src_width || !cfg->src_height || !cfg->dst_width || !cfg->dst_height)
        return efail(SP_E_CONFIG, "frame dimensions must be >= 1");
    if (cfg->dst_width > cfg->src_width || cfg->dst_height > cfg->src_height)
        return efail(SP_E_CONFIG, "upscaling is an input error (S:289)");
    if (cfg->block_size < 3 || cfg->block_size > 15 || cfg->block_size % 2 == 0)
        return efail(SP_E_CONFIG, "block_size must be odd in [3, 15]");
    if (!std::isfinite(cfg->bias) || std::fabs(cfg->bias) > 255.0f) return efail(SP_E_CONFIG, "bias out of range");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return efail(SP_E_CUDA, "no CUDA device");
    if (cfg->device < 0 || cfg->device >= ndev) return efail(SP_E_ARG, "device out of range");
    cudaSetDevice(cfg->device);
    sp_encoder* e = new sp_encoder();
    e->cfg = *cfg;
    e->device = cfg->device;
    cudaDeviceGetAttribute(&e->sm_count, cudaDevAttrMultiProcessorCount, e->device);
    int max_smem = 0;
    cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, e->device);
    int sm_smem = 0;
    cudaDeviceGetAttribute(&sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, e->device);
    sp::EncParams& p = e->p;
    p.W0 = cfg->src_width, p.H0 = cfg->src_height, p.W1 = cfg->dst_width, p.H1 = cfg->dst_height;
    p.row_bytes = 3u * p.W0;
    p.K = static_cast<int32_t>(cfg->block_size);
    p.cbias = static_cast<int32_t>(std::ceil(cfg->bias));
    gaussian_f32(p.K, p.kw);
    std::vector<uint32_t> yoff, ysy, xoff, xsx;
    std::vector<float> ybeta, xalpha;
    sp::area_table(p.H0, p.H1, yoff, ysy, ybeta);
    sp::area_table(p.W0, p.W1, xoff, xsx, xalpha);
    p.xfast = 1u;
    for (uint32_t d = 0; d < p.W1 && p.xfast; ++d) {
        if (xoff[d + 1] - xoff[d] != 4u) p.xfast = 0u;
        for (uint32_t k = xoff[d]; k < xoff[d + 1] && p.xfast; ++k)
            if (xsx[k] != 4u * d + (k - xoff[d]) || xalpha[k] != 0.25f) p.xfast = 0u;
    }
    // bands of output rows: the fewest bands (largest band_rows, stage <= 48 KiB) whose ring of
    // >= 2 stages lets 2 CTAs share an SM; then the deepest ring that keeps that occupancy
    const uint32_t gray_bytes = (p.W1 * p.H1 + 127u) & ~127u;
    p.ny_entries = static_cast<uint32_t>(ysy.size());
    p.nx_entries = static_cast<uint32_t>(xsx.size());
    // the x tables are only staged for the generic path (the 4:1 fast path does not read them)
    p.table_bytes = 4u * (p.H1 + 1u + 2u * p.ny_entries + (p.xfast ? 0u : p.W1 + 1u + 2u * p.nx_entries));
    int static_smem = 0;
    {
        cudaFuncAttributes fa{};
        if (cudaFuncGetAttributes(&fa, sp::k_encode) == cudaSuccess) static_smem = static_cast<int>(fa.sharedSizeBytes);
    }
    uint32_t best_rows = 0, best_stages = 0, best_cps = 0, best_stage_bytes = 0;
    const char* mc = std::getenv("SP_ENC_MAXCPS");  // development override (experiments)
    const uint32_t max_cps = mc ? static_cast<uint32_t>(std::atoi(mc)) : 2u;
    std::vector<uint32_t> sy0, sn;
    for (uint32_t rows = 1; rows <= p.H1; ++rows) {
        uint32_t maxn = 0;
        for (uint32_t b = 0; b * rows < p.H1; ++b) {
            const uint32_t d0 = b * rows, d1 = std::min(p.H1, d0 + rows);
            const uint32_t lo = ysy[yoff[d0]], hi = ysy[yoff[d1] - 1u];
            maxn = std::max(maxn, hi - lo + 1u);
        }
        const uint32_t stage = (maxn * p.row_bytes + 127u) & ~127u;
        if (rows > 1 && stage > 49152u) break;
        for (uint32_t stages = sp::kMaxStages; stages >= 2; --stages) {
            const uint32_t smem = gray_bytes + stages * stage + p.table_bytes;
            if (static_cast<int>(smem) > max_smem - static_smem) continue;
            const uint32_t cps = std::min<uint32_t>(max_cps, static_cast<uint32_t>(sm_smem) /
                                                                 (smem + static_smem + 1024u));
            if (cps == 0) continue;
            const bool better = cps > best_cps || (cps == best_cps && (rows > best_rows ||
                                                                         (rows == best_rows && stages > best_stages)));
            if (better) best_rows = rows, best_stages = stages, best_cps = cps, best_stage_bytes = stage;
        }
    }
    if (!best_rows) {
        delete e;
        return efail(SP_E_CONFIG, "frame rows do not fit shared memory");
    }
    p.band_rows = best_rows;
    p.stages = best_stages;
    p.stage_bytes = best_stage_bytes;
    e->ctas_per_sm = std::max<uint32_t>(1u, best_cps);
    e->smem = gray_bytes + p.stages * p.stage_bytes + p.table_bytes;
    p.bands = (p.H1 + p.band_rows - 1u) / p.band_rows;
    for (uint32_t b = 0; b < p.bands; ++b) {
        const uint32_t d0 = b * p.band_rows, d1 = std::min(p.H1, d0 + p.band_rows);
        sy0.push_back(ysy[yoff[d0]]);
        sn.push_back(ysy[yoff[d1] - 1u] - ysy[yoff[d0]] + 1u);
    }
    std::vector<uint32_t> u32;
    auto put = [&](const std::vector<uint32_t>& v) {
        const size_t o = u32.size();
        u32.insert(u32.end(), v.begin(), v.end());
        return o;
    };
    if (p.xfast)
        for (float& bta : ybeta) bta *= 0.25f;  // beta/4 is exact (R23 fast path)
    const size_t o_sy0 = put(sy0), o_sn = put(sn), o_yoff = put(yoff), o_ysy = put(ysy), o_xoff = put(xoff),
                 o_xsx = put(xsx);
    std::vector<float> f32(ybeta);
    const size_t o_xa = f32.size();
    f32.insert(f32.end(), xalpha.begin(), xalpha.end());
    cudaError_t err = cudaMalloc(&e->d_u32, u32.size() * 4u);
    if (err == cudaSuccess) err = cudaMalloc(&e->d_f32, f32.size() * 4u);
    if (err == cudaSuccess) err = cudaMemcpy(e->d_u32, u32.data(), u32.size() * 4u, cudaMemcpyHostToDevice);
    if (err == cudaSuccess) err = cudaMemcpy(e->d_f32, f32.data(), f32.size() * 4u, cudaMemcpyHostToDevice);
    if (err == cudaSuccess)
        err = cudaFuncSetAttribute(sp::k_encode, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(e->smem));
    if (err != cudaSuccess) {
        if (e->d_u32) cudaFree(e->d_u32);
        if (e->d_f32) cudaFree(e->d_f32);
        delete e;
        return efail(SP_E_CUDA, cudaGetErrorString(err));
    }
    p.band_sy0 = e->d_u32 + o_sy0;
    p.band_n = e->d_u32 + o_sn;
    p.yoff = e->d_u32 + o_yoff;
    p.ysy = e->d_u32 + o_ysy;
    p.xoff = e->d_u32 + o_xoff;
    p.xsx = e->d_u32 + o_xsx;
    p.ybeta = e->d_f32;
    p.xalpha = e->d_f32 + o_xa;
    *out = e;
    return SP_OK;
}

sp_status sp_encoder_destroy(sp_encoder* e) {
    if (!e) return SP_OK;
    cudaSetDevice(e->device);
    cudaDeviceSynchronize();
    cudaFree(e->d_u32);
    cudaFree(e->d_f32);
    if (e->d_chunk) cudaFree(e->d_chunk);
    if (e->fstream) cudaStreamDestroy(e->fstream);
    for (cudaEvent_t ev : e->fev)
        if (ev) cudaEventDestroy(ev);
    delete e;
    return SP_OK;
}

sp_status sp_encode_compute(sp_encoder* e, sp_handle* sp, const uint8_t* bgr_dev, uint32_t num_frames,
                            uint32_t* sdr_dev, uint32_t* count_dev, void* cuda_stream) {
    if (!e || !sp) return efail(SP_E_ARG, "encoder or SP handle is NULL");
    uint32_t W = 0, H = 0, P = 0, words = 0;
    int dev = 0;
    if (sp::handle_frame_dims(sp, &W, &H, &P, &words, &dev) != SP_OK) return efail(SP_E_ARG, "SP handle");
    if (W != e->p.W1 || H != e->p.H1)
        return efail(SP_E_CONFIG, "the SP's input frame must be the encoder's output frame (dst_width x dst_height)");
    if (dev != e->device) return efail(SP_E_ARG, "encoder and SP on different devices");
    if (num_frames == 0) return SP_OK;
    if (!bgr_dev || !sdr_dev || !count_dev) return efail(SP_E_ARG, "NULL buffer");
    cudaSetDevice(e->device);
    cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
    const size_t fbytes = static_cast<size_t>(e->p.W1) * e->p.H1;
    if (!e->d_chunk) {
        if (const char* ec = std::getenv("SP_ENC_CHUNK")) e->chunk = std::max(1, std::atoi(ec));
        cudaError_t err = cudaMalloc(&e->d_chunk, e->chunk * fbytes);
        if (err != cudaSuccess) {
            e->d_chunk = nullptr;
            return efail(SP_E_OOM, cudaGetErrorString(err));
        }
        // persisting L2 set-aside for the chunk buffer: raised for the duration of each call
        // and restored afterwards (a standing set-aside shrinks L2 for every other kernel)
        int max_persist = 0;
        cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, e->device);
        e->l2_window = std::min<size_t>(static_cast<size_t>(max_persist), e->chunk * fbytes);
        // an internal stream whose access-policy window is the chunk buffer (the caller's stream,
        // possibly the legacy default stream, is left untouched); ordered by events
        cudaError_t es = cudaStreamCreateWithFlags(&e->fstream, cudaStreamNonBlocking);
        if (es == cudaSuccess) es = cudaEventCreateWithFlags(&e->fev[0], cudaEventDisableTiming);
        if (es == cudaSuccess) es = cudaEventCreateWithFlags(&e->fev[1], cudaEventDisableTiming);
        if (es != cudaSuccess) return efail(SP_E_CUDA, cudaGetErrorString(es));
        if (e->l2_window > 0) {
            cudaStreamAttrValue attr{};
            attr.accessPolicyWindow.base_ptr = e->d_chunk;
            attr.accessPolicyWindow.num_bytes = e->chunk * fbytes;
            attr.accessPolicyWindow.hitRatio =
                std::min(1.0f, static_cast<float>(e->l2_window) / static_cast<float>(e->chunk * fbytes));
            attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
            attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
            e->window_set = cudaStreamSetAttribute(e->fstream, cudaStreamAttributeAccessPolicyWindow, &attr) ==
                            cudaSuccess;
        }
        (void)cudaGetLastError();
    }
    size_t old_limit = 0;
    cudaDeviceGetLimit(&old_limit, cudaLimitPersistingL2CacheSize);
    if (e->l2_window > old_limit) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, e->l2_window);
    (void)cudaGetLastError();
    cudaStream_t fs = e->fstream;
    cudaError_t ee = cudaEventRecord(e->fev[0], s);
    if (ee == cudaSuccess) ee = cudaStreamWaitEvent(fs, e->fev[0], 0);
    if (ee != cudaSuccess) return efail(SP_E_CUDA, cudaGetErrorString(ee));
    sp_status st = SP_OK;
    for (uint32_t f0 = 0; f0 < num_frames && st == SP_OK; f0 += e->chunk) {
        const uint32_t n = std::min(e->chunk, num_frames - f0);
        st = encode_impl(e, bgr_dev + static_cast<size_t>(f0) * 3u * e->p.W0 * e->p.H0, n, e->d_chunk, fs, 1u);
        if (st != SP_OK) break;
        const size_t row = static_cast<size_t>(f0) * P;
        st = sp_compute_into(sp, e->d_chunk, n, 0, sdr_dev + row * words, count_dev + row, fs);
    }
    // the caller's stream continues after the last chunk
    ee = cudaEventRecord(e->fev[1], fs);
    if (ee == cudaSuccess) ee = cudaStreamWaitEvent(s, e->fev[1], 0);
    if (e->l2_window > old_limit) {
        // the persisting lines go back to normal once the SP has read the last chunk
        cudaStreamSynchronize(fs);
        cudaCtxResetPersistingL2Cache();
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, old_limit);
        (void)cudaGetLastError();
    }
    if (st != SP_OK) return efail(st, sp_last_error());
    if (ee != cudaSuccess) return efail(SP_E_CUDA, cudaGetErrorString(ee));
    // the winners of the whole call are the SP's "last results" (sp_winners, sp_histograms)
    sp::handle_set_result(sp, sdr_dev, count_dev, static_cast<uint32_t>(static_cast<uint64_t>(num_frames) * P));
    e->fused_calls++;
    return SP_OK;
}

sp_status sp_encode(sp_encoder* e, const uint8_t* bgr_dev, uint32_t num_frames, uint8_t* out_dev, void* cuda_stream) {
    return encode_impl(e, bgr_dev, num_frames, out_dev, cuda_stream, 0u);
}

sp_status sp_encoder_get_info(sp_encoder* e, sp_encoder_info* out) {
    if (!e || !out) return efail(SP_E_ARG, "NULL argument");
    out->band_rows = e->p.band_rows;
    out->bands = e->p.bands;
    out->stages = e->p.stages;
    out->stage_bytes = e->p.stage_bytes;
    out->smem_bytes = e->smem;
    out->ctas_per_sm = e->ctas_per_sm;
    out->xfast = e->p.xfast;
    out->kernel_launches = e->launches;
    for (int i = 0; i < 16; ++i) out->kernel[i] = i < e->p.K ? e->p.kw[i] : 0.0f;
    out->chunk_frames = e->chunk;
    out->l2_window_set = e->window_set ? 1u : 0u;
    out->l2_window_bytes = e->l2_window;
    return SP_OK;
}

}  // extern "C"
