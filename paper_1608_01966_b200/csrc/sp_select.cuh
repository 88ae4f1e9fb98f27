// sp_select.cuh — warp-level k-winners building blocks shared by the batched, per-input
// and cluster-learning kernels.
//
// Local inhibition with a uniform boost (R6, R7, R9): with one boost the key order is
// (raw desc, index asc) and the floor raw*Bc > 2^23 is raw >= r_lo.  Column c wins iff
// x_c >= r_lo and fewer than k columns d != c of its truncated window [c-r, c+r] beat it,
// where d beats c iff x_d > x_c, or x_d == x_c and d < c; x = raw, zeroed below r_lo
// (a zeroed column never beats an eligible one, and never wins).
//
// Bit-sliced evaluation: the x values of each 32-column word are stored as nb bit-planes
// (one ballot per plane); a lane compares its own x with the 32 columns of a neighbour word
// at once (3 LOP3 per plane), masks the window and the tie-break, and popcounts.
#pragma once

#include <cstdint>

#include <cuda_fp16.h>

namespace sp {

// planes[cw * nb + b] = bit b of x over the 32 columns of word cw, for cw = cw0, cw0+step, ..
template <typename RowT>
__device__ __forceinline__ void build_raw_planes(const RowT* row, uint32_t* planes, uint32_t ncw,
                                                 uint32_t nb, uint32_t r_lo, uint32_t cw0,
                                                 uint32_t step, uint32_t lane) {
    for (uint32_t cw = cw0; cw < ncw; cw += step) {
        uint32_t x = row[cw * 32u + lane];
        x = x >= r_lo ? x : 0u;
        for (uint32_t b = 0; b < nb; ++b) {
            const uint32_t pl = __ballot_sync(0xffffffffu, (x >> b) & 1u);
            if (lane == b) planes[cw * nb + b] = pl;
        }
    }
}

// Number of columns of the window of c (inside word jw) that beat c, given gt/eq masks.
__device__ __forceinline__ uint32_t window_beats(int jw, int c, int lo, int hi, uint32_t gt,
                                                 uint32_t eq) {
    const int base = jw * 32;
    const int a = max(lo, base) - base, z = min(hi, base + 31) - base;
    uint32_t wm = a <= z ? (0xFFFFFFFFu >> (31 - z)) & (0xFFFFFFFFu << a) : 0u;
    const int self = c - base;
    uint32_t below = 0u;  // bits d < c inside this word
    if (self >= 32) below = 0xFFFFFFFFu;
    else if (self > 0) below = 0xFFFFFFFFu >> (32 - self);
    if (self >= 0 && self < 32) wm &= ~(1u << self);
    return __popc(gt & wm) + __popc(eq & wm & below);
}

// Winners of the 32 columns of word cw (the SDR word), all lanes of the warp call it.
template <typename RowT>
__device__ __forceinline__ uint32_t local_uniform_word(const RowT* row, const uint32_t* planes,
                                                       uint32_t ncw, uint32_t nb, uint32_t cw,
                                                       uint32_t C, uint32_t radius, uint32_t k,
                                                       uint32_t r_lo, uint32_t lane) {
    const int c = static_cast<int>(cw * 32u + lane);
    uint32_t x = row[c];
    x = x >= r_lo ? x : 0u;
    const int R = static_cast<int>(radius), Cn = static_cast<int>(C);
    const int lo = max(0, c - R), hi = min(Cn - 1, c + R);
    const int jw0 = max(0, (static_cast<int>(cw) * 32 - R) / 32);
    const int jw1 = min(static_cast<int>(ncw) - 1, (static_cast<int>(cw) * 32 + 31 + R) / 32);
    uint32_t Xm[10];  // per-plane masks of this lane's x (nb <= 10: S <= 1023)
#pragma unroll
    for (int b = 0; b < 10; ++b) Xm[b] = 0u - ((x >> b) & 1u);
    uint32_t beats = 0;
    int jw = jw0;
    for (; jw + 1 <= jw1; jw += 2) {  // two independent neighbour words (ILP)
        const uint32_t* P0 = planes + jw * nb;
        const uint32_t* P1 = P0 + nb;
        uint32_t gt0 = 0u, eq0 = 0xFFFFFFFFu, gt1 = 0u, eq1 = 0xFFFFFFFFu;
#pragma unroll
        for (int b = 9; b >= 0; --b) {
            if (b < static_cast<int>(nb)) {
                const uint32_t B0 = P0[b], B1 = P1[b], X = Xm[b];
                gt0 |= eq0 & B0 & ~X;
                eq0 &= ~(B0 ^ X);
                gt1 |= eq1 & B1 & ~X;
                eq1 &= ~(B1 ^ X);
            }
        }
        beats += window_beats(jw, c, lo, hi, gt0, eq0) + window_beats(jw + 1, c, lo, hi, gt1, eq1);
    }
    if (jw <= jw1) {
        const uint32_t* P0 = planes + jw * nb;
        uint32_t gt0 = 0u, eq0 = 0xFFFFFFFFu;
#pragma unroll
        for (int b = 9; b >= 0; --b) {
            if (b < static_cast<int>(nb)) {
                const uint32_t B0 = P0[b], X = Xm[b];
                gt0 |= eq0 & B0 & ~X;
                eq0 &= ~(B0 ^ X);
            }
        }
        beats += window_beats(jw, c, lo, hi, gt0, eq0);
    }
    return __ballot_sync(0xffffffffu, c < Cn && x > 0u && beats < k);
}

// Beats of lane's column of word cw counted over the neighbour words jw0+part, jw0+part+parts,
// .. only (several warps share one word's window); x_out = the column's value (0: ineligible)
template <typename RowT>
__device__ __forceinline__ uint32_t local_uniform_beats_part(const RowT* row, const uint32_t* planes, uint32_t ncw,
                                                             uint32_t nb, uint32_t cw, uint32_t C, uint32_t radius,
                                                             uint32_t r_lo, uint32_t lane, uint32_t part,
                                                             uint32_t parts, uint32_t& x_out) {
    const int c = static_cast<int>(cw * 32u + lane);
    uint32_t x = row[c];
    x = x >= r_lo ? x : 0u;
    x_out = c < static_cast<int>(C) ? x : 0u;
    const int R = static_cast<int>(radius), Cn = static_cast<int>(C);
    const int lo = max(0, c - R), hi = min(Cn - 1, c + R);
    const int jw0 = max(0, (static_cast<int>(cw) * 32 - R) / 32);
    const int jw1 = min(static_cast<int>(ncw) - 1, (static_cast<int>(cw) * 32 + 31 + R) / 32);
    uint32_t Xm[10];
#pragma unroll
    for (int b = 0; b < 10; ++b) Xm[b] = 0u - ((x >> b) & 1u);
    uint32_t beats = 0;
    for (int jw = jw0 + static_cast<int>(part); jw <= jw1; jw += static_cast<int>(parts)) {
        const uint32_t* P0 = planes + jw * nb;
        uint32_t gt0 = 0u, eq0 = 0xFFFFFFFFu;
#pragma unroll
        for (int b = 9; b >= 0; --b) {
            if (b < static_cast<int>(nb)) {
                const uint32_t B0 = P0[b], X = Xm[b];
                gt0 |= eq0 & B0 & ~X;
                eq0 &= ~(B0 ^ X);
            }
        }
        beats += window_beats(jw, c, lo, hi, gt0, eq0);
    }
    return beats;
}

// Local inhibition, uniform boost, by one warp with a wavelet matrix over the positions (any
// radius, O(C log range) per input instead of O(C * r)).  Values x' = x - xmin + 1 for the
// eligible columns (x >= r_lo), 0 otherwise, B = bits(xmax - xmin + 1) <= 8 levels.  For
// column c with window [lo, hi]:
//     beats(c) = #{d in [lo, hi] : x'_d > x'_c} + #{d in [lo, c) : x'_d == x'_c}
// from one descent through the levels tracking the positions lo, c and hi+1 (rank queries
// on per-level bit-vectors with per-word prefix counts).  emit(cw, word) gets the SDR words
// in order (warp-uniform).  Scratch: buf0, buf1 [C32] bytes; lv [B][ncw + 2] uint2 {bits, ones
// before} per word (entry ncw + 1: the level's zero count Z).
__device__ __forceinline__ uint32_t wm_rank2(const uint2* lvl, uint32_t p) {
    const uint2 e = lvl[p >> 5];
    return e.y + __popc(e.x & ((1u << (p & 31u)) - 1u));
}

// NI inputs of one warp at once (NI = 1 or 2; independent builds and descents interleave, so
// the latency of one input's chains hides behind the other's).  Input i: row[i], xmin[i];
// scratch buf0[i], buf1[i] [C32] bytes and lv[i] [B][ncw + 2] uint2; B = the largest of
// the inputs' level counts (extra top levels of the other input are all-zero partitions).
// emit(i, cw, word) gets input i's SDR words in order (warp-uniform).
template <int NI, typename RowT, typename Emit>
__device__ __forceinline__ void local_uniform_wavelet(const RowT* const* row, uint32_t C, uint32_t C32, uint32_t ncw,
                                                      uint32_t radius, uint32_t k, uint32_t r_lo,
                                                      const uint32_t* xmin, uint32_t B, uint8_t* const* buf0,
                                                      uint8_t* const* buf1, uint2* const* lv, uint32_t lane,
                                                      Emit emit) {
    const uint32_t stride = ncw + 2u;
    auto xval = [&](int i, uint32_t c) -> uint32_t {
        const uint32_t x = c < C ? static_cast<uint32_t>(row[i][c]) : 0u;
        return x >= r_lo ? x - xmin[i] + 1u : 0u;
    };
#pragma unroll
    for (int i = 0; i < NI; ++i)
        for (uint32_t c = lane; c < C32; c += 32u) buf0[i][c] = static_cast<uint8_t>(xval(i, c));
    __syncwarp();
    uint8_t* src[NI];
    uint8_t* dst[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) src[i] = buf0[i], dst[i] = buf1[i];
    for (int l = static_cast<int>(B) - 1; l >= 0; --l) {
        uint32_t ones[NI];
#pragma unroll
        for (int i = 0; i < NI; ++i) ones[i] = 0u;
#pragma unroll 4
        for (uint32_t j = 0; j < ncw; ++j) {
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                const uint32_t w = __ballot_sync(0xffffffffu, (src[i][j * 32u + lane] >> l) & 1u);
                if (lane == 0) lv[i][l * stride + j] = make_uint2(w, ones[i]);
                ones[i] += __popc(w);
            }
        }
        uint32_t Z[NI];
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            Z[i] = C32 - ones[i];
            if (lane == 0) lv[i][l * stride + ncw] = make_uint2(0u, ones[i]), lv[i][l * stride + ncw + 1u] = make_uint2(0u, Z[i]);
        }
        __syncwarp();
#pragma unroll 4
        for (uint32_t j = 0; j < ncw; ++j) {
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                const uint32_t c = j * 32u + lane;
                const uint32_t v = src[i][c];
                const uint2 e = lv[i][l * stride + j];
                const uint32_t r = e.y + __popc(e.x & ((1u << lane) - 1u));
                dst[i][((v >> l) & 1u) ? Z[i] + r : c - r] = static_cast<uint8_t>(v);
            }
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            uint8_t* t = src[i];
            src[i] = dst[i];
            dst[i] = t;
        }
    }
    const int R = static_cast<int>(radius), Cn = static_cast<int>(C);
    // beats of NQ columns per lane and input (independent descents interleave):
    //   greater + equal before c = (hi - lo) - less - (b - a) + (m - a)
    constexpr int NQ = NI == 1 ? 4 : 2;
    for (uint32_t cw0 = 0; cw0 < ncw; cw0 += NQ) {
        uint32_t x[NI][NQ], a[NI][NQ], m[NI][NQ], b[NI][NQ], lo[NQ], hi[NQ], less[NI][NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const uint32_t c = (cw0 + q) * 32u + lane;
            lo[q] = static_cast<uint32_t>(max(0, static_cast<int>(c) - R));
            hi[q] = static_cast<uint32_t>(min(Cn - 1, static_cast<int>(c) + R)) + 1u;
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                x[i][q] = cw0 + q < ncw ? xval(i, c) : 0u;
                a[i][q] = lo[q], m[i][q] = c, b[i][q] = hi[q], less[i][q] = 0u;
            }
        }
        for (int l = static_cast<int>(B) - 1; l >= 0; --l) {
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                const uint2* lvl = lv[i] + l * stride;
                const uint32_t Z = lvl[ncw + 1u].y;
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    const uint32_t ra = wm_rank2(lvl, a[i][q]), rm = wm_rank2(lvl, m[i][q]),
                                   rb = wm_rank2(lvl, b[i][q]);
                    if ((x[i][q] >> l) & 1u) {
                        less[i][q] += (b[i][q] - a[i][q]) - (rb - ra);
                        a[i][q] = Z + ra, m[i][q] = Z + rm, b[i][q] = Z + rb;
                    } else {
                        a[i][q] -= ra, m[i][q] -= rm, b[i][q] -= rb;
                    }
                }
            }
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            if (cw0 + q >= ncw) break;
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                const uint32_t beats = ((hi[q] - lo[q]) - less[i][q] - (b[i][q] - a[i][q])) + (m[i][q] - a[i][q]);
                emit(i, cw0 + q, __ballot_sync(0xffffffffu, x[i][q] > 0u && beats < k));
            }
        }
    }
    __syncwarp();
}

// ---- general boosts ---------------------------------------------------------------------
// Exact rank key (R4, R6): N = raw*Bc (exact), key = N << L | (2^L-1-c).
__device__ __forceinline__ uint64_t exact_key(uint32_t raw, uint32_t bc, uint32_t theta, uint32_t c,
                                              uint32_t L, uint64_t& N) {
    N = raw >= theta ? static_cast<uint64_t>(raw) * bc : 0ull;
    return (N << L) | (((1ull << L) - 1ull) - c);
}

// 16-bit coarse key of a column that passes cutoff and floor (N > 2^23 => u >= 1 for
// sh <= 23), 0 otherwise.  u is monotone in N, so u_d > u_c implies key_d > key_c.
__device__ __forceinline__ uint32_t coarse_u(uint32_t raw, uint32_t bc, uint32_t theta, uint32_t sh) {
    const uint64_t N = raw >= theta ? static_cast<uint64_t>(raw) * bc : 0ull;
    return N > (1ull << 23) ? static_cast<uint32_t>(N >> sh) : 0u;
}

// planes[cw * 16 + b] = bit b of u over the 32 columns of word cw
template <typename RowT>
__device__ __forceinline__ void build_coarse_planes(const RowT* row, const uint32_t* bc, uint32_t* planes,
                                                    uint32_t ncw, uint32_t theta, uint32_t sh,
                                                    uint32_t cw0, uint32_t step, uint32_t lane) {
    for (uint32_t cw = cw0; cw < ncw; cw += step) {
        const uint32_t c = cw * 32u + lane;
        const uint32_t u = coarse_u(row[c], bc[c], theta, sh);
#pragma unroll
        for (uint32_t b = 0; b < 16u; ++b) {
            const uint32_t pl = __ballot_sync(0xffffffffu, (u >> b) & 1u);
            if (lane == b) planes[cw * 16u + b] = pl;
        }
    }
}

// Local inhibition with per-column boosts: bit-sliced comparison of the coarse keys, then the
// exact keys only for the neighbours whose coarse key ties with c's (rare).
template <typename RowT>
__device__ __forceinline__ uint32_t local_general_word(const RowT* row, const uint32_t* bc,
                                                       const uint32_t* planes, uint32_t ncw,
                                                       uint32_t cw, uint32_t C, uint32_t radius,
                                                       uint32_t k, uint32_t theta, uint32_t sh,
                                                       uint32_t L, uint32_t lane) {
    const int c = static_cast<int>(cw * 32u + lane);
    const uint32_t u = coarse_u(row[c], bc[c], theta, sh);
    uint64_t Nc;
    const uint64_t keyc = exact_key(row[c], bc[c], theta, static_cast<uint32_t>(c), L, Nc);
    const int R = static_cast<int>(radius), Cn = static_cast<int>(C);
    const int lo = max(0, c - R), hi = min(Cn - 1, c + R);
    const int jw0 = max(0, (static_cast<int>(cw) * 32 - R) / 32);
    const int jw1 = min(static_cast<int>(ncw) - 1, (static_cast<int>(cw) * 32 + 31 + R) / 32);
    uint32_t Xm[16];
#pragma unroll
    for (int b = 0; b < 16; ++b) Xm[b] = 0u - ((u >> b) & 1u);
    uint32_t beats = 0;
    for (int jw = jw0; jw <= jw1; ++jw) {
        const uint32_t* P0 = planes + jw * 16;
        uint32_t gt = 0u, eq = 0xFFFFFFFFu;
#pragma unroll
        for (int b = 15; b >= 0; --b) {
            const uint32_t B = P0[b], X = Xm[b];
            gt |= eq & B & ~X;
            eq &= ~(B ^ X);
        }
        const int base = jw * 32;
        const int a = max(lo, base) - base, z = min(hi, base + 31) - base;
        uint32_t wm = a <= z ? (0xFFFFFFFFu >> (31 - z)) & (0xFFFFFFFFu << a) : 0u;
        const int self = c - base;
        if (self >= 0 && self < 32) wm &= ~(1u << self);
        beats += __popc(gt & wm);
        uint32_t ties = u > 0u ? (eq & wm) : 0u;  // same coarse key: compare exactly
        while (ties) {
            const int d = base + __ffs(ties) - 1;
            ties &= ties - 1u;
            uint64_t Nd;
            beats += exact_key(row[d], bc[d], theta, static_cast<uint32_t>(d), L, Nd) > keyc ? 1u : 0u;
        }
    }
    return __ballot_sync(0xffffffffu, c < Cn && u > 0u && beats < k);
}

// ---- local inhibition, per-column boosts, with a per-input coarse map ---------------------
// The coarse key is only an accelerator: exactness comes from the exact comparison of the
// columns whose coarse keys tie.  Mapping the eligible N onto 15 bits relative to the input's
// own range [Nmin, Nmax] (instead of a fixed shift) makes coarse ties rare, and a "lossless"
// flag (the dropped low bits are zero) resolves the common remaining case, equal N, by index
// alone (d beats c iff d < c): exact keys are compared only for ties involving a lossy column.
struct CoarseMap {
    uint64_t nlo;  // smallest eligible N, rounded down to a multiple of 2^sh
    uint32_t sh;   // right shift of N - nlo, so that u - 1 < 2^15
};

// umax_lim: largest u - 1 (32766: 15-bit keys; the per-warp wavelet may ask for fewer levels)
__device__ __forceinline__ CoarseMap coarse_map(uint64_t nmin, uint64_t nmax, uint32_t umax_lim = 32766u) {
    CoarseMap m{0ull, 0u};
    if (nmin > nmax) return m;  // no eligible column
    // nlo aligned to 2^sh: then "lossless" is N % 2^sh == 0, which holds for every column with a
    // boost of 1 (N = raw * 2^23) whenever sh <= 23, so equal-N ties stay index ties
    for (;; ++m.sh) {
        m.nlo = nmin & ~((1ull << m.sh) - 1ull);
        if (((nmax - m.nlo) >> m.sh) <= umax_lim) break;
    }
    return m;
}

// N of column c if it passes the cutoff and the floor (N > 2^23), else 0
__device__ __forceinline__ uint64_t eligible_N(uint32_t raw, uint32_t bc, uint32_t theta) {
    const uint64_t N = raw >= theta ? static_cast<uint64_t>(raw) * bc : 0ull;
    return N > (1ull << 23) ? N : 0ull;
}

// u in [1, 2^15] for eligible columns (0 otherwise) and whether the map dropped nonzero bits
__device__ __forceinline__ uint32_t coarse_u15(uint64_t N, const CoarseMap& m, bool& lossy) {
    if (N == 0ull) {
        lossy = false;
        return 0u;
    }
    const uint64_t d = N - m.nlo;
    lossy = (d & ((1ull << m.sh) - 1ull)) != 0ull;
    return static_cast<uint32_t>(d >> m.sh) + 1u;
}

__device__ __forceinline__ void minmax64_warp(uint64_t& mn, uint64_t& mx) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        const uint64_t a = __shfl_xor_sync(0xffffffffu, mn, d), b = __shfl_xor_sync(0xffffffffu, mx, d);
        mn = a < mn ? a : mn;
        mx = b > mx ? b : mx;
    }
}

// eligible-N range of words [w0, w1) by one warp (all lanes get the result)
template <typename RowT>
__device__ __forceinline__ CoarseMap coarse_map_warp(const RowT* row, const uint32_t* bc, uint32_t theta, uint32_t w0,
                                                     uint32_t w1, uint32_t lane, uint32_t umax_lim = 32766u) {
    uint64_t mn = ~0ull, mx = 0ull;
    for (uint32_t cw = w0; cw < w1; ++cw) {
        const uint32_t c = cw * 32u + lane;
        const uint64_t N = eligible_N(row[c], bc[c], theta);
        if (N) mn = N < mn ? N : mn, mx = N > mx ? N : mx;
    }
    minmax64_warp(mn, mx);
    return coarse_map(mn, mx, umax_lim);
}

// the same by the threads [0, nthr) of a CTA; s_mm[2] is shared scratch.  Contains barriers.
template <typename RowT>
__device__ __forceinline__ CoarseMap coarse_map_block(const RowT* row, const uint32_t* bc, uint32_t theta, uint32_t w0,
                                                      uint32_t w1, unsigned long long* s_mm) {
    const uint32_t tid = threadIdx.x, nthr = blockDim.x;
    if (tid == 0) s_mm[0] = ~0ull, s_mm[1] = 0ull;
    __syncthreads();
    uint64_t mn = ~0ull, mx = 0ull;
    for (uint32_t c = w0 * 32u + tid; c < w1 * 32u; c += nthr) {
        const uint64_t N = eligible_N(row[c], bc[c], theta);
        if (N) mn = N < mn ? N : mn, mx = N > mx ? N : mx;
    }
    minmax64_warp(mn, mx);
    if ((tid & 31u) == 0 && mn <= mx) {
        atomicMin(&s_mm[0], static_cast<unsigned long long>(mn));
        atomicMax(&s_mm[1], static_cast<unsigned long long>(mx));
    }
    __syncthreads();
    return coarse_map(s_mm[0], s_mm[1]);
}

// planes[cw*16 + 0] = lossy flags, planes[cw*16 + 1 + b] = bit b of u (b < 15)
template <typename RowT>
__device__ __forceinline__ void build_coarse_planes15(const RowT* row, const uint32_t* bc, uint32_t* planes,
                                                      uint32_t ncw, uint32_t theta, const CoarseMap& m,
                                                      uint32_t cw0, uint32_t step, uint32_t lane) {
    for (uint32_t cw = cw0; cw < ncw; cw += step) {
        const uint32_t c = cw * 32u + lane;
        bool lossy;
        const uint32_t u = coarse_u15(eligible_N(row[c], bc[c], theta), m, lossy);
        const uint32_t pl = __ballot_sync(0xffffffffu, lossy);
        if (lane == 0) planes[cw * 16u] = pl;
#pragma unroll
        for (uint32_t b = 0; b < 15u; ++b) {
            const uint32_t q = __ballot_sync(0xffffffffu, (u >> b) & 1u);
            if (lane == b + 1u) planes[cw * 16u + 1u + b] = q;
        }
    }
}

// Beats of lane's column of word cw (local inhibition, per-column boosts) over the neighbour
// words jw0+part, jw0+part+parts, ..; u_out = the column's coarse key (0: ineligible)
template <typename RowT>
__device__ __forceinline__ uint32_t local_general_beats15(const RowT* row, const uint32_t* bc, const uint32_t* planes,
                                                          uint32_t ncw, uint32_t cw, uint32_t C, uint32_t radius,
                                                          uint32_t theta, const CoarseMap& m, uint32_t L, uint32_t lane,
                                                          uint32_t part, uint32_t parts, uint32_t& u_out) {
    const int c = static_cast<int>(cw * 32u + lane);
    uint64_t Nc;
    const uint64_t keyc = exact_key(row[c], bc[c], theta, static_cast<uint32_t>(c), L, Nc);
    bool lossy_c;
    const uint32_t u = coarse_u15(Nc > (1ull << 23) ? Nc : 0ull, m, lossy_c);
    u_out = c < static_cast<int>(C) ? u : 0u;
    const int R = static_cast<int>(radius), Cn = static_cast<int>(C);
    const int lo = max(0, c - R), hi = min(Cn - 1, c + R);
    const int jw0 = max(0, (static_cast<int>(cw) * 32 - R) / 32);
    const int jw1 = min(static_cast<int>(ncw) - 1, (static_cast<int>(cw) * 32 + 31 + R) / 32);
    uint32_t Xm[15];
#pragma unroll
    for (int b = 0; b < 15; ++b) Xm[b] = 0u - ((u >> b) & 1u);
    uint32_t beats = 0;
    for (int jw = jw0 + static_cast<int>(part); jw <= jw1; jw += static_cast<int>(parts)) {
        const uint32_t* P0 = planes + jw * 16;
        uint32_t gt = 0u, eq = 0xFFFFFFFFu;
#pragma unroll
        for (int b = 14; b >= 0; --b) {
            const uint32_t B = P0[1 + b], X = Xm[b];
            gt |= eq & B & ~X;
            eq &= ~(B ^ X);
        }
        const int base = jw * 32;
        const int a = max(lo, base) - base, z = min(hi, base + 31) - base;
        uint32_t wm = a <= z ? (0xFFFFFFFFu >> (31 - z)) & (0xFFFFFFFFu << a) : 0u;
        const int self = c - base;
        if (self >= 0 && self < 32) wm &= ~(1u << self);
        beats += __popc(gt & wm);
        if (u > 0u) {
            const uint32_t ties = eq & wm;
            uint32_t exact = lossy_c ? ties : (ties & P0[0]);  // pairs with a lossy column
            uint32_t below = 0u;                                // bits d < c of this word
            if (self >= 32) below = 0xFFFFFFFFu;
            else if (self > 0) below = 0xFFFFFFFFu >> (32 - self);
            beats += __popc(ties & ~exact & below);             // equal N: the lower index wins
            while (exact) {
                const int d = base + __ffs(exact) - 1;
                exact &= exact - 1u;
                uint64_t Nd;
                beats += exact_key(row[d], bc[d], theta, static_cast<uint32_t>(d), L, Nd) > keyc ? 1u : 0u;
            }
        }
    }
    return beats;
}

// Local inhibition, per-column boosts, by one warp with a wavelet matrix over the positions (any
// radius; O(C log 2^15) per input instead of the comparator's O(C * r)).  Values: the coarse key
// u of coarse_map (0 for ineligible columns), stored as u << 1 | lossy, B = bits(max u) <= 15
// levels.  The descent of column c with window [lo, hi] gives #{d in window : u_d > u_c} (u is
// monotone in N, so these beat c) and the range [a, b) of the window's columns with u_d == u_c at
// the bottom level, stable in position ([a, m) are the ones with d < c).  Equal u between two
// lossless columns means equal N: the lower index wins, i.e. beats += m - a.  When the bottom-level
// bit-vector of the lossy flags shows a lossy column in [a, b) (c included), the ties of c are
// re-decided on the exact keys (rare: see coarse_map); the tied columns are read from the
// bottom-level positions recorded by the first pass (pos[m] = c).
// Scratch: buf0, buf1 [C32] uint16; lv [B + 1][ncw + 2] uint2 {bits, ones before} per word
// (level B: lossy flags; entry ncw + 1 holds the level's zero count Z).
template <typename RowT, typename Emit>
__device__ __forceinline__ void local_general_wavelet(const RowT* row, const uint32_t* bc, uint32_t C, uint32_t C32,
                                                      uint32_t ncw, uint32_t radius, uint32_t k, uint32_t theta,
                                                      uint32_t L, const CoarseMap& cm, uint16_t* buf0,
                                                      uint16_t* buf1, uint2* lv, uint32_t lane, Emit emit) {
    const uint32_t stride = ncw + 2u;
    auto sval = [&](uint32_t c) -> uint32_t {  // u << 1 | lossy (0: ineligible or pad column)
        if (c >= C) return 0u;
        bool lossy;
        const uint32_t u = coarse_u15(eligible_N(row[c], bc[c], theta), cm, lossy);
        return u ? (u << 1) | (lossy ? 1u : 0u) : 0u;
    };
    uint32_t umax = 0;
    for (uint32_t i = lane; i < C32; i += 32u) {
        const uint32_t v = sval(i);
        buf0[i] = static_cast<uint16_t>(v);
        umax = max(umax, v >> 1);
    }
    umax = __reduce_max_sync(0xffffffffu, umax);
    const uint32_t B = umax ? 32u - __clz(umax) : 1u;
    __syncwarp();
    uint16_t* src = buf0;
    uint16_t* dst = buf1;
    // level l partitions on bit l of u (bit l + 1 of the stored value); level B: the lossy bit
    for (int l = static_cast<int>(B) - 1; l >= -1; --l) {
        uint2* lvl = lv + (l >= 0 ? l : static_cast<int>(B)) * stride;
        const uint32_t sb = static_cast<uint32_t>(l + 1);
        uint32_t ones = 0;
#pragma unroll 8
        for (uint32_t j = 0; j < ncw; ++j) {
            const uint32_t w = __ballot_sync(0xffffffffu, (src[j * 32u + lane] >> sb) & 1u);
            if (lane == 0) lvl[j] = make_uint2(w, ones);
            ones += __popc(w);
        }
        const uint32_t Z = C32 - ones;
        if (lane == 0) lvl[ncw] = make_uint2(0u, ones), lvl[ncw + 1u] = make_uint2(0u, Z);
        __syncwarp();
        if (l < 0) break;
#pragma unroll 8
        for (uint32_t j = 0; j < ncw; ++j) {
            const uint32_t i = j * 32u + lane;
            const uint32_t v = src[i];
            const uint2 e = lvl[j];
            const uint32_t r = e.y + __popc(e.x & ((1u << lane) - 1u));
            dst[((v >> sb) & 1u) ? Z + r : i - r] = static_cast<uint16_t>(v);
        }
        __syncwarp();
        uint16_t* t = src;
        src = dst;
        dst = t;
    }
    const int R = static_cast<int>(radius), Cn = static_cast<int>(C);
    const uint2* lvL = lv + B * stride;
    auto window_of = [&](uint32_t c, uint32_t& lo, uint32_t& hi) {
        lo = static_cast<uint32_t>(max(0, static_cast<int>(c) - R));
        hi = static_cast<uint32_t>(min(Cn - 1, static_cast<int>(c) + R)) + 1u;
    };
    // pass 1: beats by the index rule for equal u (buf0[c], bit 15 = a lossy column among c's
    // ties; 0x7FFF = ineligible) and the bottom-level position of every eligible column
    // (buf1[m] = c), which lists the tied columns of pass 2.  NQ columns per lane descend
    // together (independent shared-memory chains).
    uint16_t* beats_s = buf0;
    uint16_t* pos_s = buf1;
    constexpr int NQ = 4;
    for (uint32_t cw0 = 0; cw0 < ncw; cw0 += NQ) {
        uint32_t c[NQ], u[NQ], a[NQ], m[NQ], b[NQ], lo[NQ], hi[NQ], less[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            c[q] = (cw0 + q) * 32u + lane;
            u[q] = cw0 + q < ncw ? sval(c[q]) >> 1 : 0u;
            window_of(c[q], lo[q], hi[q]);
            a[q] = lo[q], m[q] = c[q], b[q] = hi[q], less[q] = 0u;
        }
        for (int l = static_cast<int>(B) - 1; l >= 0; --l) {
            const uint2* lvl = lv + l * stride;
            const uint32_t Z = lvl[ncw + 1u].y;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const uint32_t ra = wm_rank2(lvl, a[q]), rm = wm_rank2(lvl, m[q]), rb = wm_rank2(lvl, b[q]);
                if ((u[q] >> l) & 1u) {
                    less[q] += (b[q] - a[q]) - (rb - ra);
                    a[q] = Z + ra, m[q] = Z + rm, b[q] = Z + rb;
                } else {
                    a[q] -= ra, m[q] -= rm, b[q] -= rb;
                }
            }
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            if (cw0 + q >= ncw) break;
            uint16_t out = 0x7FFFu;
            if (u[q]) {
                const uint32_t beats = ((hi[q] - lo[q]) - less[q] - (b[q] - a[q])) + (m[q] - a[q]);
                const bool fix = b[q] - a[q] > 1u && wm_rank2(lvL, b[q]) != wm_rank2(lvL, a[q]);
                out = static_cast<uint16_t>(beats | (fix ? 0x8000u : 0u));
                pos_s[m[q]] = static_cast<uint16_t>(c[q]);
            }
            beats_s[c[q]] = out;
        }
    }
    __syncwarp();
    // pass 2: ties involving a lossy column re-decided on the exact keys (rare): sum over the
    // tied d of [key_d > key_c] - [d < c] (the index rule counted the latter)
    for (uint32_t cw = 0; cw < ncw; ++cw) {
        const uint32_t c = cw * 32u + lane;
        const uint32_t v = beats_s[c];
        int beats = static_cast<int>(v & 0x7FFFu);
        if (v & 0x8000u) {
            const uint64_t Nc = eligible_N(row[c], bc[c], theta);
            bool lossy_c;
            const uint32_t uc = coarse_u15(Nc, cm, lossy_c);
            const uint64_t keyc = (Nc << L) | (((1ull << L) - 1ull) - c);
            uint32_t lo, hi;
            window_of(c, lo, hi);
            uint32_t a = lo, m = c, b = hi;
            for (int l = static_cast<int>(B) - 1; l >= 0; --l) {
                const uint2* lvl = lv + l * stride;
                const uint32_t ra = wm_rank2(lvl, a), rm = wm_rank2(lvl, m), rb = wm_rank2(lvl, b);
                if ((uc >> l) & 1u) {
                    const uint32_t Z = lvl[ncw + 1u].y;
                    a = Z + ra, m = Z + rm, b = Z + rb;
                } else {
                    a -= ra, m -= rm, b -= rb;
                }
            }
            for (uint32_t q = a; q < b; ++q) {
                const uint32_t d = pos_s[q];
                if (d == c) continue;
                const uint64_t Nd = eligible_N(row[d], bc[d], theta);
                bool lossy_d;
                coarse_u15(Nd, cm, lossy_d);
                if (lossy_c || lossy_d) {
                    const uint64_t keyd = (Nd << L) | (((1ull << L) - 1ull) - d);
                    beats += (keyd > keyc ? 1 : 0) - (d < c ? 1 : 0);
                }
            }
        }
        emit(cw, __ballot_sync(0xffffffffu, v != 0x7FFFu && beats < static_cast<int>(k)));
    }
    __syncwarp();
}

// Winners of word cw (local inhibition, per-column boosts), all lanes of the warp call it.
template <typename RowT>
__device__ __forceinline__ uint32_t local_general_word15(const RowT* row, const uint32_t* bc,
                                                         const uint32_t* planes, uint32_t ncw, uint32_t cw,
                                                         uint32_t C, uint32_t radius, uint32_t k, uint32_t theta,
                                                         const CoarseMap& m, uint32_t L, uint32_t lane) {
    uint32_t u;
    const uint32_t beats = local_general_beats15(row, bc, planes, ncw, cw, C, radius, theta, m, L, lane, 0u, 1u, u);
    return __ballot_sync(0xffffffffu, u > 0u && beats < k);
}

// ---- global inhibition by a whole CTA (cluster learning) ---------------------------------
// Exact k-winners over all C columns (R4-R7): a two-level radix select of the k-th largest
// 15-bit coarse key u (histograms of (u-1) >> 7, then of (u-1) & 127 inside the bucket, shared
// atomics), then the columns tied at the threshold Tu: if none of them is lossy they all have
// the same N and the lowest indices win (a prefix count over the tie masks); otherwise the
// need-th largest exact key T2 among them is found (a tie list, or a bitwise search with CTA
// counts when the list overflows).  Every thread of the CTA must call it (barriers);
// C <= 4 * blockDim.x.  scratch: >= 400 + 2*ncw + 1 words; ties: tie_cap keys.
struct GlobalSel {
    uint32_t Tu;     // coarse threshold (0: fewer than k eligible columns, all eligible win)
    uint32_t need;   // winners among the columns with u == Tu
    uint32_t exact;  // 1: decide the tied columns by exact key >= T2, 0: by index rank
    uint64_t T2;
};

template <typename RowT>
__device__ __forceinline__ GlobalSel global_select_cta(const RowT* row, const uint32_t* bc, uint32_t theta, uint32_t C,
                                                       uint32_t ncw, uint32_t k, uint32_t L, uint32_t keyBits,
                                                       const CoarseMap& m, uint32_t* scratch, uint64_t* ties,
                                                       uint32_t tie_cap) {
    const uint32_t tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31u, wi = tid >> 5, nw = nthr >> 5;
    uint32_t* h1 = scratch;            // [256]
    uint32_t* h2 = scratch + 256;      // [128]
    uint32_t* misc = scratch + 384;    // [16]
    uint32_t* tmask = scratch + 400;   // [ncw]
    uint32_t* tscan = tmask + ncw;     // [ncw + 1]
    for (uint32_t i = tid; i < 400u; i += nthr) scratch[i] = 0u;
    // the coarse keys of this thread's columns (c = tid + j*nthr), kept for both histograms
    constexpr int kMaxPer = 4;  // C <= 4 * blockDim.x (cluster learning: C32 <= 2048, 512 threads)
    uint32_t uc[kMaxPer];
#pragma unroll
    for (int j = 0; j < kMaxPer; ++j) {
        const uint32_t c = tid + j * nthr;
        bool lossy;
        uc[j] = c < C ? coarse_u15(eligible_N(row[c], bc[c], theta), m, lossy) : 0u;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kMaxPer; ++j)
        if (uc[j]) atomicAdd(&h1[(uc[j] - 1u) >> 7], 1u);
    __syncthreads();
    if (wi == 0) {  // bucket of the k-th largest: suffix counts from the top, 8 bins per lane
        uint32_t v[8], sum = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = h1[lane * 8u + j], sum += v[j];
        uint32_t above = sum;  // inclusive suffix over lanes >= lane
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_down_sync(0xffffffffu, above, d);
            if (lane + d < 32u) above += o;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, above, 0);
        // bin b = 8*lane + j: count of bins > b = (above - sum) + sum of v[j+1..7]
        uint32_t hi_above = above - sum, found = 0xFFFFFFFFu, f_above = 0;
#pragma unroll
        for (int j = 7; j >= 0; --j) {
            if (found == 0xFFFFFFFFu && hi_above < k && hi_above + v[j] >= k) found = lane * 8u + j, f_above = hi_above;
            hi_above += v[j];
        }
        const uint32_t who = __ballot_sync(0xffffffffu, found != 0xFFFFFFFFu);
        if (lane == 0) misc[0] = total;
        if (who && lane == static_cast<uint32_t>(__ffs(who) - 1)) misc[1] = found, misc[2] = f_above;
    }
    __syncthreads();
    GlobalSel r{0u, 0u, 0u, 0ull};
    if (misc[0] < k) return r;  // fewer than k eligible: all of them win (Tu = 0)
    const uint32_t B1 = misc[1], above1 = misc[2];
#pragma unroll
    for (int j = 0; j < kMaxPer; ++j)
        if (uc[j] && ((uc[j] - 1u) >> 7) == B1) atomicAdd(&h2[(uc[j] - 1u) & 127u], 1u);
    __syncthreads();
    if (wi == 0) {
        const uint32_t kk = k - above1;
        uint32_t v[4], sum = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = h2[lane * 4u + j], sum += v[j];
        uint32_t above = sum;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_down_sync(0xffffffffu, above, d);
            if (lane + d < 32u) above += o;
        }
        uint32_t hi_above = above - sum, found = 0xFFFFFFFFu, f_above = 0;
#pragma unroll
        for (int j = 3; j >= 0; --j) {
            if (found == 0xFFFFFFFFu && hi_above < kk && hi_above + v[j] >= kk) found = lane * 4u + j, f_above = hi_above;
            hi_above += v[j];
        }
        const uint32_t who = __ballot_sync(0xffffffffu, found != 0xFFFFFFFFu);
        if (who && lane == static_cast<uint32_t>(__ffs(who) - 1)) {
            misc[3] = ((B1 << 7) | found) + 1u;  // Tu
            misc[4] = kk - f_above;              // need (>= 1)
        }
        if (lane == 0) misc[5] = 0u, misc[6] = 0u;  // lossy-tie flag, tie count
    }
    __syncthreads();
    r.Tu = misc[3];
    r.need = misc[4];
    // the columns tied at Tu: masks per word, lossy flag, and their exact keys (list)
    for (uint32_t cw = wi; cw < ncw; cw += nw) {
        const uint32_t c = cw * 32u + lane;
        bool lossy = false;
        uint64_t N = 0;
        const uint64_t key = c < C ? exact_key(row[c], bc[c], theta, c, L, N) : 0ull;
        const uint32_t u = c < C ? coarse_u15(N > (1ull << 23) ? N : 0ull, m, lossy) : 0u;
        const bool tied = u == r.Tu;
        const uint32_t tm = __ballot_sync(0xffffffffu, tied);
        if (lane == 0) tmask[cw] = tm;
        if (__any_sync(0xffffffffu, tied && lossy) && lane == 0) atomicOr(&misc[5], 1u);
        if (tied) {
            const uint32_t pos = atomicAdd(&misc[6], 1u);
            if (pos < tie_cap) ties[pos] = key;
        }
    }
    __syncthreads();
    r.exact = misc[5];
    if (!r.exact) {
        if (wi == 0) {  // exclusive scan of the tie counts per word
            uint32_t carry = 0;
            for (uint32_t base = 0; base < ncw; base += 32u) {
                const uint32_t cw = base + lane;
                const uint32_t v = cw < ncw ? __popc(tmask[cw]) : 0u;
                uint32_t x = v;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t o = __shfl_up_sync(0xffffffffu, x, d);
                    if (lane >= static_cast<uint32_t>(d)) x += o;
                }
                if (cw < ncw) tscan[cw] = carry + x - v;
                carry += __shfl_sync(0xffffffffu, x, 31);
            }
        }
        __syncthreads();
        return r;
    }
    const uint32_t nt = misc[6];
    if (nt <= tie_cap) {
        // T2 = the need-th largest tied key: the one with exactly need-1 larger ones (distinct)
        for (uint32_t i = tid; i < nt; i += nthr) {
            const uint64_t ki = ties[i];
            uint32_t g = 0;
            for (uint32_t j = 0; j < nt; ++j) g += ties[j] > ki ? 1u : 0u;
            if (g + 1u == r.need) misc[8] = static_cast<uint32_t>(ki), misc[9] = static_cast<uint32_t>(ki >> 32);
        }
    } else {
        // bitwise search over the tied columns in place, CTA counts (rare: many lossy ties)
        uint64_t T2 = 0;
        for (int bit = static_cast<int>(keyBits) - 1; bit >= 0; --bit) {
            const uint64_t cand = T2 | (1ull << bit);
            uint32_t cnt = 0;
            for (uint32_t c = tid; c < C; c += nthr) {
                if (!((tmask[c >> 5] >> (c & 31u)) & 1u)) continue;
                uint64_t N;
                cnt += exact_key(row[c], bc[c], theta, c, L, N) >= cand ? 1u : 0u;
            }
            cnt = __reduce_add_sync(0xffffffffu, cnt);
            if (tid == 0) misc[10] = 0u;
            __syncthreads();
            if (lane == 0 && cnt) atomicAdd(&misc[10], cnt);
            __syncthreads();
            if (misc[10] >= r.need) T2 = cand;
            __syncthreads();
        }
        if (tid == 0) misc[8] = static_cast<uint32_t>(T2), misc[9] = static_cast<uint32_t>(T2 >> 32);
    }
    __syncthreads();
    r.T2 = (static_cast<uint64_t>(misc[9]) << 32) | misc[8];
    return r;
}

// Global k-winners with a uniform boost by a whole CTA: a histogram of the eligible raw counts
// (shared atomics), one warp scans it from the top for r* (the k-th largest raw); the winners
// are raw > r* plus the first `need` columns (by index) with raw == r* (R6, R7).  Every thread
// of the CTA calls it (barriers).  hist: >= S + 4 words of shared scratch.
struct UniformSel {
    uint32_t rgt;   // raw >= rgt wins outright
    uint32_t rtie;  // raw == rtie wins for the `need` lowest indices (0xFFFFFFFF: none)
    uint32_t need;
};

template <typename RowT>
__device__ __forceinline__ UniformSel global_uniform_cta(const RowT* row, uint32_t C, uint32_t S, uint32_t k,
                                                         uint32_t r_lo, uint32_t* hist) {
    const uint32_t tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31u;
    uint32_t* misc = hist + S + 1u;  // [3]
    for (uint32_t v = tid; v <= S; v += nthr) hist[v] = 0u;
    __syncthreads();
    for (uint32_t c = tid; c < C; c += nthr) {
        const uint32_t x = row[c];
        if (x >= r_lo) atomicAdd(&hist[x], 1u);
    }
    __syncthreads();
    if (tid < 32u) {
        // lane owns bins [lane*per, (lane+1)*per); suffix counts from the top
        const uint32_t per = (S + 32u) / 32u;
        uint32_t sum = 0;
        for (uint32_t j = 0; j < per; ++j) {
            const uint32_t v = lane * per + j;
            sum += v <= S ? hist[v] : 0u;
        }
        uint32_t above = sum;  // inclusive suffix over lanes >= lane
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_down_sync(0xffffffffu, above, d);
            if (lane + d < 32u) above += o;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, above, 0);
        uint32_t hi_above = above - sum, found = 0xFFFFFFFFu, f_above = 0;
        for (int j = static_cast<int>(per) - 1; j >= 0; --j) {
            const uint32_t v = lane * per + static_cast<uint32_t>(j);
            const uint32_t h = v <= S ? hist[v] : 0u;
            if (found == 0xFFFFFFFFu && hi_above < k && hi_above + h >= k) found = v, f_above = hi_above;
            hi_above += h;
        }
        const uint32_t who = __ballot_sync(0xffffffffu, found != 0xFFFFFFFFu);
        if (total < k) {  // fewer than k eligible: all of them win
            if (lane == 0) misc[0] = r_lo, misc[1] = 0xFFFFFFFFu, misc[2] = 0u;
        } else if (who && lane == static_cast<uint32_t>(__ffs(who) - 1)) {
            misc[0] = found + 1u, misc[1] = found, misc[2] = k - f_above;
        }
    }
    __syncthreads();
    return UniformSel{misc[0], misc[1], misc[2]};
}

// SDR word gcw from a UniformSel (all lanes of a warp call it)
template <typename RowT>
__device__ __forceinline__ uint32_t global_uniform_word_sel(const RowT* row, uint32_t C, uint32_t gcw,
                                                            const UniformSel& u, uint32_t lane) {
    uint32_t before = 0;  // ties at raw == rtie in lower column-words
#pragma unroll 8
    for (uint32_t d = lane; d < gcw * 32u; d += 32u) before += row[d] == u.rtie ? 1u : 0u;
    before = __reduce_add_sync(0xffffffffu, before);
    const uint32_t c = gcw * 32u + lane;
    const uint32_t r = c < C ? static_cast<uint32_t>(row[c]) : 0u;
    const uint32_t tb = __ballot_sync(0xffffffffu, r == u.rtie && c < C);
    return __ballot_sync(0xffffffffu, c < C && (r >= u.rgt ||
                                                (r == u.rtie && before + __popc(tb & ((1u << lane) - 1u)) < u.need)));
}

// SDR word cw from a GlobalSel (all lanes of a warp call it)
template <typename RowT>
__device__ __forceinline__ uint32_t global_select_word(const RowT* row, const uint32_t* bc, uint32_t theta, uint32_t C,
                                                       uint32_t cw, uint32_t L, const CoarseMap& m, const GlobalSel& r,
                                                       const uint32_t* scratch, uint32_t ncw, uint32_t lane) {
    const uint32_t c = cw * 32u + lane;
    uint64_t N = 0;
    const uint64_t key = c < C ? exact_key(row[c], bc[c], theta, c, L, N) : 0ull;
    bool lossy;
    const uint32_t u = c < C ? coarse_u15(N > (1ull << 23) ? N : 0ull, m, lossy) : 0u;
    bool win;
    if (r.Tu == 0u) {
        win = u > 0u;
    } else if (u != r.Tu) {
        win = u > r.Tu;
    } else if (r.exact) {
        win = key >= r.T2;
    } else {
        const uint32_t* tmask = scratch + 400;
        const uint32_t* tscan = tmask + ncw;
        win = tscan[cw] + __popc(tmask[cw] & ((1u << lane) - 1u)) < r.need;
    }
    return __ballot_sync(0xffffffffu, c < C && win);
}

// r_lo = smallest raw passing both the cutoff (raw >= theta) and the floor raw*Bc > 2^23.
__device__ __forceinline__ uint32_t uniform_r_lo(uint32_t theta, uint32_t bc) {
    return max(theta, (1u << 23) / bc + 1u);
}

// ---- global inhibition (r = 0), one warp ------------------------------------------------
// Uniform boost (R6, R7): the key order is (raw desc, index asc) and the floor is raw >= r_lo,
// so the k winners are: raw >= rgt, plus the first `need` columns (by index) with
// raw == rtie.  r* = largest r with #{raw >= max(r, r_lo)} >= k, by a bitwise search over
// the raw bits; the counts come from raw values packed two per half2 (exact: raw <= 1023)
// with HSET2/HADD2 (no atomics, no block barrier).  NH half2 registers cover 64*NH columns.
template <int NH, typename RowT>
__device__ __forceinline__ void global_uniform_threshold(const RowT* row, uint32_t C32, uint32_t S,
                                                         uint32_t k, uint32_t r_lo, uint32_t lane,
                                                         uint32_t& rgt, uint32_t& rtie,
                                                         uint32_t& need) {
    __half2 hr[NH];
#pragma unroll
    for (int t = 0; t < NH; ++t) {
        const uint32_t ca = (2u * t) * 32u + lane, cb = ca + 32u;
        uint32_t ra = ca < C32 ? static_cast<uint32_t>(row[ca]) : 0u;
        uint32_t rb = cb < C32 ? static_cast<uint32_t>(row[cb]) : 0u;
        ra = ra >= r_lo ? ra : 0u;
        rb = rb >= r_lo ? rb : 0u;
        hr[t] = __halves2half2(__uint2half_rn(ra), __uint2half_rn(rb));
    }
    auto count_ge = [&](uint32_t x) -> uint32_t {
        const __half2 hx = __half2half2(__uint2half_rn(x));
        __half2 acc0 = __float2half2_rn(0.0f), acc1 = acc0;  // two chains (ILP)
#pragma unroll
        for (int t = 0; t < NH; t += 2) {
            acc0 = __hadd2(acc0, __hge2(hr[t], hx));
            if (t + 1 < NH) acc1 = __hadd2(acc1, __hge2(hr[t + 1], hx));
        }
        const __half2 acc = __hadd2(acc0, acc1);
        const uint32_t mine = static_cast<uint32_t>(__low2float(acc) + __high2float(acc));
        return __reduce_add_sync(0xffffffffu, mine);
    };
    rgt = r_lo;  // raw >= rgt wins outright
    rtie = 0xFFFFFFFFu;
    need = 0;
    if (count_ge(r_lo) >= k) {
        uint32_t T = 0;
        for (int bit = 31 - __clz(S); bit >= 0; --bit)
            if (count_ge(T | (1u << bit)) >= k) T |= 1u << bit;
        rtie = T;
        need = k - count_ge(T + 1u);
        rgt = T + 1u;
    }
}

// SDR words of one input (global, uniform boost) from its threshold (rgt, rtie, need): lane j
// builds words j, j+32, .. from its own 32 raw counts (four conflict-free LDS.128: the 16-byte
// chunks are visited in a lane-rotated order), so there is no chain across words; the `need`
// lowest-index columns with raw == rtie win through a warp scan of the per-word tie counts.
// store(w, word) gets every word once (lane-parallel, coalesced); returns the winner count
// (all lanes).  row: 16-byte aligned uint16 counts [ncw * 32].
template <typename Store>
__device__ __forceinline__ uint32_t uniform_sdr_words(const uint16_t* row, uint32_t ncw, uint32_t rgt,
                                                      uint32_t rtie, uint32_t need, uint32_t lane, Store store) {
    uint32_t total = 0, carry = 0;
    for (uint32_t j0 = 0; j0 < ncw; j0 += 32u) {
        const uint32_t j = j0 + lane;
        uint32_t win = 0, tie = 0;
        if (j < ncw) {
#pragma unroll
            for (uint32_t q = 0; q < 4u; ++q) {
                const uint32_t qq = (q + (lane >> 1)) & 3u;
                const uint4 v = *reinterpret_cast<const uint4*>(row + 32u * j + 8u * qq);
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (uint32_t e = 0; e < 4u; ++e) {
                    const uint32_t lo = w[e] & 0xFFFFu, hi = w[e] >> 16;
                    const uint32_t sh = 8u * qq + 2u * e;
                    win |= (lo >= rgt ? 1u : 0u) << sh | (hi >= rgt ? 2u : 0u) << sh;
                    tie |= (lo == rtie ? 1u : 0u) << sh | (hi == rtie ? 2u : 0u) << sh;
                }
            }
        }
        const uint32_t tc = __popc(tie);
        uint32_t incl = tc;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
            if (static_cast<int>(lane) >= d) incl += y;
        }
        const uint32_t before = carry + incl - tc;
        uint32_t grant = need > before ? min(need - before, tc) : 0u;
        while (grant--) {
            win |= tie & (0u - tie);  // lowest remaining tie
            tie &= tie - 1u;
        }
        if (j < ncw) store(j, win);
        total += __reduce_add_sync(0xffffffffu, __popc(win));
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    return total;
}

// The same for two inputs at once (rows a and b): two independent count chains per step, so
// the latency of one search hides behind the other's (a warp's two inputs of the batched top-k).
template <int NH, typename RowT>
__device__ __forceinline__ void global_uniform_threshold2(const RowT* ra_row, const RowT* rb_row, uint32_t C32,
                                                          uint32_t S, uint32_t k, uint32_t r_lo, uint32_t lane,
                                                          uint32_t rgt[2], uint32_t rtie[2], uint32_t need[2]) {
    __half2 ha[NH], hb[NH];
#pragma unroll
    for (int t = 0; t < NH; ++t) {
        const uint32_t ca = (2u * t) * 32u + lane, cb = ca + 32u;
        uint32_t a0 = ca < C32 ? static_cast<uint32_t>(ra_row[ca]) : 0u;
        uint32_t a1 = cb < C32 ? static_cast<uint32_t>(ra_row[cb]) : 0u;
        uint32_t b0 = ca < C32 ? static_cast<uint32_t>(rb_row[ca]) : 0u;
        uint32_t b1 = cb < C32 ? static_cast<uint32_t>(rb_row[cb]) : 0u;
        a0 = a0 >= r_lo ? a0 : 0u;
        a1 = a1 >= r_lo ? a1 : 0u;
        b0 = b0 >= r_lo ? b0 : 0u;
        b1 = b1 >= r_lo ? b1 : 0u;
        ha[t] = __halves2half2(__uint2half_rn(a0), __uint2half_rn(a1));
        hb[t] = __halves2half2(__uint2half_rn(b0), __uint2half_rn(b1));
    }
    auto count_ge2 = [&](uint32_t xa, uint32_t xb, uint32_t& na, uint32_t& nb) {
        const __half2 hxa = __half2half2(__uint2half_rn(xa)), hxb = __half2half2(__uint2half_rn(xb));
        __half2 va[NH], vb[NH];
#pragma unroll
        for (int t = 0; t < NH; ++t) va[t] = __hge2(ha[t], hxa), vb[t] = __hge2(hb[t], hxb);
#pragma unroll
        for (int d = 1; d < NH; d <<= 1)  // pairwise tree: log2(NH) dependent adds, not NH/2
#pragma unroll
            for (int t = 0; t + d < NH; t += 2 * d) va[t] = __hadd2(va[t], va[t + d]), vb[t] = __hadd2(vb[t], vb[t + d]);
        const __half2 sa = va[0], sb = vb[0];
        na = __reduce_add_sync(0xffffffffu, static_cast<uint32_t>(__low2float(sa) + __high2float(sa)));
        nb = __reduce_add_sync(0xffffffffu, static_cast<uint32_t>(__low2float(sb) + __high2float(sb)));
    };
    uint32_t na, nb;
    count_ge2(r_lo, r_lo, na, nb);
    const bool sa = na >= k, sb = nb >= k;  // else: every eligible column wins
    uint32_t Ta = 0, Tb = 0;
    for (int bit = 31 - __clz(S); bit >= 0; --bit) {
        count_ge2(Ta | (1u << bit), Tb | (1u << bit), na, nb);
        if (na >= k) Ta |= 1u << bit;
        if (nb >= k) Tb |= 1u << bit;
    }
    count_ge2(Ta + 1u, Tb + 1u, na, nb);
    rgt[0] = sa ? Ta + 1u : r_lo;
    rtie[0] = sa ? Ta : 0xFFFFFFFFu;
    need[0] = sa ? k - na : 0u;
    rgt[1] = sb ? Tb + 1u : r_lo;
    rtie[1] = sb ? Tb : 0xFFFFFFFFu;
    need[1] = sb ? k - nb : 0u;
}

// Per-column boosts (R4, R6): (1) the k-th largest 16-bit coarse key u = N >> sh (Tu) by a
// bitwise search over keys packed two per register (columns 64t+lane, 64t+32+lane);
// (2) the exact key threshold T2 among the columns tied at u == Tu (a 64-entry list in
// tie_list, else an in-place search).  Column c wins iff N > 2^23 and
// (Tu == 0 ? u > 0 : u > Tu || (u == Tu && key >= T2)) — see global_general_wins.
template <int NU, typename RowT>
__device__ __forceinline__ void global_general_threshold(const RowT* row, const uint32_t* bc,
                                                         uint32_t C32, uint32_t ncw, uint32_t k,
                                                         uint32_t theta, uint32_t sh, uint32_t L,
                                                         uint32_t keyBits, uint64_t* tie_list,
                                                         uint32_t lane, uint32_t& Tu, uint64_t& T2) {
    Tu = 0;
    T2 = 0;
    uint32_t uu[NU];
#pragma unroll
    for (int t = 0; t < NU; ++t) {
        const uint32_t ca = (2u * t) * 32u + lane, cb = ca + 32u;
        uint64_t Na = 0, Nb = 0;
        if (ca < C32) exact_key(row[ca], bc[ca], theta, ca, L, Na);
        if (cb < C32) exact_key(row[cb], bc[cb], theta, cb, L, Nb);
        uu[t] = static_cast<uint32_t>(Na >> sh) | (static_cast<uint32_t>(Nb >> sh) << 16);
    }
    for (int bit = 15; bit >= 0; --bit) {
        const uint32_t cand = (Tu | (1u << bit)) << 16;
        uint32_t cnt0 = 0, cnt1 = 0;
#pragma unroll
        for (int t = 0; t < NU; ++t) {
            cnt0 += uu[t] >= cand ? 1u : 0u;
            cnt1 += (uu[t] << 16) >= cand ? 1u : 0u;
        }
        if (__reduce_add_sync(0xffffffffu, cnt0 + cnt1) >= k) Tu |= 1u << bit;
    }
    if (Tu == 0) return;
    // columns above the coarse threshold, and the exact keys of the columns tied at Tu
    uint32_t ngt = 0, nties = 0;
    for (uint32_t cw = 0; cw < ncw; ++cw) {
        const uint32_t c = cw * 32u + lane;
        uint64_t N;
        const uint64_t key = exact_key(row[c], bc[c], theta, c, L, N);
        const uint32_t u = static_cast<uint32_t>(N >> sh);
        ngt += u > Tu ? 1u : 0u;
        const uint32_t tie = __ballot_sync(0xffffffffu, u == Tu);
        const uint32_t pos = nties + __popc(tie & ((1u << lane) - 1u));
        if (u == Tu && pos < 64u) tie_list[pos] = key;
        nties += __popc(tie);
    }
    ngt = __reduce_add_sync(0xffffffffu, ngt);
    const uint32_t need = k - ngt;  // 1 <= need <= nties by construction of Tu
    __syncwarp();
    if (nties <= 64u) {
        // T2 = the need-th largest tied key: the one with exactly need-1 larger tied keys
        // (keys are distinct: they carry the column index)
        const uint64_t k0 = lane < nties ? tie_list[lane] : 0ull;
        const uint64_t k1 = lane + 32u < nties ? tie_list[lane + 32u] : 0ull;
        uint32_t g0 = 0, g1 = 0;
        for (uint32_t j = 0; j < nties; ++j) {
            const uint64_t kj = tie_list[j];
            g0 += kj > k0 ? 1u : 0u;
            g1 += kj > k1 ? 1u : 0u;
        }
        const bool h0 = lane < nties && g0 + 1u == need, h1 = lane + 32u < nties && g1 + 1u == need;
        const uint32_t src = __ffs(__ballot_sync(0xffffffffu, h0 || h1)) - 1u;
        const uint64_t mine = h0 ? k0 : k1;
        const uint32_t lo = __shfl_sync(0xffffffffu, static_cast<uint32_t>(mine), src);
        const uint32_t hi = __shfl_sync(0xffffffffu, static_cast<uint32_t>(mine >> 32), src);
        T2 = (static_cast<uint64_t>(hi) << 32) | lo;
    } else {  // many ties: bitwise search over all tied columns in place
        for (int bit = static_cast<int>(keyBits) - 1; bit >= 0; --bit) {
            const uint64_t cand = T2 | (1ull << bit);
            uint32_t cnt = 0;
            for (uint32_t c = lane; c < C32; c += 32u) {
                uint64_t N;
                const uint64_t key = exact_key(row[c], bc[c], theta, c, L, N);
                cnt += (static_cast<uint32_t>(N >> sh) == Tu && key >= cand) ? 1u : 0u;
            }
            if (__reduce_add_sync(0xffffffffu, cnt) >= need) T2 = cand;
        }
    }
    __syncwarp();  // tie_list is reused by the caller's next input
}

__device__ __forceinline__ bool global_general_wins(uint64_t N, uint64_t key, uint32_t sh, uint32_t Tu,
                                                    uint64_t T2) {
    if (N <= (1ull << 23)) return false;
    const uint32_t u = static_cast<uint32_t>(N >> sh);
    return Tu == 0 ? u > 0 : (u > Tu || (u == Tu && key >= T2));
}

// ---- local inhibition by candidate pruning (any boosts, one warp) -------------------------
// Column c wins iff it is eligible and fewer than k columns of W(c)\{c} have a larger exact key
// (R4-R7, R9).  Let v be monotone in the exact key (uniform boost: raw; per-column boosts: the
// coarse key u of coarse_map, < 2^15), 0 for ineligible columns, and M_t = {d : v_d >= t},
// t >= 1.  If every window W(c) with v_c < t holds >= k members of M_t, each such c has >= k
// larger keys in its window and loses: only the candidates M_t can win, and only candidates
// can beat a candidate (every other column of the window has a smaller v, hence a smaller
// key).  The largest t passing a conservative test is searched bitwise: the columns of word j
// share the window core I_j = [max(0, 32j+31-r), min(C-1, 32j+r)], which must hold >= k
// members of M_t.  The candidates are compacted in position order with their exact keys; the
// candidates of W(c) are then a contiguous range of that list, and c counts the larger keys in
// it (stopping at k).  Lane j owns the column-words j and j + 32 (NW2 = 2 when ncw > 32): v of
// its 32 columns sits two per register (columns i and i + 16), biased by 0x8000 per half, so
// the word of M_t is 16 subtractions, shifts and LOP3s with no cross-lane traffic.  Cost per
// input ~ (C/32) * bits(v) for the search plus ~ P * |range| / 32 compares per lane (P ~
// C*k/r candidates).  Returns false without emitting anything when more candidates remain
// than the scratch holds (small radii): the caller falls back to the wavelet / comparator.
// KeyT: uint32_t (uniform: raw << L | (2^L-1-c), raw <= 1023, L <= 11) or uint64_t
// (exact_key).  emit(cw, word) gets the SDR words in order (warp-uniform).  Scratch: [64] SDR
// words, then keys and positions u16.
template <int NW2, bool UNIFORM, typename KeyT, typename RowT, typename Emit>
__device__ __forceinline__ bool local_candidates(const RowT* row, const uint32_t* bc, uint32_t C, uint32_t ncw,
                                                 uint32_t radius, uint32_t k, uint32_t theta, uint32_t r_lo,
                                                 uint32_t L, const CoarseMap& cm, uint8_t* scratch,
                                                 uint32_t scratch_bytes, uint32_t lane, Emit emit, uint32_t dbg = 0) {
    static_assert(NW2 == 1 || NW2 == 2, "at most 64 column-words");
    const uint32_t full = 0xffffffffu;
    auto value = [&](uint32_t c) -> uint32_t {
        if (UNIFORM) {
            const uint32_t x = row[c];
            return x >= r_lo ? x : 0u;
        } else {
            bool lossy;
            return coarse_u15(eligible_N(row[c], bc[c], theta), cm, lossy);
        }
    };
    // vb[h][i] = (v(32j + i) | 0x8000) | (v(32j + i + 16) | 0x8000) << 16, j = lane + 32h.  The
    // values are computed column-coalesced (lane = column of each word) and staged in the scratch
    // as rows of 34 u16 per word with columns i, i+16 adjacent, then read lane-owned as u32 pairs at
    // word offset 17 j + i (conflict-free; reading them lane-owned straight from the raw counts
    // and boosts would be 16- and 32-way bank conflicts)
    constexpr uint32_t kHead = 64u * 4u;
    uint32_t vb[NW2][16];
    uint32_t vmax = 0;
    if (scratch_bytes >= kHead + ncw * 68u) {
        uint16_t* stg = reinterpret_cast<uint16_t*>(scratch + kHead);
        for (uint32_t cw = 0; cw < ncw; ++cw) {
            const uint32_t v = value(cw * 32u + lane);
            vmax = max(vmax, v);
            stg[cw * 34u + ((lane & 15u) << 1) + (lane >> 4)] = static_cast<uint16_t>(v);
        }
        __syncwarp();
#pragma unroll
        for (int h = 0; h < NW2; ++h) {
            const uint32_t j = lane + 32u * h;
            const uint32_t* rowp = reinterpret_cast<const uint32_t*>(stg) + 17u * j;
#pragma unroll
            for (int i = 0; i < 16; ++i) vb[h][i] = (j < ncw ? rowp[i] : 0u) | 0x80008000u;
        }
        __syncwarp();  // the staging area is reused below
    } else {
#pragma unroll
        for (int h = 0; h < NW2; ++h) {
            const uint32_t j = lane + 32u * h;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const uint32_t a = j < ncw ? value(32u * j + i) : 0u;
                const uint32_t b = j < ncw ? value(32u * j + i + 16u) : 0u;
                vmax = max(vmax, max(a, b));
                vb[h][i] = (a | (b << 16)) | 0x80008000u;
            }
        }
    }
    vmax = __reduce_max_sync(full, vmax);
    uint32_t* sdr = reinterpret_cast<uint32_t*>(scratch);
    if (vmax == 0u) {  // no eligible column
        for (uint32_t cw = 0; cw < ncw; ++cw) emit(cw, 0u);
        return true;
    }
    // M_t: lane j's words m[h] (natural bit order) and their exclusive prefix counts e[h]
    uint32_t m[NW2], e[NW2], total;
    auto masks = [&](uint32_t t) {
        const uint32_t tt = t | (t << 16);  // v >= t  <=>  bit 15 of (v | 0x8000) - t is set
#pragma unroll
        for (int h = 0; h < NW2; ++h) {
            uint32_t acc = 0;
#pragma unroll
            for (int i = 0; i < 16; ++i) acc |= ((vb[h][i] - tt) >> (15 - i)) & (0x00010001u << i);
            m[h] = acc;
        }
        uint32_t p[NW2];
#pragma unroll
        for (int h = 0; h < NW2; ++h) p[h] = __popc(m[h]);
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
            for (int h = 0; h < NW2; ++h) {
                const uint32_t a = __shfl_up_sync(full, p[h], d);
                if (lane >= static_cast<uint32_t>(d)) p[h] += a;
            }
        }
        const uint32_t t0 = __shfl_sync(full, p[0], 31);
        total = t0;
        e[0] = p[0] - __popc(m[0]);
        if (NW2 > 1) {
            total += __shfl_sync(full, p[NW2 - 1], 31);
            e[NW2 - 1] = t0 + p[NW2 - 1] - __popc(m[NW2 - 1]);
        }
    };
    // #{d < x : d in M_t}, x in [0, C] (warp-uniform call, per-lane x)
    auto cntlt = [&](uint32_t x) -> uint32_t {
        const uint32_t w = x >> 5, src = w & 31u;
        uint32_t ev = __shfl_sync(full, e[0], src), mv = __shfl_sync(full, m[0], src);
        if (NW2 > 1) {
            const uint32_t eb = __shfl_sync(full, e[NW2 - 1], src), mb = __shfl_sync(full, m[NW2 - 1], src);
            if (w >= 32u) ev = eb, mv = mb;
        }
        return x >= C ? total : ev + __popc(mv & ((1u << (x & 31u)) - 1u));
    };
    auto core_ok = [&](uint32_t j) -> bool {  // the window core of word j holds >= k of M_t
        const uint32_t lo = 32u * j + 31u >= radius ? 32u * j + 31u - radius : 0u;
        const uint32_t hi1 = min(C, 32u * j + radius + 1u);
        const uint32_t n = cntlt(hi1) - cntlt(lo);
        return j >= ncw || (lo < hi1 && n >= k);
    };
    // bitwise search of the largest passing t over the top 10 bits of v (the low bits would only
    // trim a few candidates more)
    const int nb = 32 - __clz(vmax);
    uint32_t t = 0;
    for (int b = nb - 1; b >= max(0, nb - 10); --b) {
        const uint32_t tt = t | (1u << b);
        if (tt > vmax) continue;
        masks(tt);
        bool ok = core_ok(lane);
        if (NW2 > 1) {
            const bool ok1 = core_ok(lane + 32u);  // not short-circuited: core_ok shuffles
            ok = ok && ok1;
        }
        if (__all_sync(full, ok)) t = tt;
    }
    t = max(t, 1u);
    if (UNIFORM && vmax - t < 160u && scratch_bytes >= kHead + 4u * 8u * 65u) {
        // Uniform boost, few levels: sweep the raw values from the top.  With G = the columns of
        // value > l and E = those of value l (bit masks over all columns, one word per lane), a
        // column c of value l has beats(c) = |G & W(c)| + |E & [lo(c), c)| (equal raw: the lower
        // index wins): two range popcounts from per-word prefix counts, no candidate list.
        uint2* sG = reinterpret_cast<uint2*>(scratch + kHead);  // [65] {word of G, exclusive prefix count}
        uint2* sE = sG + 65;                                     // [65] the same for E
        auto ge = [&](uint32_t l, uint32_t* w) {
            const uint32_t ll = l | (l << 16);
#pragma unroll
            for (int h = 0; h < NW2; ++h) {
                uint32_t acc = 0;
#pragma unroll
                for (int i = 0; i < 16; ++i) acc |= ((vb[h][i] - ll) >> (15 - i)) & (0x00010001u << i);
                w[h] = acc;
            }
        };
        // exclusive prefix counts of the words w[h] (word lane + 32h) -> sw / sp (+ total at ncw);
        // ex[h] / tot_out get this lane's exclusive prefixes and the total
        auto publish = [&](const uint32_t* w, uint2* sw, uint32_t* ex, uint32_t& tot_out) {
            uint32_t q[NW2];
#pragma unroll
            for (int h = 0; h < NW2; ++h) q[h] = __popc(w[h]);
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
                for (int h = 0; h < NW2; ++h) {
                    const uint32_t a = __shfl_up_sync(full, q[h], d);
                    if (lane >= static_cast<uint32_t>(d)) q[h] += a;
                }
            }
            const uint32_t t0 = __shfl_sync(full, q[0], 31);
            const uint32_t tot = t0 + (NW2 > 1 ? __shfl_sync(full, q[NW2 - 1], 31) : 0u);
#pragma unroll
            for (int h = 0; h < NW2; ++h) {
                const uint32_t j = lane + 32u * h;
                ex[h] = (h ? t0 : 0u) + q[h] - __popc(w[h]);
                if (j < ncw) sw[j] = make_uint2(w[h], ex[h]);
            }
            if (lane == 0) sw[ncw] = make_uint2(0u, tot);
            tot_out = tot;
        };
        auto cnt = [&](const uint2* sw, uint32_t x) {  // #{d < x}, x <= C (one 8-byte load)
            const uint2 v = sw[x >> 5];
            return v.y + __popc(v.x & ((1u << (x & 31u)) - 1u));
        };
        // G's words and exclusive prefix counts are carried from level to level (G of the next
        // level = G | E of this one, so its prefix counts are the sums): one scan per level
        uint32_t gw[NW2], gp[NW2], win[NW2], gtot = 0;
#pragma unroll
        for (int h = 0; h < NW2; ++h) gw[h] = 0u, gp[h] = 0u, win[h] = 0u;
        // LV levels per step (l, l-1, .., l-LV+1): their E scans interleave, dividing the
        // dependent shuffle chains by LV; G of level l-u = G | E of the levels above it
        constexpr int LV = 4;
        const uint32_t nlvmax = scratch_bytes >= kHead + 2u * LV * 8u * 65u ? LV : 2u;
        uint2* tabs = sG;  // [2 LV][65]: G of level u at tabs[2u], E at tabs[2u + 1]
        for (uint32_t l = vmax; l + 1u > t;) {
            const uint32_t nlv = min(nlvmax, l - t + 1u);
            uint32_t m[LV][NW2], e[LV][NW2];
            bool any = false;
#pragma unroll
            for (int u = 0; u < LV; ++u) {
                if (static_cast<uint32_t>(u) < nlv) {
                    ge(l - u, m[u]);
                } else {
#pragma unroll
                    for (int h = 0; h < NW2; ++h) m[u][h] = u ? m[u - 1][h] : gw[h];
                }
#pragma unroll
                for (int h = 0; h < NW2; ++h) {
                    e[u][h] = m[u][h] & ~(u ? m[u - 1][h] : gw[h]);
                    any |= e[u][h] != 0u;
                }
            }
            l = l >= nlv ? l - nlv : 0u;
            if (l + 1u <= t && nlv < 1u) break;
            if (!__any_sync(full, any)) {
#pragma unroll
                for (int h = 0; h < NW2; ++h) gw[h] = m[LV - 1][h];
                if (l + 1u <= t) break;
                continue;
            }
            // exclusive prefix counts of the LV E masks (interleaved scans)
            uint32_t q[LV][NW2];
#pragma unroll
            for (int u = 0; u < LV; ++u)
#pragma unroll
                for (int h = 0; h < NW2; ++h) q[u][h] = __popc(e[u][h]);
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
                for (int u = 0; u < LV; ++u)
#pragma unroll
                    for (int h = 0; h < NW2; ++h) {
                        const uint32_t a = __shfl_up_sync(full, q[u][h], d);
                        if (lane >= static_cast<uint32_t>(d)) q[u][h] += a;
                    }
            }
            uint32_t etot[LV], ep[LV][NW2];
#pragma unroll
            for (int u = 0; u < LV; ++u) {
                const uint32_t t0 = __shfl_sync(full, q[u][0], 31);
                etot[u] = t0 + (NW2 > 1 ? __shfl_sync(full, q[u][NW2 - 1], 31) : 0u);
#pragma unroll
                for (int h = 0; h < NW2; ++h) ep[u][h] = (h ? t0 : 0u) + q[u][h] - __popc(e[u][h]);
            }
            // tables: G and E of each level (G of level u = G | E of the levels before it)
            {
                uint32_t gwu[NW2], gpu[NW2], gtu = gtot;
#pragma unroll
                for (int h = 0; h < NW2; ++h) gwu[h] = gw[h], gpu[h] = gp[h];
#pragma unroll
                for (int u = 0; u < LV; ++u) {
                    if (static_cast<uint32_t>(u) < nlv) {
#pragma unroll
                        for (int h = 0; h < NW2; ++h) {
                            const uint32_t j = lane + 32u * h;
                            if (j < ncw) {
                                tabs[(2 * u) * 65 + j] = make_uint2(gwu[h], gpu[h]);
                                tabs[(2 * u + 1) * 65 + j] = make_uint2(e[u][h], ep[u][h]);
                            }
                        }
                        if (lane == 0) {
                            tabs[(2 * u) * 65 + ncw] = make_uint2(0u, gtu);
                            tabs[(2 * u + 1) * 65 + ncw] = make_uint2(0u, etot[u]);
                        }
                    }
#pragma unroll
                    for (int h = 0; h < NW2; ++h) gwu[h] |= e[u][h], gpu[h] += ep[u][h];
                    gtu += etot[u];
                }
            }
            __syncwarp();
#pragma unroll
            for (int h = 0; h < NW2; ++h) {
                uint32_t eall = 0;
#pragma unroll
                for (int u = 0; u < LV; ++u) eall |= e[u][h];
                while (eall) {
                    const uint32_t bit = __ffs(eall) - 1u, c = 32u * (lane + 32u * h) + bit;
                    eall &= eall - 1u;
                    uint32_t u = 0;
#pragma unroll
                    for (int v = LV - 1; v > 0; --v) u = ((e[v][h] >> bit) & 1u) ? static_cast<uint32_t>(v) : u;
                    const uint2* G = tabs + (2u * u) * 65u;
                    const uint2* E = G + 65;
                    const uint32_t lo = c >= radius ? c - radius : 0u, hi1 = min(C, c + radius + 1u);
                    const uint32_t beats = (cnt(G, hi1) - cnt(G, lo)) + (cnt(E, c) - cnt(E, lo));
                    if (beats < k) win[h] |= 1u << bit;
                }
            }
            __syncwarp();  // the tables are rewritten by the next step
#pragma unroll
            for (int u = 0; u < LV; ++u) {
#pragma unroll
                for (int h = 0; h < NW2; ++h) gw[h] |= e[u][h], gp[h] += ep[u][h];
                gtot += etot[u];
            }
            if (l + 1u <= t) break;
        }
#pragma unroll
        for (int h = 0; h < NW2; ++h)
            if (lane + 32u * h < ncw) sdr[lane + 32u * h] = win[h];
        __syncwarp();
        for (uint32_t cw = 0; cw < ncw; ++cw) emit(cw, sdr[cw]);
        __syncwarp();
        return true;
    }
    masks(t);
    const uint32_t P = total;
    const uint32_t cap = scratch_bytes > kHead ? (scratch_bytes - kHead) / (sizeof(KeyT) + 2u) : 0u;
    if (P > cap) return false;
    KeyT* skey = reinterpret_cast<KeyT*>(scratch + kHead);                              // [cap]
    uint16_t* spos = reinterpret_cast<uint16_t*>(scratch + kHead + cap * sizeof(KeyT));  // [cap]
    for (uint32_t w = lane; w < ncw; w += 32u) sdr[w] = 0u;
    // compaction in position order, with the exact keys: lane j writes the candidates of its words
#pragma unroll
    for (int h = 0; h < NW2; ++h) {
        uint32_t mm = m[h], at = e[h];
        const uint32_t j = lane + 32u * h;
        while (mm) {
            const uint32_t c = 32u * j + (__ffs(mm) - 1u);
            mm &= mm - 1u;
            spos[at] = static_cast<uint16_t>(c);
            if (UNIFORM) {
                skey[at] = static_cast<KeyT>((static_cast<uint32_t>(row[c]) << L) | ((1u << L) - 1u - c));
            } else {
                uint64_t N;
                skey[at] = static_cast<KeyT>(exact_key(row[c], bc[c], theta, c, L, N));
            }
            ++at;
        }
    }
    __syncwarp();
    // beats of each candidate among the candidates of its window (a contiguous range)
    for (uint32_t i0 = 0; i0 < (dbg & 1u ? 0u : P); i0 += 32u) {
        const uint32_t i = i0 + lane;
        const bool has = i < P;
        const uint32_t c = has ? spos[i] : 0u;
        const uint32_t a = cntlt(c >= radius ? c - radius : 0u);
        const uint32_t b = cntlt(min(C, c + radius + 1u));
        if (has) {
            const KeyT key = skey[i];
            uint32_t beats = 0;
            uint32_t j = a;
            for (; j + 4u <= b && beats < k; j += 4u)
                beats += (skey[j] > key ? 1u : 0u) + (skey[j + 1u] > key ? 1u : 0u) +
                         (skey[j + 2u] > key ? 1u : 0u) + (skey[j + 3u] > key ? 1u : 0u);
            for (; j < b && beats < k; ++j) beats += skey[j] > key ? 1u : 0u;
            if (beats < k) atomicOr(&sdr[c >> 5], 1u << (c & 31u));
        }
    }
    __syncwarp();
    for (uint32_t cw = 0; cw < ncw; ++cw) emit(cw, sdr[cw]);
    __syncwarp();  // the scratch is reused by the caller's next input
    return true;
}

// bits needed for raw values 0..S
__device__ __forceinline__ uint32_t raw_bits(uint32_t S) { return 32u - __clz(S); }

}  // namespace sp
