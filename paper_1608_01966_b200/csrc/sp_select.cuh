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

// r_lo = smallest raw passing both the cutoff (raw >= theta) and the floor raw*Bc > 2^23.
__device__ __forceinline__ uint32_t uniform_r_lo(uint32_t theta, uint32_t bc) {
    return max(theta, (1u << 23) / bc + 1u);
}

// bits needed for raw values 0..S
__device__ __forceinline__ uint32_t raw_bits(uint32_t S) { return 32u - __clz(S); }

}  // namespace sp
