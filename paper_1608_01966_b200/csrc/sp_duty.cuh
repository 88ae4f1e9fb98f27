// sp_duty.cuh — device building blocks of the full learning step (
// SPEC S:119(b-e); R17-R21), shared by the per-input k_full kernel and
// the cluster-resident learning kernel.
//
//   (b) duty cycles   d = (d*(P-1) + a) / P, fp32, one RN operation at a time (R17)
//   (c) boost         minA = 0.01f * max(adc over W(c)); adc < minA ->
//                     1 + ((minA - adc) / minA) * (max_boost - 1), else 1     (R19)
//   (d) bump          odc < 0.01f * max(odc over W(c)) -> perm = min(1, perm + 0.1f*tau)  (R20)
//   (e) radius        clamp(floor((sum span + nbits) / (2 nbits)), 1, C)                  (R21)
//
// W(c) = [max(0, c-r), min(C-1, c+r)] (all columns for r = 0) includes c (R18).  Window maxima
// use per-32-column-block prefix/suffix maxima (warp shuffles) plus a sparse table over the
// block maxima: two lookups per column, exact (fmaxf of non-negative floats).
#pragma once

#include <cstdint>

namespace sp {

__device__ __forceinline__ float duty_update(float d, bool a, float pm1, float P) {
    // no FMA: product, sum and quotient are each rounded (R17)
    return __fdiv_rn(__fadd_rn(__fmul_rn(d, pm1), a ? 1.0f : 0.0f), P);
}

// boost of a column from its active duty cycle and the window maximum (R19)
__device__ __forceinline__ float boost_rule(float adc, float maxA, float mb1) {
    const float minA = __fmul_rn(0.01f, maxA);
    if (!(adc < minA)) return 1.0f;
    const float t2 = __fdiv_rn(__fsub_rn(minA, adc), minA);
    return __fadd_rn(1.0f, __fmul_rn(t2, mb1));
}

// Bc = boost * 2^23, exact for boost in [1,16) (R4)
__device__ __forceinline__ uint32_t boost_bc(float b) { return static_cast<uint32_t>(__fmul_rn(b, 8388608.0f)); }

__device__ __forceinline__ bool weak_column(float odc, float maxO) { return odc < __fmul_rn(0.01f, maxO); }

__device__ __forceinline__ uint32_t adapt_radius(uint64_t span_sum, uint32_t nbits, uint32_t C) {
    const uint64_t r = (span_sum + nbits) / (2ull * nbits);
    return static_cast<uint32_t>(r < 1ull ? 1ull : (r > C ? static_cast<uint64_t>(C) : r));
}

// number of sparse-table levels for nb block maxima
__host__ __device__ __forceinline__ uint32_t wmax_levels(uint32_t nb) {
    uint32_t l = 1;
    while ((1u << l) <= nb) ++l;
    return l;
}

// Window-maximum tables of v[0..C) (values >= 0), computed by the threads [t0, t0+nt) of the
// CTA (nt a multiple of 32): pre/suf[C32] in-block prefix/suffix maxima, table[levels][nb]
// with table[l][b] = max of blocks b .. b+2^l-1.  Every participating thread must call it;
// `sync` is a barrier over those threads (called between dependent levels).
template <typename Sync>
__device__ __forceinline__ void wmax_build(const float* v, uint32_t C, uint32_t C32, float* pre, float* suf,
                                           float* table, uint32_t t0, uint32_t nt, Sync sync) {
    const uint32_t tid = threadIdx.x - t0, lane = threadIdx.x & 31u;
    const uint32_t nb = C32 / 32u;
    for (uint32_t b = tid >> 5; b < nb; b += nt >> 5) {
        const uint32_t c = b * 32u + lane;
        const float x = c < C ? v[c] : 0.0f;
        float p = x, s = x;
#pragma unroll
        for (uint32_t d = 1; d < 32u; d <<= 1) {
            const float up = __shfl_up_sync(0xffffffffu, p, d);
            const float dn = __shfl_down_sync(0xffffffffu, s, d);
            if (lane >= d) p = fmaxf(p, up);
            if (lane + d < 32u) s = fmaxf(s, dn);
        }
        pre[c] = p;
        suf[c] = s;
        if (lane == 0) table[b] = s;  // block maximum
    }
    sync();
    const uint32_t L = wmax_levels(nb);
    for (uint32_t l = 1; l < L; ++l) {
        const uint32_t half = 1u << (l - 1);
        for (uint32_t b = tid; b + (1u << l) <= nb; b += nt)
            table[l * nb + b] = fmaxf(table[(l - 1) * nb + b], table[(l - 1) * nb + b + half]);
        sync();
    }
}

// max of v over W(c) for radius r (0 = all columns), from the tables of wmax_build
__device__ __forceinline__ float wmax_query(const float* v, const float* pre, const float* suf, const float* table,
                                            uint32_t nb, uint32_t C, uint32_t c, uint32_t r) {
    const uint32_t lo = (r == 0u || c < r) ? 0u : c - r;
    const uint32_t hi = (r == 0u || c + r >= C) ? C - 1u : c + r;
    const uint32_t bl = lo >> 5, bh = hi >> 5;
    if (bl == bh) {
        float m = 0.0f;
        for (uint32_t d = lo; d <= hi; ++d) m = fmaxf(m, v[d]);
        return m;
    }
    float m = fmaxf(suf[lo], pre[hi]);
    if (bh - bl >= 2u) {
        const uint32_t a = bl + 1u, b = bh - 1u;
        const uint32_t l = 31u - __clz(b - a + 1u);
        m = fmaxf(m, fmaxf(table[l * nb + a], table[l * nb + b + 1u - (1u << l)]));
    }
    return m;
}

// Windows of radius r with 2r+1 >= C (the adapted radius is typically ~C/2, R21) always reach
// an end of the column range: W(c) = [0, hi] or [lo, C-1].  Prefix and suffix maxima answer
// them: in-block scans (warp shuffles) plus the exclusive prefix/suffix maxima of the block
// maxima (one warp), two barriers instead of the sparse table's log2(nb) + 1.
__device__ __forceinline__ void wmax_build_ends(const float* v, uint32_t C, uint32_t C32, float* pre, float* suf,
                                                float* table) {
    const uint32_t tid = threadIdx.x, lane = tid & 31u, nb = C32 / 32u;
    for (uint32_t b = tid >> 5; b < nb; b += blockDim.x >> 5) {
        const uint32_t c = b * 32u + lane;
        const float x = c < C ? v[c] : 0.0f;
        float p = x, s = x;
#pragma unroll
        for (uint32_t d = 1; d < 32u; d <<= 1) {
            const float up = __shfl_up_sync(0xffffffffu, p, d);
            const float dn = __shfl_down_sync(0xffffffffu, s, d);
            if (lane >= d) p = fmaxf(p, up);
            if (lane + d < 32u) s = fmaxf(s, dn);
        }
        pre[c] = p;
        suf[c] = s;
        if (lane == 0) table[b] = s;  // block maximum
    }
    __syncthreads();
    if (tid < 32u) {  // table[nb + b] = max of blocks < b, table[2nb + b] = max of blocks > b
        float carry = 0.0f;
        for (uint32_t base = 0; base < nb; base += 32u) {  // exclusive prefix max
            const uint32_t b = base + lane;
            const float x = b < nb ? table[b] : 0.0f;
            float p = x;
#pragma unroll
            for (uint32_t d = 1; d < 32u; d <<= 1) {
                const float up = __shfl_up_sync(0xffffffffu, p, d);
                if (lane >= d) p = fmaxf(p, up);
            }
            const float ex = fmaxf(carry, __shfl_up_sync(0xffffffffu, p, 1));
            if (b < nb) table[nb + b] = lane == 0 ? carry : ex;
            carry = fmaxf(carry, __shfl_sync(0xffffffffu, p, 31));
        }
        carry = 0.0f;
        for (int base = static_cast<int>((nb - 1u) / 32u) * 32; base >= 0; base -= 32) {  // exclusive suffix max
            const uint32_t b = static_cast<uint32_t>(base) + lane;
            const float x = b < nb ? table[b] : 0.0f;
            float s = x;
#pragma unroll
            for (uint32_t d = 1; d < 32u; d <<= 1) {
                const float dn = __shfl_down_sync(0xffffffffu, s, d);
                if (lane + d < 32u) s = fmaxf(s, dn);
            }
            const float ex = fmaxf(carry, __shfl_down_sync(0xffffffffu, s, 1));
            if (b < nb) table[2u * nb + b] = lane == 31u ? carry : ex;
            carry = fmaxf(carry, __shfl_sync(0xffffffffu, s, 0));
        }
    }
    __syncthreads();
}

__device__ __forceinline__ float wmax_query_ends(const float* pre, const float* suf, const float* table, uint32_t nb,
                                                 uint32_t C, uint32_t c, uint32_t r) {
    const uint32_t lo = c < r ? 0u : c - r;
    const uint32_t hi = c + r >= C ? C - 1u : c + r;
    if (lo == 0u) return fmaxf(pre[hi], table[nb + (hi >> 5)]);
    return fmaxf(suf[lo], table[2u * nb + (lo >> 5)]);  // hi == C-1 when 2r+1 >= C
}

// Maxima of a[0..C) and b[0..C) (values >= 0) over the whole CTA, for windows that cover all
// columns (radius 0 or >= C-1): one reduction instead of the window tables.  s_red >= 64
// floats of shared scratch; every thread of the CTA calls it and gets both maxima.
__device__ __forceinline__ void block_max2(const float* a, const float* b, uint32_t C, float* s_red, float& ma,
                                           float& mb) {
    const uint32_t tid = threadIdx.x, lane = tid & 31u, wi = tid >> 5, nw = blockDim.x >> 5;
    float x = 0.0f, y = 0.0f;
    for (uint32_t c = tid; c < C; c += blockDim.x) x = fmaxf(x, a[c]), y = fmaxf(y, b[c]);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, d));
        y = fmaxf(y, __shfl_xor_sync(0xffffffffu, y, d));
    }
    if (lane == 0) s_red[wi] = x, s_red[32 + wi] = y;
    __syncthreads();
    x = lane < nw ? s_red[lane] : 0.0f;
    y = lane < nw ? s_red[32 + lane] : 0.0f;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, d));
        y = fmaxf(y, __shfl_xor_sync(0xffffffffu, y, d));
    }
    ma = x, mb = y;
}

// span of a column from its connected synapses: lanes hold (connected, s) pairs; returns
// max - min + 1 of idx over the connected ones, 0 if none (warp-collective; idx ascending)
__device__ __forceinline__ void span_accumulate(bool conn, uint32_t s, uint32_t& smin, uint32_t& smax) {
    if (conn) {
        smin = min(smin, s);
        smax = max(smax, s);
    }
}

__device__ __forceinline__ uint32_t span_finish(uint32_t smin, uint32_t smax, const uint32_t* idx_row,
                                                uint32_t idx_mask) {
    smin = __reduce_min_sync(0xffffffffu, smin);
    smax = __reduce_max_sync(0xffffffffu, smax);
    if (smin == 0xFFFFFFFFu) return 0u;
    return (idx_row[smax] & idx_mask) - (idx_row[smin] & idx_mask) + 1u;
}

}  // namespace sp
