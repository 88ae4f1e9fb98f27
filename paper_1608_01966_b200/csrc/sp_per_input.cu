// sp_per_input.cu — the per-input CUDA path:
//   P1 k_pack     uint8 frames/patches -> input bit-planes (a1)
//   P2 k_overlap  per input: bit-plane in smem, thread-per-column gather-count (a2)
//   P3 k_inhibit  per input: exact rank keys, k-winners (global / local), SDR (a3, a4)
//   P4 k_learn    per input: fused +inc/-dec, clamp, connected-flag refresh (a5)
// plus layout maintenance (synapse-major idx|flag words, batched ELL flags).
// Learning runs P2 -> P3 -> P4 per input in order (the recurrence of P:92).
#include <algorithm>
#include <cstdlib>

#include "sp_duty.cuh"
#include "sp_internal.h"
#include "sp_select.cuh"

namespace sp {

namespace {

// ---------------------------------------------------------------------------------------
// P1: packing.  Input t = (frame t / P, tile t % P); bit y*pw + x of the input is pixel
// (ty*ph + y, tx*pw + x) of the frame (R12, R13).  One thread per output word.
// ---------------------------------------------------------------------------------------
__global__ void k_pack(const PerInputParams p) {
    const uint32_t word = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t t = blockIdx.y;  // input within the sub-batch
    if (word >= p.Wn || t >= p.num_inputs) return;
    const Geometry& g = p.g;
    const uint32_t frame = t / g.P, tile = t % g.P;
    const uint8_t* fr = p.frames + static_cast<size_t>(frame) * g.W * g.H;
    const uint32_t q0 = word * 32u;
    uint32_t out = 0;
    if (g.whole && (g.nbits % 16u) == 0 && q0 + 32u <= g.nbits &&
        (reinterpret_cast<uintptr_t>(fr) & 15u) == 0) {
        const uint4 a = *reinterpret_cast<const uint4*>(fr + q0);
        const uint4 b = *reinterpret_cast<const uint4*>(fr + q0 + 16);
        const uint32_t v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
#pragma unroll
            for (int by = 0; by < 4; ++by)
                out |= (((v[k] >> (8 * by)) & 0xFFu) != 0u ? 1u : 0u) << (4 * k + by);
        }
    } else {
        const uint32_t tilesx = g.W / g.pw;
        const uint32_t ty = tile / tilesx, tx = tile % tilesx;
        for (uint32_t j = 0; j < 32u; ++j) {
            const uint32_t q = q0 + j;
            if (q >= g.nbits) break;
            const uint32_t y = q / g.pw, x = q % g.pw;
            const uint8_t v = fr[static_cast<size_t>(ty * g.ph + y) * g.W + tx * g.pw + x];
            out |= (v != 0 ? 1u : 0u) << j;
        }
    }
    p.bits[static_cast<size_t>(t) * (p.bits_stride ? p.bits_stride : p.Wn) + word] = out;
}

// ---------------------------------------------------------------------------------------
// P2: overlap.  grid (column blocks, inputs); the input's bit-plane is staged in smem.
// syn[s][c] = idx | connected << 31 (synapse-major: coalesced across columns).
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_overlap(const PerInputParams p) {
    // 64 columns x 4 synapse quarters per CTA: reads of syn[s][c] stay coalesced across
    // the 64 consecutive columns, and large C gets 4x the CTAs of thread-per-column.
    extern __shared__ uint32_t s_bits[];
    __shared__ uint32_t s_part[4][64];
    const uint32_t t = blockIdx.y;
    const uint32_t* src = p.bits + static_cast<size_t>(t) * p.Wn;
    for (uint32_t i = threadIdx.x; i < p.Wn; i += blockDim.x) s_bits[i] = src[i];
    __syncthreads();
    const uint32_t cl = threadIdx.x & 63u, part = threadIdx.x >> 6;
    const uint32_t c = blockIdx.x * 64u + cl;
    const uint32_t C32 = p.g.C32, S = p.g.S;
    const uint32_t s0 = part * S / 4u, s1 = (part + 1u) * S / 4u;
    uint32_t raw = 0;
    if (c < C32) {
        const uint32_t* e = p.syn + c;
        uint32_t s = s0;
        for (; s + 8 <= s1; s += 8) {
            uint32_t v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = e[(s + u) * C32];
#pragma unroll
            for (int u = 0; u < 8; ++u) raw += (s_bits[(v[u] & 0x7FFFFFFFu) >> 5] >> (v[u] & 31u)) & (v[u] >> 31);
        }
        for (; s < s1; ++s) {
            const uint32_t e0 = e[s * C32];
            raw += (s_bits[(e0 & 0x7FFFFFFFu) >> 5] >> (e0 & 31u)) & (e0 >> 31);
        }
    }
    s_part[part][cl] = raw;
    __syncthreads();
    if (part == 0 && c < C32)
        p.raw[static_cast<size_t>(t) * C32 + c] = s_part[0][cl] + s_part[1][cl] + s_part[2][cl] + s_part[3][cl];
}

// ---------------------------------------------------------------------------------------
// P3: inhibition, one CTA per input.  key(c) = (N << L) | (2^L-1-c), N = raw*Bc exact
// (R4); active iff N > 2^23 (Alg. 2 floor, R7) and fewer than k columns of W(c)\{c}
// have a larger key (R5, R6, R9).
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t key_of(uint32_t raw, uint32_t bc, uint32_t theta, uint32_t c,
                                           uint32_t L, uint64_t& N) {
    N = raw >= theta ? static_cast<uint64_t>(raw) * bc : 0ull;
    return (N << L) | (((1ull << L) - 1ull) - c);
}

// Local inhibition with per-column boosts and a large radius, by the whole CTA: a wavelet
// matrix over the 15-bit coarse keys of all C32 columns (the per-warp version of sp_select.cuh
// at CTA scale: ballots by warps, a CTA scan of the per-word counts, a stable scatter of
// (value << 16 | position) pairs, so the bottom level lists the columns of every tie range).
// Every CTA of the input builds it (the build is the latency; the queries are split), then
// answers the words [w0, w1): beats(c) = #{u_d > u_c} + #{u_d = u_c, d < c} over W(c), the
// ties with a lossy column re-decided on the exact keys (R4, R6).  Scratch: 2 x C32 pairs +
// (B + 1) x (ncw + 2) uint2 levels (the last: lossy flags in the bottom order).
__device__ void inhibit_wavelet(const PerInputParams& p, uint32_t* sm, uint32_t t, uint32_t gin, uint32_t radius,
                                uint32_t w0, uint32_t w1, uint32_t* s_total) {
    const Geometry& g = p.g;
    const uint32_t tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31u, wid = tid >> 5, nw = nthr >> 5;
    const uint32_t theta = p.min_overlap, L = g.keyL, C32 = g.C32, ncw = g.ncw, stride = ncw + 2u;
    const uint32_t* row = p.raw + static_cast<size_t>(t) * C32;
    const uint32_t* bc = p.bc;
    uint32_t* bufA = sm;
    uint32_t* bufB = sm + C32;
    uint2* lv = reinterpret_cast<uint2*>(sm + 2u * C32);
    __shared__ unsigned long long s_mm[2];
    __shared__ uint32_t s_red[32];
    const CoarseMap cm = coarse_map_block(row, bc, theta, 0u, ncw, s_mm);
    uint32_t umax = 0;
    for (uint32_t c = tid; c < C32; c += nthr) {
        bool lossy;
        const uint32_t u = c < g.C ? coarse_u15(eligible_N(row[c], bc[c], theta), cm, lossy) : 0u;
        const uint32_t v = u ? (u << 1) | (lossy ? 1u : 0u) : 0u;
        bufA[c] = (v << 16) | c;
        umax = max(umax, u);
    }
    umax = __reduce_max_sync(0xffffffffu, umax);
    if (lane == 0) s_red[wid] = umax;
    __syncthreads();
    if (wid == 0) {
        const uint32_t m = __reduce_max_sync(0xffffffffu, lane < nw ? s_red[lane] : 0u);
        if (lane == 0) s_red[0] = m;
    }
    __syncthreads();
    umax = s_red[0];
    const uint32_t B = umax ? 32u - __clz(umax) : 1u;
    __syncthreads();
    uint32_t* src = bufA;
    uint32_t* dst = bufB;
    for (int l = static_cast<int>(B) - 1; l >= -1; --l) {
        uint2* lvl = lv + (l >= 0 ? l : static_cast<int>(B)) * stride;
        const uint32_t sb = static_cast<uint32_t>(l + 17);  // bit l of u (l = -1: the lossy flag)
        for (uint32_t j = wid; j < ncw; j += nw) {
            const uint32_t w = __ballot_sync(0xffffffffu, (src[j * 32u + lane] >> sb) & 1u);
            if (lane == 0) lvl[j] = make_uint2(w, static_cast<uint32_t>(__popc(w)));
        }
        __syncthreads();
        // exclusive scan of the per-word counts (ncw <= 1024 = one per thread)
        uint32_t v = tid < ncw ? lvl[tid].y : 0u, x = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
            if (static_cast<int>(lane) >= d) x += y;
        }
        if (lane == 31u) s_red[wid] = x;
        __syncthreads();
        if (wid == 0) {
            uint32_t z = lane < nw ? s_red[lane] : 0u;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, z, d);
                if (static_cast<int>(lane) >= d) z += y;
            }
            s_red[lane] = z;  // inclusive warp totals
        }
        __syncthreads();
        const uint32_t before = (wid ? s_red[wid - 1u] : 0u) + x - v;
        const uint32_t ones = s_red[nw - 1u];
        if (tid < ncw) lvl[tid].y = before;
        if (tid == 0) lvl[ncw] = make_uint2(0u, ones), lvl[ncw + 1u] = make_uint2(0u, C32 - ones);
        __syncthreads();
        if (l < 0) break;
        const uint32_t Z = C32 - ones;
        for (uint32_t i = tid; i < C32; i += nthr) {
            const uint32_t e = src[i];
            const uint2 q = lvl[i >> 5];
            const uint32_t r = q.y + __popc(q.x & ((1u << (i & 31u)) - 1u));
            dst[((e >> sb) & 1u) ? Z + r : i - r] = e;
        }
        __syncthreads();
        uint32_t* tt = src;
        src = dst;
        dst = tt;
    }
    // queries: the columns of words [w0, w1), one per thread
    const int R = static_cast<int>(radius), Cn = static_cast<int>(g.C);
    const uint2* lvL = lv + B * stride;
    uint32_t my_total = 0;
    for (uint32_t cw = w0 + wid; cw < w1; cw += nw) {
        const uint32_t c = cw * 32u + lane;
        bool lossy_c = false;
        const uint64_t Nc = c < g.C ? eligible_N(row[c], bc[c], theta) : 0ull;
        const uint32_t uc = coarse_u15(Nc, cm, lossy_c);
        bool act = false;
        if (uc) {
            const uint32_t lo = static_cast<uint32_t>(max(0, static_cast<int>(c) - R));
            const uint32_t hi = static_cast<uint32_t>(min(Cn - 1, static_cast<int>(c) + R)) + 1u;
            uint32_t a = lo, m = c, b = hi, less = 0;
            for (int l = static_cast<int>(B) - 1; l >= 0; --l) {
                const uint2* lvl = lv + l * stride;
                const uint32_t ra = wm_rank2(lvl, a), rm = wm_rank2(lvl, m), rb = wm_rank2(lvl, b);
                if ((uc >> l) & 1u) {
                    const uint32_t Z = lvl[ncw + 1u].y;
                    less += (b - a) - (rb - ra);
                    a = Z + ra, m = Z + rm, b = Z + rb;
                } else {
                    a -= ra, m -= rm, b -= rb;
                }
            }
            int beats = static_cast<int>(((hi - lo) - less - (b - a)) + (m - a));
            if (b - a > 1u && wm_rank2(lvL, b) != wm_rank2(lvL, a)) {
                // a lossy column among c's ties: exact keys (src = the bottom level, positions)
                const uint64_t keyc = (Nc << L) | (((1ull << L) - 1ull) - c);
                for (uint32_t q = a; q < b; ++q) {
                    const uint32_t d = src[q] & 0xFFFFu;
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
            act = beats < static_cast<int>(p.k);
        }
        const uint32_t word = __ballot_sync(0xffffffffu, act);
        if (lane == 0) {
            p.sdr[static_cast<size_t>(gin) * ncw + cw] = word;
            my_total += __popc(word);
        }
    }
    if (lane == 0 && my_total) atomicAdd(s_total, my_total);
}

__global__ void __launch_bounds__(1024) k_inhibit(const PerInputParams p) {
    extern __shared__ uint32_t sm[];
    const Geometry& g = p.g;
    uint32_t* s_raw = sm;               // [C32]
    uint32_t* s_bc = sm + g.C32;        // [C32]
    uint32_t* s_planes = sm + 2u * g.C32;  // [ncw][<=16] bit-planes (local inhibition)
    __shared__ uint32_t s_cnt[2];
    __shared__ uint32_t s_total;
    const uint32_t t = blockIdx.x;
    const uint32_t gin = p.first_input + t;
    // gridDim.y CTAs share an input: CTA y emits the SDR words [w0, w1) (every CTA builds the
    // full key planes / threshold its windows need); counts then meet with atomics
    const uint32_t parts = gridDim.y;
    const uint32_t w0 = blockIdx.y * g.ncw / parts, w1 = (blockIdx.y + 1u) * g.ncw / parts;
    const uint32_t tid = threadIdx.x, nthr = blockDim.x;
    const uint32_t radius = p.radius_dev ? *p.radius_dev : p.radius;  // adapted by full learning
    if (radius > 0 && radius + 1u < g.C && !p.uniform_bc && p.wm_ok && radius >= p.wm_min_radius) {
        if (p.raw_out) {
            for (uint32_t c = w0 * 32u + tid; c < min(g.C, w1 * 32u); c += nthr) {
                const uint32_t r = p.raw[static_cast<size_t>(t) * g.C32 + c];
                p.raw_out[static_cast<size_t>(gin) * g.C + c] = static_cast<uint16_t>(r);
                p.boosted_out[static_cast<size_t>(gin) * g.C + c] =
                    r >= p.min_overlap ? __fmul_rn(static_cast<float>(r), p.boost[c]) : 0.0f;
            }
        }
        if (tid == 0) s_total = 0;
        __syncthreads();
        inhibit_wavelet(p, sm, t, gin, radius, w0, w1, &s_total);
        __syncthreads();
        if (tid == 0) {
            if (parts == 1u) p.counts[gin] = s_total;
            else if (s_total) atomicAdd(p.counts + gin, s_total);  // zeroed before the launch
        }
        return;
    }
    for (uint32_t c = tid; c < g.C32; c += nthr) {
        s_raw[c] = p.raw[static_cast<size_t>(t) * g.C32 + c];
        s_bc[c] = p.bc[c];
    }
    if (tid < 2) s_cnt[tid] = 0;
    if (tid == 0) s_total = 0;
    __syncthreads();
    const uint32_t theta = p.min_overlap, L = g.keyL;
    if (p.raw_out) {
        for (uint32_t c = w0 * 32u + tid; c < min(g.C, w1 * 32u); c += nthr) {
            const uint32_t r = s_raw[c];
            p.raw_out[static_cast<size_t>(gin) * g.C + c] = static_cast<uint16_t>(r);
            p.boosted_out[static_cast<size_t>(gin) * g.C + c] =
                r >= theta ? __fmul_rn(static_cast<float>(r), p.boost[c]) : 0.0f;
        }
    }
    uint64_t T = 0;
    if (radius == 0) {
        for (int bit = static_cast<int>(g.keyBits) - 1, it = 0; bit >= 0; --bit, ++it) {
            const uint64_t cand = T | (1ull << bit);
            uint32_t cnt = 0;
            for (uint32_t c = tid; c < g.C32; c += nthr) {
                uint64_t N;
                cnt += key_of(s_raw[c], s_bc[c], theta, c, L, N) >= cand ? 1u : 0u;
            }
            cnt = __reduce_add_sync(0xffffffffu, cnt);
            if ((tid & 31u) == 0 && cnt) atomicAdd(&s_cnt[it & 1], cnt);
            __syncthreads();
            const uint32_t total = s_cnt[it & 1];
            if (tid == 0) s_cnt[(it + 1) & 1] = 0;
            if (total >= p.k) T = cand;
            __syncthreads();
        }
    }
    // SDR: warp per 32-column word
    const uint64_t one = 1ull << 23;
    uint32_t my_total = 0;
    if (radius > 0 && p.uniform_bc) {
        // local inhibition, uniform boost: bit-sliced window comparator (sp_select.cuh)
        const uint32_t r_lo = uniform_r_lo(theta, s_bc[0]);
        const uint32_t nb = raw_bits(g.S);
        build_raw_planes(s_raw, s_planes, g.ncw, nb, r_lo, tid >> 5, nthr >> 5, tid & 31u);
        __syncthreads();
        for (uint32_t cw = w0 + (tid >> 5); cw < w1; cw += nthr >> 5) {
            const uint32_t word = local_uniform_word(s_raw, s_planes, g.ncw, nb, cw, g.C, radius, p.k,
                                                     r_lo, tid & 31u);
            if ((tid & 31u) == 0) {
                p.sdr[static_cast<size_t>(gin) * g.ncw + cw] = word;
                my_total += __popc(word);
            }
        }
    } else if (radius > 0) {
        // local inhibition, per-column boosts: coarse bit-sliced + exact ties (sp_select.cuh)
        __shared__ unsigned long long s_mm[2];
        const CoarseMap cm = coarse_map_block(s_raw, s_bc, theta, 0u, g.ncw, s_mm);
        build_coarse_planes15(s_raw, s_bc, s_planes, g.ncw, theta, cm, tid >> 5, nthr >> 5, tid & 31u);
        __syncthreads();
        for (uint32_t cw = w0 + (tid >> 5); cw < w1; cw += nthr >> 5) {
            const uint32_t word = local_general_word15(s_raw, s_bc, s_planes, g.ncw, cw, g.C, radius, p.k,
                                                       theta, cm, L, tid & 31u);
            if ((tid & 31u) == 0) {
                p.sdr[static_cast<size_t>(gin) * g.ncw + cw] = word;
                my_total += __popc(word);
            }
        }
    } else {
    for (uint32_t cw = w0 + (tid >> 5); cw < w1; cw += nthr >> 5) {
        const uint32_t c = cw * 32u + (tid & 31u);
        uint64_t N;
        const uint64_t key = key_of(s_raw[c], s_bc[c], theta, c, L, N);
        bool act = N > one;
        if (act) {
            if (radius == 0) {
                act = key >= T;
            } else {
                const uint32_t lo = c >= radius ? c - radius : 0u;
                const uint32_t hi = min(g.C - 1u, c + radius);
                uint32_t beats = 0;
                for (uint32_t d = lo; d <= hi && beats < p.k; ++d) {
                    uint64_t Nd;
                    beats += (d != c && key_of(s_raw[d], s_bc[d], theta, d, L, Nd) > key) ? 1u : 0u;
                }
                act = beats < p.k;
            }
        }
        const uint32_t word = __ballot_sync(0xffffffffu, act);
        if ((tid & 31u) == 0) {
            p.sdr[static_cast<size_t>(gin) * g.ncw + cw] = word;
            my_total += __popc(word);
        }
    }
    }
    __syncthreads();
    if ((tid & 31u) == 0 && my_total) atomicAdd(&s_total, my_total);
    __syncthreads();
    if (tid == 0) {
        if (parts == 1u) p.counts[gin] = s_total;
        else if (s_total) atomicAdd(p.counts + gin, s_total);  // zeroed before the launch
    }
}

// ---------------------------------------------------------------------------------------
// P4: learning for ONE input (P:92 -> whitepaper rule, S:119(a); R3, R10).  Warp per
// column; inactive columns exit at once.  perm is fp32: one IEEE RN add/sub, then clamp.
// ---------------------------------------------------------------------------------------
__global__ void k_learn(const PerInputParams p, uint32_t t) {
    const Geometry& g = p.g;
    const uint32_t c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint32_t lane = threadIdx.x & 31u;
    if (c >= g.C) return;
    const uint32_t gin = p.first_input + t;
    const uint32_t word = p.sdr[static_cast<size_t>(gin) * g.ncw + (c >> 5)];
    if (((word >> (c & 31u)) & 1u) == 0u) return;
    const uint32_t* bits = p.bits + static_cast<size_t>(t) * p.Wn;
    const uint32_t* idx = p.idx + static_cast<size_t>(c) * g.S;
    float* perm = p.perm + static_cast<size_t>(c) * g.S;
    uint32_t smin = 0xFFFFFFFFu, smax = 0u;
    for (uint32_t s = lane; s < g.S; s += 32u) {
        const uint32_t i = idx[s];
        const bool on = ((bits[i >> 5] >> (i & 31u)) & 1u) != 0u;
        float v = on ? __fadd_rn(perm[s], p.inc) : __fsub_rn(perm[s], p.dec);
        v = fminf(fmaxf(v, 0.0f), 1.0f);
        perm[s] = v;
        p.syn_rw[static_cast<size_t>(s) * g.C32 + c] = i | (v >= p.tau ? 0x80000000u : 0u);
        span_accumulate(v >= p.tau, s, smin, smax);
    }
    if (p.fl.span) {  // full learning: the connected span of the updated column (R21)
        const uint32_t sp_c = span_finish(smin, smax, idx, 0xFFFFFFFFu);
        if (lane == 0) p.fl.span[c] = sp_c;
    }
}

// ---------------------------------------------------------------------------------------
// P5: full learning steps (b)-(e) after input t's permanence update (S:119(b-e); DESIGN
// R17-R21), one CTA of 1024 threads: duty cycles of every column, window maxima (sp_duty.cuh),
// boosts, the bump of weak columns (warp per weak column: perm, synapse-major flags, span)
// and the adapted radius from the sum of the connected spans.
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_full(const PerInputParams p, uint32_t t) {
    const Geometry& g = p.g;
    const FullLearn& fl = p.fl;
    const uint32_t tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31u;
    const uint32_t gin = p.first_input + t;
    const uint32_t* sdr = p.sdr + static_cast<size_t>(gin) * g.ncw;
    const uint32_t* raw = p.raw + static_cast<size_t>(t) * g.C32;
    const uint32_t r = *fl.radius;  // radius in force for this input (W(c) of (c), (d); R18)
    const uint32_t nb = g.C32 / 32u;
    float* pre = fl.scratch;
    float* suf = pre + g.C32;
    float* table = suf + g.C32;
    __shared__ unsigned long long s_span;
    if (tid == 0) s_span = 0ull;
    // (b) duty cycles
    for (uint32_t c = tid; c < g.C; c += nthr) {
        const bool a = ((sdr[c >> 5] >> (c & 31u)) & 1u) != 0u;
        const bool o = raw[c] >= p.min_overlap && raw[c] > 0u;  // N > 0
        fl.adc[c] = duty_update(fl.adc[c], a, fl.pm1, fl.P);
        fl.odc[c] = duty_update(fl.odc[c], o, fl.pm1, fl.P);
    }
    __syncthreads();
    auto sync = [] { __syncthreads(); };
    // (c) boosts from the active duty cycles
    wmax_build(fl.adc, g.C, g.C32, pre, suf, table, 0u, nthr, sync);
    for (uint32_t c = tid; c < g.C; c += nthr) {
        const float b = boost_rule(fl.adc[c], wmax_query(fl.adc, pre, suf, table, nb, g.C, c, r), fl.mb1);
        fl.boost[c] = b;
        fl.bc[c] = boost_bc(b);
    }
    __syncthreads();
    // (d) bump of the weak columns, warp per column
    wmax_build(fl.odc, g.C, g.C32, pre, suf, table, 0u, nthr, sync);
    for (uint32_t c = tid >> 5; c < g.C; c += nthr >> 5) {
        if (!weak_column(fl.odc[c], wmax_query(fl.odc, pre, suf, table, nb, g.C, c, r))) continue;
        const uint32_t* idx = p.idx + static_cast<size_t>(c) * g.S;
        float* perm = p.perm + static_cast<size_t>(c) * g.S;
        uint32_t smin = 0xFFFFFFFFu, smax = 0u;
        for (uint32_t s = lane; s < g.S; s += 32u) {
            const float v = fminf(__fadd_rn(perm[s], fl.bump), 1.0f);
            perm[s] = v;
            p.syn_rw[static_cast<size_t>(s) * g.C32 + c] = idx[s] | (v >= p.tau ? 0x80000000u : 0u);
            span_accumulate(v >= p.tau, s, smin, smax);
        }
        const uint32_t sp_c = span_finish(smin, smax, idx, 0xFFFFFFFFu);
        if (lane == 0) fl.span[c] = sp_c;
    }
    if (!fl.adapt) return;
    __syncthreads();
    // (e) radius from the connected spans (exact integer form of S:151, R21)
    unsigned long long part = 0;
    for (uint32_t c = tid; c < g.C; c += nthr) part += fl.span[c];
    for (uint32_t d = 16; d > 0; d >>= 1) part += __shfl_xor_sync(0xffffffffu, part, d);
    if (lane == 0 && part) atomicAdd(&s_span, part);
    __syncthreads();
    if (tid == 0) *fl.radius = adapt_radius(s_span, g.nbits, g.C);
}

// P5 for many columns (C32 >= 4096), split over the SMs in two launches:
//   k_full_a: duty cycles (b) of every column; in-block prefix/suffix maxima and block maxima of
//             both duty arrays -> global scratch
//   k_full_b: every CTA builds the sparse tables over the block maxima in shared memory, then
//             boosts (c) and bumps (d) of its column range, the span sum of its range; the last
//             CTA to finish (ticket) forms the adapted radius (e)
__global__ void __launch_bounds__(1024) k_full_a(const PerInputParams p, uint32_t t) {
    const Geometry& g = p.g;
    const FullLearn& fl = p.fl;
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x, lane = threadIdx.x & 31u;
    const uint32_t nb = g.C32 / 32u;
    float* preA = fl.scratch;
    float* sufA = preA + g.C32;
    float* preO = sufA + g.C32;
    float* sufO = preO + g.C32;
    float* bmA = sufO + g.C32;
    float* bmO = bmA + nb;
    float a = 0.0f, o = 0.0f;
    if (c < g.C) {
        const uint32_t gin = p.first_input + t;
        const bool act = ((p.sdr[static_cast<size_t>(gin) * g.ncw + (c >> 5)] >> (c & 31u)) & 1u) != 0u;
        const uint32_t r = p.raw[static_cast<size_t>(t) * g.C32 + c];
        a = duty_update(fl.adc[c], act, fl.pm1, fl.P);
        o = duty_update(fl.odc[c], r >= p.min_overlap && r > 0u, fl.pm1, fl.P);
        fl.adc[c] = a;
        fl.odc[c] = o;
    }
    if (c >= g.C32) return;  // whole warps past the padded range
    float pa = a, sa = a, po = o, so = o;
#pragma unroll
    for (uint32_t d = 1; d < 32u; d <<= 1) {
        const float ua = __shfl_up_sync(0xffffffffu, pa, d), da = __shfl_down_sync(0xffffffffu, sa, d);
        const float uo = __shfl_up_sync(0xffffffffu, po, d), dn = __shfl_down_sync(0xffffffffu, so, d);
        if (lane >= d) pa = fmaxf(pa, ua), po = fmaxf(po, uo);
        if (lane + d < 32u) sa = fmaxf(sa, da), so = fmaxf(so, dn);
    }
    preA[c] = pa, sufA[c] = sa, preO[c] = po, sufO[c] = so;
    if (lane == 0) bmA[c >> 5] = sa, bmO[c >> 5] = so;
}

__global__ void __launch_bounds__(1024) k_full_b(const PerInputParams p) {
    extern __shared__ float s_tab[];  // [2][levels][nb]
    const Geometry& g = p.g;
    const FullLearn& fl = p.fl;
    const uint32_t tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31u;
    const uint32_t nb = g.C32 / 32u, Lv = wmax_levels(nb);
    const float* preA = fl.scratch;
    const float* sufA = preA + g.C32;
    const float* preO = sufA + g.C32;
    const float* sufO = preO + g.C32;
    const float* bmA = sufO + g.C32;
    const float* bmO = bmA + nb;
    unsigned long long* acc = reinterpret_cast<unsigned long long*>(fl.scratch + 4u * g.C32 + 2u * nb + 2u);
    uint32_t* ticket = reinterpret_cast<uint32_t*>(acc + 1);
    float* tA = s_tab;
    float* tO = s_tab + Lv * nb;
    for (uint32_t b = tid; b < nb; b += nthr) tA[b] = bmA[b], tO[b] = bmO[b];
    __syncthreads();
    for (uint32_t l = 1; l < Lv; ++l) {
        const uint32_t half = 1u << (l - 1);
        for (uint32_t b = tid; b + (1u << l) <= nb; b += nthr) {
            tA[l * nb + b] = fmaxf(tA[(l - 1) * nb + b], tA[(l - 1) * nb + b + half]);
            tO[l * nb + b] = fmaxf(tO[(l - 1) * nb + b], tO[(l - 1) * nb + b + half]);
        }
        __syncthreads();
    }
    const uint32_t r = *fl.radius;  // radius in force for this input (R18)
    const uint32_t c0 = blockIdx.x * g.C / gridDim.x, c1 = (blockIdx.x + 1u) * g.C / gridDim.x;
    for (uint32_t c = c0 + tid; c < c1; c += nthr) {  // (c) boosts
        const float b = boost_rule(fl.adc[c], wmax_query(fl.adc, preA, sufA, tA, nb, g.C, c, r), fl.mb1);
        fl.boost[c] = b;
        fl.bc[c] = boost_bc(b);
    }
    for (uint32_t c = c0 + (tid >> 5); c < c1; c += nthr >> 5) {  // (d) bumps, warp per column
        if (!weak_column(fl.odc[c], wmax_query(fl.odc, preO, sufO, tO, nb, g.C, c, r))) continue;
        const uint32_t* idx = p.idx + static_cast<size_t>(c) * g.S;
        float* perm = p.perm + static_cast<size_t>(c) * g.S;
        uint32_t smin = 0xFFFFFFFFu, smax = 0u;
        for (uint32_t s = lane; s < g.S; s += 32u) {
            const float v = fminf(__fadd_rn(perm[s], fl.bump), 1.0f);
            perm[s] = v;
            p.syn_rw[static_cast<size_t>(s) * g.C32 + c] = idx[s] | (v >= p.tau ? 0x80000000u : 0u);
            span_accumulate(v >= p.tau, s, smin, smax);
        }
        const uint32_t sp_c = span_finish(smin, smax, idx, 0xFFFFFFFFu);
        if (lane == 0) fl.span[c] = sp_c;
    }
    if (!fl.adapt) return;
    __syncthreads();
    // (e) this range's span sum; the last CTA forms the radius and resets the accumulator
    __shared__ unsigned long long s_part;
    __shared__ uint32_t s_last;
    if (tid == 0) s_part = 0ull;
    __syncthreads();
    unsigned long long part = 0;
    for (uint32_t c = c0 + tid; c < c1; c += nthr) part += fl.span[c];
    for (uint32_t d = 16; d > 0; d >>= 1) part += __shfl_xor_sync(0xffffffffu, part, d);
    if (lane == 0 && part) atomicAdd(&s_part, part);
    __syncthreads();
    if (tid == 0) {
        atomicAdd(acc, s_part);
        __threadfence();
        s_last = atomicAdd(ticket, 1u) + 1u == gridDim.x ? 1u : 0u;
    }
    __syncthreads();
    if (s_last && tid == 0) {
        __threadfence();
        const unsigned long long total = atomicAdd(acc, 0ull);
        *fl.radius = adapt_radius(total, g.nbits, g.C);
        *acc = 0ull;
        *ticket = 0u;
    }
}

// spans of every column from the canonical arrays (warp per column; R21)
__global__ void k_span(const uint32_t* idx, const float* perm, float tau, uint32_t C, uint32_t S, uint32_t* span) {
    const uint32_t c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint32_t lane = threadIdx.x & 31u;
    if (c >= C) return;
    uint32_t smin = 0xFFFFFFFFu, smax = 0u;
    for (uint32_t s = lane; s < S; s += 32u) span_accumulate(perm[static_cast<size_t>(c) * S + s] >= tau, s, smin, smax);
    const uint32_t v = span_finish(smin, smax, idx + static_cast<size_t>(c) * S, 0xFFFFFFFFu);
    if (lane == 0) span[c] = v;
}

// syn[s][c] = idx | connected << 31 from the canonical arrays; pad columns point nowhere.
__global__ void k_build_syn(const uint32_t* idx, const float* perm, float tau, uint32_t C,
                            uint32_t C32, uint32_t S, uint32_t* syn) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t s = blockIdx.y;
    if (c >= C32 || s >= S) return;
    uint32_t v = 0u;  // pad column: disconnected synapse on input 0
    if (c < C) {
        const size_t k = static_cast<size_t>(c) * S + s;
        v = idx[k] | (perm[k] >= tau ? 0x80000000u : 0u);
    }
    syn[static_cast<size_t>(s) * C32 + c] = v;
}

// synT[c][s] = idx | connected << 31 (column-major, grid learning); pad columns: 0.
__global__ void k_build_synT(const uint32_t* idx, const float* perm, float tau, uint32_t C, uint32_t C32,
                             uint32_t S, uint32_t* synT) {
    const size_t k = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= static_cast<size_t>(C32) * S) return;
    synT[k] = k < static_cast<size_t>(C) * S ? (idx[k] | (perm[k] >= tau ? 0x80000000u : 0u)) : 0u;
}

// Batched ELL: slot pos[c][s] holds the window-local index if connected, else the zero slot Lw.
__global__ void k_refresh_ell(const uint32_t* idx, const float* perm, const uint32_t* pos,
                              float tau, uint32_t n, uint32_t Lw, uint16_t* ell) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint32_t i = idx[k];
    ell[pos[k]] = static_cast<uint16_t>(perm[k] >= tau ? i % Lw : Lw);
}

}  // namespace

cudaError_t launch_pack(const PerInputParams& p, cudaStream_t s) {
    dim3 grid((p.Wn + 255u) / 256u, p.num_inputs);
    k_pack<<<grid, 256, 0, s>>>(p);
    return cudaGetLastError();
}

template <typename F>
static cudaError_t allow_dynamic_smem(F* fn, int max_smem) {
    cudaFuncAttributes a{};
    cudaError_t e = cudaFuncGetAttributes(&a, fn);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                max_smem - static_cast<int>(a.sharedSizeBytes));
}

uint32_t inhibit_wavelet_smem(const Geometry& g) {
    return g.C32 * 8u + 16u * (g.ncw + 2u) * 8u;  // pairs x 2, <= 15 levels + the lossy level
}

cudaError_t configure_per_input(int max_smem) {
    cudaError_t e = allow_dynamic_smem(k_overlap, max_smem);
    if (e == cudaSuccess) e = allow_dynamic_smem(k_inhibit, max_smem);
    if (e == cudaSuccess) e = allow_dynamic_smem(k_full_b, max_smem);
    return e;
}

cudaError_t launch_overlap(const PerInputParams& p, cudaStream_t s) {
    const uint32_t smem = p.Wn * 4u;
    dim3 grid((p.g.C32 + 63u) / 64u, p.num_inputs);
    k_overlap<<<grid, 256, smem, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_inhibit(const PerInputParams& p, cudaStream_t s, uint32_t parts) {
    uint32_t smem = p.g.C32 * 8u + p.g.ncw * 16u * 4u;  // raw, Bc, bit-planes
    if (p.wm_ok) smem = max(smem, inhibit_wavelet_smem(p.g));
    const uint32_t threads = p.g.C32 < 1024u ? p.g.C32 : 1024u;
    if (parts > 1u) {
        cudaError_t e = cudaMemsetAsync(p.counts + p.first_input, 0, p.num_inputs * 4u, s);
        if (e != cudaSuccess) return e;
    }
    k_inhibit<<<dim3(p.num_inputs, parts), threads, smem, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_learn(const PerInputParams& p, uint32_t input, cudaStream_t s) {
    const uint32_t warps = 8;
    k_learn<<<(p.g.C + warps - 1) / warps, warps * 32, 0, s>>>(p, input);
    return cudaGetLastError();
}

cudaError_t launch_full(const PerInputParams& p, uint32_t input, cudaStream_t s, uint32_t* launches) {
    const uint32_t C32 = p.g.C32;
    if (C32 < 4096u || std::getenv("SP_FULL_ONE_CTA")) {
        k_full<<<1, 1024, 0, s>>>(p, input);
        *launches = 1;
        return cudaGetLastError();
    }
    const uint32_t nb = C32 / 32u;
    k_full_a<<<(C32 + 1023u) / 1024u, 1024, 0, s>>>(p, input);
    const uint32_t G = std::min<uint32_t>(148u, (p.g.C + 255u) / 256u);
    k_full_b<<<G, 1024, 2u * wmax_levels(nb) * nb * 4u, s>>>(p);
    *launches = 2;
    return cudaGetLastError();
}

cudaError_t launch_span(const uint32_t* idx, const float* perm, float tau, uint32_t C, uint32_t S,
                        uint32_t* span, cudaStream_t s) {
    k_span<<<(C + 7u) / 8u, 256, 0, s>>>(idx, perm, tau, C, S, span);
    return cudaGetLastError();
}

size_t full_scratch_floats(uint32_t C32) {
    const size_t nb = C32 / 32u;
    return std::max<size_t>(2u * C32 + wmax_levels(nb) * nb + 32u, 4u * C32 + 2u * nb + 8u);
}

cudaError_t launch_build_syn(const uint32_t* idx, const float* perm, float tau, uint32_t C,
                             uint32_t C32, uint32_t S, uint32_t* syn, cudaStream_t s) {
    dim3 grid((C32 + 255u) / 256u, S);
    k_build_syn<<<grid, 256, 0, s>>>(idx, perm, tau, C, C32, S, syn);
    return cudaGetLastError();
}

cudaError_t launch_build_synT(const uint32_t* idx, const float* perm, float tau, uint32_t C, uint32_t C32,
                              uint32_t S, uint32_t* synT, cudaStream_t s) {
    const size_t n = static_cast<size_t>(C32) * S;
    k_build_synT<<<static_cast<uint32_t>((n + 255u) / 256u), 256, 0, s>>>(idx, perm, tau, C, C32, S, synT);
    return cudaGetLastError();
}

cudaError_t launch_refresh_ell(const uint32_t* idx, const float* perm, const uint32_t* pos,
                               float tau, uint32_t C, uint32_t S, uint32_t Lw, uint16_t* ell,
                               cudaStream_t s) {
    const uint32_t n = C * S;
    k_refresh_ell<<<(n + 255u) / 256u, 256, 0, s>>>(idx, perm, pos, tau, n, Lw, ell);
    return cudaGetLastError();
}

}  // namespace sp
