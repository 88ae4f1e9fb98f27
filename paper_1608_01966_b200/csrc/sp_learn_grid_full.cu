// sp_learn_grid_full.cu — grid-resident sequential learning WITH the full learning step
// (SURVEY §8(a) a1-a5 + §8(f) NEXT-1; S:119(a-e); R17-R21, §4.2d) for SPs
// whose synapse table does not fit a cluster (BASELINE config 5: 16384 columns x 512 synapses,
// radius adapted 80 -> ~C/2).
//
// One cooperative launch, G co-resident CTAs (one per SM); CTA b owns the column-words
// [b*ncw/G, (b+1)*ncw/G) for every step.  Per input t, with R the radius in force:
//
//   a2   overlap of the owned columns (synapse slice streamed from L2 through a TMA ring, as in
//        sp_learn_grid.cu); raw counts -> global (by input parity)
//        ---- grid barrier B1 ----
//   (e') R for this input = adapt(sum of the per-CTA connected-span sums of input t-1)
//   a3/a4 k-winners of the owned columns by CTA-level candidate pruning: over the union U of
//        the owned columns' windows, v = N >> vsh (monotone in the exact key); the largest t
//        with >= k values >= t in the window core shared by every owned column (bitwise search,
//        block reductions) makes every column with v < t a loser; the candidates of U (v >= t)
//        are compacted in position order with their exact keys, and each owned candidate counts
//        the larger keys among the candidates of its window (a contiguous range), warp-wide
//   (a)  permanence update of the owned winners; their connected spans
//   (b)  duty cycles of the owned columns; in-block prefix/suffix maxima and block maxima of
//        both duty arrays -> global scratch
//        ---- grid barrier B2 ----
//   (c)  boosts of the owned columns from the window maxima of the active duty cycles (block
//        maxima of the fully covered 32-column blocks + the prefix/suffix maxima of the two
//        partial blocks)
//   (d)  bump of the owned weak columns (window maxima of the overlap duty cycles); spans
//        per-CTA span sum -> global (by input parity), read by every CTA after the next B1
//
// A CTA only updates its own columns; other CTAs read them only across a grid barrier: raw
// counts and duty tables after B1/B2 of the same input, boosts (written after B2 of t) in the
// selection of t+1 (after B1 of t+1), span sums of t after B1 of t+1.  Two grid barriers per
// input.
#include <cooperative_groups.h>

#include "sp_duty.cuh"
#include "sp_grid.cuh"
#include "sp_internal.h"
#include "sp_pack.cuh"
#include "sp_select.cuh"

namespace sp {

namespace {

constexpr uint32_t kGfThreads = 512;
constexpr uint32_t kGfWarps = kGfThreads / 32;
constexpr uint32_t kGfPer = 32;  // columns of the union window per thread (C32 <= 16384)

// block sum of x (every thread gets it); buf = 16 words of shared scratch used alternately
__device__ __forceinline__ uint32_t block_sum(uint32_t x, uint32_t* buf) {
    x = __reduce_add_sync(0xffffffffu, x);
    if ((threadIdx.x & 31u) == 0) buf[threadIdx.x >> 5] = x;
    __syncthreads();
    uint32_t s = 0;
#pragma unroll
    for (uint32_t w = 0; w < kGfWarps; ++w) s += buf[w];
    return s;
}

__device__ __forceinline__ float block_fmax(float x, float* buf) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, d));
    if ((threadIdx.x & 31u) == 0) buf[threadIdx.x >> 5] = x;
    __syncthreads();
    float m = 0.0f;
#pragma unroll
    for (uint32_t w = 0; w < kGfWarps; ++w) m = fmaxf(m, buf[w]);
    return m;
}

// first index i in [0, n) with pos[i] >= x (n if none)
__device__ __forceinline__ uint32_t lower_bound_u16(const uint16_t* pos, uint32_t n, uint32_t x) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (pos[mid] < x) lo = mid + 1u;
        else hi = mid;
    }
    return lo;
}

}  // namespace

__global__ void __launch_bounds__(kGfThreads, 1)
    sp_learn_grid_full_kernel(const __grid_constant__ LearnGridParams p) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ __align__(8) uint64_t s_bar_bits;
    __shared__ __align__(8) uint64_t s_bar_ring[8];
    __shared__ uint32_t s_red[4][kGfWarps];
    __shared__ float s_fred[4][kGfWarps];
    __shared__ uint32_t s_scan[kGfWarps];
    __shared__ uint32_t s_R, s_noc, s_P;
    __shared__ unsigned long long s_span;
    const Geometry& g = p.g;
    const FullLearn& fl = p.fl;
    const uint32_t tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31u, wi = tid >> 5, nw = nthr >> 5;
    const uint32_t b = blockIdx.x, G = p.G, n = p.num_inputs;
    const uint32_t S = g.S, C = g.C, C32 = g.C32, ncw = g.ncw;
    const uint32_t Wn4 = (p.Wn + 3u) / 4u * 4u;
    const uint32_t wb0 = b * ncw / G, wb1 = (b + 1u) * ncw / G, nown = wb1 - wb0;
    const uint32_t c0 = wb0 * 32u, ncols = nown * 32u;
    const uint32_t c1 = min(C, c0 + ncols);  // owned real columns [c0, c1)
    const uint32_t ccols = p.ccols, stages = p.stages, chunk_words = ccols * S;
    const uint32_t nchunks = ncols / ccols;
    const uint32_t wpc = kGfWarps / ccols;
    const uint32_t span = S / wpc;
    const bool vec_ok = S % wpc == 0u && span % 4u == 0u;
    const uint32_t theta = p.min_overlap, L = g.keyL, k = p.k, cap = p.cand_cap, vsh = p.vsh;

    uint32_t* s_bits = reinterpret_cast<uint32_t*>(smem);                        // [Wn4]
    uint32_t* s_ring = s_bits + Wn4;                                              // [stages][chunk]
    uint32_t* s_craw = s_ring + static_cast<size_t>(stages) * chunk_words;        // [own cols]
    uint32_t* s_sdr = s_craw + p.own_words * 32u;                                 // [own words (+1)]
    uint32_t* s_oc = s_sdr + (p.own_words + 3u) / 4u * 4u;                        // [own cols] owned candidates
    uint64_t* s_key = reinterpret_cast<uint64_t*>(s_oc + p.own_words * 32u);      // [cap] (16-byte aligned)
    uint16_t* s_rw = reinterpret_cast<uint16_t*>(s_key + cap);                    // [C32]
    uint16_t* s_pos = s_rw + C32;                                                 // [cap]
    float* preA = fl.scratch;
    float* sufA = preA + C32;
    float* preO = sufA + C32;
    float* sufO = preO + C32;
    float* bmA = sufO + C32;
    float* bmO = bmA + ncw;
    const uint32_t* my_syn = p.synT + static_cast<size_t>(c0) * S;
    const uint32_t bits_bytes = (p.Wn * 4u + 15u) & ~15u;
    auto gbits_of = [&](uint32_t t) { return p.bits_g + static_cast<size_t>(t) * Wn4; };  // prepacked
    // phase timers of CTA 0 / thread 0 (SP_TRACE): [0] bit-plane wait, [1] overlap, [2] B1 + radius,
    // [3] selection, [4] (a) + (b), [5] B2, [6] (c) (d) (e); [7] running timestamp
    // selection sub-phases (SP_TRACE): [8] raw row load, [9] values, [10] threshold, [11] compaction
    // + owned candidates, [12] beats + SDR
    __shared__ uint64_t s_tr[13];
    const bool tr = p.trace != nullptr && b == 0 && tid == 0;
    if (tr)
        for (int i = 0; i < 13; ++i) s_tr[i] = 0;
    auto stamp = [&](int i) {
        if (tr) {
            const uint64_t now = globaltimer();
            s_tr[i] += now - s_tr[7];
            s_tr[7] = now;
        }
    };

    // ---- prologue -------------------------------------------------------------------------
    if (tid == 0) {
        mbar_init(&s_bar_bits, 1);
        for (uint32_t i = 0; i < stages; ++i) mbar_init(&s_bar_ring[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        s_R = *fl.radius;
    }
    for (uint32_t i = b * nthr + tid; i < n; i += G * nthr) p.counts[p.first_input + i] = 0u;
    uint32_t nbar = 0;
    grid_barrier(p.gbar, ++nbar * G);
    uint32_t bits_phase = 0, cc = 0, ring_slot = 0, ring_par = 0;
    if (tid == 0 && n > 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        bulk_copy(s_bits, gbits_of(0), bits_bytes, &s_bar_bits);
    }

    for (uint32_t t = 0; t < n; ++t) {
        const uint32_t gin = p.first_input + t;
        const uint16_t* raw_src = p.raw_g + (t & 1u) * C32;
        if (tr) s_tr[7] = globaltimer();
        const bool ring = p.dbg & 64u;  // development: the TMA chunk ring of sp_learn_grid.cu
        if (tid == 0 && ring) {
            asm volatile("fence.proxy.async.global;" ::: "memory");  // flag stores -> TMA reads
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            for (uint32_t j = 0; j < min(stages, nchunks); ++j)
                bulk_copy(s_ring + ((cc + j) % stages) * chunk_words, my_syn + static_cast<size_t>(j) * chunk_words,
                          chunk_words * 4u, &s_bar_ring[(cc + j) % stages]);
        }
        if (tid == 0 && b == 0 && t + 2u < n) prefetch_l2(gbits_of(t + 2u), Wn4 * 4u);
        for (uint32_t i = tid; i < ncols; i += nthr) s_craw[i] = 0u;
        mbar_wait(&s_bar_bits, bits_phase);
        bits_phase ^= 1u;
        __syncthreads();
        stamp(0);
        // ---- a2: overlap of the owned columns ------------------------------------------------
        // warp per column pair: the synapse rows (idx | connected << 31, contiguous, L2-resident)
        // by 16-byte L2 loads, 8 in flight per lane; the input bits from shared memory
        auto hit = [&](uint32_t e) { return (s_bits[(e & 0x7FFFFFFFu) >> 5] >> (e & 31u)) & (e >> 31); };
        const uint32_t S4 = S / 4u;  // S % 4 == 0 (grid eligibility)
        for (uint32_t cl0 = wi; !ring && cl0 < ncols; cl0 += 2u * nw) {
            const uint32_t clb = cl0 + nw;
            const uint4* ra = reinterpret_cast<const uint4*>(p.synT + static_cast<size_t>(c0 + cl0) * S);
            const uint4* rb = reinterpret_cast<const uint4*>(p.synT + static_cast<size_t>(c0 + min(clb, ncols - 1u)) * S);
            uint32_t xa = 0, xb = 0;
            for (uint32_t q0 = 0; q0 < S4; q0 += 128u) {
                uint4 ea[4], eb[4];
#pragma unroll
                for (uint32_t u = 0; u < 4u; ++u) {
                    const uint32_t q = q0 + lane + 32u * u;
                    ea[u] = q < S4 ? __ldcg(ra + q) : make_uint4(0u, 0u, 0u, 0u);
                    eb[u] = (q < S4 && clb < ncols) ? __ldcg(rb + q) : make_uint4(0u, 0u, 0u, 0u);
                }
#pragma unroll
                for (uint32_t u = 0; u < 4u; ++u) {
                    xa += (hit(ea[u].x) + hit(ea[u].y)) + (hit(ea[u].z) + hit(ea[u].w));
                    xb += (hit(eb[u].x) + hit(eb[u].y)) + (hit(eb[u].z) + hit(eb[u].w));
                }
            }
            xa = __reduce_add_sync(0xffffffffu, xa);
            xb = __reduce_add_sync(0xffffffffu, xb);
            if (lane == 0) {
                s_craw[cl0] = xa;
                if (clb < ncols) s_craw[clb] = xb;
            }
        }
        if (!ring) __syncthreads();
        for (uint32_t j = 0; ring && j < nchunks; ++j, ++cc) {
            const uint32_t slot = ring_slot, parity = ring_par;
            if (++ring_slot == stages) ring_slot = 0, ring_par ^= 1u;
            mbar_wait(&s_bar_ring[slot], parity);
            const uint32_t* ch = s_ring + slot * chunk_words;
            const uint32_t jc = wi / wpc, part = wi % wpc;
            const uint32_t* col = ch + jc * S;
            uint32_t r0 = 0, r1 = 0;
            if (vec_ok) {
                const uint32_t lo = part * span, hi = lo + span;
                for (uint32_t s = lo + 4u * lane; s < hi; s += 256u) {
                    const uint4 a = *reinterpret_cast<const uint4*>(col + s);
                    const uint4 c2 = s + 128u < hi ? *reinterpret_cast<const uint4*>(col + s + 128u)
                                                   : make_uint4(0u, 0u, 0u, 0u);
                    r0 += (hit(a.x) + hit(a.y)) + (hit(a.z) + hit(a.w));
                    r1 += (hit(c2.x) + hit(c2.y)) + (hit(c2.z) + hit(c2.w));
                }
            } else {
                uint32_t s = part * 32u + lane;
                const uint32_t step = wpc * 32u;
                for (; s + step < S; s += 2u * step) {
                    r0 += hit(col[s]);
                    r1 += hit(col[s + step]);
                }
                if (s < S) r0 += hit(col[s]);
            }
            const uint32_t raw = __reduce_add_sync(0xffffffffu, r0 + r1);
            if (lane == 0 && raw) atomicAdd(&s_craw[j * ccols + jc], raw);
            __syncthreads();
            if (tid == 0 && j + stages < nchunks) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                bulk_copy(s_ring + slot * chunk_words, my_syn + static_cast<size_t>(j + stages) * chunk_words,
                          chunk_words * 4u, &s_bar_ring[slot]);
            }
        }
        for (uint32_t i = tid; i < ncols; i += nthr) {
            const uint32_t c = c0 + i, raw = s_craw[i];
            p.raw_g[(t & 1u) * C32 + c] = static_cast<uint16_t>(raw);
            if (p.raw_out && c < C) {
                p.raw_out[static_cast<size_t>(gin) * C + c] = static_cast<uint16_t>(raw);
                p.boosted_out[static_cast<size_t>(gin) * C + c] =
                    raw >= theta ? __fmul_rn(static_cast<float>(raw), p.boost[c]) : 0.0f;
            }
        }
        stamp(1);
        grid_barrier(p.gbar, ++nbar * G);  // B1: raw counts of t; span sums of t-1
        // (e) the radius in force for input t, from the span sums of input t-1 (R21)
        if (t > 0 && fl.adapt) {
            if (wi == 0) {
                unsigned long long sum = 0;
                for (uint32_t i = lane; i < G; i += 32u) sum += __ldcg(p.span_part + ((t - 1u) & 1u) * G + i);
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, d);
                if (lane == 0) s_R = adapt_radius(sum, g.nbits, C);
            }
            __syncthreads();
        }
        stamp(2);
        const uint32_t R = s_R;
        const uint32_t Re = (R == 0u || R >= C) ? C : R;  // 0 = global (all columns)
        // ---- a3/a4: k-winners of the owned columns (candidate pruning) ---------------------
        const uint32_t ulo = c0 >= Re ? c0 - Re : 0u, uhi = min(C - 1u, c1 - 1u + Re);  // union window
        const uint32_t klo = c1 - 1u >= Re ? c1 - 1u - Re : 0u, khi = min(C - 1u, c0 + Re);  // common core
        const bool core = klo <= khi;
        // U aligned down to 32 columns; raw counts -> s_rw, Bc -> the synapse ring (idle until the
        // next input's overlap) when it holds U, both by 16-byte coalesced loads
        const uint32_t ua = ulo & ~31u, nu = uhi - ua + 1u;
        for (uint32_t c8 = ua / 8u + tid; c8 <= uhi / 8u; c8 += nthr)
            reinterpret_cast<uint4*>(s_rw)[c8] = __ldcg(reinterpret_cast<const uint4*>(raw_src) + c8);
        const bool bc_smem = stages * chunk_words >= ((nu + 3u) & ~3u);
        uint32_t* s_bcu = s_ring - ua;  // s_bcu[c], c in U (when bc_smem)
        if (bc_smem)
            for (uint32_t c4 = ua / 4u + tid; c4 <= uhi / 4u; c4 += nthr)
                reinterpret_cast<uint4*>(s_ring)[c4 - ua / 4u] = __ldcg(reinterpret_cast<const uint4*>(p.bc) + c4);
        for (uint32_t i = tid; i < nown; i += nthr) s_sdr[i] = 0u;
        if (tid == 0) s_noc = 0u, s_P = 0u;
        __syncthreads();
        auto bc_of = [&](uint32_t c) { return bc_smem ? s_bcu[c] : __ldcg(p.bc + c); };
        stamp(8);
        // thread i: columns ua + i + 512 j (conflict-free shared loads), v two per register
        uint32_t vv[kGfPer / 2];
        uint32_t tmax = 0;  // largest v of this thread's core columns
#pragma unroll
        for (uint32_t j = 0; j < kGfPer; j += 2u) {
            uint32_t v2[2];
#pragma unroll
            for (uint32_t e2 = 0; e2 < 2u; ++e2) {
                const uint32_t c = ua + tid + kGfThreads * (j + e2);
                uint32_t v = 0;
                if (c >= ulo && c <= uhi) {
                    const uint64_t N = eligible_N(s_rw[c], bc_of(c), theta);
                    v = N ? max(1u, static_cast<uint32_t>(N >> vsh)) : 0u;
                    if (c >= klo && c <= khi) tmax = max(tmax, v);
                }
                v2[e2] = v;
            }
            vv[j / 2u] = v2[0] | (v2[1] << 16);
        }
        stamp(9);
        // t: the largest value with >= k threads whose core maximum reaches it -- then >= k core
        // columns have v >= t (valid), and t is close to the core's k-th largest value
        uint32_t tthr = 0;
        if (core) {
            for (int bit = 15; bit >= 0; --bit) {
                const uint32_t tt = tthr | (1u << bit);
                if (__syncthreads_count(tmax >= tt) >= static_cast<int>(k)) tthr = tt;
            }
        }
        tthr = max(tthr, 1u);
        stamp(10);
        // the candidates of U (v >= t), unordered (warp-aggregated appends), with exact keys; the
        // owned ones also into s_oc
#pragma unroll
        for (uint32_t j = 0; j < kGfPer; ++j) {
            const uint32_t c = ua + tid + kGfThreads * j;
            const bool is = ((vv[j / 2u] >> (16u * (j & 1u))) & 0xFFFFu) >= tthr;
            const uint32_t bal = __ballot_sync(0xffffffffu, is);
            if (bal == 0u) continue;
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(&s_P, static_cast<uint32_t>(__popc(bal)));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (is) {
                const uint32_t at = base + __popc(bal & ((1u << lane) - 1u));
                uint64_t N;
                const uint64_t key = exact_key(s_rw[c], bc_of(c), theta, c, L, N);
                if (at < cap) s_pos[at] = static_cast<uint16_t>(c), s_key[at] = key;
                if (c >= c0 && c < c1) s_oc[atomicAdd(&s_noc, 1u)] = c;
            }
        }
        __syncthreads();
        stamp(11);
        const uint32_t P = s_P;
        const bool listed = P <= cap;
        // beats of each owned candidate among the candidates of its window: a warp per candidate
        const uint32_t noc = s_noc;
        for (uint32_t q = wi; q < noc; q += nw) {
            const uint32_t c = s_oc[q];
            const uint32_t lo = c >= Re ? c - Re : 0u, hi = min(C - 1u, c + Re);
            uint64_t N;
            const uint64_t key = exact_key(s_rw[c], bc_of(c), theta, c, L, N);
            uint32_t beats = 0;
            if (listed) {
                for (uint32_t j0 = 0; j0 < P && beats < k; j0 += 32u) {
                    const uint32_t j = j0 + lane;
                    bool gt = false;
                    if (j < P) {
                        const uint32_t d = s_pos[j];
                        gt = d >= lo && d <= hi && s_key[j] > key;
                    }
                    beats += __popc(__ballot_sync(0xffffffffu, gt));
                }
            } else {  // direct scan of the window (every column of it)
                for (uint32_t d0 = lo; d0 <= hi && beats < k; d0 += 32u) {
                    const uint32_t d = d0 + lane;
                    bool gt = false;
                    if (d <= hi) {
                        uint64_t Nd;
                        gt = exact_key(s_rw[d], __ldcg(p.bc + d), theta, d, L, Nd) > key;
                    }
                    beats += __popc(__ballot_sync(0xffffffffu, gt));
                }
            }
            if (lane == 0 && beats < k) atomicOr(&s_sdr[(c - c0) >> 5], 1u << (c & 31u));
        }
        __syncthreads();  // s_sdr complete
        for (uint32_t i = tid; i < nown; i += nthr) {
            const uint32_t word = s_sdr[i];
            p.sdr[static_cast<size_t>(gin) * ncw + wb0 + i] = word;
            if (word) atomicAdd(p.counts + gin, static_cast<uint32_t>(__popc(word)));
        }
        stamp(12);
        // ---- (a) permanence update of the owned winners (warp per column) + their spans ----
        for (uint32_t cl = wi; cl < ncols; cl += nw) {
            const uint32_t c = c0 + cl;
            if (c >= C) break;
            if (((s_sdr[cl >> 5] >> (cl & 31u)) & 1u) == 0u) continue;
            float* __restrict__ perm = p.perm + static_cast<size_t>(c) * S;
            uint32_t* __restrict__ syn = p.synT + static_cast<size_t>(c) * S;
            uint32_t smin = 0xFFFFFFFFu, smax = 0u;
            for (uint32_t s0 = 0; s0 < S; s0 += 512u) {
                float4 v[4];
                uint4 e[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t s = s0 + 128u * q + 4u * lane;
                    if (s < S) {
                        v[q] = __ldcg(reinterpret_cast<const float4*>(perm + s));
                        e[q] = __ldcg(reinterpret_cast<const uint4*>(syn + s));
                    }
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t s = s0 + 128u * q + 4u * lane;
                    if (s < S) {
                        float* vq = &v[q].x;
                        uint32_t* eq = &e[q].x;
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) {
                            const uint32_t i = eq[kk] & 0x7FFFFFFFu;
                            const bool on = ((s_bits[i >> 5] >> (i & 31u)) & 1u) != 0u;
                            float x = on ? __fadd_rn(vq[kk], p.inc) : __fsub_rn(vq[kk], p.dec);
                            x = fminf(fmaxf(x, 0.0f), 1.0f);
                            vq[kk] = x;
                            eq[kk] = i | (x >= p.tau ? 0x80000000u : 0u);
                            span_accumulate(x >= p.tau, s + kk, smin, smax);
                        }
                        *reinterpret_cast<float4*>(perm + s) = v[q];
                        *reinterpret_cast<uint4*>(syn + s) = e[q];
                    }
                }
            }
            const uint32_t sp_c = span_finish(smin, smax, syn, 0x7FFFFFFFu);
            if (lane == 0) fl.span[c] = sp_c;
        }
        // ---- (b) duty cycles of the owned columns; window-maximum tables -> global ---------
        for (uint32_t ow = wi; ow < nown; ow += nw) {
            const uint32_t c = c0 + ow * 32u + lane;
            float a = 0.0f, o = 0.0f;
            if (c < C) {
                const bool act = ((s_sdr[ow] >> lane) & 1u) != 0u;
                const uint32_t raw = s_craw[ow * 32u + lane];
                a = duty_update(fl.adc[c], act, fl.pm1, fl.P);
                o = duty_update(fl.odc[c], raw >= theta && raw > 0u, fl.pm1, fl.P);  // N > 0
                fl.adc[c] = a;
                fl.odc[c] = o;
            }
            float pa = a, sa = a, po = o, so = o;
#pragma unroll
            for (uint32_t d = 1; d < 32u; d <<= 1) {
                const float ua = __shfl_up_sync(0xffffffffu, pa, d), da = __shfl_down_sync(0xffffffffu, sa, d);
                const float uo = __shfl_up_sync(0xffffffffu, po, d), dn = __shfl_down_sync(0xffffffffu, so, d);
                if (lane >= d) pa = fmaxf(pa, ua), po = fmaxf(po, uo);
                if (lane + d < 32u) sa = fmaxf(sa, da), so = fmaxf(so, dn);
            }
            const uint32_t cc2 = c0 + ow * 32u + lane;
            preA[cc2] = pa, sufA[cc2] = sa, preO[cc2] = po, sufO[cc2] = so;
            if (lane == 0) bmA[wb0 + ow] = sa, bmO[wb0 + ow] = so;
        }
        stamp(4);
        grid_barrier(p.gbar, ++nbar * G);  // B2: duty tables of t complete
        stamp(5);
        // ---- (c) boosts and (d) weak-column bumps of the owned columns ----------------------
        // window maxima over W(c) = [lo, hi]: partial blocks by the in-block prefix/suffix maxima,
        // the fully covered blocks by the block maxima; the blocks covered for every owned column
        // (core K) are reduced once per CTA
        const uint32_t kb0 = ((c1 - 1u >= Re ? c1 - 1u - Re : 0u) >> 5) + 1u;       // bl(c1-1) + 1
        const uint32_t kb1 = (min(C - 1u, c0 + Re) >> 5);                            // bh(c0) (exclusive)
        float mcA = 0.0f, mcO = 0.0f;
        const bool kcore = kb0 + 8u < kb1;
        if (kcore) {
            float xa = 0.0f, xo = 0.0f;
            for (uint32_t bk = kb0 + tid; bk < kb1; bk += nthr) xa = fmaxf(xa, __ldcg(bmA + bk)), xo = fmaxf(xo, __ldcg(bmO + bk));
            mcA = block_fmax(xa, s_fred[0]);
            mcO = block_fmax(xo, s_fred[1]);
        }
        auto wmax = [&](const float* v, const float* pre, const float* suf, const float* bm, float mc, uint32_t c) {
            const uint32_t lo = c >= Re ? c - Re : 0u, hi = min(C - 1u, c + Re);
            const uint32_t bl = lo >> 5, bh = hi >> 5;
            if (bl == bh) {
                float m = 0.0f;
                for (uint32_t d = lo; d <= hi; ++d) m = fmaxf(m, __ldcg(v + d));
                return m;
            }
            float m = fmaxf(__ldcg(suf + lo), __ldcg(pre + hi));
            if (kcore) {
                m = fmaxf(m, mc);
                for (uint32_t bk = bl + 1u; bk < kb0; ++bk) m = fmaxf(m, __ldcg(bm + bk));
                for (uint32_t bk = kb1; bk < bh; ++bk) m = fmaxf(m, __ldcg(bm + bk));
            } else {
                for (uint32_t bk = bl + 1u; bk < bh; ++bk) m = fmaxf(m, __ldcg(bm + bk));
            }
            return m;
        };
        for (uint32_t c = c0 + tid; c < c1; c += nthr) {
            const float bst = boost_rule(__ldcg(fl.adc + c), wmax(fl.adc, preA, sufA, bmA, mcA, c), fl.mb1);
            fl.boost[c] = bst;
            fl.bc[c] = boost_bc(bst);
            const bool weak = weak_column(__ldcg(fl.odc + c), wmax(fl.odc, preO, sufO, bmO, mcO, c));
            s_craw[c - c0] = weak ? 1u : 0u;  // the raw counts are no longer needed
        }
        __syncthreads();
        for (uint32_t cl = wi; cl < c1 - c0; cl += nw) {
            if (!s_craw[cl]) continue;
            const uint32_t c = c0 + cl;
            float* __restrict__ perm = p.perm + static_cast<size_t>(c) * S;
            uint32_t* __restrict__ syn = p.synT + static_cast<size_t>(c) * S;
            uint32_t smin = 0xFFFFFFFFu, smax = 0u;
            for (uint32_t s = lane; s < S; s += 32u) {
                const float v = fminf(__fadd_rn(__ldcg(perm + s), fl.bump), 1.0f);
                perm[s] = v;
                syn[s] = (syn[s] & 0x7FFFFFFFu) | (v >= p.tau ? 0x80000000u : 0u);
                span_accumulate(v >= p.tau, s, smin, smax);
            }
            __syncwarp();
            const uint32_t sp_c = span_finish(smin, smax, syn, 0x7FFFFFFFu);
            if (lane == 0) fl.span[c] = sp_c;
        }
        __syncthreads();
        // (e) this CTA's span sum (read by every CTA after the next B1)
        if (fl.adapt) {
            if (tid == 0) s_span = 0ull;
            __syncthreads();
            unsigned long long part = 0;
            for (uint32_t c = c0 + tid; c < c1; c += nthr) part += __ldcg(fl.span + c);
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) part += __shfl_xor_sync(0xffffffffu, part, d);
            if (lane == 0 && part) atomicAdd(&s_span, part);
            __syncthreads();
            if (tid == 0) p.span_part[(t & 1u) * G + b] = s_span;
        }
        // the next input's bit-plane (the permanence update read this one)
        if (t + 1u < n) {
            __syncthreads();
            if (tid == 0) {
                asm volatile("fence.proxy.async.global;" ::: "memory");
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                bulk_copy(s_bits, gbits_of(t + 1u), bits_bytes, &s_bar_bits);
            }
        }
        stamp(6);
    }
    // the radius in force after the call
    if (fl.adapt && n > 0) {
        grid_barrier(p.gbar, ++nbar * G);
        if (b == 0 && wi == 0) {
            unsigned long long sum = 0;
            for (uint32_t i = lane; i < G; i += 32u) sum += __ldcg(p.span_part + ((n - 1u) & 1u) * G + i);
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, d);
            if (lane == 0) *fl.radius = adapt_radius(sum, g.nbits, C);
        }
    }
    if (tr) {
        for (int i = 0; i < 7; ++i) p.trace[i] = s_tr[i];
        p.trace[7] = n;
        for (int i = 8; i < 13; ++i) p.trace[i] = s_tr[i];
    }
}

// dynamic smem of the full-learning grid kernel with G CTAs (0 if it cannot run): a single
// bit-plane buffer, `stages` ring stages, the whole raw row (u16) and `cap` candidates
uint32_t learn_grid_full_smem(const Geometry& g, uint32_t G, uint32_t stages, uint32_t cap, uint32_t* own_words,
                              uint32_t* ccols) {
    const uint32_t Wn4 = ((g.nbits + 31u) / 32u + 3u) / 4u * 4u;
    const uint32_t own = (g.ncw + G - 1u) / G;
    const uint32_t cc = learn_grid_chunk_cols(g.S);
    if (own_words) *own_words = own;
    if (ccols) *ccols = cc;
    if (g.C32 > kGfThreads * kGfPer || g.C32 > 65536u) return 0u;  // union window per thread / u16 positions
    const uint32_t own_cols = own * 32u;
    return 4u * (Wn4 + stages * cc * g.S + own_cols + (own + 3u) / 4u * 4u + own_cols) + 8u * cap + 2u * g.C32 +
           2u * cap;
}

cudaError_t configure_learn_grid_full(int max_smem) {
    cudaFuncAttributes a{};
    cudaError_t e = cudaFuncGetAttributes(&a, sp_learn_grid_full_kernel);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(sp_learn_grid_full_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 max_smem - static_cast<int>(a.sharedSizeBytes));
    return e;
}

cudaError_t learn_grid_full_max_ctas(uint32_t smem, int* n) {
    int per_sm = 0, dev = 0, sms = 0;
    cudaError_t e =
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sp_learn_grid_full_kernel, kGfThreads, smem);
    if (e == cudaSuccess) e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    *n = e == cudaSuccess ? per_sm * sms : 0;
    if (e != cudaSuccess) (void)cudaGetLastError();
    return cudaSuccess;
}

cudaError_t launch_learn_grid_full(const LearnGridParams& p, uint32_t smem, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(p.gbar, 0, sizeof(uint32_t), s);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.G);
    cfg.blockDim = dim3(kGfThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, sp_learn_grid_full_kernel, p);
}

}  // namespace sp
