// sp_learn.cu — cluster-resident sequential learning (learn=1).
//
// Learning is a recurrence over inputs (input t+1 sees input t's permanence
// update), so it cannot be batched.  One launch processes the whole stream with a
// thread-block cluster of Q CTAs (Q <= 16) that keeps the synapse table idx|connected
// (column-major, the CTA's column slice) resident in shared memory:
//
//   per input t:  every CTA loads the bit-plane of t (global, L2) into smem, and packs a
//                 1/Q slice of input t+1 into the other global bit-plane buffer
//                 overlap of the CTA's columns; raw counts are broadcast to every CTA's
//                 smem through DSMEM (double-buffered by input parity)
//                 cluster barrier: all raw counts of t, and the bit-plane of t+1, complete
//                 every CTA runs the same exact k-winners (warp-level, sp_select.cuh), writes
//                 the SDR words of its columns, and updates the permanences of its winners
//                 (fp32 RN add/sub + clamp, R3) and their connected flags in smem
//
// One cluster barrier per input; the frame of t+2 is prefetched into L2 (bulk prefetch)
// two inputs ahead.
//
// Full learning (SP_FLAG_FULL_LEARNING, NEXT-1; S:119(b-e); DESIGN R17-R21) adds, after the
// permanence update of input t: the SDR words of every CTA are broadcast (DSMEM) -> a second
// cluster barrier -> every CTA updates the duty cycles of ALL columns and recomputes ALL boosts
// (the same fp32 operations in every CTA, so the replicas stay identical and the next
// selection needs no exchange), bumps its own weak columns, and sends the sum of its columns'
// connected spans to every CTA; the radius of input t+1 is formed after the overlap barrier.  Only the frame bytes and the winners' permanence rows touch memory
// below L2.  DESIGN.md §4.2.
#include <algorithm>

#include <cooperative_groups.h>

#include "sp_duty.cuh"
#include "sp_internal.h"
#include "sp_pack.cuh"
#include "sp_select.cuh"

namespace cg = cooperative_groups;

namespace sp {

namespace {

constexpr uint32_t kLearnThreads = 512;

// store one SDR word of this CTA (lane 0): smem copy for the learning step, the global SDR
// and the input's winner count
__device__ __forceinline__ void emit_word(const LearnParams& p, uint32_t* s_sdr, uint32_t cw, uint32_t gcw,
                                          uint32_t gin, uint32_t word, uint32_t lane) {
    if (lane != 0u) return;
    s_sdr[cw] = word;
    if (gcw < p.g.ncw) {
        p.sdr[static_cast<size_t>(gin) * p.g.ncw + gcw] = word;
        if (word) atomicAdd(p.counts + gin, static_cast<uint32_t>(__popc(word)));
    }
}

}  // namespace

// overlap of this CTA's columns for the input whose bit-plane is in bits; raw counts go
// to every CTA's raw buffer (DSMEM).  tpc consecutive lanes share a column (synapses
// s = part, part+tpc, ..) with a shuffle reduction; the padded column-major slice keeps
// the reads conflict-free
// L2 prefetch ahead of use: the prepacked bit-plane of input t (CTA 0 only: every CTA reads the
// whole plane), else this CTA's share of the frame bytes it will pack
__device__ __forceinline__ void prefetch_plane_or_input(const LearnParams& p, uint32_t t, uint32_t wbeg, uint32_t wend,
                                                        uint32_t q, uint32_t Q, const uint32_t* plane, uint32_t Wn4) {
    if (!p.prepacked) {
        prefetch_input(p, t, wbeg, wend, q, Q);
        return;
    }
    if (q == 0 && t < p.num_inputs && !(p.dbg & 2u)) prefetch_l2(plane, Wn4 * 4u);
}

__device__ __forceinline__ void overlap_step(const LearnParams& p, cg::cluster_group& cluster, const uint32_t* s_syn,
                                             const uint32_t* bits, uint16_t* raw_buf, uint32_t c0, uint32_t gin,
                                             const uint32_t* s_bc) {
    const Geometry& g = p.g;
    const uint32_t cpc = p.cols_per_cta, ss = p.syn_stride, tpc = p.tpc, Q = p.Q;
    for (uint32_t base = 0; base < cpc * tpc; base += blockDim.x) {
        const uint32_t slot = base + threadIdx.x;
        const uint32_t cl = slot / tpc, part = slot % tpc;
        uint32_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;
        if (cl < cpc) {
            const uint32_t* col = s_syn + cl * ss;
            uint32_t s = part;
            for (; s + 3u * tpc < g.S; s += 4u * tpc) {  // four independent lookups
                const uint32_t e0 = col[s], e1 = col[s + tpc], e2 = col[s + 2u * tpc], e3 = col[s + 3u * tpc];
                r0 += (bits[(e0 & 0x7FFFFFFFu) >> 5] >> (e0 & 31u)) & (e0 >> 31);
                r1 += (bits[(e1 & 0x7FFFFFFFu) >> 5] >> (e1 & 31u)) & (e1 >> 31);
                r2 += (bits[(e2 & 0x7FFFFFFFu) >> 5] >> (e2 & 31u)) & (e2 >> 31);
                r3 += (bits[(e3 & 0x7FFFFFFFu) >> 5] >> (e3 & 31u)) & (e3 >> 31);
            }
            for (; s < g.S; s += tpc) {
                const uint32_t e = col[s];
                r0 += (bits[(e & 0x7FFFFFFFu) >> 5] >> (e & 31u)) & (e >> 31);
            }
        }
        uint32_t raw = (r0 + r1) + (r2 + r3);
        for (uint32_t d = tpc >> 1; d > 0; d >>= 1) raw += __shfl_xor_sync(0xffffffffu, raw, d);
        const uint32_t c = c0 + cl;
        // the tpc lanes of a column all hold its count: they share the Q remote stores
        if (cl < cpc && c < g.C32)
            for (uint32_t r = part; r < Q; r += tpc) cluster.map_shared_rank(raw_buf, r)[c] = static_cast<uint16_t>(raw);
        if (part == 0 && cl < cpc && c < g.C32) {
            if (p.raw_out && c < g.C) {
                p.raw_out[static_cast<size_t>(gin) * g.C + c] = static_cast<uint16_t>(raw);
                // boost = Bc * 2^-23 exactly (Bc has <= 24 significant bits); the boost in
                // force for this input (full learning updates s_bc between inputs)
                const float b = __fmul_rn(__uint2float_rn(s_bc[c]), 1.1920928955078125e-07f);
                p.boosted_out[static_cast<size_t>(gin) * g.C + c] =
                    raw >= p.min_overlap ? __fmul_rn(static_cast<float>(raw), b) : 0.0f;
            }
        }
    }
}

__global__ void __launch_bounds__(kLearnThreads, 1) sp_learn_cluster_kernel(const __grid_constant__ LearnParams p) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ __align__(8) uint64_t s_bar;  // bulk-copy completion of the bit-plane
    cg::cluster_group cluster = cg::this_cluster();
    const Geometry& g = p.g;
    const uint32_t tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31u;
    const uint32_t wi = tid >> 5, nw = nthr >> 5;
    const uint32_t q = cluster.block_rank(), Q = p.Q;
    const uint32_t cpc = p.cols_per_cta;        // columns owned by this CTA (multiple of 32)
    const uint32_t ncl = cpc / 32u;              // column-words owned
    const uint32_t c0 = q * cpc;                 // first column owned
    const uint32_t Wn = p.Wn, Wn4 = (Wn + 3u) / 4u * 4u;
    const uint32_t C32r = (g.C32 + 3u) / 4u * 4u;
    const uint32_t n = p.num_inputs;

    const uint32_t ss = p.syn_stride;                               // >= S, == 8 mod 32
    uint32_t* s_syn = reinterpret_cast<uint32_t*>(smem);           // [cpc][ss] idx | connected<<31
    uint32_t* s_bits = s_syn + static_cast<size_t>(ss) * cpc;      // [1 or 2][Wn4] input bit-planes
    uint32_t* s_bc = s_bits + (p.dbl_bits ? 2u : 1u) * Wn4;         // [C32]
    uint16_t* s_raw = reinterpret_cast<uint16_t*>(s_bc + g.C32);    // [2][C32r] raw, by input parity
    uint64_t* s_ties = reinterpret_cast<uint64_t*>(s_raw + 2u * C32r);  // [ncl][64] tie lists
    uint32_t* s_sdr = reinterpret_cast<uint32_t*>(s_ties + ncl * 64u);  // [ncl] SDR words
    uint32_t* s_planes = s_sdr + ncl;                               // [ncw][16] key bit-planes
    // full learning (p.fl.on): replicated duty cycles and window-maximum tables, the SDR of
    // the whole input, own spans, per-CTA span sums
    const FullLearn& fl = p.fl;
    const uint32_t nb = g.C32 / 32u;
    float* s_adc = reinterpret_cast<float*>(s_planes + max(g.ncw * 16u, 512u));  // [C32]
    float* s_odc = s_adc + g.C32;                                       // [C32]
    float* s_pre = s_odc + g.C32;                                       // [C32]
    float* s_suf = s_pre + g.C32;                                       // [C32]
    float* s_table = s_suf + g.C32;                                     // [levels + 3][nb]
    uint32_t* s_sdr_all = reinterpret_cast<uint32_t*>(s_table + (wmax_levels(nb) + 3u) * nb);  // [ncw]
    uint32_t* s_span = s_sdr_all + g.ncw;                               // [cpc]
    unsigned long long* s_spanpart =
        reinterpret_cast<unsigned long long*>((reinterpret_cast<uintptr_t>(s_span + cpc) + 7u) & ~uintptr_t(7));  // [Q]
    __shared__ unsigned long long s_myspan;
    __shared__ unsigned long long s_mm[2];  // eligible-N range of the coarse map
    auto bits_of = [&](uint32_t t) { return s_bits + (p.dbl_bits ? (t & 1u) * Wn4 : 0u); };
    // bit-planes in global memory: prepacked by k_pack for the whole launch (p.prepacked), or
    // packed by the CTAs themselves into two buffers by input parity
    auto gbits_of = [&](uint32_t t) { return p.bits_g + (p.prepacked ? t : (t & 1u)) * Wn4; };

    // ---- resident state: this CTA's synapse slice, Bc; counts zeroed ---------------------
    for (uint32_t i = tid; i < g.S * cpc; i += nthr) {
        const uint32_t s = i / cpc, cl = i % cpc, c = c0 + cl;
        s_syn[cl * ss + s] = c < g.C32 ? p.syn[static_cast<size_t>(s) * g.C32 + c] : 0u;
    }
    for (uint32_t c = tid; c < g.C32; c += nthr) s_bc[c] = p.bc[c];
    uint32_t R = p.radius;  // radius in force (full learning: adapted after every input)
    if (fl.on) {
        R = *fl.radius;
        for (uint32_t c = tid; c < g.C32; c += nthr) {
            s_adc[c] = c < g.C ? fl.adc[c] : 0.0f;
            s_odc[c] = c < g.C ? fl.odc[c] : 0.0f;
        }
        for (uint32_t cl = tid; cl < cpc; cl += nthr) s_span[cl] = c0 + cl < g.C ? fl.span[c0 + cl] : 0u;
    }
    if (q == 0)
        for (uint32_t i = tid; i < n; i += nthr) p.counts[p.first_input + i] = 0u;
    if (tid == 0) {
        mbar_init(&s_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }

    const uint32_t theta = p.min_overlap, L = g.keyL;
    const uint32_t wbeg = q * Wn / Q, wend = (q + 1) * Wn / Q;  // packed words of this CTA
    uint64_t* trace = (p.trace && q == 0 && tid == 0) ? p.trace : nullptr;
    // phase accumulators of the traced threads live in smem (no registers held in the loop)
    __shared__ uint64_t s_tr[9];
    uint64_t& t_ld = s_tr[0];
    uint64_t& t_ov = s_tr[1];
    uint64_t& t_bar = s_tr[2];
    uint64_t& t_sel = s_tr[3];
    uint64_t& t_learn = s_tr[4];
    uint64_t& t_ph = s_tr[5];
    uint64_t& t_sub = s_tr[6];
    uint64_t& t_pk = s_tr[7];
    uint64_t& t_full = s_tr[8];
    if (tid == 0)
        for (int i = 0; i < 9; ++i) s_tr[i] = 0;
    uint32_t phase = 0;  // parity of s_bar's next completion
    // selection warps (global inhibition): one per owned column-word; the others pack
    const uint32_t nsel = ncl < nw ? ncl : nw;
    const uint32_t tpk0 = nsel < nw ? nsel * 32u : 0u, npk = nthr - tpk0;
    // the first packing thread also traces its own phase (selection vs pack)
    uint64_t* trace_pk = (p.trace && q == 0 && tid == tpk0 && tpk0 != 0u) ? p.trace : nullptr;

    // ---- prologue: bit-planes of inputs 0 and 1; overlap of input 0 ----------------------
    if (tid == 0)
        for (uint32_t t = 0; t < 3u; ++t) prefetch_plane_or_input(p, t, wbeg, wend, q, Q, gbits_of(t), Wn4);
    if (!p.prepacked) {
        if (n > 0) pack_slice(p, 0, wbeg, wend, gbits_of(0), 0, nthr);
        if (n > 1) pack_slice(p, 1, wbeg, wend, gbits_of(1), 0, nthr);
    }
    cluster.sync();  // bit-planes 0 (and 1) complete; smem and counts initialised
    if (n > 0) {
        if (tid == 0) bulk_load_bits(bits_of(0), gbits_of(0), Wn, &s_bar);
        mbar_wait(&s_bar, phase);
        phase ^= 1u;
        overlap_step(p, cluster, s_syn, bits_of(0), s_raw, c0, p.first_input, s_bc);
    }
    cluster.sync();  // raw counts of input 0 everywhere

    for (uint32_t t = 0; t < n; ++t) {
        const uint32_t gin = p.first_input + t;
        const uint16_t* raw_t = s_raw + (t & 1u) * C32r;
        const bool more = t + 1u < n;
        if (fl.adapt && t > 0u) {  // radius of input t from the span sums of input t-1 (R21)
            unsigned long long sum = 0;
            for (uint32_t r = 0; r < Q; ++r) sum += s_spanpart[r];
            R = adapt_radius(sum, g.nbits, g.C);
        }
        if (trace) t_ph = globaltimer();
        if (tid == 0) {
            prefetch_plane_or_input(p, t + 3u, wbeg, wend, q, Q, gbits_of(t + 3u), Wn4);
            // bit-plane of t+1 (complete since the last barrier) into its smem buffer; with
            // one buffer it must wait until learning of t is done with the current plane
            if (more && p.dbl_bits && !(p.dbg & 16u)) bulk_load_bits(bits_of(t + 1u), gbits_of(t + 1u), Wn, &s_bar);
        }
        // ---- a3/a4: the same exact k-winners in every CTA (sp_select.cuh), while the
        //      other warps pack input t+2 into the global buffer input t used ----------
        if (R > 0) {
            const bool uni = p.uniform_bc != 0u;
            const uint32_t r_lo = uniform_r_lo(theta, s_bc[0]);
            const uint32_t rb = raw_bits(g.S);
            CoarseMap cm{0ull, 0u};
            if (uni) {
                build_raw_planes(raw_t, s_planes, g.ncw, rb, r_lo, wi, nw, lane);
            } else {
                cm = coarse_map_block(raw_t, s_bc, theta, 0u, g.ncw, s_mm);
                build_coarse_planes15(raw_t, s_bc, s_planes, g.ncw, theta, cm, wi, nw, lane);
            }
            const uint32_t parts = nw / ncl;  // warps per owned word (its window split between them)
            uint32_t* s_beats = reinterpret_cast<uint32_t*>(s_ties);  // [ncl][32]
            if (parts > 1u)
                for (uint32_t i = tid; i < ncl * 32u; i += nthr) s_beats[i] = 0u;
            __syncthreads();
            if (parts > 1u && !(p.dbg & 128u)) {
                if (wi < ncl * parts) {
                    const uint32_t cw = wi % ncl, part = wi / ncl, gcw = c0 / 32u + cw;
                    if (gcw < g.ncw) {
                        uint32_t v;
                        const uint32_t b =
                            uni ? local_uniform_beats_part(raw_t, s_planes, g.ncw, rb, gcw, g.C, R, r_lo, lane, part,
                                                           parts, v)
                                : local_general_beats15(raw_t, s_bc, s_planes, g.ncw, gcw, g.C, R, theta, cm, L, lane,
                                                        part, parts, v);
                        if (b) atomicAdd(&s_beats[cw * 32u + lane], b);
                    }
                }
                __syncthreads();
                for (uint32_t cw = wi; cw < ncl; cw += nw) {
                    const uint32_t gcw = c0 / 32u + cw, c = gcw * 32u + lane;
                    bool elig = false;
                    if (gcw < g.ncw && c < g.C) {
                        if (uni) {
                            elig = raw_t[c] >= r_lo;
                        } else {
                            bool lossy;
                            elig = coarse_u15(eligible_N(raw_t[c], s_bc[c], theta), cm, lossy) > 0u;
                        }
                    }
                    const uint32_t word = __ballot_sync(0xffffffffu, elig && s_beats[cw * 32u + lane] < p.k);
                    emit_word(p, s_sdr, cw, gcw, gin, word, lane);
                }
            } else {
                for (uint32_t cw = wi; cw < ncl; cw += nw) {
                    const uint32_t gcw = c0 / 32u + cw;
                    uint32_t word = 0u;
                    if (gcw < g.ncw)
                        word = uni ? local_uniform_word(raw_t, s_planes, g.ncw, rb, gcw, g.C, R, p.k, r_lo, lane)
                                   : local_general_word15(raw_t, s_bc, s_planes, g.ncw, gcw, g.C, R, p.k, theta,
                                                          cm, L, lane);
                    emit_word(p, s_sdr, cw, gcw, gin, word, lane);
                }
            }
        } else if (p.prepacked && p.uniform_bc && g.S + 4u <= max(g.ncw * 16u, 512u) && !(p.dbg & 64u)) {
            // uniform boost, no packing to overlap: the whole CTA builds the raw histogram
            const UniformSel us = global_uniform_cta(raw_t, g.C, g.S, p.k, uniform_r_lo(theta, s_bc[0]), s_planes);
            for (uint32_t cw = wi; cw < ncl; cw += nw) {
                const uint32_t gcw = c0 / 32u + cw;
                uint32_t word = 0u;
                if (gcw < g.ncw) word = global_uniform_word_sel(raw_t, g.C, gcw, us, lane);
                emit_word(p, s_sdr, cw, gcw, gin, word, lane);
            }
        } else if (p.prepacked && !p.uniform_bc && !(p.dbg & 64u)) {
            // per-column boosts and no packing to overlap: the whole CTA selects (two-level
            // radix select, sp_select.cuh) instead of one warp per owned word
            const CoarseMap cm = coarse_map_block(raw_t, s_bc, theta, 0u, g.ncw, s_mm);
            const GlobalSel gs = global_select_cta(raw_t, s_bc, theta, g.C, g.ncw, p.k, L, g.keyBits, cm, s_planes,
                                                   s_ties, ncl * 64u);
            for (uint32_t cw = wi; cw < ncl; cw += nw) {
                const uint32_t gcw = c0 / 32u + cw;
                uint32_t word = 0u;
                if (gcw < g.ncw) word = global_select_word(raw_t, s_bc, theta, g.C, gcw, L, cm, gs, s_planes, g.ncw, lane);
                emit_word(p, s_sdr, cw, gcw, gin, word, lane);
            }
        } else {
            for (uint32_t cw = wi; cw < ncl; cw += nw) {
                const uint32_t gcw = c0 / 32u + cw;
                uint32_t word = 0u;
                if (gcw < g.ncw && !(p.dbg & 8u)) {
                    uint64_t* ties = s_ties + cw * 64u;
                    // NR registers hold 64 * NR columns (two per register)
                    word = g.C32 <= 512u    ? global_word<8>(p, raw_t, s_bc, ties, gcw, lane)
                           : g.C32 <= 1024u ? global_word<16>(p, raw_t, s_bc, ties, gcw, lane)
                                            : global_word<32>(p, raw_t, s_bc, ties, gcw, lane);
                }
                emit_word(p, s_sdr, cw, gcw, gin, word, lane);
            }
        }
        if (trace) t_sub += globaltimer() - t_ph;  // selection alone (warp 0)
        uint64_t tp0 = 0;
        if (trace_pk) tp0 = globaltimer();
        if (!p.prepacked && t + 2u < n && !(p.dbg & 4u))
            pack_slice(p, t + 2u, wbeg, wend, gbits_of(t + 2u), tpk0, npk);
        if (trace_pk) t_pk += globaltimer() - tp0;
        __syncthreads();  // s_sdr complete
        if (trace) {
            t_sel += globaltimer() - t_ph;
            t_ph = globaltimer();
        }
        // ---- a5: permanence update of this CTA's winners (warp per column) ---------------
        // idx from the resident slice; the perm row is read in batches of 8 values per lane
        // (independent loads, one L2 round trip), updated (fp32 RN add/sub + clamp, R3) and
        // written back with the refreshed connected flags
        const uint32_t* bits_t = bits_of(t);
        for (uint32_t cl = wi; cl < cpc; cl += nw) {
            const uint32_t c = c0 + cl;
            if (c >= g.C) break;
            if (((s_sdr[cl >> 5] >> (cl & 31u)) & 1u) == 0u) continue;
            float* __restrict__ perm = p.perm + static_cast<size_t>(c) * g.S;
            uint32_t* col = s_syn + cl * ss;
            uint32_t smin = 0xFFFFFFFFu, smax = 0u;
            for (uint32_t s0 = 0; s0 < g.S; s0 += 256u) {
                float v[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint32_t s = s0 + 32u * j + lane;
                    v[j] = s < g.S ? __ldcg(perm + s) : 0.0f;
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint32_t s = s0 + 32u * j + lane;
                    if (s < g.S) {
                        const uint32_t i = col[s] & 0x7FFFFFFFu;
                        const bool on = ((bits_t[i >> 5] >> (i & 31u)) & 1u) != 0u;
                        float x = on ? __fadd_rn(v[j], p.inc) : __fsub_rn(v[j], p.dec);
                        x = fminf(fmaxf(x, 0.0f), 1.0f);
                        perm[s] = x;
                        col[s] = i | (x >= p.tau ? 0x80000000u : 0u);
                        span_accumulate(x >= p.tau, s, smin, smax);
                    }
                }
            }
            if (fl.on) {  // connected span of the updated column (R21)
                const uint32_t v = span_finish(smin, smax, col, 0x7FFFFFFFu);
                if (lane == 0) s_span[cl] = v;
            }
        }
        __syncthreads();  // flags updated (and, with one buffer, the plane of t released)
        if (fl.on) {
            if (trace) {
                t_learn += globaltimer() - t_ph;
                t_ph = globaltimer();
            }
            // ---- full learning (b)-(e) of input t (S:119(b-e); DESIGN R17-R21) -------------
            for (uint32_t i = tid; i < ncl * Q; i += nthr) {  // this CTA's SDR words to every CTA
                const uint32_t gcw = c0 / 32u + i % ncl;
                if (gcw < g.ncw) cluster.map_shared_rank(s_sdr_all, i / ncl)[gcw] = s_sdr[i % ncl];
            }
            if (tid == 0) s_myspan = 0ull;
            cluster.sync();  // the whole SDR of input t everywhere
            // (b) duty cycles of every column (replicated)
            for (uint32_t c = tid; c < g.C; c += nthr) {
                const bool a = ((s_sdr_all[c >> 5] >> (c & 31u)) & 1u) != 0u;
                const uint32_t r = raw_t[c];
                s_adc[c] = duty_update(s_adc[c], a, fl.pm1, fl.P);
                s_odc[c] = duty_update(s_odc[c], r >= theta && r > 0u, fl.pm1, fl.P);
            }
            __syncthreads();
            auto sync = [] { __syncthreads(); };
            // (c) boosts of every column (replicated): the keys of input t+1.  A window that
            // covers every column (radius 0 or >= C-1) needs only the two maxima.
            const bool gwin = R == 0u || R + 1u >= g.C;
            const bool ends = !gwin && 2u * R + 1u >= g.C;  // every window reaches an end
            float gA = 0.0f, gO = 0.0f;
            auto wq = [&](const float* v, uint32_t c) {
                return ends ? wmax_query_ends(s_pre, s_suf, s_table, nb, g.C, c, R)
                            : wmax_query(v, s_pre, s_suf, s_table, nb, g.C, c, R);
            };
            if (gwin) block_max2(s_adc, s_odc, g.C, s_pre, gA, gO);
            else if (ends) wmax_build_ends(s_adc, g.C, g.C32, s_pre, s_suf, s_table);
            else wmax_build(s_adc, g.C, g.C32, s_pre, s_suf, s_table, 0u, nthr, sync);
            for (uint32_t c = tid; c < g.C; c += nthr)
                s_bc[c] = boost_bc(boost_rule(s_adc[c], gwin ? gA : wq(s_adc, c), fl.mb1));
            __syncthreads();
            // (d) bump of this CTA's weak columns, warp per column
            if (ends) wmax_build_ends(s_odc, g.C, g.C32, s_pre, s_suf, s_table);
            else if (!gwin) wmax_build(s_odc, g.C, g.C32, s_pre, s_suf, s_table, 0u, nthr, sync);
            for (uint32_t cl = wi; cl < cpc; cl += nw) {
                const uint32_t c = c0 + cl;
                if (c >= g.C) break;
                if (!weak_column(s_odc[c], gwin ? gO : wq(s_odc, c))) continue;
                float* __restrict__ perm = p.perm + static_cast<size_t>(c) * g.S;
                uint32_t* col = s_syn + cl * ss;
                uint32_t smin = 0xFFFFFFFFu, smax = 0u;
                for (uint32_t s = lane; s < g.S; s += 32u) {
                    const float x = fminf(__fadd_rn(__ldcg(perm + s), fl.bump), 1.0f);
                    perm[s] = x;
                    col[s] = (col[s] & 0x7FFFFFFFu) | (x >= p.tau ? 0x80000000u : 0u);
                    span_accumulate(x >= p.tau, s, smin, smax);
                }
                const uint32_t v = span_finish(smin, smax, col, 0x7FFFFFFFu);
                if (lane == 0) s_span[cl] = v;
            }
            if (fl.adapt) {
                __syncthreads();
                // (e) this CTA's span sum to every CTA; the radius of t+1 is formed after the
                // next barrier
                unsigned long long part = 0;
                for (uint32_t cl = tid; cl < cpc; cl += nthr) part += c0 + cl < g.C ? s_span[cl] : 0u;
                for (uint32_t d = 16; d > 0; d >>= 1) part += __shfl_xor_sync(0xffffffffu, part, d);
                if (lane == 0 && part) atomicAdd(&s_myspan, part);
                __syncthreads();
                if (tid < Q) cluster.map_shared_rank(s_spanpart, tid)[q] = s_myspan;
            }
            __syncthreads();  // bumped flags and new boosts visible to the overlap of t+1
            if (trace) {
                t_full += globaltimer() - t_ph;
                t_ph = globaltimer();
            }
        }
        if (trace) {
            t_learn += globaltimer() - t_ph;
            t_ph = globaltimer();
        }
        if (!more) break;
        // ---- a1/a2 of input t+1: its bit-plane, then the overlap of this CTA's columns ------
        if (tid == 0 && (!p.dbl_bits || (p.dbg & 16u))) bulk_load_bits(bits_of(t + 1u), gbits_of(t + 1u), Wn, &s_bar);
        mbar_wait(&s_bar, phase);
        phase ^= 1u;
        if (trace) {
            t_ld += globaltimer() - t_ph;
            t_ph = globaltimer();
        }
        // raw counts of t+1 go to the other parity buffer: a CTA still selecting input t
        // reads this one; the buffer of t is rewritten (input t+2) only after every CTA has
        // passed the barrier below
        overlap_step(p, cluster, s_syn, bits_of(t + 1u), s_raw + ((t + 1u) & 1u) * C32r, c0, gin + 1u, s_bc);
        if (trace) {
            t_ov += globaltimer() - t_ph;
            t_ph = globaltimer();
        }
        cluster.sync();  // raw counts of t+1 everywhere; bit-plane of t+2 complete
        if (trace) t_bar += globaltimer() - t_ph;
    }
    if (trace) {
        trace[0] = t_ld;
        trace[1] = t_ov;
        trace[2] = t_bar;
        trace[3] = t_sel;
        trace[4] = t_learn;
        trace[5] = n;
        trace[6] = t_sub;
        trace[8] = t_full;
    }
    if (trace_pk) trace_pk[7] = t_pk;
    if (fl.on) {  // ---- full-learning state back to global (replicas are identical) ---------
        if (fl.adapt) {
            cluster.sync();  // span sums of the last input everywhere
            unsigned long long sum = 0;
            for (uint32_t r = 0; r < Q; ++r) sum += s_spanpart[r];
            R = adapt_radius(sum, g.nbits, g.C);
        }
        if (n > 0 && q == 0) {
            for (uint32_t c = tid; c < g.C; c += nthr) {
                fl.adc[c] = s_adc[c];
                fl.odc[c] = s_odc[c];
                fl.bc[c] = s_bc[c];
                fl.boost[c] = __fmul_rn(__uint2float_rn(s_bc[c]), 1.1920928955078125e-07f);
            }
            if (tid == 0) *fl.radius = R;
        }
        for (uint32_t cl = tid; cl < cpc; cl += nthr)
            if (c0 + cl < g.C) fl.span[c0 + cl] = s_span[cl];
    }
    // ---- write the resident connected flags back (the per-input path reads them) ---------
    for (uint32_t i = tid; i < g.S * cpc; i += nthr) {
        const uint32_t s = i / cpc, cl = i % cpc, c = c0 + cl;
        if (c < g.C32) p.syn[static_cast<size_t>(s) * g.C32 + c] = s_syn[cl * ss + s];
    }
}

uint32_t learn_syn_stride(uint32_t S) { return (S + 31u) / 32u * 32u + 8u; }

// threads per column in the overlap: a power of two <= 32 with cpc * tpc <= 512
uint32_t learn_threads_per_column(uint32_t cpc) {
    uint32_t t = 1;
    while (t < 32u && cpc * t * 2u <= kLearnThreads) t *= 2u;
    return t;
}

uint32_t learn_cluster_smem(const Geometry& g, uint32_t Q, uint32_t* cols_per_cta, bool dbl_bits, bool full) {
    const uint32_t cpc = ((g.C32 + Q - 1u) / Q + 31u) / 32u * 32u;
    const uint32_t Wn4 = ((g.nbits + 31u) / 32u + 3u) / 4u * 4u;
    if (cols_per_cta) *cols_per_cta = cpc;
    const uint32_t nb = g.C32 / 32u;
    const uint32_t full_bytes = full ? 4u * (4u * g.C32 + (wmax_levels(nb) + 3u) * nb + g.ncw + cpc) + 8u + 8u * Q : 0u;
    return 4u * (learn_syn_stride(g.S) * cpc + (dbl_bits ? 2u : 1u) * Wn4 + g.C32) +
           4u * ((g.C32 + 3u) / 4u * 4u) + 8u * (cpc / 32u * 64u) + 4u * (cpc / 32u) +
           4u * std::max(g.ncw * 16u, 512u) + full_bytes;
}

cudaError_t configure_learn(int max_smem) {
    cudaFuncAttributes a{};
    cudaError_t e = cudaFuncGetAttributes(&a, sp_learn_cluster_kernel);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(sp_learn_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 max_smem - static_cast<int>(a.sharedSizeBytes));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(sp_learn_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    return e;
}

cudaError_t learn_max_clusters(uint32_t Q, uint32_t smem, int* n) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(Q);
    cfg.blockDim = dim3(kLearnThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = Q;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    *n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(n, sp_learn_cluster_kernel, &cfg);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        *n = 0;
    }
    return cudaSuccess;
}

cudaError_t launch_learn_cluster(const LearnParams& p, uint32_t smem, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.Q);
    cfg.blockDim = dim3(kLearnThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.Q;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, sp_learn_cluster_kernel, p);
}

}  // namespace sp
