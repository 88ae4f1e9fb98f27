// sp_learn_grid.cu — grid-resident sequential learning for SPs whose synapse table does not
// fit a cluster's shared memory (SURVEY §8(a) rows a1-a5 with learn=1; BASELINE config 5:
// 16384 columns x 512 synapses, local inhibition).  DESIGN.md §4.2.
//
// One cooperative launch processes the whole stream with G co-resident CTAs (one per SM).
// CTA b owns the contiguous column-words [b*ncw/G, (b+1)*ncw/G) for every step of the path:
//
//   per input t:  bulk-copy the bit-plane of t (global, L2) into smem; pack this CTA's share
//                 of input t+1 into the other global bit-plane buffer
//                 a2: stream the CTA's column-major synapse slice idx|connected (contiguous,
//                 L2-resident) through a TMA chunk ring; warps gather-count their columns;
//                 raw counts -> global raw buffer (double-buffered by input parity)
//                 grid barrier (raw counts of t and bit-plane of t+1 complete)
//                 a3/a4: load the raw counts of the CTA's words +- r into smem, bit-sliced
//                 local (or warp-level global) k-winners of its own words -> SDR, counts
//                 a5: warp per winning column: fp32 RN add/sub + clamp of the perm row and
//                 the connected flags of its synapse row (both contiguous rows)
//
// A CTA only ever updates and re-reads its own columns, so the learning of t and the
// overlap of t+1 need no barrier between CTAs: one grid barrier per input.
#include <cooperative_groups.h>

#include "sp_grid.cuh"
#include "sp_internal.h"
#include "sp_pack.cuh"
#include "sp_select.cuh"

namespace sp {

namespace {

constexpr uint32_t kGridThreads = 512;
constexpr uint32_t kGridWarps = kGridThreads / 32;

}  // namespace

__global__ void __launch_bounds__(kGridThreads, 1) sp_learn_grid_kernel(const __grid_constant__ LearnGridParams p) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ unsigned long long s_mm[2];  // eligible-N range of the coarse map
    __shared__ __align__(8) uint64_t s_bar_bits;
    __shared__ __align__(8) uint64_t s_bar_ring[8];
    const Geometry& g = p.g;
    const uint32_t tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31u, wi = tid >> 5, nw = nthr >> 5;
    const uint32_t b = blockIdx.x, G = p.G, n = p.num_inputs;
    const uint32_t S = g.S, C32 = g.C32, ncw = g.ncw;
    const uint32_t Wn = p.Wn, Wn4 = (Wn + 3u) / 4u * 4u;
    // owned column-words / columns, and the raw window [jlo, jhi] the inhibition reads
    const uint32_t wb0 = b * ncw / G, wb1 = (b + 1u) * ncw / G, nown = wb1 - wb0;
    const uint32_t c0 = wb0 * 32u, ncols = nown * 32u;
    const uint32_t R = p.radius;
    const uint32_t jlo = R == 0u ? 0u : (c0 >= R ? (c0 - R) / 32u : 0u);
    const uint32_t jhi = R == 0u ? ncw - 1u : min(ncw - 1u, (c0 + ncols - 1u + R) / 32u);
    const uint32_t nwin = jhi - jlo + 1u, cwin = jlo * 32u;
    const uint32_t ccols = p.ccols, stages = p.stages, chunk_words = ccols * S;
    const uint32_t nchunks = ncols / ccols;
    const uint32_t wpc = kGridWarps / ccols;  // warps per column of a chunk
    const uint32_t span = S / wpc;             // synapses per warp (vector path)
    const bool vec_ok = S % wpc == 0u && span % 4u == 0u;

    uint32_t* s_bits = reinterpret_cast<uint32_t*>(smem);                         // [1|2][Wn4]
    uint32_t* s_ring = s_bits + (p.dbl_bits ? 2u : 1u) * Wn4;                      // [stages][chunk]
    uint32_t* s_bcw = s_ring + static_cast<size_t>(stages) * chunk_words;          // [win*32]
    uint32_t* s_planes = s_bcw + p.win_words * 32u;                                // [win][16]
    uint32_t* s_craw = s_planes + p.win_words * 16u;                               // [own cols]
    uint32_t* s_sdr = s_craw + p.own_words * 32u;                                  // [own words]
    uint64_t* s_ties = reinterpret_cast<uint64_t*>(s_sdr + (p.own_words + 1u) / 2u * 2u);  // [own][64]
    uint16_t* s_rw = reinterpret_cast<uint16_t*>(s_ties + p.own_words * 64u);      // [win*32]
    auto bits_of = [&](uint32_t t) { return s_bits + (p.dbl_bits ? (t & 1u) * Wn4 : 0u); };
    const uint32_t pb0_ = b * Wn / G, pb1_ = (b + 1u) * Wn / G;  // packed words of this CTA
    // global bit-planes: prepacked by k_pack for the whole launch, or two by input parity
    auto gbits_of = [&](uint32_t t) { return p.bits_g + (p.prepacked ? t : (t & 1u)) * Wn4; };
    auto prefetch = [&](uint32_t t) {  // L2 prefetch ahead of use (thread 0)
        if (!p.prepacked) prefetch_input(p, t, pb0_, pb1_, b, G);
        else if (b == 0 && t < n) prefetch_l2(gbits_of(t), Wn4 * 4u);
    };
    const uint32_t* my_syn = p.synT + static_cast<size_t>(c0) * S;
    const uint32_t bits_bytes = (Wn * 4u + 15u) & ~15u;
    // phase timers of CTA 0 / thread 0 (SP_TRACE): [0] start..bits ready, [1] overlap,
    // [2] grid barrier, [3] selection, [4] learning
    __shared__ uint64_t s_tr[6];
    const bool tr = p.trace != nullptr && b == 0 && tid == 0;
    if (tr)
        for (int i = 0; i < 6; ++i) s_tr[i] = 0;

    // ---- prologue -------------------------------------------------------------------------
    if (tid == 0) {
        mbar_init(&s_bar_bits, 1);
        for (uint32_t i = 0; i < stages; ++i) mbar_init(&s_bar_ring[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (p.uniform_bc == 0u || R == 0u)
        for (uint32_t i = tid; i < nwin * 32u; i += nthr) s_bcw[i] = p.bc[cwin + i];
    for (uint32_t i = b * nthr + tid; i < n; i += G * nthr) p.counts[p.first_input + i] = 0u;
    if (tid == 0) {
        prefetch(0);
        prefetch(1);
    }
    if (n > 0 && !p.prepacked) pack_slice(p, 0, pb0_, pb1_, gbits_of(0), 0, nthr);
    uint32_t nbar = 0;  // grid barriers passed
    grid_barrier(p.gbar, ++nbar * G);
    uint32_t bits_phase = 0, cc = 0;  // s_bar_bits parity; chunks consumed
    uint32_t ring_slot = 0, ring_par = 0;  // = cc % stages, (cc / stages) & 1
    if (tid == 0 && n > 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        bulk_copy(bits_of(0), gbits_of(0), bits_bytes, &s_bar_bits);
    }

    for (uint32_t t = 0; t < n; ++t) {
        const uint32_t gin = p.first_input + t;
        const uint16_t* raw_src = p.raw_g + (t & 1u) * C32;
        if (tr) s_tr[5] = globaltimer();
        // ---- a2 pipeline start: the first chunks of this CTA's synapse slice (TMA ring;
        // development switch SP_LEARN_DBG & 64 -- the default reads the rows directly below) ----
        const bool ring = (p.dbg & 64u) != 0u;
        if (tid == 0 && !ring) prefetch(t + 2u);
        if (tid == 0 && ring) {
            asm volatile("fence.proxy.async.global;" ::: "memory");  // learning's flag stores
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            for (uint32_t j = 0; j < min(stages, nchunks); ++j)
                bulk_copy(s_ring + ((cc + j) % stages) * chunk_words, my_syn + static_cast<size_t>(j) * chunk_words,
                          chunk_words * 4u, &s_bar_ring[(cc + j) % stages]);
            prefetch(t + 2u);
        }
        // ---- a1: this CTA's share of input t+1 -> global plane (read after the barrier) ----
        if (t + 1u < n && !p.prepacked) pack_slice(p, t + 1u, pb0_, pb1_, gbits_of(t + 1u), 0, nthr);
        for (uint32_t i = tid; i < ncols; i += nthr) s_craw[i] = 0u;
        mbar_wait(&s_bar_bits, bits_phase);
        bits_phase ^= 1u;
        __syncthreads();  // s_craw zeroed; bit-plane of t visible to all threads
        if (tr) {
            const uint64_t now = globaltimer();
            s_tr[0] += now - s_tr[5];
            s_tr[5] = now;
        }
        const uint32_t* bits = bits_of(t);
        // ---- a2: overlap of the owned columns ---------------------------------------------
        // warp per column pair: the synapse rows (idx | connected << 31, contiguous, L2-resident)
        // by 16-byte L2 loads, 8 in flight per lane (2x faster than the TMA chunk ring with its
        // CTA barrier per chunk: config 5 overlap 9.6 -> 4.8 us per input)
        auto hitd = [&](uint32_t e) { return (bits[(e & 0x7FFFFFFFu) >> 5] >> (e & 31u)) & (e >> 31); };
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
                    xa += (hitd(ea[u].x) + hitd(ea[u].y)) + (hitd(ea[u].z) + hitd(ea[u].w));
                    xb += (hitd(eb[u].x) + hitd(eb[u].y)) + (hitd(eb[u].z) + hitd(eb[u].w));
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
            if (++ring_slot == stages) {
                ring_slot = 0;
                ring_par ^= 1u;
            }
            mbar_wait(&s_bar_ring[slot], parity);
            const uint32_t* ch = s_ring + slot * chunk_words;
            const uint32_t jc = wi / wpc, part = wi % wpc;  // column of the chunk, synapse part
            const uint32_t* col = ch + jc * S;
            uint32_t r0 = 0, r1 = 0;
            auto hit = [&](uint32_t e) { return (bits[(e & 0x7FFFFFFFu) >> 5] >> (e & 31u)) & (e >> 31); };
            if (vec_ok) {
                // this warp's contiguous synapse range, 16-byte vectors: 8 independent gathers
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
            __syncthreads();  // every warp is done with this slot
            if (tid == 0 && j + stages < nchunks) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                bulk_copy(s_ring + slot * chunk_words, my_syn + static_cast<size_t>(j + stages) * chunk_words,
                          chunk_words * 4u, &s_bar_ring[slot]);
            }
        }
        for (uint32_t i = tid; i < ncols; i += nthr) {
            const uint32_t c = c0 + i, raw = s_craw[i];
            p.raw_g[(t & 1u) * C32 + c] = static_cast<uint16_t>(raw);
            if (p.raw_out && c < g.C) {
                p.raw_out[static_cast<size_t>(gin) * g.C + c] = static_cast<uint16_t>(raw);
                p.boosted_out[static_cast<size_t>(gin) * g.C + c] =
                    raw >= p.min_overlap ? __fmul_rn(static_cast<float>(raw), p.boost[c]) : 0.0f;
            }
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");  // packed words -> TMA readers
        if (tr) {
            const uint64_t now = globaltimer();
            s_tr[1] += now - s_tr[5];
            s_tr[5] = now;
        }
        grid_barrier(p.gbar, ++nbar * G);  // raw counts of t and the bit-plane of t+1 complete
        if (tr) {
            const uint64_t now = globaltimer();
            s_tr[2] += now - s_tr[5];
            s_tr[5] = now;
        }
        if (tid == 0 && t + 1u < n && p.dbl_bits) {
            asm volatile("fence.proxy.async.global;" ::: "memory");
            bulk_copy(bits_of(t + 1u), gbits_of(t + 1u), bits_bytes, &s_bar_bits);
        }
        // ---- a3/a4: k-winners of the owned words over the raw window -----------------------
        for (uint32_t i = tid; i < nwin * 32u; i += nthr) s_rw[i] = __ldcg(raw_src + cwin + i);
        __syncthreads();
        const uint16_t* row = s_rw - cwin;   // row[c], c in the window
        const uint32_t* bcr = s_bcw - cwin;  // bc[c], c in the window
        const uint32_t theta = p.min_overlap, L = g.keyL;
        if (R > 0u) {
            const bool uni = p.uniform_bc != 0u;
            const uint32_t r_lo = uniform_r_lo(theta, uni ? p.bc[0] : 1u);
            const uint32_t nb = raw_bits(S);
            uint32_t* planes = s_planes - jlo * (uni ? nb : 16u);
            CoarseMap cm{0ull, 0u};
            if (uni) {
                build_raw_planes(row, planes, jhi + 1u, nb, r_lo, jlo + wi, nw, lane);
            } else {
                cm = coarse_map_block(row, bcr, theta, jlo, jhi + 1u, s_mm);
                build_coarse_planes15(row, bcr, planes, jhi + 1u, theta, cm, jlo + wi, nw, lane);
            }
            __syncthreads();
            for (uint32_t cw = wi; cw < nown; cw += nw) {
                const uint32_t gcw = wb0 + cw;
                const uint32_t word =
                    uni ? local_uniform_word(row, planes, ncw, nb, gcw, g.C, R, p.k, r_lo, lane)
                        : local_general_word15(row, bcr, planes, ncw, gcw, g.C, R, p.k, theta, cm, L, lane);
                if (lane == 0) {
                    s_sdr[cw] = word;
                    p.sdr[static_cast<size_t>(gin) * ncw + gcw] = word;
                    if (word) atomicAdd(p.counts + gin, static_cast<uint32_t>(__popc(word)));
                }
            }
        } else {
            for (uint32_t cw = wi; cw < nown; cw += nw) {
                const uint32_t gcw = wb0 + cw;
                uint64_t* ties = s_ties + cw * 64u;
                const uint32_t word = C32 <= 512u    ? global_word<8>(p, row, bcr, ties, gcw, lane)
                                      : C32 <= 1024u ? global_word<16>(p, row, bcr, ties, gcw, lane)
                                                     : global_word<32>(p, row, bcr, ties, gcw, lane);
                if (lane == 0) {
                    s_sdr[cw] = word;
                    p.sdr[static_cast<size_t>(gin) * ncw + gcw] = word;
                    if (word) atomicAdd(p.counts + gin, static_cast<uint32_t>(__popc(word)));
                }
            }
        }
        __syncthreads();  // s_sdr complete
        if (tr) {
            const uint64_t now = globaltimer();
            s_tr[3] += now - s_tr[5];
            s_tr[5] = now;
        }
        // ---- a5: permanence update of the owned winners (warp per column) -----------------
        for (uint32_t cl = wi; cl < ncols; cl += nw) {
            const uint32_t c = c0 + cl;
            if (c >= g.C) break;
            if (((s_sdr[cl >> 5] >> (cl & 31u)) & 1u) == 0u) continue;
            float* __restrict__ perm = p.perm + static_cast<size_t>(c) * S;
            uint32_t* __restrict__ syn = p.synT + static_cast<size_t>(c) * S;
            // rows of S values, 16-byte vectors: lane covers s = s0 + 128q + 4 lane + (0..3);
            // all loads of a 512-synapse block are issued before any use (one L2 round trip)
            for (uint32_t s0 = 0; s0 < S; s0 += 512u) {
                float4 v[4];
                uint4 e[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t s = s0 + 128u * q + 4u * lane;
                    if (s < S) {  // S % 4 == 0: whole vectors
                        v[q] = __ldcg(reinterpret_cast<const float4*>(perm + s));
                        e[q] = __ldcg(reinterpret_cast<const uint4*>(syn + s));
                    }
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t s = s0 + 128u * q + 4u * lane;
                    if (s < S) {
                        float* vv = &v[q].x;
                        uint32_t* ee = &e[q].x;
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const uint32_t i = ee[k] & 0x7FFFFFFFu;
                            const bool on = ((bits[i >> 5] >> (i & 31u)) & 1u) != 0u;
                            float x = on ? __fadd_rn(vv[k], p.inc) : __fsub_rn(vv[k], p.dec);
                            x = fminf(fmaxf(x, 0.0f), 1.0f);
                            vv[k] = x;
                            ee[k] = i | (x >= p.tau ? 0x80000000u : 0u);
                        }
                        *reinterpret_cast<float4*>(perm + s) = v[q];
                        *reinterpret_cast<uint4*>(syn + s) = e[q];
                    }
                }
            }
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");  // flag stores -> next TMA reads
        if (t + 1u < n) {
            // the next input's bit-plane: with one smem buffer only now (learning used it)
            __syncthreads();
            if (tid == 0 && !p.dbl_bits) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                bulk_copy(bits_of(t + 1u), gbits_of(t + 1u), bits_bytes, &s_bar_bits);
            }
        }
        if (tr) s_tr[4] += globaltimer() - s_tr[5];
    }
    if (tr) {
        for (int i = 0; i < 5; ++i) p.trace[i] = s_tr[i];
        p.trace[5] = n;
    }
}

uint32_t learn_grid_chunk_cols(uint32_t S) {
    uint32_t c = 16;
    while (c > 1u && c * S * 4u > 16384u) c >>= 1;
    return c;
}

// dynamic smem of the grid learning kernel with G CTAs; 0 if it cannot run (see host plan)
uint32_t learn_grid_smem(const Geometry& g, uint32_t radius, uint32_t G, bool dbl_bits, uint32_t* own_words,
                         uint32_t* win_words, uint32_t* ccols, uint32_t* stages) {
    const uint32_t Wn4 = ((g.nbits + 31u) / 32u + 3u) / 4u * 4u;
    const uint32_t own = (g.ncw + G - 1u) / G;
    const uint32_t win = radius == 0u ? g.ncw : std::min(g.ncw, own + 2u * ((radius + 31u) / 32u) + 1u);
    const uint32_t cc = learn_grid_chunk_cols(g.S);
    const uint32_t st = *stages;  // requested ring depth (the host tries 8 down to 2)
    if (own_words) *own_words = own;
    if (win_words) *win_words = win;
    if (ccols) *ccols = cc;
    return 4u * ((dbl_bits ? 2u : 1u) * Wn4 + st * cc * g.S + win * 32u + win * 16u + own * 32u +
                 (own + 1u) / 2u * 2u) +
           8u * own * 64u + 2u * win * 32u;
}

cudaError_t configure_learn_grid(int max_smem) {
    cudaFuncAttributes a{};
    cudaError_t e = cudaFuncGetAttributes(&a, sp_learn_grid_kernel);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(sp_learn_grid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 max_smem - static_cast<int>(a.sharedSizeBytes));
    return e;
}

cudaError_t learn_grid_max_ctas(uint32_t smem, int* n) {
    int per_sm = 0, dev = 0, sms = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sp_learn_grid_kernel, kGridThreads, smem);
    if (e == cudaSuccess) e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    *n = e == cudaSuccess ? per_sm * sms : 0;
    if (e != cudaSuccess) (void)cudaGetLastError();
    return cudaSuccess;
}

cudaError_t launch_learn_grid(const LearnGridParams& p, uint32_t smem, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(p.gbar, 0, sizeof(uint32_t), s);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.G);
    cfg.blockDim = dim3(kGridThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, sp_learn_grid_kernel, p);
}

}  // namespace sp
