// sp_learn.cu — cluster-resident sequential learning (learn=1).
//
// Learning is a recurrence over inputs (input t+1 sees input t's permanence
// update), so it cannot be batched.  One launch processes the whole stream with a
// thread-block cluster of Q CTAs (Q <= 16) that keeps the synapse table idx|connected
// (synapse-major, the CTA's column slice) resident in shared memory:
//
//   per input t:  pack a 1/Q slice of the frame -> global bit-plane (L2)
//                 cluster barrier #1
//                 every CTA loads the bit-plane into smem (ld.global.cg)
//                 overlap of the CTA's columns (thread per column), raw counts are
//                 broadcast to every CTA's smem through DSMEM
//                 cluster barrier #2
//                 every CTA runs the same exact k-winners over all columns, writes the
//                 SDR words of its columns, and updates the permanences of its winners
//                 (fp32 RN add/sub + clamp, R3) and their connected flags in smem
//
// Two cluster barriers per input; only the frame bytes and the winners' permanence rows
// touch memory below L2.  DESIGN.md §4.2.
#include <cooperative_groups.h>

#include "sp_internal.h"
#include "sp_select.cuh"

namespace cg = cooperative_groups;

namespace sp {

namespace {

constexpr uint32_t kLearnThreads = 512;

__device__ __forceinline__ uint64_t key_of(uint32_t raw, uint32_t bc, uint32_t theta, uint32_t c,
                                           uint32_t L, uint64_t& N) {
    N = raw >= theta ? static_cast<uint64_t>(raw) * bc : 0ull;
    return (N << L) | (((1ull << L) - 1ull) - c);
}

// Block-wide sum of one value per thread (all threads call it).
__device__ __forceinline__ uint32_t block_sum(uint32_t v, uint32_t* scratch) {
    const uint32_t lane = threadIdx.x & 31u, wi = threadIdx.x >> 5;
    v = __reduce_add_sync(0xffffffffu, v);
    __syncthreads();
    if (lane == 0) scratch[wi] = v;
    __syncthreads();
    uint32_t t = 0;
    for (uint32_t i = 0; i < (blockDim.x >> 5); ++i) t += scratch[i];
    return t;
}

}  // namespace

__global__ void __launch_bounds__(kLearnThreads, 1) sp_learn_cluster_kernel(const LearnParams p) {
    extern __shared__ __align__(16) uint8_t smem[];
    cg::cluster_group cluster = cg::this_cluster();
    const Geometry& g = p.g;
    const uint32_t tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31u;
    const uint32_t q = cluster.block_rank(), Q = p.Q;
    const uint32_t cpc = p.cols_per_cta;        // columns owned by this CTA (multiple of 32)
    const uint32_t c0 = q * cpc;                 // first column owned
    const uint32_t Wn = p.Wn;

    const uint32_t ss = p.syn_stride;                               // >= S, == 8 mod 32
    uint32_t* s_syn = reinterpret_cast<uint32_t*>(smem);           // [cpc][ss] idx | connected<<31
    uint32_t* s_bits = s_syn + static_cast<size_t>(ss) * cpc;      // [Wn] input bit-plane
    uint32_t* s_bc = s_bits + Wn;                                   // [C32]
    uint16_t* s_raw = reinterpret_cast<uint16_t*>(s_bc + g.C32);    // [C32] all columns' raw
    uint32_t* s_hist = reinterpret_cast<uint32_t*>(s_raw + g.C32 + (g.C32 & 1u));  // [S+1]
    uint32_t* s_red = s_hist + g.S + 1u;                            // [32] block reductions
    uint32_t* s_misc = s_red + 32u;                                 // [4]
    uint32_t* s_sdr = s_misc + 4u;                                  // [cpc/32] this CTA's SDR words
    uint32_t* s_planes = s_sdr + cpc / 32u;                         // [ncw][nb] raw bit-planes

    // ---- resident state: this CTA's synapse slice, Bc -----------------------------------
    for (uint32_t i = tid; i < g.S * cpc; i += nthr) {
        const uint32_t s = i / cpc, cl = i % cpc, c = c0 + cl;
        s_syn[cl * ss + s] = c < g.C32 ? p.syn[static_cast<size_t>(s) * g.C32 + c] : 0u;
    }
    for (uint32_t c = tid; c < g.C32; c += nthr) s_bc[c] = p.bc[c];
    __syncthreads();

    const uint32_t theta = p.min_overlap, L = g.keyL;
    const uint64_t one = 1ull << 23;
    const uint32_t wbeg = q * Wn / Q, wend = (q + 1) * Wn / Q;  // packed words of this CTA

    for (uint32_t t = 0; t < p.num_inputs; ++t) {
        const uint32_t gin = p.first_input + t;
        if (q == 0 && tid == 0) p.counts[gin] = 0u;  // winners are added after barrier #2
        // ---- a1: pack this CTA's slice of input t into the global bit-plane --------------
        {
            const uint32_t frame = t / g.P, tile = t % g.P;
            const uint8_t* fr = p.frames + static_cast<size_t>(frame) * g.W * g.H;
            const bool vec = g.whole && (g.nbits % 16u) == 0 && (reinterpret_cast<uintptr_t>(fr) & 15u) == 0;
            const uint32_t tilesx = g.W / g.pw;
            const uint32_t ty = tile / tilesx, tx = tile % tilesx;
            for (uint32_t w = wbeg + tid; w < wend; w += nthr) {
                const uint32_t q0 = w * 32u;
                uint32_t out = 0;
                if (vec && q0 + 32u <= g.nbits) {
                    const uint4 a = __ldcs(reinterpret_cast<const uint4*>(fr + q0));
                    const uint4 b = __ldcs(reinterpret_cast<const uint4*>(fr + q0 + 16));
                    const uint32_t v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
                    for (int k = 0; k < 8; ++k)
#pragma unroll
                        for (int by = 0; by < 4; ++by)
                            out |= (((v[k] >> (8 * by)) & 0xFFu) != 0u ? 1u : 0u) << (4 * k + by);
                } else {
                    for (uint32_t jj = 0; jj < 32u; ++jj) {
                        const uint32_t qq = q0 + jj;
                        if (qq >= g.nbits) break;
                        const uint32_t y = qq / g.pw, x = qq % g.pw;
                        out |= (fr[static_cast<size_t>(ty * g.ph + y) * g.W + tx * g.pw + x] != 0 ? 1u : 0u) << jj;
                    }
                }
                p.bits_g[w] = out;
            }
        }
        cluster.sync();  // #1: the whole bit-plane of input t is in global memory (L2)
        {
            const uint32_t n4 = Wn / 4u;
            const uint4* src = reinterpret_cast<const uint4*>(p.bits_g);
            for (uint32_t w = tid; w < n4; w += nthr) reinterpret_cast<uint4*>(s_bits)[w] = __ldcg(src + w);
            for (uint32_t w = n4 * 4u + tid; w < Wn; w += nthr) s_bits[w] = __ldcg(p.bits_g + w);
        }
        __syncthreads();

        // ---- a2: overlap of this CTA's columns; raw counts to every CTA (DSMEM) ----------
        // tpc consecutive lanes share a column (synapses s = part, part+tpc, ..), then a
        // shuffle reduction; the padded column-major slice keeps the reads conflict-free
        for (uint32_t base = 0; base < cpc * p.tpc; base += nthr) {
            const uint32_t slot = base + tid;
            const uint32_t cl = slot / p.tpc, part = slot % p.tpc;
            uint32_t raw = 0;
            if (cl < cpc) {
                const uint32_t* col = s_syn + cl * ss;
                for (uint32_t s = part; s < g.S; s += p.tpc) {
                    const uint32_t e = col[s];
                    raw += (s_bits[(e & 0x7FFFFFFFu) >> 5] >> (e & 31u)) & (e >> 31);
                }
            }
            for (uint32_t d = p.tpc >> 1; d > 0; d >>= 1) raw += __shfl_xor_sync(0xffffffffu, raw, d);
            const uint32_t c = c0 + cl;
            if (part == 0 && cl < cpc && c < g.C32) {
                for (uint32_t r = 0; r < Q; ++r) cluster.map_shared_rank(s_raw, r)[c] = static_cast<uint16_t>(raw);
                if (p.raw_out && c < g.C) {
                    p.raw_out[static_cast<size_t>(gin) * g.C + c] = static_cast<uint16_t>(raw);
                    p.boosted_out[static_cast<size_t>(gin) * g.C + c] =
                        raw >= theta ? __fmul_rn(static_cast<float>(raw), p.boost[c]) : 0.0f;
                }
            }
        }
        cluster.sync();  // #2: every CTA holds all raw counts of input t

        // ---- a3/a4: the same exact k-winners in every CTA ---------------------------------
        int rstar = -1;
        uint32_t need = 0;
        uint64_t T = 0;
        if (p.radius == 0 && p.uniform_bc) {
            // histogram of the eligible raw counts; r* = largest r with #{raw >= r} >= k
            for (uint32_t b = tid; b <= g.S; b += nthr) s_hist[b] = 0u;
            __syncthreads();
            for (uint32_t c = tid; c < g.C; c += nthr) {
                const uint32_t r = s_raw[c];
                if (r >= theta) atomicAdd(&s_hist[r], 1u);
            }
            __syncthreads();
            if (tid < 32) {
                const uint32_t B = (g.S + 1u + 31u) / 32u;
                const uint32_t lo = tid * B;
                uint32_t mine = 0;
                for (uint32_t b = 0; b < B; ++b)
                    if (lo + b <= g.S) mine += s_hist[lo + b];
                uint32_t incl = mine;
#pragma unroll
                for (uint32_t d = 1; d < 32u; d <<= 1) {
                    const uint32_t v = __shfl_down_sync(0xffffffffu, incl, d);
                    if (tid + d < 32u) incl += v;
                }
                const uint32_t crossing = __ballot_sync(0xffffffffu, incl >= p.k);
                int rs = -1;
                uint32_t nd = 0;
                if (crossing) {
                    const uint32_t Lc = 31u - __clz(crossing);
                    uint32_t acc = __shfl_sync(0xffffffffu, incl - mine, Lc);
                    if (tid == Lc) {
                        for (int b = static_cast<int>(B) - 1; b >= 0; --b) {
                            const uint32_t r = lo + b;
                            if (r > g.S) continue;
                            if (acc + s_hist[r] >= p.k) {
                                rs = static_cast<int>(r);
                                nd = p.k - acc;
                                break;
                            }
                            acc += s_hist[r];
                        }
                    }
                    rs = __shfl_sync(0xffffffffu, rs, Lc);
                    nd = __shfl_sync(0xffffffffu, nd, Lc);
                }
                if (tid == 0) {
                    s_misc[0] = static_cast<uint32_t>(rs);
                    s_misc[1] = nd;
                }
            }
            __syncthreads();
            rstar = static_cast<int>(s_misc[0]);
            need = s_misc[1];
        } else if (p.radius == 0) {
            // exact bitwise search of the k-th largest key with block-wide counts
            for (int bit = static_cast<int>(g.keyBits) - 1; bit >= 0; --bit) {
                const uint64_t cand = T | (1ull << bit);
                uint32_t cnt = 0;
                for (uint32_t c = tid; c < g.C32; c += nthr) {
                    uint64_t N;
                    cnt += key_of(s_raw[c], s_bc[c], theta, c, L, N) >= cand ? 1u : 0u;
                }
                if (block_sum(cnt, s_red) >= p.k) T = cand;
            }
        }
        // winners of this CTA's columns -> SDR words; ties among raw == r* go to the lowest
        // indices over ALL columns, so count the ties before this CTA's range first
        uint32_t ties_before = 0;
        if (p.radius == 0 && p.uniform_bc && rstar >= 0) {
            uint32_t cnt = 0;
            for (uint32_t c = tid; c < c0 && c < g.C; c += nthr) {
                const uint32_t r = s_raw[c];
                cnt += (static_cast<int>(r) == rstar && static_cast<uint64_t>(r) * s_bc[c] > one) ? 1u : 0u;
            }
            ties_before = block_sum(cnt, s_red);
        }
        const uint32_t wi = tid >> 5, nw = nthr >> 5;
        if (p.radius > 0 && p.uniform_bc) {
            // local inhibition, uniform boost: bit-sliced window comparator (sp_select.cuh)
            const uint32_t r_lo = uniform_r_lo(theta, s_bc[0]);
            const uint32_t nb = raw_bits(g.S);
            build_raw_planes(s_raw, s_planes, g.ncw, nb, r_lo, wi, nw, lane);
            __syncthreads();
            for (uint32_t cw = wi; cw < cpc / 32u; cw += nw) {
                const uint32_t gcw = c0 / 32u + cw;
                uint32_t word = 0u;
                if (gcw < g.ncw)
                    word = local_uniform_word(s_raw, s_planes, g.ncw, nb, gcw, g.C, p.radius, p.k, r_lo, lane);
                if (lane == 0) {
                    s_sdr[cw] = word;
                    if (gcw < g.ncw) {
                        p.sdr[static_cast<size_t>(gin) * g.ncw + gcw] = word;
                        if (word) atomicAdd(p.counts + gin, static_cast<uint32_t>(__popc(word)));
                    }
                }
            }
        } else if (p.radius > 0) {
            // local inhibition, per-column boosts: coarse bit-sliced + exact ties
            const uint32_t sh = g.keyBits - L - 16u;
            build_coarse_planes(s_raw, s_bc, s_planes, g.ncw, theta, sh, wi, nw, lane);
            __syncthreads();
            for (uint32_t cw = wi; cw < cpc / 32u; cw += nw) {
                const uint32_t gcw = c0 / 32u + cw;
                uint32_t word = 0u;
                if (gcw < g.ncw)
                    word = local_general_word(s_raw, s_bc, s_planes, g.ncw, gcw, g.C, p.radius, p.k, theta,
                                              sh, L, lane);
                if (lane == 0) {
                    s_sdr[cw] = word;
                    if (gcw < g.ncw) {
                        p.sdr[static_cast<size_t>(gin) * g.ncw + gcw] = word;
                        if (word) atomicAdd(p.counts + gin, static_cast<uint32_t>(__popc(word)));
                    }
                }
            }
        } else
        for (uint32_t cw = wi; cw < cpc / 32u; cw += nw) {
            const uint32_t c = c0 + cw * 32u + lane;
            bool act = false;
            uint32_t tb = 0;
            if (c < g.C) {
                uint64_t N;
                const uint64_t key = key_of(s_raw[c], s_bc[c], theta, c, L, N);
                act = N > one;
                if (act) {
                    if (p.radius == 0 && p.uniform_bc) {
                        act = rstar < 0 || static_cast<int>(s_raw[c]) > rstar;
                    } else if (p.radius == 0) {
                        act = key >= T;
                    } else {
                        const uint32_t lo = c >= p.radius ? c - p.radius : 0u;
                        const uint32_t hi = min(g.C - 1u, c + p.radius);
                        uint32_t beats = 0;
                        for (uint32_t d = lo; d <= hi && beats < p.k; ++d) {
                            uint64_t Nd;
                            beats += (d != c && key_of(s_raw[d], s_bc[d], theta, d, L, Nd) > key) ? 1u : 0u;
                        }
                        act = beats < p.k;
                    }
                }
            }
            if (p.radius == 0 && p.uniform_bc && rstar >= 0) {
                // ties at raw == r*: rank by column index across the whole SP
                const bool tie = c < g.C && static_cast<int>(s_raw[c]) == rstar &&
                                 static_cast<uint64_t>(s_raw[c]) * s_bc[c] > one;
                tb = __ballot_sync(0xffffffffu, tie);
                // ties in earlier column-words of this CTA
                uint32_t earlier = 0;
                for (uint32_t cw2 = 0; cw2 < cw; ++cw2) {
                    const uint32_t c2 = c0 + cw2 * 32u + lane;
                    const bool t2 = c2 < g.C && static_cast<int>(s_raw[c2]) == rstar &&
                                    static_cast<uint64_t>(s_raw[c2]) * s_bc[c2] > one;
                    earlier += __popc(__ballot_sync(0xffffffffu, t2));
                }
                if (tie) act = ties_before + earlier + __popc(tb & ((1u << lane) - 1u)) < need;
            }
            const uint32_t word = __ballot_sync(0xffffffffu, act);
            if (lane == 0) {
                s_sdr[cw] = word;
                if (c0 / 32u + cw < g.ncw) {
                    p.sdr[static_cast<size_t>(gin) * g.ncw + c0 / 32u + cw] = word;
                    if (word) atomicAdd(p.counts + gin, static_cast<uint32_t>(__popc(word)));
                }
            }
        }
        // ---- a5: permanence update of this CTA's winners (warp per column) ---------------
        __syncthreads();  // s_sdr complete
        for (uint32_t cl = wi; cl < cpc; cl += nw) {
            const uint32_t c = c0 + cl;
            if (c >= g.C) break;
            if (((s_sdr[cl >> 5] >> (cl & 31u)) & 1u) == 0u) continue;
            const uint32_t* idx = p.idx + static_cast<size_t>(c) * g.S;
            float* perm = p.perm + static_cast<size_t>(c) * g.S;
            for (uint32_t s = lane; s < g.S; s += 32u) {
                const uint32_t i = idx[s];
                const bool on = ((s_bits[i >> 5] >> (i & 31u)) & 1u) != 0u;
                float v = on ? __fadd_rn(perm[s], p.inc) : __fsub_rn(perm[s], p.dec);
                v = fminf(fmaxf(v, 0.0f), 1.0f);
                perm[s] = v;
                s_syn[cl * ss + s] = i | (v >= p.tau ? 0x80000000u : 0u);
            }
        }
        __syncthreads();  // smem flags updated before the next input's overlap
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

uint32_t learn_cluster_smem(const Geometry& g, uint32_t Q, uint32_t* cols_per_cta) {
    const uint32_t cpc = ((g.C32 + Q - 1u) / Q + 31u) / 32u * 32u;
    const uint32_t Wn = (g.nbits + 31u) / 32u;
    if (cols_per_cta) *cols_per_cta = cpc;
    return 4u * (learn_syn_stride(g.S) * cpc + (Wn + 3u) / 4u * 4u + g.C32) + 2u * (g.C32 + (g.C32 & 1u)) +
           4u * (g.S + 1u + 32u + 4u) + 4u * (cpc / 32u) + 4u * (g.ncw * 16u);
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
