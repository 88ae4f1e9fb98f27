// sp_topk.cuh -- rows a3/a4 for a group of SP inputs whose raw counts sit in shared memory
// (u16 rawbuf[input][C32]): cutoff, exact boost keys, k-winners (global / local, uniform /
// per-column boosts) and the SDR words, one warp per input.  Shared by the
// bit-sliced batched and patch kernels (sp_batched.cu) and the tensor-core patch kernel
// (sp_patch_mma.cu).  Selection building blocks: sp_select.cuh.
#pragma once

#include <cooperative_groups.h>
#include <cuda_fp16.h>

#include "sp_internal.h"
#include "sp_select.cuh"

namespace sp {

// Rank key of column c (R4/R6): exact boosted overlap N = raw*Bc over 2^23,
// ties broken towards the lower index.
__device__ __forceinline__ uint64_t rank_key(uint32_t raw, uint32_t bc, uint32_t theta, uint32_t c,
                                             uint32_t L, uint64_t& N) {
    N = raw >= theta ? static_cast<uint64_t>(raw) * bc : 0ull;
    return (N << L) | (((1ull << L) - 1ull) - c);
}


// a3/a4 for the inputs of this CTA: (cluster-sum of partial counts), exact keys, k-winners,
// SDR.  Kept out of line so its register needs do not shape the streaming loop's allocation.
// big / big_bytes: shared memory idle during the top-k (region plus, in the whole-frame kernel,
// the ring behind the raw counts) for the per-column-boost wavelet.
template <int CPT, uint32_t NW>
__device__ __noinline__ void batched_topk(const BatchedParams& p, uint16_t* rawbuf, uint8_t* region,
                                          uint8_t* big, uint32_t big_bytes,
                                          const uint32_t* s_bc, uint32_t in0, uint32_t gs,
                                          uint32_t rank, uint32_t K, uint32_t wi, uint32_t lane) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const uint32_t theta = p.min_overlap, L = p.keyL;
    const uint64_t one = 1ull << 23;
    uint32_t radius = p.radius_dev ? *p.radius_dev : p.radius;  // adapted by full learning
    if (radius + 1u >= p.C) radius = 0u;  // every window holds all columns: global inhibition (R9)
    const uint32_t nbN = p.keyBits - L;             // significant bits of N
    const uint32_t sh = nbN > 16u ? nbN - 16u : 0u;  // coarse key u = N >> sh has <= 16 bits
    uint64_t* tie_list = reinterpret_cast<uint64_t*>(region) + wi * 64u;  // X window is idle now
    // local inhibition with a uniform boost: per-warp wavelet slots (sized for 8 levels; below).
    // When 16 slots fit neither in the windows nor in `big` (C32 = 2048: the raw counts fill the
    // ring), only the warps whose slots fit in `big` take inputs ("narrow"), so every input
    // still gets the O(C log range) wavelet instead of the O(C r) comparator.
    const uint32_t wbytes = (2u * p.C32 + 8u * 8u * (p.ncw + 2u) + 127u) & ~127u;
    const uint32_t slot2 = max(2u * wbytes, 2560u), slot1 = max(wbytes, 2560u);
    uint32_t nwork = NW;
    bool narrow = false;
    if (radius > 0 && p.uniform_bc && slot1 * NW > p.region_bytes && slot2 * NW > big_bytes &&
        slot1 * NW > big_bytes && slot1 * (NW / 2u) <= big_bytes) {
        nwork = big_bytes / slot1;
        narrow = true;
    }
    for (uint32_t f = rank + K * wi; wi < nwork && f < gs; f += K * nwork) {
        uint16_t* row = rawbuf + f * p.C32;
        if (K > 1 && !p.gsplit) {
            // sum the K partial rows (DSMEM): 16-byte loads of 8 counts, packed u16 adds (a sum
            // is a raw count <= S < 2^16, so no carry crosses a half); every load of a pass is
            // issued before its stores, so the remote latencies overlap
            uint4* row4 = reinterpret_cast<uint4*>(row);
            const uint32_t nv = p.C32 / 8u;
            for (uint32_t v0 = lane; v0 < nv; v0 += 128u) {
                uint4 acc[4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    acc[i] = v0 + 32u * i < nv ? row4[v0 + 32u * i] : make_uint4(0u, 0u, 0u, 0u);
                for (uint32_t q = 0; q < K; ++q) {
                    if (q == rank) continue;
                    const uint4* rr = cluster.map_shared_rank(row4, q);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        if (v0 + 32u * i < nv) {
                            const uint4 t = rr[v0 + 32u * i];
                            acc[i].x += t.x, acc[i].y += t.y, acc[i].z += t.z, acc[i].w += t.w;
                        }
                    }
                }
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (v0 + 32u * i < nv) row4[v0 + 32u * i] = acc[i];
            }
            __syncwarp();
        }
        const uint32_t gin = in0 + f;
        // optional test outputs (SP_FLAG_RECORD_OVERLAPS); the paired branches below record
        // their second input too, so recording does not change which selection code runs
        auto record = [&](const uint16_t* rw, uint32_t g) {
            if (!p.raw_out) return;
            for (uint32_t c = lane; c < p.C; c += 32u) {
                const uint32_t r = rw[c];
                p.raw_out[static_cast<size_t>(g) * p.C + c] = static_cast<uint16_t>(r);
                p.boosted_out[static_cast<size_t>(g) * p.C + c] =
                    r >= theta ? __fmul_rn(static_cast<float>(r), p.boost[c]) : 0.0f;
            }
        };
        record(row, gin);
        if (radius == 0 && p.uniform_bc) {
            // Uniform boost: the key order is (raw desc, index asc), so the k-th largest key
            // is found from a histogram of the raw counts: with one boost
            // the floor raw*Bc > 2^23 (R7) is raw >= r_lo; r* = largest r with
            // #{raw >= max(r, r_lo)} >= k; winners = raw > r*, plus the lowest indices among
            // raw == r* up to k.  Exact; O(C/32 + S/32) per lane.
            const uint32_t r_lo = max(theta, (1u << 23) / s_bc[0] + 1u);
            // raw counts (<= 1023, exact in fp16) of this lane's columns, two per half2,
            // zeroed below r_lo; counts of raw >= x with HSET2/HADD2 (FMA pipe, no atomics)
            constexpr int NH = (CPT * NW + 1) / 2;
            const uint32_t f2 = f + K * NW;
            if (CPT * NW <= 32 && f2 < gs && K == 1u) {  // NH <= 16 half2 registers per input
                // this warp's next input too: both searches and SDR loops interleaved
                const uint16_t* row2 = rawbuf + f2 * p.C32;
                const uint32_t gin2 = in0 + f2;
                record(row2, gin2);
                uint32_t rgt[2], rtie[2], need[2];
                global_uniform_threshold2<NH>(row, row2, p.C32, p.S, p.k, r_lo, lane, rgt, rtie, need);
                const uint32_t tot0 = uniform_sdr_words(row, p.ncw, rgt[0], rtie[0], need[0], lane,
                                                        [&](uint32_t w, uint32_t word) {
                                                            p.sdr[static_cast<size_t>(gin) * p.ncw + w] = word;
                                                        });
                const uint32_t tot1 = uniform_sdr_words(row2, p.ncw, rgt[1], rtie[1], need[1], lane,
                                                        [&](uint32_t w, uint32_t word) {
                                                            p.sdr[static_cast<size_t>(gin2) * p.ncw + w] = word;
                                                        });
                if (lane == 0) p.counts[gin] = tot0, p.counts[gin2] = tot1;
                f = f2;  // the loop's increment moves past f2
                continue;
            }
            uint32_t rgt, rtie, need;
            global_uniform_threshold<NH>(row, p.C32, p.S, p.k, r_lo, lane, rgt, rtie, need);
            const uint32_t total = uniform_sdr_words(row, p.ncw, rgt, rtie, need, lane, [&](uint32_t w, uint32_t word) {
                p.sdr[static_cast<size_t>(gin) * p.ncw + w] = word;
            });
            if (lane == 0) p.counts[gin] = total;
            continue;
        }
        if (radius > 0 && p.uniform_bc) {
            const uint32_t r_lo = uniform_r_lo(theta, s_bc[0]);
            // range of the eligible raw counts of an input: the wavelet path needs <= 8 levels
            auto range_of = [&](const uint16_t* rw, uint32_t& xmn, uint32_t& Bo) {
                uint32_t mn = 0xFFFFFFFFu, mx = 0u;
                for (uint32_t c = lane; c < p.C; c += 32u) {
                    const uint32_t x = rw[c];
                    if (x >= r_lo) mn = min(mn, x), mx = max(mx, x);
                }
                mn = __reduce_min_sync(0xffffffffu, mn);
                mx = __reduce_max_sync(0xffffffffu, mx);
                xmn = mn;
                Bo = mn <= mx ? 32u - __clz(mx - mn + 1u) : 1u;
            };
            // per-warp scratch slots sized for the largest B (8), so the warps' regions do not
            // depend on their inputs' ranges; a warp's comparator fallback uses its own slot too.
            // With room in the idle ring + windows (`big`), a slot holds two wavelets and the warp
            // runs its two inputs together.
            const bool pairs = !narrow && K == 1u && slot2 * NW <= big_bytes;
            const bool slotted = pairs || narrow || slot1 * NW <= p.region_bytes;
            uint8_t* wslot = pairs ? big + wi * slot2 : narrow ? big + wi * slot1 : region + wi * slot1;
            if (radius >= p.cand_min_radius_u && slotted) {
                // candidate pruning (sp_select.cuh): O(C k / r) per input
                constexpr int NW2 = CPT * NW > 32 ? 2 : 1;
                uint32_t total = 0, myword = 0;
                const CoarseMap cm0{0ull, 0u};
                if (local_candidates<NW2, true, uint32_t>(row, s_bc, p.C, p.ncw, radius, p.k, theta, r_lo, L, cm0,
                                                         wslot, pairs ? slot2 : slot1, lane,
                                                         [&](uint32_t cw, uint32_t word) {
                                                             if ((cw & 31u) == lane) myword = word;
                                                             total += __popc(word);
                                                             if ((cw & 31u) == 31u || cw + 1u == p.ncw) {
                                                                 const uint32_t w0 = cw & ~31u;
                                                                 if (lane <= (cw & 31u))
                                                                     p.sdr[static_cast<size_t>(gin) * p.ncw + w0 +
                                                                           lane] = myword;
                                                             }
                                                         }, p.cand_dbg)) {
                    if (lane == 0) p.counts[gin] = total;
                    continue;
                }
            }
            uint32_t xmn, B;
            range_of(row, xmn, B);
            const uint32_t f2 = f + K * NW;
            if (pairs && f2 < gs && B <= 8u) {
                const uint16_t* row2 = rawbuf + f2 * p.C32;
                uint32_t xmn2, B2;
                range_of(row2, xmn2, B2);
                if (B2 <= 8u) {
                    const uint32_t gin2 = in0 + f2;
                    record(row2, gin2);
                    const uint16_t* rows[2] = {row, row2};
                    const uint32_t xmins[2] = {xmn, xmn2};
                    uint8_t* b0s[2] = {wslot, wslot + wbytes};
                    uint8_t* b1s[2] = {wslot + p.C32, wslot + wbytes + p.C32};
                    uint2* lvs[2] = {reinterpret_cast<uint2*>(wslot + 2u * p.C32),
                                     reinterpret_cast<uint2*>(wslot + wbytes + 2u * p.C32)};
                    uint32_t total[2] = {0u, 0u}, myw[2] = {0u, 0u};
                    const uint32_t gins[2] = {gin, gin2};
                    local_uniform_wavelet<2>(rows, p.C, p.C32, p.ncw, radius, p.k, r_lo, xmins, max(B, B2), b0s, b1s,
                                             lvs, lane, [&](int i, uint32_t cw, uint32_t word) {
                                                 if ((cw & 31u) == lane) myw[i] = word;
                                                 total[i] += __popc(word);
                                                 if ((cw & 31u) == 31u || cw + 1u == p.ncw) {
                                                     const uint32_t w0 = cw & ~31u;
                                                     if (lane <= (cw & 31u))
                                                         p.sdr[static_cast<size_t>(gins[i]) * p.ncw + w0 + lane] = myw[i];
                                                 }
                                             });
                    if (lane == 0) p.counts[gin] = total[0], p.counts[gin2] = total[1];
                    f = f2;  // the loop's increment moves past f2
                    continue;
                }
            }
            if (B <= 8u && slotted) {
                // wavelet matrix over the positions (sp_select.cuh): O(C log range) per input
                const uint16_t* rows[1] = {row};
                const uint32_t xmins[1] = {xmn};
                uint8_t* b0s[1] = {wslot};
                uint8_t* b1s[1] = {wslot + p.C32};
                uint2* lvs[1] = {reinterpret_cast<uint2*>(wslot + 2u * p.C32)};
                uint32_t total = 0, myword = 0;
                local_uniform_wavelet<1>(rows, p.C, p.C32, p.ncw, radius, p.k, r_lo, xmins, B, b0s, b1s, lvs, lane,
                                         [&](int, uint32_t cw, uint32_t word) {
                                             if ((cw & 31u) == lane) myword = word;
                                             total += __popc(word);
                                             if ((cw & 31u) == 31u || cw + 1u == p.ncw) {
                                                 const uint32_t w0 = cw & ~31u;
                                                 if (lane <= (cw & 31u))
                                                     p.sdr[static_cast<size_t>(gin) * p.ncw + w0 + lane] = myword;
                                             }
                                         });
                if (lane == 0) p.counts[gin] = total;
                continue;
            }
            // local inhibition, uniform boost: bit-sliced window comparator (sp_select.cuh)
            const uint32_t nb = raw_bits(p.S);
            uint32_t* planes = reinterpret_cast<uint32_t*>(slotted ? wslot : region + wi * 2560u);  // [ncw <= 64][nb <= 10]
            build_raw_planes(row, planes, p.ncw, nb, r_lo, 0u, 1u, lane);
            __syncwarp();
            uint32_t total = 0, myword = 0;
            for (uint32_t cw = 0; cw < p.ncw; ++cw) {
                const uint32_t word = local_uniform_word(row, planes, p.ncw, nb, cw, p.C, radius, p.k,
                                                         r_lo, lane);
                if ((cw & 31u) == lane) myword = word;
                total += __popc(word);
                if ((cw & 31u) == 31u || cw + 1u == p.ncw) {
                    const uint32_t base = cw & ~31u;
                    if (lane <= (cw & 31u)) p.sdr[static_cast<size_t>(gin) * p.ncw + base + lane] = myword;
                }
            }
            if (lane == 0) p.counts[gin] = total;
            __syncwarp();  // planes are rewritten by this warp's next input
            continue;
        }
        const uint32_t gwb = (4u * p.C32 + 2u * 16u * (p.ncw + 2u) * 4u + 127u) & ~127u;  // <= 15 levels + lossy
        // this warp's scratch slot for local inhibition with per-column boosts; every selector of
        // the warp (candidates, wavelet, comparator fallback) uses it, so warps that take
        // different selectors for different inputs never overlap
        uint8_t* cs = nullptr;
        uint32_t cbytes = 0;
        if (gwb * NW <= big_bytes) cs = big + wi * gwb, cbytes = gwb;
        else if (NW * 4096u <= p.region_bytes) cs = region + wi * 4096u, cbytes = 4096u;
        if (radius > 0 && radius >= p.cand_min_radius) {
            // local inhibition, per-column boosts: candidate pruning (sp_select.cuh), O(C k / r)
            if (cs) {
                constexpr int NW2 = CPT * NW > 32 ? 2 : 1;
                const CoarseMap cm = coarse_map_warp(row, s_bc, theta, 0u, p.ncw, lane, p.wm_umax);
                uint32_t total = 0, myword = 0;
                if (local_candidates<NW2, false, uint64_t>(row, s_bc, p.C, p.ncw, radius, p.k, theta, 0u, L, cm, cs,
                                                          cbytes, lane, [&](uint32_t cw, uint32_t word) {
                                                              if ((cw & 31u) == lane) myword = word;
                                                              total += __popc(word);
                                                              if ((cw & 31u) == 31u || cw + 1u == p.ncw) {
                                                                  const uint32_t w0 = cw & ~31u;
                                                                  if (lane <= (cw & 31u))
                                                                      p.sdr[static_cast<size_t>(gin) * p.ncw + w0 +
                                                                            lane] = myword;
                                                              }
                                                          }, p.cand_dbg)) {
                    if (lane == 0) p.counts[gin] = total;
                    continue;
                }
            }
        }
        if (radius > 0 && radius >= p.wm_min_radius && gwb * NW <= big_bytes) {
            // local inhibition, per-column boosts: wavelet matrix over the coarse keys + exact
            // lossy ties (sp_select.cuh), O(C log 2^15) per input
            uint8_t* base = big + wi * gwb;
            uint16_t* b0 = reinterpret_cast<uint16_t*>(base);
            uint2* lv = reinterpret_cast<uint2*>(base + 4u * p.C32);
            const CoarseMap cm = coarse_map_warp(row, s_bc, theta, 0u, p.ncw, lane, p.wm_umax);
            uint32_t total = 0, myword = 0;
            local_general_wavelet(row, s_bc, p.C, p.C32, p.ncw, radius, p.k, theta, L, cm, b0, b0 + p.C32, lv,
                                  lane, [&](uint32_t cw, uint32_t word) {
                                      if ((cw & 31u) == lane) myword = word;
                                      total += __popc(word);
                                      if ((cw & 31u) == 31u || cw + 1u == p.ncw) {
                                          const uint32_t w0 = cw & ~31u;
                                          if (lane <= (cw & 31u))
                                              p.sdr[static_cast<size_t>(gin) * p.ncw + w0 + lane] = myword;
                                      }
                                  });
            if (lane == 0) p.counts[gin] = total;
            continue;
        }
        if (radius > 0 && p.ncw * 16u <= 1024u && cs) {
            // local inhibition, per-column boosts: coarse bit-sliced + exact ties
            uint32_t* planes = reinterpret_cast<uint32_t*>(cs);  // [ncw][16] (ncw * 64 <= 4096 bytes)
            const CoarseMap cm = coarse_map_warp(row, s_bc, theta, 0u, p.ncw, lane);
            build_coarse_planes15(row, s_bc, planes, p.ncw, theta, cm, 0u, 1u, lane);
            __syncwarp();
            uint32_t total = 0, myword = 0;
            for (uint32_t cw = 0; cw < p.ncw; ++cw) {
                const uint32_t word = local_general_word15(row, s_bc, planes, p.ncw, cw, p.C, radius,
                                                           p.k, theta, cm, L, lane);
                if ((cw & 31u) == lane) myword = word;
                total += __popc(word);
                if ((cw & 31u) == 31u || cw + 1u == p.ncw) {
                    const uint32_t base = cw & ~31u;
                    if (lane <= (cw & 31u)) p.sdr[static_cast<size_t>(gin) * p.ncw + base + lane] = myword;
                }
            }
            if (lane == 0) p.counts[gin] = total;
            __syncwarp();
            continue;
        }
        uint32_t Tu = 0;       // k-th largest coarse key
        uint64_t T2 = 0;       // exact key threshold among the columns with u == Tu
        if (radius == 0) {
            constexpr int NU = (CPT * NW + 1) / 2;  // column-warps of this CTA, two per register
            global_general_threshold<NU>(row, s_bc, p.C32, p.ncw, p.k, theta, sh, L, p.keyBits, tie_list,
                                         lane, Tu, T2);
        }
        uint32_t total = 0;
        for (uint32_t cw = 0; cw < p.ncw; ++cw) {
            const uint32_t c = cw * 32u + lane;
            uint64_t N;
            const uint64_t key = rank_key(row[c], s_bc[c], theta, c, L, N);
            bool act = N > one;
            if (act) {
                if (radius == 0) {
                    act = global_general_wins(N, key, sh, Tu, T2);
                } else {
                    const uint32_t lo = c >= radius ? c - radius : 0u;
                    const uint32_t hi = min(p.C - 1u, c + radius);
                    uint32_t beats = 0;
                    for (uint32_t d = lo; d <= hi && beats < p.k; ++d) {
                        uint64_t Nd;
                        beats += (d != c && rank_key(row[d], s_bc[d], theta, d, L, Nd) > key) ? 1u : 0u;
                    }
                    act = beats < p.k;
                }
            }
            const uint32_t word = __ballot_sync(0xffffffffu, act);
            if (lane == 0) p.sdr[static_cast<size_t>(gin) * p.ncw + cw] = word;
            total += __popc(word);
        }
        if (lane == 0) p.counts[gin] = total;
    }
}

}  // namespace sp
