// sp_pack.cuh — device helpers shared by the learning kernels (sp_learn.cu, sp_learn_grid.cu):
// input staging (a1: byte frames/tiles -> input bit-planes, R12/R13), L2 prefetch, TMA
// bulk copies with mbarrier completion, and the warp-level global k-winners word (a4).
// PP is the kernel's parameter struct (fields frames, g, num_inputs, dbg, min_overlap, k,
// uniform_bc).
#pragma once

#include <cstdint>

#include "sp_internal.h"
#include "sp_select.cuh"

namespace sp {

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// L2 prefetch of [ptr, ptr + bytes) by the bulk-copy engine (one instruction; a hint)
__device__ __forceinline__ void prefetch_l2(const void* ptr, uint32_t bytes) {
    if (bytes == 0u || (reinterpret_cast<uintptr_t>(ptr) & 15u) != 0u || (bytes & 15u) != 0u) return;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ptr), "r"(bytes) : "memory");
}

// L2 prefetch of this CTA's share of the bytes input t reads (whole frame: the CTA's
// slice; patch mode: the CTA's share of the tile-row band, once per band)
template <typename PP>
__device__ __forceinline__ void prefetch_input(const PP& p, uint32_t t, uint32_t wbeg, uint32_t wend,
                                               uint32_t q, uint32_t Q) {
    const Geometry& g = p.g;
    if (t >= p.num_inputs || (p.dbg & 2u)) return;
    const uint32_t frame = t / g.P, tile = t % g.P;
    const uint8_t* fr = p.frames + static_cast<size_t>(frame) * g.W * g.H;
    if (g.whole) {
        const uint32_t b0 = wbeg * 32u, b1 = min(wend * 32u, g.nbits);
        if (b1 > b0) prefetch_l2(fr + b0, (b1 - b0) & ~15u);
        return;
    }
    const uint32_t tilesx = g.W / g.pw;
    if (t != 0u && tile % tilesx != 0u) return;  // band already prefetched
    const uint32_t band = g.ph * g.W, ty = tile / tilesx;
    const uint32_t lo = (band * q / Q) & ~15u, hi = q + 1u == Q ? band : (band * (q + 1u) / Q) & ~15u;
    if (hi > lo) prefetch_l2(fr + static_cast<size_t>(ty) * band + lo, (hi - lo) & ~15u);
}

// byte-nonzero flags of the 4 bytes of v as a nibble (bit j = byte j != 0): the high bit
// of each byte of f is set iff the byte is nonzero; the multiply gathers the four flags
// (at bits 0, 8, 16, 24 after the shift) into bits 21..24 without carries
__device__ __forceinline__ uint32_t nz_nibble(uint32_t v) {
    const uint32_t f = (((v & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | v) & 0x80808080u;
    return (((f >> 7) * 0x00204081u) >> 21) & 0xFu;
}

// address of the first byte of word w of input t; run = its 32 bytes are contiguous
template <typename PP>
__device__ __forceinline__ const uint8_t* word_src(const PP& p, uint32_t t, uint32_t w, bool& run) {
    const Geometry& g = p.g;
    const uint32_t frame = t / g.P, tile = t % g.P;
    const uint8_t* fr = p.frames + static_cast<size_t>(frame) * g.W * g.H;
    const uint32_t q0 = w * 32u;
    if (g.whole) {
        run = q0 + 32u <= g.nbits;
        return fr + q0;
    }
    const uint32_t tilesx = g.W / g.pw, ty = tile / tilesx, tx = tile % tilesx;
    const uint32_t y = q0 / g.pw, x = q0 % g.pw;
    run = x + 32u <= g.pw && q0 + 32u <= g.nbits;
    return fr + static_cast<size_t>(ty * g.ph + y) * g.W + tx * g.pw + x;
}

// word w of input t bit by bit (ragged tails, patches narrower than 32 bits)
template <typename PP>
__device__ __forceinline__ uint32_t pack_word_slow(const PP& p, uint32_t t, uint32_t w) {
    const Geometry& g = p.g;
    const uint32_t frame = t / g.P, tile = t % g.P;
    const uint8_t* fr = p.frames + static_cast<size_t>(frame) * g.W * g.H;
    const uint32_t tilesx = g.W / g.pw, ty = tile / tilesx, tx = tile % tilesx;
    uint32_t out = 0;
#pragma unroll 1
    for (uint32_t jj = 0; jj < 32u; ++jj) {
        const uint32_t qq = w * 32u + jj;
        if (qq >= g.nbits) break;
        uint8_t b;
        if (g.whole) {
            b = fr[qq];
        } else {
            const uint32_t y = qq / g.pw, x = qq % g.pw;
            b = fr[static_cast<size_t>(ty * g.ph + y) * g.W + tx * g.pw + x];
        }
        out |= (b != 0 ? 1u : 0u) << jj;
    }
    return out;
}

// this CTA's share (words [wbeg, wend)) of the bit-plane of input t -> global buffer dst
// (bit j of word w = byte 32w+j != 0, R12), by threads [t0, t0 + nt) of the CTA; the loads
// of U words per thread are issued before any is used (one L2 round trip per U words).
// The stores are then made visible to the bulk-copy (async) proxy of the CTAs that read
// the buffer after the next cluster barrier.
template <typename PP>
__device__ __forceinline__ void pack_slice(const PP& p, uint32_t t, uint32_t wbeg, uint32_t wend,
                                           uint32_t* dst, uint32_t t0, uint32_t nt) {
    if (threadIdx.x < t0 || threadIdx.x >= t0 + nt) return;
    constexpr int U = 4;
    for (uint32_t base = wbeg + threadIdx.x - t0; base < wend; base += U * nt) {
        uint4 a[U], b[U];
        bool vec[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t w = base + u * nt;
            bool run = false;
            const uint8_t* src = w < wend ? word_src(p, t, w, run) : nullptr;
            vec[u] = run && (reinterpret_cast<uintptr_t>(src) & 15u) == 0;
            if (vec[u]) {
                if (p.dbg & 32u) {
                    a[u] = __ldcg(reinterpret_cast<const uint4*>(src));
                    b[u] = __ldcg(reinterpret_cast<const uint4*>(src + 16));
                } else {
                    a[u] = __ldcs(reinterpret_cast<const uint4*>(src));
                    b[u] = __ldcs(reinterpret_cast<const uint4*>(src + 16));
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t w = base + u * nt;
            if (vec[u])
                dst[w] = nz_nibble(a[u].x) | nz_nibble(a[u].y) << 4 | nz_nibble(a[u].z) << 8 |
                         nz_nibble(a[u].w) << 12 | nz_nibble(b[u].x) << 16 | nz_nibble(b[u].y) << 20 |
                         nz_nibble(b[u].z) << 24 | nz_nibble(b[u].w) << 28;
        }
        // ragged / unaligned words bit by bit, after the vector registers are dead
#pragma unroll 1
        for (int u = 0; u < U; ++u) {
            const uint32_t w = base + u * nt;
            if (w < wend && !vec[u]) dst[w] = pack_word_slow(p, t, w);
        }
    }
    if (!(p.dbg & 1u)) asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
                 "r"(count)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
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

// one thread: bulk copy (TMA engine) of the global bit-plane src[0, Wn) into smem dst,
// completion counted on bar (expect_tx)
__device__ __forceinline__ void bulk_load_bits(uint32_t* dst, const uint32_t* src, uint32_t Wn, uint64_t* bar) {
    const uint32_t bytes = (Wn * 4u + 15u) & ~15u;
    const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
    asm volatile("fence.proxy.async.global;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    constexpr uint32_t kChunk = 16384u;
    for (uint32_t off = 0; off < bytes; off += kChunk) {
        const uint32_t n = min(kChunk, bytes - off);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                static_cast<uint32_t>(__cvta_generic_to_shared(reinterpret_cast<uint8_t*>(dst) + off))),
            "l"(reinterpret_cast<const uint8_t*>(src) + off), "r"(n), "r"(b)
            : "memory");
    }
}

// warp-level global k-winners of column-word gcw (r = 0); NR registers hold 64 * NR columns
template <int NR, typename PP>
__device__ __forceinline__ uint32_t global_word(const PP& p, const uint16_t* row, const uint32_t* s_bc,
                                                uint64_t* ties, uint32_t gcw, uint32_t lane) {
    const Geometry& g = p.g;
    const uint32_t theta = p.min_overlap, L = g.keyL;
    const uint32_t c = gcw * 32u + lane;
    if (p.uniform_bc) {
        const uint32_t r_lo = uniform_r_lo(theta, s_bc[0]);
        uint32_t rgt, rtie, need;
        global_uniform_threshold<NR>(row, g.C32, g.S, p.k, r_lo, lane, rgt, rtie, need);
        uint32_t before = 0;  // ties at raw == r* in lower column-words
        for (uint32_t d = lane; d < gcw * 32u; d += 32u) before += row[d] == rtie ? 1u : 0u;
        before = __reduce_add_sync(0xffffffffu, before);
        const uint32_t r = c < g.C ? row[c] : 0u;
        const uint32_t tb = __ballot_sync(0xffffffffu, r == rtie);
        return __ballot_sync(0xffffffffu,
                             r >= rgt || (r == rtie && before + __popc(tb & ((1u << lane) - 1u)) < need));
    }
    const uint32_t sh = g.keyBits - L - 16u;
    uint32_t Tu;
    uint64_t T2;
    global_general_threshold<NR>(row, s_bc, g.C32, g.ncw, p.k, theta, sh, L, g.keyBits, ties, lane, Tu, T2);
    uint64_t N = 0, key = 0;
    if (c < g.C) key = exact_key(row[c], s_bc[c], theta, c, L, N);
    return __ballot_sync(0xffffffffu, c < g.C && global_general_wins(N, key, sh, Tu, T2));
}


}  // namespace sp
