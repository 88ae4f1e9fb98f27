// sp_batched.cu — bit-sliced batched inference: staging + overlap + boost + inhibition
// fused in one kernel.
//
// Idea: the potential pools are the same for every frame, so a
// group of up to 32 SP inputs is processed together with one BIT per input in
// a 32-bit lane word.  For each pixel i the CTA builds, in shared memory, the
// word X[i] whose bit f is pixel i of input f (a 32x32 bit transpose of the
// uint8 frames, done with warp shuffles).  The overlap of column c for all 32
// inputs is then the bit-sliced ("vertical") population count of
//     X[idx[c,s]]  over its connected synapses s                 (Alg. 1 l.1-5)
// accumulated with carry-save adders (Harley-Seal), so ONE shared-memory
// gather serves 32 inputs.  The frames stream from HBM exactly once through a
// ring of 2-D TMA boxes (128 pixels x 32 inputs, 128B swizzle, mbarrier
// complete_tx), so the kernel is HBM-bound.
//
// Shared memory per CTA:
//   [stages x 32 KiB]   TMA ring (8 boxes per stage); after streaming it holds the
//                       raw counts uint16[32][C32]
//   [region]            window of Lw bit-sliced words + zero slot (later: tie lists)
//   [C32 x u32]         Bc = boost * 2^23
//   [stages x u64/u32]  mbarriers, release counters
// A cluster of K CTAs can split one group's pixel windows; partial counts are
// then summed through distributed shared memory (DSMEM) before inhibition.
#include <cooperative_groups.h>
#include <cuda_fp16.h>

#include "sp_internal.h"
#include "sp_select.cuh"
#include "sp_topk.cuh"

namespace cg = cooperative_groups;

#ifndef SP_BATCHED_DBG_ON  // development builds only: honour SP_BATCHED_DBG (timing switches)
#define SP_BATCHED_DBG_ON 0
#endif
constexpr bool kDbg = SP_BATCHED_DBG_ON != 0;

namespace sp {

namespace {

__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait_s(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}

// 16-byte shared load at a shared-window address (hoisted once per kernel: a generic pointer
// made ptxas re-derive the window base, S2UR SR_CgaCtaId, every chunk)
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}

// One 2-D TMA box {128 pixels, 32 inputs} at (x, row) of the frames' tensor map.
__device__ __forceinline__ void tma_box_g2s(void* dst, const CUtensorMap* map, uint32_t x,
                                            uint32_t row, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(row), "r"(smem_addr(bar))
        : "memory");
}

// 32x32 bit-matrix transpose across a warp (row = lane, column = bit):
// afterwards lane j bit f = lane f bit j.  Recursive block swap, 5 stages of SHFL + merge with
// per-lane constants precomputed once: the 16- and 8-bit stages move whole
// bytes, so one PRMT (byte permute of x and the partner's y, per-lane selector) does the
// rotate + select; the 4-, 2- and 1-bit stages rotate (SHF.L.W) and select (LOP3).
#ifndef SP_PRMT_TRANSPOSE  // development A/B: 0 = rotate + select in all five stages
#define SP_PRMT_TRANSPOSE 1
#endif
struct TransposeLane {
    uint32_t rot[5], keep[5];
    uint32_t sel16, sel8;
    __device__ __forceinline__ explicit TransposeLane(uint32_t lane) {
        const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            const uint32_t s = 16u >> i;
            const bool lo = (lane & s) == 0;
            rot[i] = lo ? s : 32u - s;
            keep[i] = lo ? masks[i] : ~masks[i];
        }
        // bytes of x (0-3) and y (4-7): lo lanes keep their low half / even bytes and take the
        // partner's low half / even bytes above them; hi lanes the mirror image
        sel16 = (lane & 16u) == 0 ? 0x5410u : 0x3276u;
        sel8 = (lane & 8u) == 0 ? 0x6240u : 0x3715u;
    }
};

__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, const TransposeLane& t) {
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const uint32_t y = __shfl_xor_sync(0xffffffffu, x, 16u >> i);
        if (SP_PRMT_TRANSPOSE && i < 2) {
            x = __byte_perm(x, y, i == 0 ? t.sel16 : t.sel8);
        } else {
            const uint32_t r = __funnelshift_l(y, y, t.rot[i]);
            x = (x & t.keep[i]) | (r & ~t.keep[i]);
        }
    }
    return x;
}

// One elected lane of the (converged) warp adds 1 to a shared counter with acq_rel
// semantics; returns true on that lane iff the counter was at NW-1 mod NW (i.e. this warp
// is the last of the CTA's NW warps to release the stage; NW is a power of two).
// RELAXED: a relaxed add, for callers whose reads of the stage have all returned (their values
// consumed into registers before the call, the warp converged): nothing is left to order, and
// the acq_rel fence waited on every outstanding load of the thread (the ELL prefetch).
template <uint32_t NW, bool RELAXED = false>
__device__ __forceinline__ bool warp_release_is_last(uint32_t addr) {
    uint32_t last;
    if (RELAXED) {
        asm volatile(
            "{\n"
            ".reg .pred P1, P2;\n"
            ".reg .b32 old;\n"
            "elect.sync _|P1, 0xffffffff;\n"
            "mov.u32 old, 0;\n"
            "@P1 atom.relaxed.cta.shared::cta.add.u32 old, [%1], 1;\n"
            "and.b32 old, old, %2;\n"
            "setp.eq.and.u32 P2, old, %2, P1;\n"
            "selp.u32 %0, 1, 0, P2;\n"
            "}\n"
            : "=r"(last)
            : "r"(addr), "n"(NW - 1)
            : "memory");
        return last != 0;
    }
    asm volatile(
        "{\n"
        ".reg .pred P1, P2;\n"
        ".reg .b32 old;\n"
        "elect.sync _|P1, 0xffffffff;\n"
        "mov.u32 old, 0;\n"
        "@P1 atom.acq_rel.cta.shared::cta.add.u32 old, [%1], 1;\n"
        "and.b32 old, old, %2;\n"
        "setp.eq.and.u32 P2, old, %2, P1;\n"
        "selp.u32 %0, 1, 0, P2;\n"
        "}\n"
        : "=r"(last)
        : "r"(addr), "n"(NW - 1)
        : "memory");
    return last != 0;
}

// Byte-nonzero flags of 32 consecutive pixels (two uint4) merged into one word.
// Flag of byte b of word k sits at bit 8b+7 after the carry trick (bit = byte != 0, R12);
// words k < 7 are moved into place with one IMAD.HI (a right shift by a multiply on the
// FMA pipe) and word 7 with one IMAD, then masked in with a LOP3.
// Resulting position of pixel 4k+b: k, 7+k, 15+k, 23+k (k < 7); 14, 22, 30, 31 (k = 7).
// `one` is 1 at run time (a kernel parameter): the add becomes an IMAD on the FMA pipe
// instead of an IADD on the ALU pipe, which is this loop's bottleneck.
__device__ __forceinline__ uint32_t nz_flags(uint32_t v, uint32_t one, uint32_t okm = 0x80808080u) {
    uint32_t t;
    asm("mad.lo.u32 %0, %1, %2, 0x7F7F7F7F;" : "=r"(t) : "r"(v & 0x7F7F7F7Fu), "r"(one));
    return (t | v) & okm;
}

#ifndef SP_MASK_SHIFT  // development A/B: 0 = the round-1 IMAD.HI merge
#define SP_MASK_SHIFT 1
#endif
#ifndef SP_MADHI_RT  // development A/B: 1 = multiplier through `one` (IMAD.HI), 0 = LEA.HI
#define SP_MADHI_RT 0
#endif
#if SP_MASK_SHIFT
// Round 2: word k's flags (bits 8b+7) shifted right by k and added (disjoint bits): pixel 4k+b
// lands at bit 8b+7-k, all 32 distinct; 7 IMAD.HI instead of 7 (IMAD.HI + LOP3) + IMAD + LOP3.
// okm = 0x80808080 for an input lane, 0 for a lane past the group (its row is another
// group's or stale): the flag mask doubles as the lane mask, no extra AND per block.
__device__ __forceinline__ uint32_t nonzero_mask32(const uint4 a, const uint4 b, uint32_t one,
                                                   uint32_t okm = 0x80808080u) {
    const uint32_t v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    // the shifted flags are disjoint, so OR = ADD: one mad.hi (FMA pipe) per word shifts by
    // multiplying with 2^(32-k) and accumulates; no ALU op for the merge
    uint32_t m = nz_flags(v[0], one, okm);
    // (SP_MADHI_RT: the multiplier goes through the run-time `one`, else ptxas turns the mad.hi
    // into LEA.HI on the ALU pipe)
#if SP_MADHI_RT
#define SP_MADHI_ACC(k) asm("mad.hi.u32 %0, %1, %2, %0;" : "+r"(m) : "r"(nz_flags(v[k], one, okm)), "r"(one << (32 - (k))))
#else
#define SP_MADHI_ACC(k) asm("mad.hi.u32 %0, %1, %2, %0;" : "+r"(m) : "r"(nz_flags(v[k], one, okm)), "n"(1u << (32 - (k))))
#endif
    SP_MADHI_ACC(1);
    SP_MADHI_ACC(2);
    SP_MADHI_ACC(3);
    SP_MADHI_ACC(4);
    SP_MADHI_ACC(5);
    SP_MADHI_ACC(6);
    SP_MADHI_ACC(7);
#undef SP_MADHI_ACC
    return m;
}

// Pixel (0..31 within a block) whose flag ends at bit j of nonzero_mask32's result.
__device__ __forceinline__ uint32_t pixel_of_bit(uint32_t j) { return 4u * (7u - (j & 7u)) + (j >> 3); }
#else
__device__ __forceinline__ uint32_t nonzero_mask32(const uint4 a, const uint4 b, uint32_t one) {
    const uint32_t v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    uint32_t m = 0;
#pragma unroll
    for (int k = 0; k < 7; ++k) {
        const uint32_t mk = (1u << (k + 25)) | (1u << (k + 24));
        m |= __umulhi(nz_flags(v[k], one), mk) &
             ((1u << k) | (1u << (7 + k)) | (1u << (15 + k)) | (1u << (23 + k)));
    }
    m |= (nz_flags(v[7], one) * 0x81u) & 0xC0404000u;
    return m;
}

// Pixel (0..31 within a block) whose flag ends at bit j of nonzero_mask32's result.
__device__ __forceinline__ uint32_t pixel_of_bit(uint32_t j) {
    if (j == 31) return 31;
    if (j == 30) return 30;
    if (j == 22) return 29;
    if (j == 14) return 28;
    const uint32_t b = j < 7 ? 0u : (j < 14 ? 1u : (j < 22 ? 2u : 3u));
    const uint32_t base = b == 0 ? 0u : (b == 1 ? 7u : (b == 2 ? 15u : 23u));
    return 4u * (j - base) + b;
}
#endif

struct Planes {
    uint32_t ones, twos, fours;
    uint32_t hi[kHiPlanes];  // weights 8, 16, ..., 512
};

__device__ __forceinline__ void full_add(uint32_t& s, uint32_t& c, uint32_t a, uint32_t b,
                                         uint32_t d) {
    const uint32_t u = a ^ b;
    s = u ^ d;
    c = (a & b) | (u & d);
}

// Harley-Seal carry-save accumulation of 8 bit-sliced words into the counter.
__device__ __forceinline__ void accumulate8(Planes& P, uint32_t x0, uint32_t x1, uint32_t x2,
                                            uint32_t x3, uint32_t x4, uint32_t x5, uint32_t x6,
                                            uint32_t x7) {
    uint32_t c1, c2, c3, c4, f1, f2, e;
    full_add(P.ones, c1, P.ones, x0, x1);
    full_add(P.ones, c2, P.ones, x2, x3);
    full_add(P.twos, f1, P.twos, c1, c2);
    full_add(P.ones, c3, P.ones, x4, x5);
    full_add(P.ones, c4, P.ones, x6, x7);
    full_add(P.twos, f2, P.twos, c3, c4);
    full_add(P.fours, e, P.fours, f1, f2);
#pragma unroll
    for (int h = 0; h < (int)kHiPlanes; ++h) {
        const uint32_t t = P.hi[h] & e;
        P.hi[h] ^= e;
        e = t;
    }
}

// Raw counts of column c for the gs inputs of a group into rawbuf[f][c].
__device__ __forceinline__ void store_counts(const Planes& P, uint16_t* rawbuf, uint32_t C32, uint32_t c,
                                             uint32_t gs) {
    // all 32 counts of column c at once: the 10 planes as a 16 x 32 bit matrix (rows b,
    // bit f = input f), transposed in registers as two 16 x 16 blocks side by side;
    // then y_j holds count_j (low half) and count_{j+16} (high half)
    uint32_t y0, y1, y2, y3, y4, y5, y6, y7, y8, y9, y10, y11, y12, y13, y14, y15;
    static_assert(kHiPlanes == 7, "10 count planes (ones, twos, fours, 7 high)");
    y0 = P.ones, y1 = P.twos, y2 = P.fours;
    y3 = P.hi[0], y4 = P.hi[1], y5 = P.hi[2], y6 = P.hi[3], y7 = P.hi[4], y8 = P.hi[5], y9 = P.hi[6];
    y10 = 0u, y11 = 0u, y12 = 0u, y13 = 0u, y14 = 0u, y15 = 0u;
    { const uint32_t t = ((y0 >> 8) ^ y8) & 0x00FF00FFu; y8 ^= t; y0 ^= t << 8; }
    { const uint32_t t = ((y1 >> 8) ^ y9) & 0x00FF00FFu; y9 ^= t; y1 ^= t << 8; }
    { const uint32_t t = ((y2 >> 8) ^ y10) & 0x00FF00FFu; y10 ^= t; y2 ^= t << 8; }
    { const uint32_t t = ((y3 >> 8) ^ y11) & 0x00FF00FFu; y11 ^= t; y3 ^= t << 8; }
    { const uint32_t t = ((y4 >> 8) ^ y12) & 0x00FF00FFu; y12 ^= t; y4 ^= t << 8; }
    { const uint32_t t = ((y5 >> 8) ^ y13) & 0x00FF00FFu; y13 ^= t; y5 ^= t << 8; }
    { const uint32_t t = ((y6 >> 8) ^ y14) & 0x00FF00FFu; y14 ^= t; y6 ^= t << 8; }
    { const uint32_t t = ((y7 >> 8) ^ y15) & 0x00FF00FFu; y15 ^= t; y7 ^= t << 8; }
    { const uint32_t t = ((y0 >> 4) ^ y4) & 0x0F0F0F0Fu; y4 ^= t; y0 ^= t << 4; }
    { const uint32_t t = ((y1 >> 4) ^ y5) & 0x0F0F0F0Fu; y5 ^= t; y1 ^= t << 4; }
    { const uint32_t t = ((y2 >> 4) ^ y6) & 0x0F0F0F0Fu; y6 ^= t; y2 ^= t << 4; }
    { const uint32_t t = ((y3 >> 4) ^ y7) & 0x0F0F0F0Fu; y7 ^= t; y3 ^= t << 4; }
    { const uint32_t t = ((y8 >> 4) ^ y12) & 0x0F0F0F0Fu; y12 ^= t; y8 ^= t << 4; }
    { const uint32_t t = ((y9 >> 4) ^ y13) & 0x0F0F0F0Fu; y13 ^= t; y9 ^= t << 4; }
    { const uint32_t t = ((y10 >> 4) ^ y14) & 0x0F0F0F0Fu; y14 ^= t; y10 ^= t << 4; }
    { const uint32_t t = ((y11 >> 4) ^ y15) & 0x0F0F0F0Fu; y15 ^= t; y11 ^= t << 4; }
    { const uint32_t t = ((y0 >> 2) ^ y2) & 0x33333333u; y2 ^= t; y0 ^= t << 2; }
    { const uint32_t t = ((y1 >> 2) ^ y3) & 0x33333333u; y3 ^= t; y1 ^= t << 2; }
    { const uint32_t t = ((y4 >> 2) ^ y6) & 0x33333333u; y6 ^= t; y4 ^= t << 2; }
    { const uint32_t t = ((y5 >> 2) ^ y7) & 0x33333333u; y7 ^= t; y5 ^= t << 2; }
    { const uint32_t t = ((y8 >> 2) ^ y10) & 0x33333333u; y10 ^= t; y8 ^= t << 2; }
    { const uint32_t t = ((y9 >> 2) ^ y11) & 0x33333333u; y11 ^= t; y9 ^= t << 2; }
    { const uint32_t t = ((y12 >> 2) ^ y14) & 0x33333333u; y14 ^= t; y12 ^= t << 2; }
    { const uint32_t t = ((y13 >> 2) ^ y15) & 0x33333333u; y15 ^= t; y13 ^= t << 2; }
    { const uint32_t t = ((y0 >> 1) ^ y1) & 0x55555555u; y1 ^= t; y0 ^= t << 1; }
    { const uint32_t t = ((y2 >> 1) ^ y3) & 0x55555555u; y3 ^= t; y2 ^= t << 1; }
    { const uint32_t t = ((y4 >> 1) ^ y5) & 0x55555555u; y5 ^= t; y4 ^= t << 1; }
    { const uint32_t t = ((y6 >> 1) ^ y7) & 0x55555555u; y7 ^= t; y6 ^= t << 1; }
    { const uint32_t t = ((y8 >> 1) ^ y9) & 0x55555555u; y9 ^= t; y8 ^= t << 1; }
    { const uint32_t t = ((y10 >> 1) ^ y11) & 0x55555555u; y11 ^= t; y10 ^= t << 1; }
    { const uint32_t t = ((y12 >> 1) ^ y13) & 0x55555555u; y13 ^= t; y12 ^= t << 1; }
    { const uint32_t t = ((y14 >> 1) ^ y15) & 0x55555555u; y15 ^= t; y14 ^= t << 1; }
    const uint32_t ys[16] = {y0, y1, y2, y3, y4, y5, y6, y7, y8, y9, y10, y11, y12, y13, y14, y15};
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        if (static_cast<uint32_t>(j) < gs) rawbuf[j * C32 + c] = static_cast<uint16_t>(ys[j]);
        if (static_cast<uint32_t>(j) + 16u < gs)
            rawbuf[(j + 16) * C32 + c] = static_cast<uint16_t>(ys[j] >> 16);
    }
}

}  // namespace

// Global split (p.gsplit): the K CTAs of a group are not a cluster but members of
// a cooperative launch (all resident).  Each writes its partial counts rawbuf[f < gs] to
// part[group][rank], arrives on the group's counter and waits for the K arrivals; then CTA rank
// sums the K partial rows of its inputs f = rank, rank + K, .. into its own rawbuf (the rows
// batched_topk then reads), and departs; the last departure zeroes both counters for the next
// launch (stream order: it starts after this one has finished).
__device__ __noinline__ void global_split_sum(const BatchedParams& p, uint16_t* rawbuf, uint32_t group,
                                              uint32_t rank, uint32_t K, uint32_t gs, uint32_t tid,
                                              uint32_t nt) {
    const uint32_t nv = p.C32 / 8u;  // uint4 per row
    uint4* mine = p.part + (static_cast<size_t>(group) * K + rank) * 32u * nv;
    const uint4* raw4 = reinterpret_cast<const uint4*>(rawbuf);
    for (uint32_t i = tid; i < gs * nv; i += nt) __stcg(mine + i, raw4[i]);
    __threadfence();
    __syncthreads();
    uint32_t* arr = p.gbar + group;
    uint32_t* dep = p.gbar + p.groups + group;
    if (tid == 0) {
        atomicAdd(arr, 1u);
        uint32_t seen = 0, spins = 0;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(arr) : "memory");
            if (++spins > (1u << 22)) __trap();  // a missing peer (seconds of spinning): fail loudly, never hang
        } while (seen < K);
    }
    __syncthreads();
    const uint32_t mine_n = gs > rank ? (gs - rank + K - 1u) / K : 0u;  // inputs rank, rank+K, ..
    uint4* sum4 = reinterpret_cast<uint4*>(rawbuf);
    const uint4* base = p.part + static_cast<size_t>(group) * K * 32u * nv;
    for (uint32_t i = tid; i < mine_n * nv; i += nt) {
        const uint32_t f = rank + K * (i / nv), v = i % nv;
        // packed u16 adds (every sum is a raw count <= S); four L2 loads in flight per thread
        // (a serial loop over K waited one L2 round trip per partial row)
        const uint4* src = base + static_cast<size_t>(f) * nv + v;
        const size_t rs = 32u * static_cast<size_t>(nv);  // between the K partial rows of f
        uint4 acc = make_uint4(0u, 0u, 0u, 0u);
        uint32_t q = 0;
        for (; q + 4u <= K; q += 4u) {
            const uint4 t0 = __ldcg(src + q * rs), t1 = __ldcg(src + (q + 1u) * rs);
            const uint4 t2 = __ldcg(src + (q + 2u) * rs), t3 = __ldcg(src + (q + 3u) * rs);
            acc.x += (t0.x + t1.x) + (t2.x + t3.x), acc.y += (t0.y + t1.y) + (t2.y + t3.y);
            acc.z += (t0.z + t1.z) + (t2.z + t3.z), acc.w += (t0.w + t1.w) + (t2.w + t3.w);
        }
        for (; q < K; ++q) {
            const uint4 t = __ldcg(src + q * rs);
            acc.x += t.x, acc.y += t.y, acc.z += t.z, acc.w += t.w;
        }
        sum4[f * nv + v] = acc;
    }
    __syncthreads();
    if (tid == 0 && atomicAdd(dep, 1u) == K - 1u) {
        atomicExch(arr, 0u);
        atomicExch(dep, 0u);
    }
}

// NT threads per CTA (1024: 1 block of 32 pixels per warp per chunk, 64 registers;
// 512: 2 blocks per warp per chunk, 128 registers); CPT column-warps per warp.
// PK: the frames arrive as bit-planes (sp_compute_packed; P:502's boolean representation):
// uint32[inputs][Wn4], bit i of word w = pixel 32w + i.  A stage is then one 4 KiB TMA box
// {32 words, 32 inputs} (= one chunk of kChunkBits pixels), 8x as many stages in the same ring,
// and the byte flags disappear: lane f's word of a block is already its 32 pixels.
template <int CPT, int NT, bool PK>
__global__ void __launch_bounds__(NT, 1)
    sp_batched_kernel(const __grid_constant__ BatchedParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr uint32_t NW = NT / 32;        // warps
    constexpr uint32_t BPW = 32u / NW;      // 32-pixel blocks per warp per chunk
    constexpr uint32_t SB = PK ? 32u * (kChunkBits / 8u) : kStageBytes;  // bytes per 32-row stage
    static_assert(!PK || NW == 16, "the packed staging splits 16 warps into two halves of 8 x 4 blocks");
    const uint32_t tid = threadIdx.x, lane = tid & 31u, wi = tid >> 5;
    const uint32_t NST = p.stages;
    // uint8 frames: a stage is 8 boxes of `rows` x 128 B packed back to back (rows * 1 KiB), so
    // groups of fewer than 32 inputs fit more stages in the ring; packed: 4 KiB boxes of 32 rows
    const uint32_t SBs = PK ? SB : p.rows * 1024u;
    const uint32_t box_pitch = p.rows * kBoxBytes;  // bytes between the boxes of a stage

    uint8_t* stage_base = smem;  // 1024-aligned (swizzle-128B boxes)
    uint16_t* rawbuf = reinterpret_cast<uint16_t*>(stage_base);  // after streaming
    uint8_t* region = smem + p.ring_bytes;
    uint32_t* words = reinterpret_cast<uint32_t*>(region);
    uint32_t* s_bc = reinterpret_cast<uint32_t*>(region + p.region_bytes);
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_bc + p.C32);
    uint32_t* released = reinterpret_cast<uint32_t*>(bars + NST);  // per-stage release counters

    const uint32_t K = p.K;
    const uint32_t group = blockIdx.x / K, rank = blockIdx.x % K;
    const uint32_t in0 = group * p.rows;
    const uint32_t in1 = min(p.num_inputs, in0 + p.rows);
    const uint32_t gs = in1 - in0;  // 1..rows inputs in this group
    // bytes a stage's boxes deliver: rows past the batch are zero-filled by TMA and counted
    const uint32_t tx_bytes = PK ? SB / 32u * p.rows : SBs;
    // a group's K CTAs split its chunks (not its windows: 51 windows over 9 CTAs is 5 or 6 each,
    // 507 chunks 56 or 57): CTA rank streams chunks [c0, c1), windows w0 .. w1-1, the first and
    // last of which may be partial (X is zeroed outside the CTA's chunks, so the window's full
    // ELL cell counts only them)
    const uint32_t cpw = p.Lw / kChunkBits;  // chunks per window (Lw is a multiple of the chunk)
    const uint32_t nct = (p.nbits + kChunkBits - 1) / kChunkBits;
    const uint32_t c0 = rank * nct / K, c1 = (rank + 1) * nct / K;
    const uint32_t w0 = c0 / cpw, w1 = c1 > c0 ? (c1 + cpw - 1u) / cpw : w0;
    const uint32_t pix_begin = c0 * kChunkBits;
    const uint32_t nchunks = c1 - c0;

    // ---- setup ---------------------------------------------------------------------------
    uint64_t* trace = p.trace ? p.trace + blockIdx.x * 6u : nullptr;
    uint64_t t_win = 0;  // phase timestamps (dev aid)
    if (trace && tid == 0) trace[0] = global_ns();
    if (tid == 0 && (smem_addr(smem) & 1023u)) __trap();  // swizzled boxes need 1 KiB alignment
    if (tid < NST) {
        mbar_init(&bars[tid], 1);
        released[tid] = 0u;
    }
    for (uint32_t c = tid; c < p.C32; c += NT) s_bc[c] = p.bc[c];
    if (tid == 0) {  // the zero slot(s) padding / disconnected synapses point to
        words[p.Lw] = 0u;
        if (p.xbufs == 2) words[2u * p.Lw + 1u] = 0u;
    }
    if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();

    // Producer step for chunk j (one thread): expect the stage's bytes, then 8 TMA boxes of
    // 128 pixels x `rows` inputs back to back (rows beyond the batch and pixels beyond nbits are
    // zero-filled; lanes >= gs read the next box's rows and are masked by lane_ok).
    // Called by thread 0 for the prologue and afterwards by the lane that releases a stage
    // last, so the ring refills without any CTA-wide barrier.
    auto issue = [&](uint32_t j, uint32_t st) {
        if (kDbg && (p.bdbg & 8u)) return;  // development: consumer-only timing (no loads)
        const uint32_t x0 = pix_begin + j * kChunkBits;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive_expect_tx(&bars[st], tx_bytes);
        uint8_t* dst = stage_base + st * SBs;
        if (PK) {
            tma_box_g2s(dst, &p.tmap, x0 / 32u, in0, &bars[st]);  // {32 words, rows inputs}
        } else {
#pragma unroll
            for (uint32_t b = 0; b < kChunkBits / kBoxBytes; ++b)
                tma_box_g2s(dst + b * box_pitch, &p.tmap, x0 + b * kBoxBytes, in0, &bars[st]);
        }
    };
    if (tid == 0) {
        const uint32_t pre = min(NST, nchunks);
        for (uint32_t j = 0; j < pre; ++j) issue(j, j);
    }

    const uint32_t released_addr = smem_addr(released);
    const uint32_t bars_s = smem_addr(bars), stage_s = smem_addr(stage_base);  // shared addresses
    const TransposeLane tl(lane);
    const uint32_t lane_ok = lane < gs ? 0xFFFFFFFFu : 0u;
    const uint32_t okm = lane_ok & 0x80808080u;  // flag mask of this lane (0 past the group)
    const uint32_t pob = pixel_of_bit(lane);  // pixel of the word this lane writes per block
    // lane f reads its 32 bytes of block blk from box blk/4, row f, 16-byte slots
    // 2*(blk%4) and +1, swizzled by XOR with bits 7..9 of the row's shared-memory address
    // (CU_TENSOR_MAP_SWIZZLE_128B; a stage starts 1 KiB-aligned, a box at a multiple of
    // rows x 128 B, so row f of box b is 128-byte row b*rows + f of the stage); the second
    // slot is the first XOR 16 bytes
    uint32_t rd[BPW];
#pragma unroll
    for (uint32_t i = 0; i < BPW; ++i) {
        const uint32_t blk = wi + NW * i;
        const uint32_t r128 = (blk >> 2) * p.rows + lane;
        rd[i] = r128 * kBoxBytes + (((2u * (blk & 3u)) ^ (r128 & 7u)) << 4);
    }
    // packed: lane f reads words 4(wi%8) .. +3 of row f (16-byte slot wi%8 of the 128 B row,
    // swizzled by XOR with f % 8: the 8 lanes of each LDS.128 phase hit 8 distinct slots)
    const uint32_t rdp = lane * 128u + (((wi & 7u) ^ (lane & 7u)) << 4);

    Planes P[CPT];
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
        P[i].ones = P[i].twos = P[i].fours = 0u;
#pragma unroll
        for (int h = 0; h < (int)kHiPlanes; ++h) P[i].hi[h] = 0u;
    }

    // ---- stream the windows: transpose chunks into X, then gather ----------------------
    // With two X buffers (p.xbufs == 2) window w+1 is transposed into the other buffer
    // while slower warps still gather window w: one CTA barrier per window.
    uint32_t j = 0, st = 0, phase = 0;
    // ELL prefetch depth: the first PE blocks of each of this thread's cells for window w are
    // loaded into registers when the window starts, so their L2 latency hides behind the
    // window's chunk transposes instead of stalling the gather (profiles/r01_step7*.txt)
    constexpr uint32_t PE = CPT <= 2 ? 2u : 0u;
    // cell sizes/offsets are loaded one window ahead so the block prefetch never waits
    uint32_t nnb[CPT], noff[CPT];
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
        const uint32_t cw = wi + NW * i;
        nnb[i] = cw < p.ncw && w0 < w1 ? p.ell_nb[w0 * p.ncw + cw] : 0u;
        noff[i] = cw < p.ncw && w0 < w1 ? p.ell_off[w0 * p.ncw + cw] : 0u;
    }
    for (uint32_t w = w0; w < w1; ++w) {
        uint32_t* X = words + (p.xbufs == 2 ? (w & 1u) * (p.Lw + 1u) : 0u);
        uint4 pre[CPT][PE > 0 ? PE : 1];
        uint32_t pnb[CPT], poff[CPT];
#pragma unroll
        for (int i = 0; i < CPT; ++i) {
            const uint32_t cw = wi + NW * i;
            pnb[i] = nnb[i];
            poff[i] = noff[i];
#pragma unroll
            for (uint32_t b = 0; b < PE; ++b)
                if (b < pnb[i]) pre[i][b] = __ldg(p.ell + poff[i] + lane + b * 32u);
            const bool more = cw < p.ncw && w + 1u < w1;
            nnb[i] = more ? p.ell_nb[(w + 1u) * p.ncw + cw] : 0u;
            noff[i] = more ? p.ell_off[(w + 1u) * p.ncw + cw] : 0u;
        }
        const uint32_t wbase = w * p.Lw;
        const uint32_t wlen = min(p.Lw, p.nbits - wbase);
        const uint32_t nch = (wlen + kChunkBits - 1) / kChunkBits;
        // this CTA's chunks of the window: [qa, qb); zero X outside them (partial windows of a
        // split group only; the buffer is free: every warp passed the previous window's barrier)
        const uint32_t qa = c0 > w * cpw ? c0 - w * cpw : 0u;
        const uint32_t qb = min(nch, c1 - w * cpw);
        if (qa > 0u || qb < nch) {
            for (uint32_t i = tid; i < qa * kChunkBits; i += NT) X[i] = 0u;
            for (uint32_t i = qb * kChunkBits + tid; i < nch * kChunkBits; i += NT) X[i] = 0u;
        }
        const uint32_t nmine = qb - qa;
        if (PK) {
            // packed: the warps of half (wi >> 3) take the chunks of that parity (global chunk
            // index), 4 blocks each (one conflict-free LDS.128); lane j of a transpose holds
            // pixel 32*blk + j.  NST is even, so a half always sees stages of one parity.
            const uint32_t q0 = ((wi >> 3) - j) & 1u;
            uint32_t jj = j + q0, sq = st + q0, ph = phase;
            if (sq >= NST) sq -= NST, ph ^= 1u;
            for (uint32_t q = qa + q0; q < qb; q += 2u) {
                mbar_wait_s(bars_s + 8u * sq, ph);
                const uint4 v = lds128(stage_s + sq * SB + rdp);
                const uint32_t t0 = warp_transpose32(v.x & lane_ok, tl);
                const uint32_t t1 = warp_transpose32(v.y & lane_ok, tl);
                const uint32_t t2 = warp_transpose32(v.z & lane_ok, tl);
                const uint32_t t3 = warp_transpose32(v.w & lane_ok, tl);
                uint32_t* xo = X + q * kChunkBits + (4u * (wi & 7u)) * 32u + lane;
                xo[0] = t0;
                xo[32] = t1;
                xo[64] = t2;
                xo[96] = t3;
                if (warp_release_is_last<NW / 2>(released_addr + 4u * sq) && jj + NST < nchunks)
                    issue(jj + NST, sq);
                jj += 2u;
                sq += 2u;
                if (sq >= NST) sq -= NST, ph ^= 1u;
            }
            j += nmine;  // every warp: the window's chunks are consumed
            st += nmine % NST;
            phase ^= (nmine / NST) & 1u;
            if (st >= NST) st -= NST, phase ^= 1u;
        }
        for (uint32_t q = qa; q < (PK ? 0u : qb); ++q) {
            if (!(kDbg && (p.bdbg & 8u))) mbar_wait_s(bars_s + 8u * st, phase);
            // a1: warp wi turns blocks wi, wi+NW, .. (32 pixels x 32 inputs each) into 32
            // bit-sliced words per block
            const uint32_t stg = stage_s + st * SBs;
            uint32_t m[BPW];
#pragma unroll
            for (uint32_t i = 0; i < BPW; ++i) {
                const uint4 a = lds128(stg + rd[i]);
                const uint4 b = lds128(stg + (rd[i] ^ 16u));
                m[i] = SP_MASK_SHIFT ? nonzero_mask32(a, b, p.one, okm) : nonzero_mask32(a, b, p.one) & lane_ok;
            }
            // release the stage as soon as the warp's bytes are in registers (the flags consume
            // every loaded value; the warp converges before the elected lane's relaxed add); the
            // warp that releases it last refills it (chunk j + NST) at once (reading the add's
            // result only after the transposes measured 10% slower: once this loop is trimmed
            // the stream bounds the kernel)
            if (!(kDbg && (p.bdbg & 36u))) {  // (development: 32 = no release at all, with 8 only)
#pragma unroll
                for (uint32_t i = 0; i < BPW; ++i) asm volatile("" ::"r"(m[i]));
                __syncwarp();
                if (warp_release_is_last<NW, true>(released_addr + 4u * st) && j + NST < nchunks) issue(j + NST, st);
            }
            if (!(kDbg && (p.bdbg & 2u))) {
#pragma unroll
                for (uint32_t i = 0; i < BPW; ++i)
                    X[q * kChunkBits + (wi + NW * i) * 32u + pob] = warp_transpose32(m[i], tl);
            }
            ++j;
            if (++st == NST) {
                st = 0;
                phase ^= 1u;
            }
        }
        const uint64_t tb = trace ? global_ns() : 0;
        __syncthreads();  // all words of window w written (and, double-buffered, all gathers
                          // of window w-1 finished, so its buffer may be overwritten next)
        // a2: bit-sliced gather-count of this window's synapses (ELL, 8 slots per block)
#pragma unroll
        for (int i = 0; i < CPT; ++i) {
            const uint32_t nb = (kDbg && (p.bdbg & 1u)) ? 0u : pnb[i];
            const uint4* e = p.ell + poff[i] + lane;
#pragma unroll
            for (uint32_t bk = 0; bk < PE; ++bk) {
                if (bk < nb) {
                    const uint4 s8 = pre[i][bk];
                    accumulate8(P[i], X[s8.x & 0xFFFFu], X[s8.x >> 16], X[s8.y & 0xFFFFu],
                                X[s8.y >> 16], X[s8.z & 0xFFFFu], X[s8.z >> 16],
                                X[s8.w & 0xFFFFu], X[s8.w >> 16]);
                }
            }
#pragma unroll 2
            for (uint32_t bk = PE; bk < nb; ++bk) {
                const uint4 s8 = __ldg(e + bk * 32u);
                accumulate8(P[i], X[s8.x & 0xFFFFu], X[s8.x >> 16], X[s8.y & 0xFFFFu],
                            X[s8.y >> 16], X[s8.z & 0xFFFFu], X[s8.z >> 16],
                            X[s8.w & 0xFFFFu], X[s8.w >> 16]);
            }
        }
        if (p.xbufs == 1) __syncthreads();  // before the next window overwrites X
        if (trace) {
            const uint64_t te = global_ns();
            t_win += te - tb;
        }
    }

    if (trace) {
        __syncthreads();
        if (tid == 0) {
            trace[1] = global_ns();
            trace[4] = t_win;
            trace[5] = w1 - w0;
        }
    }
    // ---- raw counts per input (partial if K > 1) into rawbuf[f][c] ----------------------
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
        const uint32_t cw = wi + NW * i;
        if (cw < p.ncw) {
            const uint32_t c = cw * 32u + lane;
            store_counts(P[i], rawbuf, p.C32, c, gs);
        }
    }
    cg::cluster_group cluster = cg::this_cluster();
    if (K > 1 && !p.gsplit) cluster.sync();
    else __syncthreads();
    if (K > 1 && p.gsplit) global_split_sum(p, rawbuf, group, rank, K, gs, tid, NT);
    if (trace && tid == 0) trace[2] = global_ns();

    // idle shared memory behind the raw counts: the rest of the ring and the X windows
    const uint32_t raw_bytes = (32u * p.C32 * 2u + 127u) & ~127u;
    const uint32_t big_bytes = p.ring_bytes >= raw_bytes ? p.ring_bytes - raw_bytes + p.region_bytes : 0u;
    batched_topk<CPT, NW>(p, rawbuf, region, smem + raw_bytes, big_bytes, s_bc, in0, gs, rank, K, wi, lane);
    if (K > 1 && !p.gsplit) cluster.sync();  // peers may still read this CTA's partial counts
    if (trace) {
        __syncthreads();
        if (tid == 0) trace[3] = global_ns();
    }
}

// ---------------------------------------------------------------------------------------
// Patch mode: every pw x ph tile of a frame is an SP
// input (R13).  A group = up to 32 consecutive tiles of one tile-row; one 4-D TMA box
// {pw, 32 tiles, ph, 1} brings its pixels (stage layout [y][tile][x]); the whole tile is one
// window of X, so each group is transposed, gathered, counted and ranked in turn by a
// persistent CTA while the ring prefetches the next groups.
// ---------------------------------------------------------------------------------------
template <int CPT, int NT>
__global__ void __launch_bounds__(NT, 1) sp_patch_kernel(const __grid_constant__ BatchedParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr uint32_t NW = NT / 32;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, wi = tid >> 5;
    const uint32_t NST = p.stages;
    const uint32_t stage_bytes = p.patch_stage_bytes;  // 32 * nbits rounded to 1 KiB
    uint8_t* stage_base = smem;
    uint32_t* X = reinterpret_cast<uint32_t*>(smem + NST * stage_bytes);         // [Lw + 1]
    uint16_t* rawbuf = reinterpret_cast<uint16_t*>(X + ((p.Lw + 4u) & ~3u));  // [32][C32], 16-byte aligned
    uint8_t* scratch = reinterpret_cast<uint8_t*>(rawbuf + 32u * p.C32);         // top-k scratch
    uint32_t* s_bc = reinterpret_cast<uint32_t*>(scratch + p.region_bytes);
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_bc + p.C32);
    uint32_t* released = reinterpret_cast<uint32_t*>(bars + NST);

    const uint32_t tpr = p.tiles_x;                     // tiles per tile-row
    const uint32_t gpr = (tpr + 31u) / 32u;             // groups per tile-row
    const uint32_t G = p.groups;                        // rows * gpr
    const uint32_t pw = p.patch_w, ph = p.patch_h;

    if (tid < NST) {
        mbar_init(&bars[tid], 1);
        released[tid] = 0u;
    }
    for (uint32_t c = tid; c < p.C32; c += NT) s_bc[c] = p.bc[c];
    if (tid == 0) X[p.Lw] = 0u;  // zero slot
    if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();

    // the j-th group of this CTA is g = blockIdx.x + j * gridDim.x
    auto issue = [&](uint32_t j, uint32_t st) {
        const uint32_t g = blockIdx.x + j * gridDim.x;
        const uint32_t row = g / gpr, px0 = (g % gpr) * 32u;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive_expect_tx(&bars[st], 32u * pw * ph);
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_addr(stage_base + st * stage_bytes)),
            "l"(reinterpret_cast<uint64_t>(&p.tmap)), "r"(0u), "r"(px0), "r"(0u), "r"(row),
            "r"(smem_addr(&bars[st]))
            : "memory");
    };
    const uint32_t ngroups = blockIdx.x < G ? (G - blockIdx.x + gridDim.x - 1u) / gridDim.x : 0u;
    if (tid == 0)
        for (uint32_t j = 0; j < min(NST, ngroups); ++j) issue(j, j);

    const TransposeLane tl(lane);
    const uint32_t pob = pixel_of_bit(lane);
    const uint32_t released_addr = smem_addr(released);
    const uint32_t bars_s = smem_addr(bars), stage_s = smem_addr(stage_base);  // shared addresses
    const uint32_t bpr = pw / 32u;            // 32-pixel blocks per tile row
    const uint32_t nblk = bpr * ph;           // blocks per tile
    uint32_t st = 0, phase = 0;
    for (uint32_t j = 0; j < ngroups; ++j) {
        const uint32_t g = blockIdx.x + j * gridDim.x;
        const uint32_t row = g / gpr, px0 = (g % gpr) * 32u;
        const uint32_t gs = min(32u, tpr - px0);
        const uint32_t in0 = row * tpr + px0;
        const uint32_t okm = lane < gs ? 0x80808080u : 0u;  // flag mask (0 past the group)
        mbar_wait_s(bars_s + 8u * st, phase);
        // a1: lane f = tile f of the group; block b = row y, pixels 32*xb .. 32*xb+31
        {
            const uint32_t stg = stage_s + st * stage_bytes;
            for (uint32_t b = wi; b < nblk; b += NW) {
                const uint32_t y = b / bpr, xb = b % bpr;
                const uint32_t src = stg + (y * 32u + lane) * pw + xb * 32u;
                const uint4 a = lds128(src);
                const uint4 bb = lds128(src + 16u);
                X[y * pw + xb * 32u + pob] = warp_transpose32(nonzero_mask32(a, bb, p.one, okm), tl);
            }
        }
        if (warp_release_is_last<NW>(released_addr + 4u * st) && j + NST < ngroups) issue(j + NST, st);
        if (++st == NST) {
            st = 0;
            phase ^= 1u;
        }
        __syncthreads();  // X of this group complete
        // a2: gather-count of all synapses (one window)
        Planes P[CPT];
#pragma unroll
        for (int i = 0; i < CPT; ++i) {
            P[i].ones = P[i].twos = P[i].fours = 0u;
#pragma unroll
            for (int h = 0; h < (int)kHiPlanes; ++h) P[i].hi[h] = 0u;
            const uint32_t cw = wi + NW * i;
            if (cw < p.ncw) {
                const uint32_t nb = (p.cand_dbg & 4u) ? 0u : p.ell_nb[cw];  // development: skip the gathers
                const uint4* e = p.ell + p.ell_off[cw] + lane;
#pragma unroll 4
                for (uint32_t bk = 0; bk < nb; ++bk) {
                    const uint4 s8 = __ldg(e + bk * 32u);
                    accumulate8(P[i], X[s8.x & 0xFFFFu], X[s8.x >> 16], X[s8.y & 0xFFFFu],
                                X[s8.y >> 16], X[s8.z & 0xFFFFu], X[s8.z >> 16],
                                X[s8.w & 0xFFFFu], X[s8.w >> 16]);
                }
                const uint32_t c = cw * 32u + lane;
                store_counts(P[i], rawbuf, p.C32, c, gs);
            }
        }
        __syncthreads();  // raw counts of the group complete; X may be overwritten
        // a3/a4: per tile
        if (!(p.cand_dbg & 2u))  // development: skip the selection
            batched_topk<CPT, NW>(p, rawbuf, scratch, scratch, p.region_bytes, s_bc, in0, gs, 0u, 1u, wi, lane);
        __syncthreads();  // rawbuf / scratch reused by the next group
    }
}

template <typename F>
static cudaError_t allow_dynamic_smem(F* fn, int max_smem) {
    cudaFuncAttributes a{};
    cudaError_t e = cudaFuncGetAttributes(&a, fn);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                max_smem - static_cast<int>(a.sharedSizeBytes));
}

cudaError_t configure_batched(int max_smem) {
    cudaError_t e = allow_dynamic_smem(sp_patch_kernel<2, 512>, max_smem);
    if (e == cudaSuccess) e = allow_dynamic_smem(sp_batched_kernel<1, 1024, false>, max_smem);
    if (e == cudaSuccess) e = allow_dynamic_smem(sp_batched_kernel<2, 1024, false>, max_smem);
    if (e == cudaSuccess) e = allow_dynamic_smem(sp_batched_kernel<2, 512, false>, max_smem);
    if (e == cudaSuccess) e = allow_dynamic_smem(sp_batched_kernel<4, 512, false>, max_smem);
    if (e == cudaSuccess) e = allow_dynamic_smem(sp_batched_kernel<2, 512, true>, max_smem);
    if (e == cudaSuccess) e = allow_dynamic_smem(sp_batched_kernel<4, 512, true>, max_smem);
    return e;
}

cudaError_t launch_batched(const BatchedParams& p, uint32_t smem_bytes, cudaStream_t s) {
    const uint32_t nt = p.threads == 512 || p.packed ? 512u : 1024u;
    const uint32_t cpt = (p.ncw + nt / 32u - 1u) / (nt / 32u);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.groups * p.K);
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = smem_bytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    if (p.gsplit) {  // every CTA resident (one per SM): the group barrier cannot deadlock
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
    } else {
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = p.K;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
    }
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (p.packed)
        return cpt <= 2 ? cudaLaunchKernelEx(&cfg, sp_batched_kernel<2, 512, true>, p)
                        : cudaLaunchKernelEx(&cfg, sp_batched_kernel<4, 512, true>, p);
    if (nt == 512)
        return cpt <= 2 ? cudaLaunchKernelEx(&cfg, sp_batched_kernel<2, 512, false>, p)
                        : cudaLaunchKernelEx(&cfg, sp_batched_kernel<4, 512, false>, p);
    return cpt <= 1 ? cudaLaunchKernelEx(&cfg, sp_batched_kernel<1, 1024, false>, p)
                    : cudaLaunchKernelEx(&cfg, sp_batched_kernel<2, 1024, false>, p);
}

cudaError_t launch_patch(const BatchedParams& p, uint32_t smem_bytes, uint32_t ctas, cudaStream_t s) {
    sp_patch_kernel<2, 512><<<ctas, 512, smem_bytes, s>>>(p);
    return cudaGetLastError();
}

// Maximum co-resident clusters for K = 1..8 at this smem size (index K).
cudaError_t batched_max_clusters(uint32_t smem_bytes, int max_clusters[9]) {
    for (int K = 0; K <= 8; ++K) max_clusters[K] = 0;
    cudaError_t e = cudaSuccess;
    for (int K = 1; K <= 8; ++K) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(K * 64);
        cfg.blockDim = dim3(1024);
        cfg.dynamicSmemBytes = smem_bytes;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = K;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        e = cudaOccupancyMaxActiveClusters(&n, sp_batched_kernel<1, 1024, false>, &cfg);
        if (e != cudaSuccess) {
            (void)cudaGetLastError();
            n = 0;
        }
        max_clusters[K] = n;
    }
    return cudaSuccess;
}

}  // namespace sp
