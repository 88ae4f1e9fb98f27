// sp_patch_mma.cu — patch mode on the 5th-generation tensor cores (
// DESIGN.md §4.7b).
//
// In patch mode every pw x ph tile of a frame is an SP input (R13), so the overlap of
// Alg. 1 l.1-5 for all tiles is one dense 0/1 product
//     raw[c][t] = sum_k conn[c][k] * x_t[k],   conn[c][k] = [c has a connected synapse on bit k]
// (idx is distinct within a column, so the sum counts each connected synapse once): a
// [C x nbits] . [nbits x tiles] GEMM with exact integer accumulation (sums <= S <= 1023).
// P:480 names the synapse reduction as the kernel's work; at 960 bits per 32x30 tile the
// dense form is 27% dense (256 of 960) and 1.06 G MACs per 960x540 frame.
//
// Kernel (one thread-block cluster of Q = C32/128 CTAs per block of 128 tile slots):
//  * A = conn, u8, CTA q keeps its 128 columns resident in TENSOR memory (lane = column,
//    4 bytes of K per TMEM column; written once with tcgen05.st), next to two accumulators;
//  * B = the tiles: a block is 4 consecutive tile-rows x 32 tile slots (slot = 32*row + tx,
//    tx >= tiles_x stay zero); a stage = SPS rows y of the 4 tile-rows, fetched as whole frame
//    rows (one 4-D TMA box {W/k, k, SPS, 4}: few long TMA rows -- 32-byte rows capped the TMA
//    at ~0.5 us per 8 KiB); two converter warps turn the bytes into 0/1 (R12: bit = byte != 0)
//    and scatter them into the K-major SWIZZLE_32B layout (slab = 32 pixels of one tile row for
//    all 128 slots, [128 rows][32 B]);
//  * one thread issues tcgen05.mma.cta_group::1.kind::i8 (M 128 columns from TMEM, N 128
//    slots from shared memory, K 32) per slab into a TMEM accumulator (2 x 128 columns);
//    commits free the converted slot and, after the last slab, the accumulator;
//  * the drain (same warpgroup) reads the accumulator with tcgen05.ld (lane = column) and
//    stores the u16 counts straight into the raw-count buffer of the CTA that owns each
//    slot (DSMEM, st.shared::cluster; CTA q owns slots [q*128/Q, (q+1)*128/Q));
//  * 8 top-k warps run rows a3/a4 (sp_topk.cuh, the same selection code as the bit-sliced
//    kernels) on the CTA's slots and write the SDR words.
// mbarriers: full/conv/empty per ring slot, a_full, tmem_full/empty per accumulator,
// raw_full/empty per raw buffer (cluster-scope arrivals from every CTA).
#include <cuda_fp16.h>

#include "sp_internal.h"
#include "sp_select.cuh"
#include "sp_topk.cuh"

namespace sp {

namespace {

constexpr uint32_t kMmaThreads = 512;
constexpr uint32_t kTopkWarps = 8;          // warps 8..15
constexpr uint32_t kSlots = 128;            // tile slots per block (MMA N)
constexpr uint32_t kSlabBytes = 128u * 32u; // one K-slab of A (128 columns) or B (128 slots)
constexpr uint32_t kConvChunks = 8;         // 16-byte chunks per converter thread per stage (<= 64 x 8 x 16 B)

__device__ __forceinline__ uint32_t saddr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(n) : "memory");
}

__device__ __forceinline__ void bar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}

// arrive on the mbarrier at the same offset in CTA `cta` of the cluster.  Relaxed: it only says
// "this CTA's top-k has read its raw buffer" (the reads have returned before the arrive issues);
// a release at cluster scope costs a MEMBAR.GPU per arrive.
__device__ __forceinline__ void bar_arrive_remote(uint64_t* b, uint32_t cta) {
    asm volatile(
        "{\n.reg .b32 ra;\n"
        "mapa.shared::cluster.u32 ra, %0, %1;\n"
        "mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [ra];\n}" ::"r"(saddr(b)),
        "r"(cta)
        : "memory");
}

__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n}" ::"r"(saddr(b)),
        "r"(parity)
        : "memory");
}

// wait with cluster-scope acquire (the phase was completed by other CTAs' release arrivals)
__device__ __forceinline__ void bar_wait_cluster(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n}" ::"r"(saddr(b)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ bool bar_test(uint64_t* b, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred P1;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n}"
        : "=r"(ok)
        : "r"(saddr(b)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ uint64_t global_timer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// asynchronous u32 store into CTA `cta`'s shared memory at the local offset of `p`; its 4 bytes
// count towards the complete_tx of the mbarrier at the local offset of `bar` in that CTA (no
// fence: the consumer's wait on that mbarrier makes the data visible, as for TMA)
__device__ __forceinline__ void st_async_u32(const void* p, const uint64_t* bar, uint32_t cta, uint32_t v) {
    asm volatile(
        "{\n.reg .b32 ra, rb;\n"
        "mapa.shared::cluster.u32 ra, %0, %2;\n"
        "mapa.shared::cluster.u32 rb, %1, %2;\n"
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.u32 [ra], %3, [rb];\n}" ::"r"(saddr(p)),
        "r"(saddr(bar)), "r"(cta), "r"(v)
        : "memory");
}

// K-major SWIZZLE_32B shared-memory matrix descriptor (tcgen05): rows of 32 bytes, 8-row
// groups 256 B apart (SBO), leading offset unused for swizzled K-major (1), version 1.
__device__ __forceinline__ uint64_t sw32_desc(uint32_t addr) {
    return static_cast<uint64_t>((addr >> 4) & 0x3FFFu) | (1ull << 16) | (16ull << 32) | (1ull << 46) |
           (6ull << 61);
}

// kind::i8 instruction descriptor: D s32, A/B u8, both K-major, N = 128, M = 128
constexpr uint32_t kIdesc = (2u << 4) | (0u << 7) | (0u << 10) | ((kSlots >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate)
        : "memory");
}

// the same with A read from tensor memory (lane = column of conn, 4 bytes of K per TMEM column)
__device__ __forceinline__ void mma_i8_ta(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\n"
        "setp.ne.b32 p, %3, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %4, p;\n}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b), "r"(accumulate), "r"(kIdesc)
        : "memory");
}

// 32 lanes x 8 columns: this thread's 8 registers -> TMEM lane (taddr lane + laneid), 8 columns
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint4& a, const uint4& b) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                 "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
                 : "memory");
}

__device__ __forceinline__ void mma_commit_local(uint64_t* b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(b))
                 : "memory");
}

__device__ __forceinline__ void mma_commit_multicast(uint64_t* b, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            saddr(b)),
        "h"(mask)
        : "memory");
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

// 32 lanes x 32 columns of 32-bit TMEM cells -> 32 registers per thread (lane = TMEM lane)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr)
        : "memory");
}

// bytes -> 0/1 (R12: bit = byte != 0), four at a time
__device__ __forceinline__ uint32_t nz01(uint32_t v) {
    return ((((v & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | v) & 0x80808080u) >> 7;
}

}  // namespace

__global__ void __launch_bounds__(kMmaThreads, 1) sp_patch_mma_kernel(const __grid_constant__ PatchMmaParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const BatchedParams& bp = p.bp;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
    const uint32_t Q = p.Q, q = cluster_rank();
    const uint32_t cid = blockIdx.x / Q, ncl = gridDim.x / Q;
    const uint32_t nblk = cid < p.nblocks ? (p.nblocks - cid + ncl - 1u) / ncl : 0u;
    const uint32_t NR = p.raw_stages, NC = p.conv_stages;
    const uint32_t SPS = p.sps, XC = p.xchunks;
    const uint32_t RS = p.raw_stage_bytes;        // W * SPS * 4 bytes: 4 tile-rows x SPS frame rows
    const uint32_t CB = SPS * XC * kSlabBytes;    // converted stage: SPS * XC K-slabs
    const uint32_t units = p.patch_h / SPS;       // stages per block
    const uint32_t SQ = kSlots / Q;               // slots owned by this CTA

    // shared memory: [conv ring NC x CB][raw ring NR x RS][raw counts 2 x SQ x C32][Bc][scratch][bars]
    uint8_t* cring = smem;
    uint8_t* rring = cring + NC * CB;
    uint16_t* raw = reinterpret_cast<uint16_t*>(rring + NR * RS);
    const uint32_t raw_elems = SQ * bp.C32;
    uint32_t* s_bc = reinterpret_cast<uint32_t*>(raw + 2u * raw_elems);
    uint8_t* region = reinterpret_cast<uint8_t*>(s_bc + bp.C32);
    uint64_t* bars = reinterpret_cast<uint64_t*>(region + p.region_bytes);
    uint64_t* rfull = bars;            // [NR] TMA -> converters
    uint64_t* rempty = rfull + NR;     // [NR] converters -> producer
    uint64_t* cfull = rempty + NR;     // [NC] converters -> MMA
    uint64_t* cempty = cfull + NC;     // [NC] MMA commit -> converters
    uint64_t* t_full = cempty + NC;    // [2] MMA -> drain
    uint64_t* t_empty = t_full + 2;    // [2] drain -> MMA
    uint64_t* r_full = t_empty + 2;    // [2] drains' st.async -> top-k
    uint64_t* r_empty = r_full + 2;    // [2] top-k of every CTA -> drains
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(r_empty + 2);

    if (tid == 0) {
        for (uint32_t i = 0; i < NR; ++i) {
            bar_init(&rfull[i], 1);
            bar_init(&rempty[i], p.multicast ? 2u * Q : 2u);  // the converter warps (of every CTA)
        }
        for (uint32_t i = 0; i < NC; ++i) {
            bar_init(&cfull[i], 2);
            bar_init(&cempty[i], 1);
        }
        for (uint32_t i = 0; i < 2; ++i) {
            bar_init(&t_full[i], 1);
            bar_init(&t_empty[i], 4);
            bar_init(&r_full[i], 1);  // the owner's expect_tx; the drains' st.async complete it
            bar_init(&r_empty[i], Q);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // the converted ring's slots tx >= tiles_x are never written: zero them once
    for (uint32_t i = tid; i < NC * CB / 16u; i += kMmaThreads) reinterpret_cast<uint4*>(cring)[i] = make_uint4(0, 0, 0, 0);
    for (uint32_t c = tid; c < bp.C32; c += kMmaThreads) s_bc[c] = bp.bc[c];
    if (warp == 1) {  // TMEM: 2 accumulators x 128 columns + A (nbits / 4 columns)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(saddr(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // every CTA's barriers are initialised before any remote arrive
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t a_col = tmem + 2u * kSlots;  // A: K-slab s at columns a_col + 8 s
    if (warp >= 4 && warp < 8) {
        // A = this CTA's 128 columns of conn: row 128 q + 32 qd + lane -> TMEM lane 32 qd + lane
        const uint32_t qd = warp - 4u;
        const uint4* row = reinterpret_cast<const uint4*>(p.conn + static_cast<size_t>(128u * q + 32u * qd + lane) *
                                                                      p.nbits);
        for (uint32_t s = 0; s < p.nbits / 32u; ++s) {
            const uint4 a = __ldg(row + 2u * s), b = __ldg(row + 2u * s + 1u);
            tmem_st8(a_col + ((32u * qd) << 16) + 8u * s, a, b);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // zeroed ring -> tensor-core reads
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    uint64_t* trace = p.trace ? p.trace + static_cast<size_t>(blockIdx.x) * p.trace_blocks * 8u : nullptr;
    auto stamp = [&](uint32_t j, uint32_t k) {
        if (trace && j < p.trace_blocks) trace[j * 8u + k] = global_timer();
    };
    if (warp == 0) {
        // ---------------- TMA producer: whole frame rows (few, long TMA rows) ----------------
        if (lane == 0) {
            uint32_t rs = 0, ph = 0, issuer = 0;
            for (uint32_t j = 0; j < nblk; ++j) {
                const uint32_t tr0 = 4u * (cid + j * ncl);  // first tile-row of the block
                for (uint32_t yg = 0; yg < units; ++yg) {
                    bar_wait(&rempty[rs], ph ^ 1u);
                    bar_expect_tx(&rfull[rs], RS);
                    if (!p.multicast)
                        asm volatile(
                            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                            " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(saddr(rring + rs * RS)),
                            "l"(reinterpret_cast<uint64_t>(&p.tmap_b)), "r"(0u), "r"(0u), "r"(yg * SPS), "r"(tr0),
                            "r"(saddr(&rfull[rs]))
                            : "memory");
                    else if (issuer == q)  // one CTA fetches the stage for the whole cluster
                        asm volatile(
                            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                            ".multicast::cluster [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(saddr(rring + rs * RS)),
                            "l"(reinterpret_cast<uint64_t>(&p.tmap_b)), "r"(0u), "r"(0u), "r"(yg * SPS), "r"(tr0),
                            "r"(saddr(&rfull[rs])), "h"(static_cast<uint16_t>((1u << Q) - 1u))
                            : "memory");
                    if (++issuer == Q) issuer = 0;
                    if (++rs == NR) rs = 0, ph ^= 1u;
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            uint32_t cs = 0, ph = 0, tb = 0, tph = 0;
            for (uint32_t j = 0; j < nblk; ++j) {
                bar_wait(&t_empty[tb], tph ^ 1u);
                tc_fence_after();
                const uint32_t d = tmem + tb * kSlots;
                for (uint32_t yg = 0; yg < units; ++yg) {
                    bar_wait(&cfull[cs], ph);
                    tc_fence_after();
                    if (yg == 0) stamp(j, 0);
                    for (uint32_t yy = 0; yy < SPS; ++yy)
                        for (uint32_t xc = 0; xc < XC; ++xc) {
                            const uint32_t i = yy * XC + xc;                  // slab of the stage
                            const uint32_t sa = (yg * SPS + yy) * XC + xc;    // K-slab of A
                            if (!(p.dbg & 4u))
                                mma_i8_ta(d, a_col + 8u * sa, sw32_desc(saddr(cring + cs * CB + i * kSlabBytes)),
                                          (yg | i) != 0u ? 1u : 0u);
                        }
                    mma_commit_local(&cempty[cs]);
                    if (++cs == NC) cs = 0, ph ^= 1u;
                }
                stamp(j, 1);
                mma_commit_local(&t_full[tb]);
                if (++tb == 2u) tb = 0, tph ^= 1u;
            }
        }
    } else if (warp == 2 || warp == 3) {
        // ---------------- converters: frame rows -> 0/1 bytes in the K-major SW32 layout ----------
        // raw stage: [t 4][yy SPS][W bytes]; converted stage: slab yy * XC + xc = [128 slots][32 B],
        // slot n = 32 t + tx, 16-byte chunk h at (h ^ ((n >> 2) & 1)) (SWIZZLE_32B)
        const uint32_t ct = 32u * (warp - 2u) + lane;
        const uint32_t cpr = p.W / 16u;                    // 16-byte chunks per frame row
        const uint32_t total = 4u * SPS * cpr;             // chunks per stage
        const uint32_t pw_shift = 31u - __clz(p.patch_w);  // pw is a power of two
        // the scatter is the same for every stage: destination of this thread's chunks, once
        uint32_t doff[kConvChunks];
#pragma unroll
        for (uint32_t m = 0; m < kConvChunks; ++m) {
            const uint32_t i = ct + 64u * m;
            const uint32_t r = i / cpr, cr = i - r * cpr;  // frame row (t, yy), 16-byte chunk
            const uint32_t t = SPS == 2u ? r >> 1 : r, yy = SPS == 2u ? r & 1u : 0u;
            const uint32_t px = 16u * cr, tx = px >> pw_shift, within = px & (p.patch_w - 1u);
            const uint32_t n = 32u * t + tx, h = (within >> 4) & 1u;
            doff[m] = (yy * XC + (within >> 5)) * kSlabBytes + 32u * n + ((h ^ ((n >> 2) & 1u)) << 4);
        }
        uint32_t rs = 0, rph = 0, cs = 0, cph = 0;
        for (uint32_t j = 0; j < nblk; ++j) {
            uint64_t w_raw = 0, w_conv = 0;  // trace: time spent waiting for data / for a slot
            for (uint32_t yg = 0; yg < units; ++yg) {
                const uint64_t t0 = trace ? global_timer() : 0;
                bar_wait(&rfull[rs], rph);
                const uint64_t t1 = trace ? global_timer() : 0;
                bar_wait(&cempty[cs], cph ^ 1u);
                if (trace) w_raw += t1 - t0, w_conv += global_timer() - t1;
                if (!(p.dbg & 8u)) {
                    const uint8_t* __restrict__ src = rring + rs * RS;
                    uint8_t* __restrict__ dst = cring + cs * CB;
                    uint4 v[kConvChunks];
#pragma unroll
                    for (uint32_t m = 0; m < kConvChunks; ++m)
                        if (ct + 64u * m < total) v[m] = *reinterpret_cast<const uint4*>(src + 16u * (ct + 64u * m));
#pragma unroll
                    for (uint32_t m = 0; m < kConvChunks; ++m)
                        if (ct + 64u * m < total) {
                            uint4 w = v[m];
                            w.x = nz01(w.x), w.y = nz01(w.y), w.z = nz01(w.z), w.w = nz01(w.w);
                            *reinterpret_cast<uint4*>(dst + doff[m]) = w;
                        }
                }
                if (!(p.dbg & 32u)) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    if (p.multicast)  // the raw slot is rewritten in every CTA at once
                        for (uint32_t r = 0; r < Q; ++r) bar_arrive_remote(&rempty[rs], r);
                    else
                        bar_arrive(&rempty[rs]);
                    bar_arrive(&cfull[cs]);
                }
                if (++rs == NR) rs = 0, rph ^= 1u;
                if (++cs == NC) cs = 0, cph ^= 1u;
            }
            if (trace && ct == 0 && j < p.trace_blocks) trace[j * 8u + 6] = w_raw, trace[j * 8u + 7] = w_conv;
        }
    } else if (warp >= 4 && warp < 8) {
        // ---------------- drain (warpgroup; quadrant = TMEM lanes) ----------------
        const uint32_t qd = warp - 4u;
        const uint32_t col = 32u * qd + lane;          // column within this CTA's 128
        const uint32_t sq_shift = 31u - __clz(SQ);     // SQ = 128 / Q is a power of two
        uint32_t tb = 0, tph = 0;
        for (uint32_t jd = 0; jd < nblk; ++jd) {
            const uint32_t rb = jd & 1u;
            // accumulator ready and every owner CTA done with raw buffer rb (block jd - 2)
            bar_wait(&t_full[tb], tph);
            if (!(p.dbg & 16u)) bar_wait(&r_empty[rb], ((jd >> 1) & 1u) ^ 1u);
            tc_fence_after();
            if (qd == 0 && lane == 0) stamp(jd, 2);
            uint16_t* rbuf = raw + rb * raw_elems + ((128u * q + col) & ~1u);
            const bool odd = lane & 1u;
            for (uint32_t cc = 0; cc < kSlots / 32u; ++cc) {
                uint32_t v[32];
                tmem_ld32(tmem + ((32u * qd) << 16) + tb * kSlots + 32u * cc, v);
                // lanes pair up so each stores (column c, c+1) of one slot as a u32:
                // even lane takes slot n of (c, c+1), odd lane slot n+1 of (c-1, c)
#pragma unroll
                for (uint32_t i = 0; i < 32u; i += 2u) {
                    const uint32_t give = odd ? v[i] : v[i + 1u];
                    const uint32_t got = __shfl_xor_sync(0xffffffffu, give, 1);
                    const uint32_t n = 32u * cc + i + (odd ? 1u : 0u);  // slot
                    const uint32_t pair = odd ? (got & 0xFFFFu) | (v[i + 1u] << 16) : (v[i] & 0xFFFFu) | (got << 16);
                    if (!(p.dbg & 2u))
                        st_async_u32(rbuf + (n & (SQ - 1u)) * bp.C32, &r_full[rb], n >> sq_shift, pair);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) bar_arrive(&t_empty[tb]);
            if (qd == 0 && lane == 0) stamp(jd, 3);
            if (++tb == 2u) tb = 0, tph ^= 1u;
        }
    } else if (warp >= 8) {
        // ---------------- top-k (rows a3/a4) ----------------
        const uint32_t wi = warp - 8u;
        const uint32_t seg = min(SQ, 32u);
        for (uint32_t j = 0; j < nblk && !(p.dbg & 16u); ++j) {
            const uint32_t rb = j & 1u;
            if (wi == 0 && lane == 0)
                bar_expect_tx(&r_full[rb], (p.dbg & 2u) ? 0u : raw_elems * 2u);  // SQ slots x C32 counts
            bar_wait(&r_full[rb], (j >> 1) & 1u);
            if (wi == 0 && lane == 0) stamp(j, 4);
            uint16_t* rbuf = raw + rb * raw_elems;
            const uint32_t tr0 = 4u * (cid + j * ncl);
            // the CTA's slots [q*SQ, (q+1)*SQ) as tile-row segments of <= 32 slots
            for (uint32_t n0 = q * SQ; n0 < (q + 1u) * SQ; n0 += seg) {
                const uint32_t tr = tr0 + (n0 >> 5), tx0 = n0 & 31u;
                const uint32_t gs = tr < p.tile_rows && tx0 < p.tiles_x ? min(seg, p.tiles_x - tx0) : 0u;
                if (gs == 0u || (p.dbg & 1u)) continue;
                batched_topk<4, kTopkWarps>(bp, rbuf + (n0 - q * SQ) * bp.C32, region, region, p.region_bytes, s_bc,
                                            tr * p.tiles_x + tx0, gs, 0u, 1u, wi, lane);
            }
            asm volatile("bar.sync 1, %0;" ::"n"(kTopkWarps * 32u) : "memory");
            if (wi == 0 && lane == 0) {
                stamp(j, 5);
                for (uint32_t r = 0; r < Q; ++r) bar_arrive_remote(&r_empty[rb], r);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // no CTA leaves while others may still write its shared memory
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

uint32_t patch_mma_smem(uint32_t W, uint32_t sps, uint32_t xchunks, uint32_t raw_stages, uint32_t conv_stages,
                        uint32_t Q, uint32_t C32, uint32_t region_bytes) {
    return conv_stages * sps * xchunks * kSlabBytes + raw_stages * W * sps * 4u + 2u * (kSlots / Q) * C32 * 2u +
           C32 * 4u + region_bytes + (2u * raw_stages + 2u * conv_stages + 8u) * 8u + 16u;
}

cudaError_t configure_patch_mma(int max_smem) {
    cudaFuncAttributes a{};
    cudaError_t e = cudaFuncGetAttributes(&a, sp_patch_mma_kernel);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(sp_patch_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                max_smem - static_cast<int>(a.sharedSizeBytes));
}

cudaError_t launch_patch_mma(const PatchMmaParams& p, uint32_t smem_bytes, uint32_t clusters, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(clusters * p.Q);
    cfg.blockDim = dim3(kMmaThreads);
    cfg.dynamicSmemBytes = smem_bytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.Q;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, sp_patch_mma_kernel, p);
}

cudaError_t patch_mma_max_clusters(uint32_t smem_bytes, uint32_t Q, int* n) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(Q * 16u);
    cfg.blockDim = dim3(kMmaThreads);
    cfg.dynamicSmemBytes = smem_bytes;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = Q;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaOccupancyMaxActiveClusters(n, sp_patch_mma_kernel, &cfg);
}

// conn[c][k] = 1 iff column c has a connected synapse (perm >= tau) on bit k; pad columns 0.
__global__ void k_build_conn(const uint32_t* __restrict__ idx, const float* __restrict__ perm, float tau,
                             uint32_t C, uint32_t S, uint32_t nbits, uint8_t* __restrict__ conn) {
    const uint32_t c = blockIdx.x;
    uint8_t* row = conn + static_cast<size_t>(c) * nbits;
    for (uint32_t k = threadIdx.x; k < nbits; k += blockDim.x) row[k] = 0;
    __syncthreads();
    if (c >= C) return;
    for (uint32_t s = threadIdx.x; s < S; s += blockDim.x) {
        const size_t o = static_cast<size_t>(c) * S + s;
        if (perm[o] >= tau) row[idx[o]] = 1;
    }
}

cudaError_t launch_build_conn(const uint32_t* idx, const float* perm, float tau, uint32_t C, uint32_t C32, uint32_t S,
                              uint32_t nbits, uint8_t* conn, cudaStream_t s) {
    k_build_conn<<<C32, 256, 0, s>>>(idx, perm, tau, C, S, nbits, conn);
    return cudaGetLastError();
}

}  // namespace sp
