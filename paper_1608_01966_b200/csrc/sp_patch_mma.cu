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
//  * A = conn, K-major u8, CTA q keeps its 128 columns resident in shared memory
//    (nbits/32 slabs of [128 rows][32 B], 2-D TMA, SWIZZLE_32B), loaded once per launch;
//  * B = the tiles: a block is 4 consecutive tile-rows x 32 tile slots (slot = 32*row + tx,
//    tx >= tiles_x zero-filled by TMA); slab s = 32 pixels of one tile row (y, x-chunk) for
//    all 128 slots, one 4-D TMA box {32 px, 32 tiles, 1 row, 4 tile-rows}, SWIZZLE_32B,
//    multicast to every CTA of the cluster (CTA s % Q issues slab s);
//  * the converter warpgroup turns bytes into 0/1 in place (R12: bit = byte != 0);
//  * one thread issues tcgen05.mma.cta_group::1.kind::i8 (M 128 columns, N 128 slots,
//    K 32) per slab into a TMEM accumulator (4 buffers of 128 columns), commits free the
//    ring slot in every CTA (multicast commit) and, after the last slab, the accumulator;
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
constexpr uint32_t kTmemBufs = 4;           // accumulators of 128 TMEM columns

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

// arrive on the mbarrier at the same offset in CTA `cta` of the cluster (release, cluster scope)
__device__ __forceinline__ void bar_arrive_remote(uint64_t* b, uint32_t cta) {
    asm volatile(
        "{\n.reg .b32 ra;\n"
        "mapa.shared::cluster.u32 ra, %0, %1;\n"
        "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n}" ::"r"(saddr(b)),
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
        "mbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n}"
        : "=r"(ok)
        : "r"(saddr(b)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// u32 store into CTA `cta`'s shared memory at the local offset of `p`
__device__ __forceinline__ void st_remote_u32(const void* p, uint32_t cta, uint32_t v) {
    asm volatile(
        "{\n.reg .b32 ra;\n"
        "mapa.shared::cluster.u32 ra, %0, %1;\n"
        "st.shared::cluster.u32 [ra], %2;\n}" ::"r"(saddr(p)),
        "r"(cta), "r"(v)
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
    const uint32_t slabs = p.slabs, NST = p.stages;
    const uint32_t SQ = kSlots / Q;  // slots owned by this CTA
    const uint16_t all = static_cast<uint16_t>((1u << Q) - 1u);

    uint8_t* sA = smem;                                   // slabs x 4 KiB
    uint8_t* ring = sA + slabs * kSlabBytes;              // NST x 4 KiB
    uint16_t* raw = reinterpret_cast<uint16_t*>(ring + NST * kSlabBytes);  // 2 x [SQ][C32]
    const uint32_t raw_elems = SQ * bp.C32;
    uint32_t* s_bc = reinterpret_cast<uint32_t*>(raw + 2u * raw_elems);
    uint8_t* region = reinterpret_cast<uint8_t*>(s_bc + bp.C32);
    uint64_t* bars = reinterpret_cast<uint64_t*>(region + p.region_bytes);
    uint64_t* full = bars;
    uint64_t* conv = full + NST;
    uint64_t* empty = conv + NST;
    uint64_t* a_full = empty + NST;
    uint64_t* t_full = a_full + 1;
    uint64_t* t_empty = t_full + kTmemBufs;
    uint64_t* r_full = t_empty + kTmemBufs;
    uint64_t* r_empty = r_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(r_empty + 2);

    if (tid == 0) {
        for (uint32_t i = 0; i < NST; ++i) {
            bar_init(&full[i], 1);
            bar_init(&conv[i], 4);
            bar_init(&empty[i], Q);
        }
        bar_init(a_full, 1);
        for (uint32_t i = 0; i < kTmemBufs; ++i) {
            bar_init(&t_full[i], 1);
            bar_init(&t_empty[i], 4);
        }
        for (uint32_t i = 0; i < 2; ++i) {
            bar_init(&r_full[i], 4u * Q);
            bar_init(&r_empty[i], Q);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (uint32_t c = tid; c < bp.C32; c += kMmaThreads) s_bc[c] = bp.bc[c];
    if (warp == 1) {  // TMEM: 4 accumulators x 128 columns
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(saddr(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // every CTA's barriers are initialised before any remote arrive / multicast
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            bar_expect_tx(a_full, slabs * kSlabBytes);
            for (uint32_t s = 0; s < slabs; ++s)
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3}], [%4];" ::"r"(saddr(sA + s * kSlabBytes)),
                    "l"(reinterpret_cast<uint64_t>(&p.tmap_a)), "r"(32u * s), "r"(128u * q), "r"(saddr(a_full))
                    : "memory");
            uint32_t g = 0;
            for (uint32_t j = 0; j < nblk; ++j) {
                const uint32_t tr0 = 4u * (cid + j * ncl);  // first tile-row of the block
                for (uint32_t s = 0; s < slabs; ++s, ++g) {
                    const uint32_t st = g % NST, ph = (g / NST) & 1u;
                    bar_wait(&empty[st], ph ^ 1u);
                    bar_expect_tx(&full[st], kSlabBytes);
                    if (g % Q == q) {
                        const uint32_t y = s / p.xchunks, xo = (s % p.xchunks) * 32u;
                        if (Q > 1)
                            asm volatile(
                                "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                                ".multicast::cluster [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(
                                    saddr(ring + st * kSlabBytes)),
                                "l"(reinterpret_cast<uint64_t>(&p.tmap_b)), "r"(xo), "r"(0u), "r"(y), "r"(tr0),
                                "r"(saddr(&full[st])), "h"(all)
                                : "memory");
                        else
                            asm volatile(
                                "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                                " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(saddr(ring + st * kSlabBytes)),
                                "l"(reinterpret_cast<uint64_t>(&p.tmap_b)), "r"(xo), "r"(0u), "r"(y), "r"(tr0),
                                "r"(saddr(&full[st]))
                                : "memory");
                    }
                }
            }
            // every remote commit aimed at this CTA's ring has landed before the final cluster
            // barrier (the last phase of each slot's empty barrier)
            for (uint32_t st = 0; st < NST && st < g; ++st) {
                const uint32_t uses = (g - st + NST - 1u) / NST;
                bar_wait(&empty[st], (uses - 1u) & 1u);
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            bar_wait(a_full, 0);
            tc_fence_after();
            uint32_t g = 0;
            for (uint32_t j = 0; j < nblk; ++j) {
                const uint32_t tb = j % kTmemBufs;
                bar_wait(&t_empty[tb], ((j / kTmemBufs) & 1u) ^ 1u);
                tc_fence_after();
                const uint32_t d = tmem + tb * kSlots;
                for (uint32_t s = 0; s < slabs; ++s, ++g) {
                    const uint32_t st = g % NST, ph = (g / NST) & 1u;
                    bar_wait(&conv[st], ph);
                    tc_fence_after();
                    mma_i8(d, sw32_desc(saddr(sA + s * kSlabBytes)), sw32_desc(saddr(ring + st * kSlabBytes)),
                           s > 0 ? 1u : 0u);
                    if (Q > 1)
                        mma_commit_multicast(&empty[st], all);  // the slot is free in every CTA
                    else
                        mma_commit_local(&empty[st]);
                }
                mma_commit_local(&t_full[tb]);
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ---------------- converter + drain (warpgroup; quadrant = TMEM lanes) ----------------
        const uint32_t qd = warp - 4u;
        const uint32_t col = 32u * qd + lane;          // column within this CTA's 128
        const uint32_t total_slabs = nblk * slabs;
        uint32_t gc = 0, jd = 0;                       // next slab to convert, next block to drain
        while (gc < total_slabs || jd < nblk) {
            bool did = false;
            if (gc < total_slabs) {
                const uint32_t st = gc % NST, ph = (gc / NST) & 1u;
                if (bar_test(&full[st], ph)) {
                    // this warp's quarter of the slab: 32 rows x 32 B, one row per lane
                    uint4* r = reinterpret_cast<uint4*>(ring + st * kSlabBytes + (32u * qd + lane) * 32u);
                    uint4 a = r[0], b = r[1];
                    a.x = nz01(a.x), a.y = nz01(a.y), a.z = nz01(a.z), a.w = nz01(a.w);
                    b.x = nz01(b.x), b.y = nz01(b.y), b.z = nz01(b.z), b.w = nz01(b.w);
                    r[0] = a;
                    r[1] = b;
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) bar_arrive(&conv[st]);
                    ++gc;
                    did = true;
                }
            }
            if (jd < nblk) {
                const uint32_t tb = jd % kTmemBufs, rb = jd & 1u;
                // accumulator ready and every owner CTA done with raw buffer rb (block jd - 2)
                if (bar_test(&t_full[tb], (jd / kTmemBufs) & 1u) && bar_test(&r_empty[rb], ((jd >> 1) & 1u) ^ 1u)) {
                    tc_fence_after();
                    uint16_t* rbuf = raw + rb * raw_elems;
                    const uint32_t cglob = 128u * q + col;  // column index (C32 space)
                    for (uint32_t cc = 0; cc < kSlots / 32u; ++cc) {
                        uint32_t v[32];
                        tmem_ld32(tmem + ((32u * qd) << 16) + tb * kSlots + 32u * cc, v);
                        // lanes pair up so each stores (column c, c+1) of one slot as a u32:
                        // even lane takes slot n of (c, c+1), odd lane slot n+1 of (c-1, c)
                        const bool odd = lane & 1u;
#pragma unroll
                        for (uint32_t i = 0; i < 32u; i += 2u) {
                            const uint32_t give = odd ? v[i] : v[i + 1u];
                            const uint32_t got = __shfl_xor_sync(0xffffffffu, give, 1);
                            const uint32_t n = 32u * cc + i + (odd ? 1u : 0u);  // slot
                            const uint32_t pair = odd ? (got & 0xFFFFu) | (v[i + 1u] << 16)
                                                      : (v[i] & 0xFFFFu) | (got << 16);
                            const uint32_t dst = n / SQ;
                            const uint32_t c0 = cglob & ~1u;
                            st_remote_u32(rbuf + (n % SQ) * bp.C32 + c0, dst, pair);
                        }
                    }
                    tc_fence_before();
                    asm volatile("fence.acq_rel.cluster;" ::: "memory");  // this lane's DSMEM stores
                    __syncwarp();
                    if (lane == 0) {
                        bar_arrive(&t_empty[tb]);
                        for (uint32_t r = 0; r < Q; ++r) bar_arrive_remote(&r_full[rb], r);
                    }
                    ++jd;
                    did = true;
                }
            }
            if (!did) __nanosleep(20);
        }
    } else if (warp >= 8) {
        // ---------------- top-k (rows a3/a4) ----------------
        const uint32_t wi = warp - 8u;
        for (uint32_t j = 0; j < nblk; ++j) {
            const uint32_t rb = j & 1u;
            bar_wait_cluster(&r_full[rb], (j >> 1) & 1u);
            uint16_t* rbuf = raw + rb * raw_elems;
            const uint32_t tr0 = 4u * (cid + j * ncl);
            // the CTA's slots [q*SQ, (q+1)*SQ) as tile-row segments of <= 32 slots
            for (uint32_t n0 = q * SQ; n0 < (q + 1u) * SQ; n0 += min(SQ, 32u)) {
                const uint32_t tr = tr0 + n0 / 32u, tx0 = n0 % 32u;
                const uint32_t gs = tr < p.tile_rows && tx0 < p.tiles_x ? min(min(SQ, 32u), p.tiles_x - tx0) : 0u;
                if (gs == 0u) continue;
                batched_topk<4, kTopkWarps>(bp, rbuf + (n0 - q * SQ) * bp.C32, region, region, p.region_bytes, s_bc,
                                            tr * p.tiles_x + tx0, gs, 0u, 1u, wi, lane);
            }
            asm volatile("bar.sync 1, %0;" ::"n"(kTopkWarps * 32u) : "memory");
            if (wi == 0 && lane == 0)
                for (uint32_t r = 0; r < Q; ++r) bar_arrive_remote(&r_empty[rb], r);
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

uint32_t patch_mma_smem(uint32_t slabs, uint32_t stages, uint32_t Q, uint32_t C32, uint32_t region_bytes) {
    return slabs * kSlabBytes + stages * kSlabBytes + 2u * (kSlots / Q) * C32 * 2u + C32 * 4u + region_bytes +
           (3u * stages + 1u + 2u * kTmemBufs + 4u) * 8u + 16u;
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
