// gather.cu -- feature rows of the input vertices.
//
// "CPU feature copy ... fetches data from both local machines and remote machines
// for each mini-batch and stores data in contiguous memory" / "GPU feature copy"
// (P:563-565): here one HBM->HBM gather per batch; rows owned by another rank are
// read in place over NVLink (peer mapping, eg_import_shards).  out_u[i] =
// rows_u[tid(src_nodes_{L-1}[u][i])], verbatim bytes (input order,
// duplicates allowed).
//
// Two implementations of the same copy (EG_GATHER=tma|ldg|auto):
//  * gather_tma_kernel (default): rows are staged through shared memory by the Tensor
//    Memory Accelerator -- one cp.async.bulk.tensor tile::gather4 per four rows of a
//    type whose table is local (a 2-D tensor map per type), else one cp.async.bulk per
//    row (e.g. rows in peer shards, over NVLink) -- and leave by one bulk store per stage
//    (the output of a tile of consecutive rows is contiguous).  A producer warp (ids of
//    the next tile prefetched) and a consumer thread around a ring of mbarrier-guarded
//    stages; 64 threads per CTA, so the sampling kernels of the other pipeline lanes
//    keep running beside it (measured: the path is faster although this gather alone is
//    slightly slower than the LDG one).
//  * gather_ldg_kernel: warp per group of 32 rows, 16-B vector loads, 8 independent
//    16-B loads per lane in flight; used at world 1 when a type has no gather4 map
//    (local per-row bulk copies are issue-bound: one UBLKCP per row).
#include <cstdlib>
#include <cstring>

#include "kernels.h"

namespace eg {

// ----------------------------------------------------------------------------- LDG path

// A warp copies groups of 32 consecutive output rows of one type: one coalesced load of
// the 32 ids, then "items" of one warp-wide 16-B access each (rows of >= 512 B take
// ceil(U/32) items per row; shorter rows pack 32/U rows per item), kBatch items in
// flight per lane before their stores.  Consecutive lanes touch consecutive 16-B units
// of a row, so every row read and the output write are coalesced.
constexpr int kBatch = 8;
#ifndef EG_GATHER_MIN_BLOCKS
#define EG_GATHER_MIN_BLOCKS 1
#endif
constexpr int kGatherMinBlocks = EG_GATHER_MIN_BLOCKS;   // CTAs per SM the register budget must allow

__device__ __forceinline__ int32_t seg_rows(const GatherSet &gs, int b, int u)
{
    const GatherDev &gd = gs.b[b];
    return gd.out[u] ? gd.meta[kMetaNodes + gd.level * EG_MAX_VT + u] : 0;
}

__global__ void __launch_bounds__(256, kGatherMinBlocks) gather_ldg_kernel(const __grid_constant__ GraphDev g,
                                                         const __grid_constant__ FeatDev f,
                                                         const __grid_constant__ GatherSet gs)
{
    const int lane = lane_id();
    const int V = g.n_vt, S = gs.nb * V;                 // segments: (batch, type)
    int64_t total = 0;
    for (int sg = 0; sg < S; ++sg) total += ((int64_t)seg_rows(gs, sg / V, sg % V) + 31) / 32;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    int sg = 0;
    int64_t seg_lo = 0, seg_hi = (seg_rows(gs, 0, 0) + 31) / 32;
    for (int64_t grp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); grp < total; grp += nw) {
        while (grp >= seg_hi) {                          // groups are visited in increasing order
            ++sg;
            seg_lo = seg_hi;
            seg_hi += (seg_rows(gs, sg / V, sg % V) + 31) / 32;
        }
        const int u = sg % V;
        const GatherDev &gd = gs.b[sg / V];
        const int64_t row0 = (grp - seg_lo) * 32;
        const int nrows = (int)min((int64_t)32, (int64_t)seg_rows(gs, sg / V, u) - row0);
        const int64_t rb = f.row_bytes[u];
        const int U = (int)(rb >> 4);
        const uint8_t *srow = nullptr;
        if (lane < nrows) {
            const int64_t tid = __ldg(gd.nodes[u] + row0 + lane) - g.off[u];
            srow = feature_row(g, f, u, tid);
        }
        uint8_t *dbase = gd.out[u] + row0 * rb;
        const bool wide = U >= 32;
        const int cpr = wide ? (U + 31) >> 5 : 1;        // items per row (wide rows)
        const int rpi = wide ? 1 : 32 / U;               // rows per item (narrow rows)
        const int lrow = wide ? 0 : lane / U, lunit = wide ? lane : lane % U;
        const int items = wide ? nrows * cpr : (nrows + rpi - 1) / rpi;
        for (int k0 = 0; k0 < items; k0 += kBatch) {
            int4 v[kBatch];
            uint32_t off[kBatch];   // output byte offset from dbase (< 32 rows x row_bytes), ~0u: none
#pragma unroll
            for (int q = 0; q < kBatch; ++q) {
                const int k = k0 + q;
                int row, unit;
                if (wide) {
                    row = k / cpr;
                    unit = (k - row * cpr) * 32 + lane;
                } else {
                    row = k * rpi + lrow;
                    unit = lunit;
                }
                const bool ok = k < items && row < nrows && unit < U && (wide || lane < rpi * U);
                const uint8_t *sp = (const uint8_t *)__shfl_sync(0xffffffffu, (unsigned long long)srow, row & 31);
                off[q] = ~0u;
                if (ok) {
                    v[q] = ld_nc_v4(sp + 16 * unit);
                    off[q] = (uint32_t)(row * rb + 16 * unit);
                }
            }
#pragma unroll
            for (int q = 0; q < kBatch; ++q)
                if (off[q] != ~0u) st_v4(dbase + off[q], v[q]);
        }
    }
}

// ----------------------------------------------------------------------------- TMA path

#ifndef EG_TMA_STAGES
#define EG_TMA_STAGES 4
#endif
#ifndef EG_TMA_STAGE_BYTES
#define EG_TMA_STAGE_BYTES 16384
#endif
constexpr int kStages = EG_TMA_STAGES;           // ring depth per CTA
constexpr int kStageBytes = EG_TMA_STAGE_BYTES;  // bytes per stage
constexpr int kMaxRowsPerTile = 128;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Bounded: a transfer that never completes (a bad tensor map, a faulting address) traps
// after ~2 s instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    uint64_t t0 = 0;
    for (uint32_t it = 0;; ++it) {
        uint32_t done;
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n"
            "}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (done) return;
        if ((it & 1023) == 1023) {
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (!t0) t0 = t;
            else if (t - t0 > 2000000000ull) __trap();
        }
    }
}

#ifndef EG_TMA_L2_HINT
#define EG_TMA_L2_HINT 0   // 1: row loads and output stores evict-first in L2 (A/B builds)
#endif

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes)
{
#if EG_TMA_L2_HINT
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes), "l"(pol)
                 : "memory");
#else
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
#endif
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// Four rows (type-local indices r0..r3 of the map's table) of a 2-D tensor map into
// shared memory, row after row: one TMA operation (tile::gather4, sm_100).
__device__ __forceinline__ void gather4_g2s(void *dst, const CUtensorMap *map, int32_t r0, int32_t r1, int32_t r2,
                                            int32_t r3, uint64_t *bar)
{
#if EG_TMA_L2_HINT
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(smem_u32(dst)),
        "l"(map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
#else
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
        : "memory");
#endif
}

// Tiles of consecutive rows of one (batch, type) segment; segments in (batch, type) order.
struct TileCursor {
    int sg = 0;
    int64_t lo = 0, hi = 0;
};

// Stage stride of a gather4 group of type u: 4 rows, rounded up to 128 B (the TMA writes
// each group to a 128-B aligned shared address; rows of 400 B leave 64 B of padding).
__device__ __forceinline__ int64_t group_stride(const FeatDev &f, int u)
{
    return (4 * f.row_bytes[u] + 127) & ~(int64_t)127;
}

// Rows per tile: gather4 types fill the stage with whole groups (a multiple of 4 rows);
// per-row types with whole rows.
__device__ __forceinline__ int32_t rows_per_tile(const FeatDev &f, const GatherMaps &m, int u)
{
    const int64_t rb = f.row_bytes[u];
    if (m.grp[u]) return (int32_t)min((int64_t)kMaxRowsPerTile, 4 * ((int64_t)kStageBytes / group_stride(f, u)));
    const int32_t r = rb ? (int32_t)min((int64_t)kMaxRowsPerTile, (int64_t)kStageBytes / rb) : 1;
    return r > 0 ? r : 1;
}

__device__ __forceinline__ int64_t seg_tiles(const GatherSet &gs, const FeatDev &f, const GatherMaps &m, int V, int sg)
{
    const int32_t n = seg_rows(gs, sg / V, sg % V);
    const int32_t rpt = rows_per_tile(f, m, sg % V);
    return (n + rpt - 1) / rpt;
}

// tiles are visited in increasing order by each block: advance the cursor
__device__ __forceinline__ void tile_of(const GatherSet &gs, const FeatDev &f, const GatherMaps &m, int V, TileCursor &cur, int64_t t,
                                        int &b, int &u, int64_t &row0, int32_t &nrows)
{
    while (t >= cur.hi) {
        ++cur.sg;
        cur.lo = cur.hi;
        cur.hi += seg_tiles(gs, f, m, V, cur.sg);
    }
    b = cur.sg / V;
    u = cur.sg % V;
    const int32_t rpt = rows_per_tile(f, m, u);
    row0 = (t - cur.lo) * rpt;
    nrows = (int32_t)min((int64_t)rpt, (int64_t)seg_rows(gs, b, u) - row0);
}

__global__ void __launch_bounds__(64, 1) gather_tma_kernel(const __grid_constant__ GraphDev g,
                                                           const __grid_constant__ FeatDev f,
                                                           const __grid_constant__ GatherSet gs,
                                                           const __grid_constant__ GatherMaps m)
{
    extern __shared__ __align__(128) uint8_t stage_mem[];
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int V = g.n_vt, S = gs.nb * V;
    int64_t total = 0;
    for (int sg = 0; sg < S; ++sg) total += seg_tiles(gs, f, m, V, sg);
    const int64_t n_my = total > blockIdx.x ? (total - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    TileCursor cur;
    cur.hi = seg_tiles(gs, f, m, V, 0);
    if (warp == 0) {
        // producer: ids -> TMA loads of rows into the stage.  The ids of tile j + 1 are
        // loaded before waiting for tile j's stage (one id-load latency per tile was the
        // producer's bound).  A lane holds 4 ids of a tile: rows 4 lane .. 4 lane + 3 (one
        // gather4 group; rows_per_tile <= 128) or rows lane + 32 q (per-row copies).
        struct Pre {
            int b, u;
            int64_t row0;
            int32_t nrows;
            int64_t id[4];
        };
        auto prefetch = [&](int64_t j, Pre &p) {
            tile_of(gs, f, m, V, cur, blockIdx.x + j * gridDim.x, p.b, p.u, p.row0, p.nrows);
            const int64_t *ids = gs.b[p.b].nodes[p.u] + p.row0;
            const bool grp = m.grp[p.u] != 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int rr = grp ? min(4 * lane + q, p.nrows - 1) : lane + 32 * q;
                const bool ok = grp ? 4 * lane < p.nrows : rr < p.nrows;
                p.id[q] = ok ? __ldg(ids + rr) : 0;
            }
        };
        Pre nx;
        if (n_my > 0) prefetch(0, nx);
        for (int64_t j = 0; j < n_my; ++j) {
            const Pre cu = nx;
            if (j + 1 < n_my) prefetch(j + 1, nx);
            const int s = (int)(j % kStages);
            mbar_wait(&empty[s], (uint32_t)(((j / kStages) & 1) ^ 1));
            const int u = cu.u;
            const int32_t nrows = cu.nrows;
            const int64_t rb = f.row_bytes[u];
            uint8_t *dst = stage_mem + s * kStageBytes;
            if (m.grp[u]) {
                // groups of 4 rows, one gather4 each, at 128-B aligned group strides (a
                // ragged last group repeats its last row: 4 rows always land, inside the
                // stage since rows_per_tile counts whole groups).  A group whose rows span
                // two owner shards is fetched row by row into the same layout.
                const int ng = (nrows + 3) >> 2;
                if (lane == 0) mbar_expect_tx(&full[s], (uint32_t)(ng * 4 * rb));
                __syncwarp();
                if (lane < ng) {
                    uint8_t *gdst = dst + lane * group_stride(f, u);
                    int64_t tid[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) tid[q] = cu.id[q] - g.off[u];
                    int p0 = 0;
                    bool same = true;
                    if (!m.whole[u]) {
                        p0 = owner_of(g, u, tid[0]);
#pragma unroll
                        for (int q = 1; q < 4; ++q) same &= tid[q] >= g.bounds[u][p0] && tid[q] < g.bounds[u][p0 + 1];
                    }
                    if (same) {
                        const int64_t lo = m.whole[u] ? 0 : g.bounds[u][p0];
                        gather4_g2s(gdst, &m.map[u][p0], (int32_t)(tid[0] - lo), (int32_t)(tid[1] - lo),
                                    (int32_t)(tid[2] - lo), (int32_t)(tid[3] - lo), &full[s]);
                    } else {
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            bulk_g2s(gdst + q * rb, feature_row(g, f, u, tid[q]), (uint32_t)rb, &full[s]);
                    }
                }
            } else {
                if (lane == 0) mbar_expect_tx(&full[s], (uint32_t)(nrows * rb));
                __syncwarp();
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int rr = lane + 32 * q;
                    if (rr < nrows)
                        bulk_g2s(dst + rr * rb, feature_row(g, f, u, cu.id[q] - g.off[u]), (uint32_t)rb, &full[s]);
                }
            }
        }
    } else if (lane == 0) {
        // consumer: one bulk store of the staged rows (contiguous in the output); a stage
        // is released once the NEXT store is issued and this one has been read
        for (int64_t j = 0; j < n_my; ++j) {
            const int s = (int)(j % kStages);
            mbar_wait(&full[s], (uint32_t)((j / kStages) & 1));
            int b, u;
            int64_t row0;
            int32_t nrows;
            tile_of(gs, f, m, V, cur, blockIdx.x + j * gridDim.x, b, u, row0, nrows);
            const int64_t rb = f.row_bytes[u];
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            const int64_t gsz = group_stride(f, u);
            if (!m.grp[u] || gsz == 4 * rb) {   // rows contiguous in the stage: one store
                bulk_s2g(gs.b[b].out[u] + row0 * rb, stage_mem + s * kStageBytes, (uint32_t)(nrows * rb));
            } else {                             // padded groups: one store per group
                for (int q = 0; 4 * q < nrows; ++q)
                    bulk_s2g(gs.b[b].out[u] + (row0 + 4 * q) * rb, stage_mem + s * kStageBytes + q * gsz,
                             (uint32_t)(min(4, nrows - 4 * q) * rb));
            }
            if (j > 0) {
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                mbar_arrive(&empty[(int)((j - 1) % kStages)]);
            }
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

int launch_gather(const GraphDev &g, const FeatDev &f, const GatherSet &gd, const GatherMaps &m, cudaStream_t s,
                  int mode)
{
    // The TMA kernel stages whole rows (per-row copies) or 4-row groups (gather4) in one
    // stage of kStageBytes: a requested type with wider rows goes to the LDG kernel, which
    // copies rows of any width in 16-B units (whatever EG_GATHER says).
    for (int b = 0; b < gd.nb; ++b)
        for (int u = 0; u < g.n_vt; ++u)
            if (gd.b[b].out[u] && f.row_bytes[u] > kStageBytes) mode = 1;
    if (mode == 2) {
        // TMA unless a requested type would be read from LOCAL memory by per-row bulk copies
        // (world 1 without a gather4 map: issue-bound, measured C3 12.7k vs 13.5k with LDG).
        // Peer rows (world > 1) are NVLink-bound either way, and the TMA kernel leaves the
        // SMs to the sampling kernels (measured N = 2: C2 +7 %, C3 +3 %, C4 +8 %, C5 +5 %).
        bool ldg = false;
        for (int b = 0; b < gd.nb; ++b)
            for (int u = 0; u < g.n_vt; ++u)
                if (gd.b[b].out[u] && !m.grp[u] && g.world == 1) ldg = true;
        mode = ldg ? 1 : 0;
    }
    if (mode == 1) {
        static int blocks = 0;
        if (!blocks) {
            int per_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gather_ldg_kernel, 256, 0);
            const char *e = getenv("EG_GATHER_CTAS");   // CTAs per SM (A/B runs); default: max resident
            if (e && atoi(e) > 0 && atoi(e) < per_sm) per_sm = atoi(e);
            blocks = kSMs * (per_sm > 0 ? per_sm : 4);
        }
        gather_ldg_kernel<<<blocks, 256, 0, s>>>(g, f, gd);
        return 1;
    }
    static bool attr = false;
    const int smem = kStages * kStageBytes;
    if (!attr) {
        cudaFuncSetAttribute(gather_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    static int per_sm = 0;
    if (!per_sm) {
        const char *e = getenv("EG_TMA_CTAS");   // CTAs per SM (A/B runs); default 2
        per_sm = (e && atoi(e) > 0 && atoi(e) <= 3) ? atoi(e) : 2;
    }
    gather_tma_kernel<<<kSMs * per_sm, 64, smem, s>>>(g, f, gd, m);
    return 0;
}

}  // namespace eg
