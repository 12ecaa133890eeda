// gather.cu -- feature rows of the input vertices.
//
// "CPU feature copy ... fetches data from both local machines and remote machines
// for each mini-batch and stores data in contiguous memory" / "GPU feature copy"
// (P:563-565): here one HBM->HBM gather per batch; rows owned by another rank are
// read in place over NVLink (peer mapping, eg_import_shards).  out_u[i] =
// rows_u[tid(src_nodes_{L-1}[u][i])], verbatim bytes (input order,
// duplicates allowed).
//
// Two implementations of the same copy:
//  * gather_tma_kernel (default): rows are staged through shared memory by the
//    Tensor Memory Accelerator -- one cp.async.bulk per row into a stage, one bulk
//    store per stage (the output of a tile of consecutive rows is contiguous) --
//    with a producer warp (ids + bulk loads) and a consumer warp (bulk stores)
//    around a ring of mbarrier-guarded stages.  Few instructions per byte and up to
//    kStages * kStageBytes in flight per SM.
//  * gather_ldg_kernel: 16-byte vector loads / stores, kUnroll per thread in flight.
#include <cstdlib>
#include <cstring>

#include "kernels.h"

namespace eg {

// ----------------------------------------------------------------------------- LDG path

constexpr int kUnroll = 8;

__global__ void __launch_bounds__(256) gather_ldg_kernel(const __grid_constant__ GraphDev g,
                                                         const __grid_constant__ FeatDev f,
                                                         const __grid_constant__ GatherDev gd)
{
    const int32_t *n = gd.meta + kMetaNodes + gd.level * EG_MAX_VT;
    int64_t cum[EG_MAX_VT + 1];
    uint32_t units[EG_MAX_VT];
    cum[0] = 0;
    for (int u = 0; u < g.n_vt; ++u) {
        units[u] = (uint32_t)(f.row_bytes[u] >> 4);
        cum[u + 1] = cum[u] + (gd.out[u] ? (int64_t)n[u] * units[u] : 0);
    }
    const int64_t total = cum[g.n_vt];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q0 < total; q0 += stride * kUnroll) {
        int4 val[kUnroll];
        uint8_t *dst[kUnroll];
#pragma unroll
        for (int k = 0; k < kUnroll; ++k) {
            const int64_t q = q0 + k * stride;
            dst[k] = nullptr;
            if (q < total) {
                int u = 0;
                while (q >= cum[u + 1]) ++u;
                const uint32_t local = (uint32_t)(q - cum[u]);
                const uint32_t i = local / units[u], c = local - i * units[u];
                const int64_t tid = __ldg(gd.nodes[u] + i) - g.off[u];
                const int p = owner_of(g, u, tid);
                const uint8_t *src = f.rows[u][p] + (tid - g.bounds[u][p]) * f.row_bytes[u] + 16 * (int64_t)c;
                val[k] = ld_nc_v4(src);
                dst[k] = gd.out[u] + (int64_t)local * 16;
            }
        }
#pragma unroll
        for (int k = 0; k < kUnroll; ++k)
            if (dst[k]) st_v4(dst[k], val[k]);
    }
}

// ----------------------------------------------------------------------------- TMA path

constexpr int kStages = 4;
constexpr int kStageBytes = 16384;
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

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

struct TileMap {
    int64_t tcum[EG_MAX_VT + 1];   // tiles before type u
    int32_t rpt[EG_MAX_VT];        // rows per tile
    int32_t n[EG_MAX_VT];
};

__device__ __forceinline__ void tile_of(const TileMap &m, int n_vt, int64_t t, int &u, int64_t &row0, int32_t &nrows)
{
    u = 0;
    while (t >= m.tcum[u + 1]) ++u;
    row0 = (t - m.tcum[u]) * m.rpt[u];
    nrows = (int32_t)min((int64_t)m.rpt[u], (int64_t)m.n[u] - row0);
}

__global__ void __launch_bounds__(64, 1) gather_tma_kernel(const __grid_constant__ GraphDev g,
                                                           const __grid_constant__ FeatDev f,
                                                           const __grid_constant__ GatherDev gd)
{
    extern __shared__ __align__(128) uint8_t stage_mem[];
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
    const int warp = threadIdx.x >> 5, lane = lane_id();
    TileMap m;
    const int32_t *nn = gd.meta + kMetaNodes + gd.level * EG_MAX_VT;
    m.tcum[0] = 0;
    for (int u = 0; u < g.n_vt; ++u) {
        const int64_t rb = f.row_bytes[u];
        m.rpt[u] = rb ? (int32_t)min((int64_t)kMaxRowsPerTile, (int64_t)kStageBytes / rb) : 1;
        m.n[u] = gd.out[u] ? nn[u] : 0;
        m.tcum[u + 1] = m.tcum[u] + (m.n[u] + m.rpt[u] - 1) / m.rpt[u];
    }
    const int64_t total = m.tcum[g.n_vt];
    const int64_t n_my = total > blockIdx.x ? (total - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 0) {
        // producer: ids -> bulk loads of rows into the stage
        for (int64_t j = 0; j < n_my; ++j) {
            const int s = (int)(j % kStages);
            mbar_wait(&empty[s], (uint32_t)(((j / kStages) & 1) ^ 1));
            int u;
            int64_t row0;
            int32_t nrows;
            tile_of(m, g.n_vt, blockIdx.x + j * gridDim.x, u, row0, nrows);
            const int64_t rb = f.row_bytes[u];
            if (lane == 0) mbar_expect_tx(&full[s], (uint32_t)(nrows * rb));
            __syncwarp();
            uint8_t *dst = stage_mem + s * kStageBytes;
            for (int rr = lane; rr < nrows; rr += 32) {
                const int64_t tid = __ldg(gd.nodes[u] + row0 + rr) - g.off[u];
                const int p = owner_of(g, u, tid);
                bulk_g2s(dst + rr * rb, f.rows[u][p] + (tid - g.bounds[u][p]) * rb, (uint32_t)rb, &full[s]);
            }
        }
    } else if (lane == 0) {
        // consumer: one bulk store of the staged rows (contiguous in the output)
        for (int64_t j = 0; j < n_my; ++j) {
            const int s = (int)(j % kStages);
            mbar_wait(&full[s], (uint32_t)((j / kStages) & 1));
            int u;
            int64_t row0;
            int32_t nrows;
            tile_of(m, g.n_vt, blockIdx.x + j * gridDim.x, u, row0, nrows);
            const int64_t rb = f.row_bytes[u];
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            bulk_s2g(gd.out[u] + row0 * rb, stage_mem + s * kStageBytes, (uint32_t)(nrows * rb));
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            mbar_arrive(&empty[s]);
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

static int gather_mode()
{
    static int mode = -1;
    if (mode < 0) {
        const char *e = getenv("EG_GATHER");
        mode = (e && !strcmp(e, "ldg")) ? 1 : 0;
    }
    return mode;
}

void launch_gather(const GraphDev &g, const FeatDev &f, const GatherDev &gd, cudaStream_t s)
{
    if (gather_mode() == 1) {
        static int blocks = 0;
        if (!blocks) {
            int per_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gather_ldg_kernel, 256, 0);
            blocks = kSMs * (per_sm > 0 ? per_sm : 4);
        }
        gather_ldg_kernel<<<blocks, 256, 0, s>>>(g, f, gd);
        return;
    }
    static bool attr = false;
    const int smem = kStages * kStageBytes;
    if (!attr) {
        cudaFuncSetAttribute(gather_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    gather_tma_kernel<<<kSMs * 2, 64, smem, s>>>(g, f, gd);
}

}  // namespace eg
