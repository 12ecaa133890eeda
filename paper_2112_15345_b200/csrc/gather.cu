// gather.cu -- feature rows of the input vertices.
//
// "CPU feature copy ... fetches data from both local machines and remote machines
// for each mini-batch and stores data in contiguous memory" / "GPU feature copy"
// (P:563-565): here one HBM->HBM gather per batch; rows owned by another rank are
// read in place over NVLink (peer mapping, eg_import_shards).  out_u[i] =
// rows_u[tid(src_nodes_{L-1}[u][i])], verbatim bytes (input order,
// duplicates allowed).
//
// Each thread moves 16-byte units (row_bytes % 16 == 0); consecutive threads take
// consecutive units of a row so both the row read and the output write coalesce;
// kUnroll independent loads are in flight per thread before their stores.
#include "kernels.h"

namespace eg {

constexpr int kUnroll = 4;

__global__ void __launch_bounds__(256) gather_kernel(const __grid_constant__ GraphDev g,
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
                const int64_t tid = gd.nodes[u][i] - g.off[u];
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

void launch_gather(const GraphDev &g, const FeatDev &f, const GatherDev &gd, cudaStream_t s)
{
    gather_kernel<<<kSMs * 8, 256, 0, s>>>(g, f, gd);
}

}  // namespace eg
