/*
 * synth/synth_dev.cu -- device side of the SYNTHETIC INPUT GENERATOR.
 *
 * Fills a GPU shard's src-tid array and feature rows with exactly the bytes
 * synth.c produces on the host (same synth_hash.h formulas), so shards of the
 * large configs never have to be materialised on the host.  Input generation
 * only; not part of the sampling path and not called inside any timed region.
 */
#include <cuda_runtime.h>
#include <stdint.h>

#include "synth_hash.h"

__global__ void sy_indices_kernel(uint64_t G, int32_t r, int64_t n_src, int64_t e_lo, int64_t n,
                                  int32_t *out)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = sy_src_tid(G, r, e_lo + i, n_src);
}

__global__ void sy_features_kernel(uint64_t G, int32_t u, int64_t tid_lo, int64_t n_rows, int64_t dim,
                                   int32_t dtype, void *out)
{
    const int64_t n = n_rows * dim;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t t = tid_lo + i / dim, c = i % dim;
        if (dtype == 0) ((uint32_t *)out)[i] = sy_feat_f32(G, u, t, c);
        else ((uint16_t *)out)[i] = sy_feat_f16(G, u, t, c);
    }
}

extern "C" int sy_indices_dev(uint64_t G, int32_t r, int64_t n_src, int64_t e_lo, int64_t e_hi,
                              int32_t *out, void *stream)
{
    if (e_hi <= e_lo) return 0;
    sy_indices_kernel<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(G, r, n_src, e_lo, e_hi - e_lo, out);
    return (int)cudaGetLastError();
}

extern "C" int sy_features_dev(uint64_t G, int32_t u, int64_t tid_lo, int64_t tid_hi, int64_t dim,
                               int32_t dtype, void *out, void *stream)
{
    if (tid_hi <= tid_lo) return 0;
    sy_features_kernel<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(G, u, tid_lo, tid_hi - tid_lo, dim,
                                                                   dtype, out);
    return (int)cudaGetLastError();
}
