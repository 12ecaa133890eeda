// compact.cu -- per-hop frontier + block compaction.
//
// "After sampling all neighbors within a hop, it computes the frontier (i.e., the
// unique set of vertices)" and "performs graph compaction to remove
// empty vertices and relabel vertices and edges".  Reading (DESIGN.md
// §3 #6, #7): S_h[u] = F_h[u] ++ sorted-by-gid(unique(srcs of type u) \ F_h[u]);
// every sampled src is relabelled to its position in S_h[s(r)].
//
// B200 design: instead of sorting, new sources are marked in a bitmap indexed by
// gid (type ranges chunk-aligned); a popcount scan over the bitmap yields the new
// vertices already in gid order and their ranks.  pos[gid] (int32, -1 = absent)
// holds the position of every vertex of the batch, so "not in F_h" is pos < 0 and
// the relabel is one gather.  The bitmap is cleared while it is read; pos is reset
// from the node arrays at the end of the batch.
#include "kernels.h"

namespace eg {

__device__ __forceinline__ int64_t edges_cum(const GraphDev &g, const int32_t *nnz, int64_t *cum)
{
    cum[0] = 0;
    for (int r = 0; r < g.n_rel; ++r) cum[r + 1] = cum[r] + nnz[r];
    return cum[g.n_rel];
}

// Mark every sampled src that is not yet in the batch.
__global__ void __launch_bounds__(256) mark_kernel(const __grid_constant__ GraphDev g,
                                                   const __grid_constant__ HopDev hd)
{
    int64_t cum[EG_MAX_REL + 1];
    const int64_t total = edges_cum(g, meta_nnz(hd.meta, hd.h), cum);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        int r = 0;
        while (e >= cum[r + 1]) ++r;
        const uint32_t s = hd.src[r][e - cum[r]];
        if (__ldg(hd.pos + s) < 0) {
            const int u = g.rel[r].src_vt;
            const int64_t bit = g.boff[u] + ((int64_t)s - g.off[u]);
            const uint32_t m = 1u << (bit & 31);
            uint32_t *wp = hd.bitmap + (bit >> 5);
            if (!(*wp & m)) atomicOr(wp, m);
        }
    }
}

// Popcount of each bitmap chunk (one CTA, one uint4 per thread); the last CTA to
// finish turns the counts into per-type exclusive prefixes (chunk_pre).
__global__ void __launch_bounds__(256) bitcount_kernel(const __grid_constant__ GraphDev g,
                                                       const __grid_constant__ HopDev hd, int32_t n_chunks)
{
    static_assert(kChunkWords == 4 * 256, "one uint4 per thread");
    __shared__ int32_t sh[33];
    __shared__ bool last;
    const uint4 x = reinterpret_cast<const uint4 *>(hd.bitmap + (int64_t)blockIdx.x * kChunkWords)[threadIdx.x];
    int32_t c = __popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w);
    c = block_sum(c, sh);
    if (threadIdx.x == 0) {
        hd.chunk_cnt[blockIdx.x] = c;
        __threadfence();
        last = atomicAdd(hd.ticket, 1u) == (uint32_t)n_chunks - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    // exclusive scan over all chunks, then rebase each type at its first chunk
    __shared__ int32_t type_base[EG_MAX_VT];
    int32_t carry = 0;
    for (int c0 = 0; c0 < n_chunks; c0 += blockDim.x) {
        const int ci = c0 + threadIdx.x;
        const int32_t v = ci < n_chunks ? *((volatile int32_t *)hd.chunk_cnt + ci) : 0;
        int32_t tot;
        const int32_t ex = block_excl_scan(v, sh, &tot);
        if (ci < n_chunks) hd.chunk_pre[ci] = carry + ex;
        carry += tot;
    }
    __threadfence_block();
    __syncthreads();
    if (threadIdx.x < g.n_vt) type_base[threadIdx.x] = hd.chunk_pre[g.boff[threadIdx.x] / kChunkBits];
    __syncthreads();
    for (int ci = threadIdx.x; ci < n_chunks; ci += blockDim.x) {
        int u = 0;
        while ((int64_t)ci * kChunkBits >= g.boff[u + 1]) ++u;
        hd.chunk_pre[ci] -= type_base[u];
    }
    if (threadIdx.x == 0) *hd.ticket = 0;   // ready for the next hop
}

// New vertices of each chunk, in gid order: append to the node array of their type,
// set pos[], clear the bitmap words.  One CTA per chunk, 4 words per thread.
__global__ void __launch_bounds__(256) emit_kernel(const __grid_constant__ GraphDev g,
                                                   const __grid_constant__ HopDev hd)
{
    __shared__ int32_t sh[33];
    const int c = blockIdx.x;
    const int32_t mine = hd.chunk_cnt[c];
    if (mine == 0) return;
    const int64_t bit0 = (int64_t)c * kChunkBits;
    int u = 0;
    while (bit0 >= g.boff[u + 1]) ++u;
    const int32_t prior = hd.chunk_pre[c];
    const int32_t nF = meta_nodes(hd.meta, hd.h)[u];
    const int64_t wi = (int64_t)c * kChunkWords + 4 * threadIdx.x;
    uint4 *wp = reinterpret_cast<uint4 *>(hd.bitmap + wi);
    const uint4 x = *wp;
    uint32_t w[4] = {x.x, x.y, x.z, x.w};
    const int32_t pc = __popc(w[0]) + __popc(w[1]) + __popc(w[2]) + __popc(w[3]);
    int32_t tot;
    int32_t position = nF + prior + block_excl_scan(pc, sh, &tot);
    if (pc) {
        const int64_t gbase = (g.off[u] - g.boff[u]) + wi * 32;   // gid of bit 0 of word wi
        int64_t *nodes = hd.nodes[u];
        const int32_t cap = hd.cap_nodes[u];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t word = w[q];
            while (word) {
                const int b = __ffs(word) - 1;
                word &= word - 1;
                const int64_t gid = gbase + 32 * q + b;
                if (position < cap) {
                    nodes[position] = gid;
                    hd.pos[gid] = position;
                } else {
                    atomicOr(hd.meta + kMetaErr, kErrCapacity);
                }
                ++position;
            }
        }
        *wp = make_uint4(0, 0, 0, 0);
    }
    if (threadIdx.x == 0) atomicAdd(meta_nodes(hd.meta, hd.h + 1) + u, mine);
}

// indices = pos[src]: the local id of every sampled src in S_h[s(r)].
__global__ void __launch_bounds__(256) relabel_kernel(const __grid_constant__ GraphDev g,
                                                      const __grid_constant__ HopDev hd)
{
    int64_t cum[EG_MAX_REL + 1];
    const int64_t total = edges_cum(g, meta_nnz(hd.meta, hd.h), cum);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        int r = 0;
        while (e >= cum[r + 1]) ++r;
        const int64_t le = e - cum[r];
        hd.indices[r][le] = __ldg(hd.pos + hd.src[r][le]);
    }
}

// End of batch: pos[] back to -1 for every vertex of the batch.
__global__ void __launch_bounds__(256) reset_kernel(const __grid_constant__ GraphDev g,
                                                    const __grid_constant__ HopDev hd, int32_t level)
{
    const int32_t *n = meta_nodes(hd.meta, level);
    int64_t cum[EG_MAX_VT + 1];
    cum[0] = 0;
    for (int u = 0; u < g.n_vt; ++u) cum[u + 1] = cum[u] + min(n[u], hd.cap_nodes[u]);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cum[g.n_vt];
         i += (int64_t)gridDim.x * blockDim.x) {
        int u = 0;
        while (i >= cum[u + 1]) ++u;
        const int64_t gid = hd.nodes[u][i - cum[u]];
        if (gid >= 0 && gid < g.off[g.n_vt]) hd.pos[gid] = -1;
    }
}

void launch_mark(const GraphDev &g, const HopDev &hd, cudaStream_t s)
{
    mark_kernel<<<kSMs * 8, 256, 0, s>>>(g, hd);
}

void launch_bitcount(const GraphDev &g, const HopDev &hd, int32_t n_chunks, cudaStream_t s)
{
    bitcount_kernel<<<n_chunks, 256, 0, s>>>(g, hd, n_chunks);
}

void launch_emit(const GraphDev &g, const HopDev &hd, int32_t n_chunks, cudaStream_t s)
{
    emit_kernel<<<n_chunks, 256, 0, s>>>(g, hd);
}

void launch_relabel(const GraphDev &g, const HopDev &hd, cudaStream_t s)
{
    relabel_kernel<<<kSMs * 8, 256, 0, s>>>(g, hd);
}

void launch_reset(const GraphDev &g, const HopDev &hd, int32_t level, cudaStream_t s)
{
    reset_kernel<<<kSMs * 4, 256, 0, s>>>(g, hd, level);
}

}  // namespace eg
