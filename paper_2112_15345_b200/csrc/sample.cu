// sample.cu -- seeds -> frontier, per-hop counts / scan, and the sampling kernel.
//
// The sampling step follows P:282-285 ("randomly pick at most K
// (called fanout) neighbor vertices for each target vertex") per edge type, hop by
// hop, under the key32 reading: for a dst v with
// in-degree d in relation r at hop h, k = fanout[h][r]: all d edges when k == -1 or
// d <= k, else the k offsets j with the smallest composites (key32 << 32 | j),
// emitted in ascending j.  One warp per (dst, relation).
#include "kernels.h"

namespace eg {

// ----------------------------------------------------------------------------- hop 0

// Seeds (caller order, mixed types) -> F_0[u] (stable per type) + pos[] for the
// dst-prefix relabel; flags out-of-range and duplicate seeds.  One CTA.
__global__ void __launch_bounds__(1024) seed_split_kernel(const __grid_constant__ GraphDev g,
                                                          const int64_t *__restrict__ seeds,
                                                          const __grid_constant__ HopDev hd)
{
    const int64_t n = (int64_t)hd.dyn[1];
    __shared__ int32_t sh[33];
    __shared__ int32_t base[EG_MAX_VT];
    if (threadIdx.x < EG_MAX_VT) base[threadIdx.x] = 0;
    __syncthreads();
    const int64_t n_total = g.off[g.n_vt];
    for (int64_t t0 = 0; t0 < n; t0 += blockDim.x) {
        const int64_t i = t0 + threadIdx.x;
        int64_t gid = -1;
        int vt = -1;
        if (i < n) {
            gid = seeds[i];
            if (gid < 0 || gid >= n_total) {
                atomicOr(hd.meta + kMetaErr, kErrSeedRange);
            } else {
                vt = 0;
                while (gid >= g.off[vt + 1]) ++vt;
            }
        }
        for (int u = 0; u < g.n_vt; ++u) {
            const int32_t flag = (vt == u);
            int32_t tot;
            const int32_t ex = block_excl_scan(flag, sh, &tot);
            if (flag) {
                const int32_t p = base[u] + ex;
                if (p < hd.cap_nodes[u]) {
                    hd.nodes[u][p] = gid;
                    if (atomicCAS(hd.pos + gid, -1, p) != -1) atomicOr(hd.meta + kMetaErr, kErrSeedDup);
                } else {
                    atomicOr(hd.meta + kMetaErr, kErrCapacity);
                }
            }
            if (threadIdx.x == 0) base[u] += tot;
            __syncthreads();
        }
    }
    if (threadIdx.x < g.n_vt)
        meta_nodes(hd.meta, 0)[threadIdx.x] = min(base[threadIdx.x], hd.cap_nodes[threadIdx.x]);
}

void launch_seed_split(const GraphDev &g, const int64_t *seeds, const HopDev &hd, cudaStream_t s)
{
    seed_split_kernel<<<1, 1024, 0, s>>>(g, seeds, hd);
}

// ----------------------------------------------------------------------------- counts + scan

// Phase 1: count c(r, i) = min(d, k) (or d) for every dst i of F_h[t(r)], written
// into the block indptr slot i; per-block sums into partial[r][b].
__global__ void __launch_bounds__(256) count_kernel(const __grid_constant__ GraphDev g,
                                                    const __grid_constant__ HopDev hd)
{
    __shared__ int32_t sh[33];
    const int r = blockIdx.y, b = blockIdx.x;
    const RelDev &R = g.rel[r];
    const int t = R.dst_vt;
    const int k = hd.fanout[r];
    const int32_t *nF = meta_nodes(hd.meta, hd.h);
    if (r == 0 && b == 0 && threadIdx.x < g.n_vt)   // S_h starts as F_h; emit adds the new ones
        meta_nodes(hd.meta, hd.h + 1)[threadIdx.x] = nF[threadIdx.x];
    const int64_t n = nF[t];
    const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
    const int64_t lo = b * chunk, hi = min(n, lo + chunk);
    int32_t sum = 0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        int32_t c = 0;
        if (k != 0) {
            const int64_t tid = hd.nodes[t][i] - g.off[t];
            const int p = owner_of(g, t, tid);
            const int64_t x = tid - g.bounds[t][p];
            const int64_t *ip = R.indptr[p];
            const int64_t b0 = ip[x], d = ip[x + 1] - b0;
            c = (int32_t)((k < 0 || d <= k) ? d : k);
            hd.ibase[r][i] = ((int64_t)p << 56) | b0;
            hd.ideg[r][i] = (int32_t)d;
        }
        hd.indptr[r][i] = c;
        sum += c;
    }
    sum = block_sum(sum, sh);
    if (threadIdx.x == 0) hd.partial[r * kScanBlocks + b] = sum;
}

// Phase 2: exclusive scan of the counts in place -> block indptr; nnz(h, r).
__global__ void __launch_bounds__(256) scan_kernel(const __grid_constant__ GraphDev g,
                                                   const __grid_constant__ HopDev hd)
{
    __shared__ int32_t sh[33];
    const int r = blockIdx.y, b = blockIdx.x;
    const int t = g.rel[r].dst_vt;
    const int64_t n = meta_nodes(hd.meta, hd.h)[t];
    const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
    const int64_t lo = b * chunk, hi = min(n, lo + chunk);
    int32_t s = 0;
    for (int j = threadIdx.x; j < b; j += blockDim.x) s += hd.partial[r * kScanBlocks + j];
    int32_t carry = block_sum(s, sh);
    int32_t *ip = hd.indptr[r];
    for (int64_t t0 = lo; t0 < hi; t0 += blockDim.x) {
        const int64_t i = t0 + threadIdx.x;
        const int32_t v = i < hi ? ip[i] : 0;
        int32_t tot;
        const int32_t ex = block_excl_scan(v, sh, &tot);
        if (i < hi) ip[i] = carry + ex;
        carry += tot;
    }
    if (b == gridDim.x - 1 && threadIdx.x == 0) {
        ip[n] = carry;
        meta_nnz(hd.meta, hd.h)[r] = carry;
    }
}

void launch_count(const GraphDev &g, const HopDev &hd, cudaStream_t s)
{
    count_kernel<<<dim3(kScanBlocks, g.n_rel), 256, 0, s>>>(g, hd);
}

void launch_scan(const GraphDev &g, const HopDev &hd, cudaStream_t s)
{
    scan_kernel<<<dim3(kScanBlocks, g.n_rel), 256, 0, s>>>(g, hd);
}

// ----------------------------------------------------------------------------- sampling

struct Item {
    int64_t bit_base;       // boff[s(r)] - off[s(r)]: bitmap bit of gid = bit_base + gid
    uint32_t soff;          // off[s(r)]
    int64_t ebase;          // global CSC position of this dst's first edge
    const int32_t *ix;      // src tids of this dst's in-edges
    uint32_t *src_out;      // this item's output slots
    int64_t *eid_out;
};

// Write one sampled edge and, if its source is not yet in the batch, mark it in
// the new-vertex bitmap (the first step of the hop's compaction, fused here).
__device__ __forceinline__ void mark_new(const HopDev &hd, uint32_t gid, int64_t bit_base)
{
    if (__ldg(hd.pos + gid) < 0) {
        const int64_t bit = bit_base + gid;
        const uint32_t m = 1u << (bit & 31);
        uint32_t *wp = hd.bitmap + (bit >> 5);
        if (!(*wp & m)) atomicOr(wp, m);
    }
}

__device__ __forceinline__ void emit_edge(const HopDev &hd, const Item &it, int32_t slot, int64_t j)
{
    const uint32_t gid = it.soff + (uint32_t)__ldg(it.ix + j);
    it.src_out[slot] = gid;
    it.eid_out[slot] = it.ebase + j;
    mark_new(hd, gid, it.bit_base);
}

// Four keys key32(seed, h, r, v, 4q .. 4q+3) from one Philox call.
__device__ __forceinline__ void keys4(uint32_t q, uint32_t v_lo, uint32_t v_hi, uint32_t hr, uint32_t k0,
                                      uint32_t k1, uint32_t w[4])
{
    uint32_t c0 = q, c1 = v_lo, c2 = v_hi, c3 = hr;
    philox4x32_10(c0, c1, c2, c3, k0, k1);
    w[0] = c0; w[1] = c1; w[2] = c2; w[3] = c3;
}

__device__ __forceinline__ uint32_t lanemask_lt() { return (1u << lane_id()) - 1u; }

// Generic exact selection for any k < d: binary search of the k-th smallest key
// value T (33 counting passes over the d keys), then one ascending-j emission
// pass taking key < T and the first (k - #{key < T}) offsets with key == T.
__device__ __noinline__ void select_generic(const HopDev &hd, const Item &it, int64_t d, int k, uint32_t v_lo, uint32_t v_hi, uint32_t hr,
                               uint32_t k0, uint32_t k1)
{
    const int64_t nq = (d + 3) >> 2;
    auto count_lt = [&](uint64_t x) -> int64_t {
        int64_t c = 0;
        for (int64_t q = lane_id(); q < nq; q += 32) {
            uint32_t w[4];
            keys4((uint32_t)q, v_lo, v_hi, hr, k0, k1, w);
#pragma unroll
            for (int t = 0; t < 4; ++t) c += (4 * q + t < d && (uint64_t)w[t] < x);
        }
        return warp_sum(c);
    };
    uint64_t lo = 0, hi = 1ull << 32;   // count_lt(lo) < k <= count_lt(hi)
    while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) >> 1;
        if (count_lt(mid) < k) lo = mid; else hi = mid;
    }
    const uint32_t T = (uint32_t)lo;
    const int64_t need_eq = k - count_lt(lo);
    int32_t out = 0;
    int64_t eq_seen = 0;
    for (int64_t q0 = 0; q0 < nq; q0 += 32) {
        const int64_t q = q0 + lane_id();
        uint32_t w[4] = {0, 0, 0, 0};
        if (q < nq) keys4((uint32_t)q, v_lo, v_hi, hr, k0, k1, w);
        uint32_t lt = 0, eq = 0;
#pragma unroll
        for (int t = 0; t < 4; ++t)
            if (q < nq && 4 * q + t < d) {
                lt |= (w[t] < T) << t;
                eq |= (w[t] == T) << t;
            }
        // equal keys in ascending j: rank among equal keys of this chunk
        const int ceq = __popc(eq);
        const int eq_ex = warp_incl_scan(ceq) - ceq;
        uint32_t sel = lt;
        int er = (int)(eq_seen + eq_ex);
#pragma unroll
        for (int t = 0; t < 4; ++t)
            if (eq >> t & 1) {
                if (er < need_eq) sel |= 1u << t;
                ++er;
            }
        eq_seen += __shfl_sync(0xffffffffu, eq_ex + ceq, 31);
        const int cs = __popc(sel);
        const int ex = warp_incl_scan(cs) - cs;
        int slot = out + ex;
#pragma unroll
        for (int t = 0; t < 4; ++t)
            if (sel >> t & 1) emit_edge(hd, it, slot++, 4 * q + t);
        out += __shfl_sync(0xffffffffu, ex + cs, 31);
    }
}

// Fast selection for k <= kSelMaxK: one pass over the d keys keeps the candidates
// below a threshold T (expected 2k + 32 of them) in shared memory, in ascending j;
// the k smallest composites among them are found by rank counting and emitted in
// ascending j.  Falls back to select_generic if the candidate count is < k or
// exceeds the slots (both astronomically rare; the result is identical).
__device__ void select_fast(const HopDev &hd, const Item &it, int64_t d, int k, uint32_t v_lo, uint32_t v_hi, uint32_t hr,
                            uint32_t k0, uint32_t k1, uint64_t *cand)
{
    const uint64_t E = 2ull * (uint64_t)k + 32;
    const uint64_t T = (E >= (uint64_t)d) ? (1ull << 32) : ((E << 32) / (uint64_t)d);
    const int64_t nq = (d + 3) >> 2;
    int m = 0;
    for (int64_t q0 = 0; q0 < nq; q0 += 32) {
        const int64_t q = q0 + lane_id();
        uint32_t w[4] = {0, 0, 0, 0};
        uint32_t f = 0;
        if (q < nq) {
            keys4((uint32_t)q, v_lo, v_hi, hr, k0, k1, w);
#pragma unroll
            for (int t = 0; t < 4; ++t) f |= (uint32_t)(4 * q + t < d && (uint64_t)w[t] < T) << t;
        }
        const int c = __popc(f);
        const int ex = warp_incl_scan(c) - c;
        const int tot = __shfl_sync(0xffffffffu, ex + c, 31);
        if (m + tot <= kSelCap) {
            int slot = m + ex;
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (f >> t & 1) cand[slot++] = ((uint64_t)w[t] << 32) | (uint64_t)(4 * q + t);
        }
        m += tot;
    }
    __syncwarp();
    if (m < k || m > kSelCap) {
        select_generic(hd, it, d, k, v_lo, v_hi, hr, k0, k1);
        return;
    }
    int32_t out = 0;
    for (int c0 = 0; c0 < m; c0 += 32) {
        const int c = c0 + lane_id();
        bool sel = false;
        uint64_t mine = 0;
        if (c < m) {
            mine = cand[c];
            int rank = 0;
            for (int o = 0; o < m; ++o) rank += cand[o] < mine;
            sel = rank < k;
        }
        const uint32_t b = __ballot_sync(0xffffffffu, sel);
        if (sel) emit_edge(hd, it, out + __popc(b & lanemask_lt()), (int64_t)(uint32_t)mine);
        out += __popc(b);
    }
    __syncwarp();
}

constexpr int kSampleWarps = 8;

// The items of a hop are the (relation, dst) pairs, relation-major.  A warp takes 32
// consecutive items at a time: lane l loads item l's block row (pos0, cnt) and the
// CSC row start / degree the count kernel recorded.  Items that take their whole
// neighbourhood (d <= k or k = -1; most of a power-law graph) are copied as one
// segmented copy spread over all 32 lanes; items that need a selection (d > k) are
// appended to the hop's selection queue, drained warp-per-item by select_kernel.
__global__ void __launch_bounds__(kSampleWarps * 32) sample_kernel(const __grid_constant__ GraphDev g,
                                                                   const __grid_constant__ HopDev hd)
{
    const int warp = threadIdx.x >> 5, lane = lane_id();
    const int32_t *nF = meta_nodes(hd.meta, hd.h);
    int64_t cum[EG_MAX_REL + 1];
    cum[0] = 0;
    for (int r = 0; r < g.n_rel; ++r) cum[r + 1] = cum[r] + (hd.fanout[r] != 0 ? nF[g.rel[r].dst_vt] : 0);
    const int64_t total = cum[g.n_rel];
    for (int64_t g0 = ((int64_t)blockIdx.x * kSampleWarps + warp) * 32; g0 < total;
         g0 += (int64_t)gridDim.x * kSampleWarps * 32) {
        const int64_t it = g0 + lane;
        int r = 0;
        int32_t pos0 = 0, cnt = 0, d = 0;
        int64_t ib = 0, i = 0;
        if (it < total) {
            while (it >= cum[r + 1]) ++r;
            i = it - cum[r];
            pos0 = hd.indptr[r][i];
            cnt = hd.indptr[r][i + 1] - pos0;
            if (cnt > 0) {
                ib = hd.ibase[r][i];
                d = hd.ideg[r][i];
            }
        }
        const int k = hd.fanout[r];
        const bool sel = cnt > 0 && k >= 0 && d > k;
        // ---- items that need a selection -> queue (one atomic per warp)
        const uint32_t selmask = __ballot_sync(0xffffffffu, sel);
        if (selmask) {
            uint32_t qbase = 0;
            if (lane == 0) qbase = atomicAdd((uint32_t *)(hd.meta + kMetaSel + hd.h), (uint32_t)__popc(selmask));
            qbase = __shfl_sync(0xffffffffu, qbase, 0);
            if (sel) hd.selq[qbase + __popc(selmask & lanemask_lt())] = ((uint64_t)r << 32) | (uint64_t)i;
        }
        // ---- segmented copy of the full neighbourhoods of this group
        const int32_t c = (cnt > 0 && !sel) ? cnt : 0;
        const int32_t incl = warp_incl_scan(c);
        const int32_t tot = __shfl_sync(0xffffffffu, incl, 31);
        const int32_t excl = incl - c;
        for (int32_t b = 0; b < tot; b += 32) {
            const int32_t s = b + lane;
            int L = 0;   // the lane whose item holds output slot s: last lane with excl <= s
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const int cand = L + step;
                const int32_t ex = __shfl_sync(0xffffffffu, excl, cand & 31);
                if (cand < 32 && ex <= s) L = cand;
            }
            const int32_t exL = __shfl_sync(0xffffffffu, excl, L);
            const int32_t posL = __shfl_sync(0xffffffffu, pos0, L);
            const int64_t ibL = __shfl_sync(0xffffffffu, ib, L);
            const int rL = __shfl_sync(0xffffffffu, r, L);
            if (s < tot) {
                const int p = (int)(ibL >> 56);
                const int64_t base = ibL & ((1ll << 56) - 1);
                const int32_t j = s - exL;
                const RelDev &R = g.rel[rL];
                const uint32_t gid = (uint32_t)g.off[R.src_vt] + (uint32_t)__ldg(R.indices[p] + base + j);
                hd.src[rL][posL + j] = gid;
                hd.eids[rL][posL + j] = R.edge_base[p] + base + j;
                mark_new(hd, gid, g.boff[R.src_vt] - g.off[R.src_vt]);
            }
        }
    }
}

// Selection items (d > k): one warp per item, any order (each item owns its slots).
__global__ void __launch_bounds__(kSampleWarps * 32) select_kernel(const __grid_constant__ GraphDev g,
                                                                   const __grid_constant__ HopDev hd)
{
    __shared__ uint64_t s_cand[kSampleWarps][kSelCap];
    const int warp = threadIdx.x >> 5;
    const uint32_t seed_lo = (uint32_t)hd.dyn[0], seed_hi = (uint32_t)(hd.dyn[0] >> 32);
    const int64_t n = *(const uint32_t *)(hd.meta + kMetaSel + hd.h);
    for (int64_t w = (int64_t)blockIdx.x * kSampleWarps + warp; w < n; w += (int64_t)gridDim.x * kSampleWarps) {
        const uint64_t e = hd.selq[w];
        const int r = (int)(e >> 32);
        const int64_t i = (int64_t)(e & 0xFFFFFFFFu);
        const RelDev &R = g.rel[r];
        const int32_t pos0 = hd.indptr[r][i];
        const int64_t ib = hd.ibase[r][i];
        const int64_t d = hd.ideg[r][i];
        const int64_t v = hd.nodes[R.dst_vt][i];
        const int p = (int)(ib >> 56);
        const int64_t base = ib & ((1ll << 56) - 1);
        Item itm;
        itm.bit_base = g.boff[R.src_vt] - g.off[R.src_vt];
        itm.soff = (uint32_t)g.off[R.src_vt];
        itm.ebase = R.edge_base[p] + base;
        itm.ix = R.indices[p] + base;
        itm.src_out = hd.src[r] + pos0;
        itm.eid_out = hd.eids[r] + pos0;
        const int k = hd.fanout[r];
        const uint32_t hr = ((uint32_t)hd.h << 16) | (uint32_t)r;
        if (k <= kSelMaxK)
            select_fast(hd, itm, d, k, (uint32_t)v, (uint32_t)((uint64_t)v >> 32), hr, seed_lo, seed_hi, s_cand[warp]);
        else
            select_generic(hd, itm, d, k, (uint32_t)v, (uint32_t)((uint64_t)v >> 32), hr, seed_lo, seed_hi);
    }
}

void launch_sample(const GraphDev &g, const HopDev &hd, cudaStream_t s)
{
    sample_kernel<<<kSMs * 8, kSampleWarps * 32, 0, s>>>(g, hd);
    select_kernel<<<kSMs * 4, kSampleWarps * 32, 0, s>>>(g, hd);
}

}  // namespace eg
