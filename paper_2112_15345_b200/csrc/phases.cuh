// phases.cuh -- the phases of one mini-batch as device functions over a virtual grid.
//
// Each phase distributes its work over `nb` blocks (block index `bid`), so the same
// code runs as one persistent cooperative kernel (batch.cu: grid barriers between
// phases) or as one kernel per phase (bid = blockIdx.x).
//
// Method:
//   seed split        F_0[u] = seeds of type u in caller order
//   count             c = min(d, k) (all d if k == -1 or d <= k) per (dst, r)
//   scan              block CSC indptr = exclusive prefix of c
//   sample            d <= k: the whole in-neighbourhood in CSC order; d > k: the
//                     k offsets with the smallest (key32 << 32 | j), ascending j P:284-285
//   compaction        new sources of the hop in gid order after the dst prefix,
//                     local src ids = positions in src_nodes (compact.cuh)
#pragma once
#include "common.cuh"

namespace eg {

__device__ __forceinline__ uint32_t lanemask_lt() { return (1u << lane_id()) - 1u; }

// ============================================================================ seed split

// Seeds (caller order, mixed types) -> F_0[u] (stable per type); every placed seed is a
// key of the level-0 compaction (compact.cuh, kModeSeeds: sorted member list, duplicate
// check).  Flags out-of-range seeds.  One block.
// sort: batches of at most blockDim.x seeds (one round) skip the level-0 compaction kernels:
// the seeds are sorted here by a block-wide bitonic sort of (gid << 32 | position), which
// gives the level-0 member list (mg[0], mp[0]) and its bucket counts, and a repeated gid
// is a duplicate seed.  Otherwise every placed seed is a key of the level-0 compaction.
__device__ __forceinline__ void phase_seed_split(const GraphDev &g, const HopDev &hd, const int64_t *__restrict__ slot_seeds,
                                                 bool sort)
{
    // the caller's buffer when it is device-accessible, else the slot's staged copy
    const int64_t *__restrict__ seeds = hd.dyn[2] ? (const int64_t *)hd.dyn[2] : slot_seeds;
    __shared__ int32_t wcnt[32][EG_MAX_VT];   // per warp, per type: count, then exclusive offset
    __shared__ int32_t base[EG_MAX_VT];
    // pointers hoisted into registers: HopDev lives in global memory and every store
    // below could alias it, so reading fields inside the loops would reload them
    uint32_t *const kcnt = hd.cd.kcnt;
    int32_t *const meta = hd.meta;
    const int64_t n = (int64_t)hd.dyn[1];
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5, lane = lane_id();
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
                atomicOr(meta + kMetaErr, kErrSeedRange);
            } else {
                vt = 0;
                while (gid >= g.off[vt + 1]) ++vt;
            }
        }
        // stable placement per type: ballot ranks within the warp, warp offsets per type
        int rank = 0;
        for (int u = 0; u < g.n_vt; ++u) {
            const uint32_t m = __ballot_sync(0xffffffffu, vt == u);
            if (vt == u) rank = __popc(m & lanemask_lt());
            if (lane == 0) wcnt[w][u] = __popc(m);
        }
        __syncthreads();
        if (threadIdx.x < g.n_vt) {
            const int u = threadIdx.x;
            int32_t run = base[u];
            for (int ww = 0; ww < nw; ++ww) {
                const int32_t cnt = wcnt[ww][u];
                wcnt[ww][u] = run;
                run += cnt;
            }
            base[u] = run;
        }
        __syncthreads();
        unsigned long long key = ~0ull;   // (gid << 32) | position, or none
        if (vt >= 0) {
            const int32_t p = wcnt[w][vt] + rank;
            if (p < hd.cap_nodes[vt]) {
                hd.nodes[vt][p] = gid;
                if (sort)
                    key = ((unsigned long long)gid << 32) | (uint32_t)p;
                else
                    atomicAdd(kcnt + bucket_of(g, vt, gid), 1u);
            } else {
                atomicOr(meta + kMetaErr, kErrCapacity);
            }
        }
        if (sort) {   // n <= blockDim.x: this is the only round
            __shared__ unsigned long long sk[1024];
            const int tid = threadIdx.x;
            for (int k = 2; k <= (int)blockDim.x; k <<= 1)
                for (int j = k >> 1; j > 0; j >>= 1) {
                    unsigned long long y;
                    if (j >= 32) {
                        sk[tid] = key;
                        __syncthreads();
                        y = sk[tid ^ j];
                        __syncthreads();
                    } else {
                        y = __shfl_xor_sync(0xffffffffu, key, j);
                    }
                    const bool up = (tid & k) == 0, low = (tid & j) == 0;
                    key = (low == up) ? min(key, y) : max(key, y);
                }
            sk[tid] = key;
            __syncthreads();
            if (key != ~0ull) {
                const uint32_t sg = (uint32_t)(key >> 32);
                EG_DCHECK(tid < hd.cd.cap_members);
                if (tid > 0 && (uint32_t)(sk[tid - 1] >> 32) == sg) atomicOr(meta + kMetaErr, kErrSeedDup);
                hd.cd.mg[0][tid] = sg;
                hd.cd.mp[0][tid] = (int32_t)(uint32_t)key;
                int u = 0;
                while (u + 1 < g.n_vt && (int64_t)sg >= g.off[u + 1]) ++u;
                atomicAdd(hd.cd.mcnt + bucket_of(g, u, sg), 1u);   // members of level 1's buckets
            }
        }
        __syncthreads();
    }
    if (threadIdx.x < g.n_vt)
        meta_nodes(meta, 0)[threadIdx.x] = min(base[threadIdx.x], hd.cap_nodes[threadIdx.x]);
    __syncthreads();
}

// ============================================================================ count

// Single pass per hop: tiles of kCountTile consecutive dst items of one relation, taken by
// ticket (relation-major).  Per item: c = min(d, k) (all d if k == -1 or d <= k) from the
// owner's CSC row bounds; the tile's exclusive prefix comes from a decoupled look-back over
// the relation's earlier tiles (window of 32), so the block indptr is final here and every
// item that needs sampling is queued with its output slot: full neighbourhoods to copyq,
// selections to selq (d > kTinyD from the bottom, the rest from the top), hubs as chunk
// tasks.  The last tile of a relation writes indptr[n] and nnz(h, r).
__device__ __forceinline__ unsigned long long clb_word(unsigned long long st, uint32_t v)
{
    return (st << 62) | v;
}

__device__ __forceinline__ void phase_count(const GraphDev &g, const HopDev &hd)
{
    __shared__ int32_t sh[kCountThreads / 32 + 1];
    __shared__ int32_t s_vt;
    __shared__ int32_t s_excl;
    const int32_t *nF = meta_nodes(hd.meta, hd.h);
    int32_t cumT[EG_MAX_REL + 1];
    cumT[0] = 0;
    for (int r = 0; r < g.n_rel; ++r) cumT[r + 1] = cumT[r] + (nF[g.rel[r].dst_vt] + kCountTile - 1) / kCountTile;
    const int lane = lane_id();
    uint32_t *const selc = (uint32_t *)(hd.meta + kMetaSel + hd.h);
    uint32_t *const tinyc = (uint32_t *)(hd.meta + kMetaTiny + hd.h);
    uint32_t *const copyc = (uint32_t *)(hd.meta + kMetaCopy + hd.h);
    uint32_t *const tiny16c = (uint32_t *)(hd.meta + kMetaTiny16 + hd.h);
    QEntry *const selq = hd.selq;
    QEntry *const tinyq16 = hd.tinyq16;
    QEntry *const copyq = hd.copyq;
    volatile unsigned long long *const clb = hd.clb;
    for (;;) {
        if (threadIdx.x == 0) s_vt = (int32_t)atomicAdd((uint32_t *)(hd.meta + kMetaCntTicket + hd.h), 1u);
        __syncthreads();
        const int32_t vt = s_vt;
        if (vt >= cumT[g.n_rel]) break;
        int r = 0;
        while (vt >= cumT[r + 1]) ++r;
        const int32_t tile = vt - cumT[r];
        const RelDev &R = g.rel[r];
        const int t = R.dst_vt;
        const int k = hd.fanout[r];
        const int64_t n = nF[t];
        const int64_t i0 = (int64_t)tile * kCountTile + (int64_t)threadIdx.x * kCountItems;
        const int64_t *const nodes = hd.nodes[t];
        int32_t c[kCountItems], d[kCountItems], v[kCountItems];
        int64_t ib[kCountItems];
        int64_t b0[kCountItems];
        const int64_t *ip[kCountItems];
#pragma unroll
        for (int q = 0; q < kCountItems; ++q) {
            c[q] = d[q] = v[q] = 0;
            ib[q] = 0;
            ip[q] = nullptr;
            const int64_t i = i0 + q;
            if (i < n && k != 0) {
                const int64_t gid = nodes[i];
                const int64_t tid = gid - g.off[t];
                const int p = owner_of(g, t, tid);
                const int64_t x = tid - g.bounds[t][p];
                ip[q] = R.indptr[p] + x;
                v[q] = (int32_t)gid;
                ib[q] = (int64_t)p << 56;
            }
        }
#pragma unroll
        for (int q = 0; q < kCountItems; ++q)
            if (ip[q]) {
                b0[q] = ip[q][0];
                d[q] = (int32_t)(ip[q][1] - b0[q]);
            }
        int32_t sum = 0;
#pragma unroll
        for (int q = 0; q < kCountItems; ++q)
            if (ip[q]) {
                ib[q] |= b0[q];
                c[q] = (k < 0 || d[q] <= k) ? d[q] : k;
                sum += c[q];
            }
        int32_t ttot;
        const int32_t texcl = block_excl_scan(sum, sh, &ttot);
        // decoupled look-back over the relation's earlier tiles (warp 0)
        if (threadIdx.x < 32) {
            if (lane == 0) clb[vt] = clb_word(tile == 0 ? 2 : 1, (uint32_t)ttot);
            uint32_t excl = 0;
            for (int32_t top = vt - 1; top >= cumT[r]; top -= 32) {
                const int32_t p = top - lane;
                unsigned long long w = 0;
                if (p >= cumT[r]) {
                    SpinGuard sg;
                    do {
                        w = clb[p];
                        sg.step();
                    } while ((w >> 62) == 0);
                }
                const uint32_t incl = __ballot_sync(0xffffffffu, p >= cumT[r] && (w >> 62) == 2);
                const int lim = incl ? __ffs(incl) - 1 : 31;
                excl += warp_sum(p >= cumT[r] && lane <= lim ? (uint32_t)w : 0u);
                if (incl) break;
            }
            if (lane == 0) {
                if (tile > 0) {
                    __threadfence();
                    clb[vt] = clb_word(2, excl + (uint32_t)ttot);
                }
                s_excl = (int32_t)excl;
            }
        }
        __syncthreads();
        int32_t pos = s_excl + texcl;
        int32_t *const bip = hd.indptr[r];
        // classify the lane's items; queue slots are reserved once per warp for all of them
        // (three independent atomics instead of one dependent round trip per item and queue)
        QEntry e[kCountItems];
        uint32_t mc[kCountItems], ms[kCountItems], mt[kCountItems], m16[kCountItems];
        uint32_t nc = 0, ns = 0, ntn = 0, n16 = 0;
#pragma unroll
        for (int q = 0; q < kCountItems; ++q) {
            const int64_t i = i0 + q;
            const bool ok = i < n;
            e[q].ib = ib[q];
            e[q].pos0 = pos;
            e[q].d = d[q];
            e[q].v = v[q];
            e[q].r = r;
            if (ok) bip[i] = pos;
            const bool all = ok && c[q] > 0 && c[q] == d[q];
            bool sel = ok && c[q] > 0 && c[q] < d[q];
            // heavy items (d > kHeavyD): split into tasks of kHeavyChunk keys for several warps
            if (sel && k <= kHeavyMaxK && d[q] > kHeavyD) {
                const uint32_t nch = (uint32_t)((d[q] + kHeavyChunk - 1) / kHeavyChunk);
                const uint32_t hs = atomicAdd((uint32_t *)(hd.meta + kMetaHeavy + hd.h), 1u);
                if (hs < (uint32_t)hd.max_heavy) {
                    const uint32_t t0 = atomicAdd((uint32_t *)(hd.meta + kMetaHeavyQ + hd.h), nch);
                    if (t0 + nch <= (uint32_t)hd.max_heavy_tasks) {
                        hd.heavy_items[hs] = e[q];
                        hd.heavy_cnt[hs] = 0;
                        hd.heavy_done[hs] = 0;
                        for (uint32_t ch = 0; ch < nch; ++ch) hd.heavyq[t0 + ch] = (hs << 16) | ch;
                        sel = false;
                    } else {   // task list full: mark the reserved entries void, item goes to the normal queue
                        for (uint32_t ch = 0; ch < nch && t0 + ch < (uint32_t)hd.max_heavy_tasks; ++ch)
                            hd.heavyq[t0 + ch] = 0xFFFFFFFFu;
                    }
                }
            }
            const bool tiny16 = sel && d[q] <= kTinyD16;             // 4 lanes per item (phase_tiny)
            const bool tiny = sel && !tiny16 && d[q] <= kTinyD;     // 8 lanes per item
            mc[q] = __ballot_sync(0xffffffffu, all);
            ms[q] = __ballot_sync(0xffffffffu, sel && !tiny && !tiny16);
            mt[q] = __ballot_sync(0xffffffffu, tiny);
            m16[q] = __ballot_sync(0xffffffffu, tiny16);
            nc += __popc(mc[q]);
            ns += __popc(ms[q]);
            ntn += __popc(mt[q]);
            n16 += __popc(m16[q]);
            pos += c[q];
        }
        uint32_t oc = 0, os = 0, ot = 0, o16 = 0;
        if (lane == 0) {
            if (nc) oc = atomicAdd(copyc, nc);
            if (ns) os = atomicAdd(selc, ns);
            if (ntn) ot = atomicAdd(tinyc, ntn);
            if (n16) o16 = atomicAdd(tiny16c, n16);
        }
        oc = __shfl_sync(0xffffffffu, oc, 0);
        os = __shfl_sync(0xffffffffu, os, 0);
        ot = __shfl_sync(0xffffffffu, ot, 0);
        o16 = __shfl_sync(0xffffffffu, o16, 0);
        const uint32_t lt = lanemask_lt();
        EG_DCHECK(oc + nc <= (uint32_t)hd.selq_cap && os + ns + ot + ntn <= (uint32_t)hd.selq_cap &&
                  o16 + n16 <= (uint32_t)hd.selq_cap);
#pragma unroll
        for (int q = 0; q < kCountItems; ++q) {
            if (mc[q] >> lane & 1) copyq[oc + __popc(mc[q] & lt)] = e[q];
            if (ms[q] >> lane & 1) selq[os + __popc(ms[q] & lt)] = e[q];
            if (mt[q] >> lane & 1) selq[hd.selq_cap - 1 - (ot + __popc(mt[q] & lt))] = e[q];
            if (m16[q] >> lane & 1) tinyq16[hd.selq_cap - 1 - (o16 + __popc(m16[q] & lt))] = e[q];
            oc += __popc(mc[q]);
            os += __popc(ms[q]);
            ot += __popc(mt[q]);
            o16 += __popc(m16[q]);
        }
        if (threadIdx.x == 0 && tile == cumT[r + 1] - cumT[r] - 1) {   // the relation's last tile
            const int32_t tot = s_excl + ttot;
            bip[n] = tot;
            meta_nnz(hd.meta, hd.h)[r] = tot;
        }
        __syncthreads();   // s_vt / s_excl reuse
    }
    // relations whose dst frontier is empty: indptr = [0], nnz = 0
    if (blockIdx.x == 0 && threadIdx.x < g.n_rel && nF[g.rel[threadIdx.x].dst_vt] == 0) {
        hd.indptr[threadIdx.x][0] = 0;
        meta_nnz(hd.meta, hd.h)[threadIdx.x] = 0;
    }
}

// ============================================================================ sampling

struct Item {
    uint32_t *kcnt;         // the batch's keys per compaction bucket
    int32_t bbase;          // first bucket of s(r)
    int32_t bshift;         // log2 gids per bucket
    uint32_t soff;          // off[s(r)]
    int64_t ebase;          // global CSC position of this dst's first edge
    const int32_t *ix;      // src tids of this dst's in-edges
    uint32_t *src_out;      // this item's output slots
    int64_t *eid_out;
};

// Count the source as a key of the hop's compaction (its first step, fused into sampling):
// fire-and-forget RED.ADD on the batch's bucket counts (L2-resident, sized by the graph's
// bucket count, ~2^16).
__device__ __forceinline__ void mark_src(const Item &it, uint32_t gid)
{
    atomicAdd(it.kcnt + it.bbase + ((gid - it.soff) >> it.bshift), 1u);   // result unused: RED
}

__device__ __forceinline__ void item_common(const GraphDev &g, const HopDev &hd, const RelDev &R, Item &it)
{
    it.kcnt = hd.cd.kcnt;
    it.bbase = (int32_t)g.bbase[R.src_vt];
    it.bshift = g.bshift;
    it.soff = (uint32_t)g.off[R.src_vt];
}

__device__ __forceinline__ void emit_edge(const HopDev &, const Item &it, int32_t slot, int64_t j)
{
    const uint32_t gid = it.soff + (uint32_t)__ldg(it.ix + j);
    it.src_out[slot] = gid;
    it.eid_out[slot] = it.ebase + j;
    mark_src(it, gid);
}

// Up to four selected edges of one lane: the source-id loads are issued together before
// any store (the stores could alias them as far as the compiler knows, so the per-edge
// form serialised load -> store chains; measured, ncu: the emission was the top stall
// of the tiny-item kernel).  Edge t (bit t of sel) has offset j[t] and output slot
// slot[t].
__device__ __forceinline__ void emit_edges4(const Item &it, uint32_t sel, const int64_t j[4], const int32_t slot[4])
{
    uint32_t ix[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) ix[t] = (sel >> t & 1) ? __ldg(it.ix + j[t]) : 0u;
#pragma unroll
    for (int t = 0; t < 4; ++t)
        if (sel >> t & 1) {
            const uint32_t gid = it.soff + ix[t];
            it.src_out[slot[t]] = gid;
            it.eid_out[slot[t]] = it.ebase + j[t];
            mark_src(it, gid);
        }
}

// Consecutive offsets j0 .. j0+3 (bits of sel), emitted in ascending order from `slot`.
__device__ __forceinline__ void emit_run4(const Item &it, uint32_t sel, int32_t slot, int64_t j0)
{
    int64_t j[4];
    int32_t s[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        j[t] = j0 + t;
        s[t] = slot;
        slot += (sel >> t) & 1;
    }
    emit_edges4(it, sel, j, s);
}

// Four keys key32(seed, h, r, v, 4q .. 4q+3) from one Philox call.
__device__ __forceinline__ void keys4(uint32_t q, uint32_t v_lo, uint32_t v_hi, uint32_t hr, uint32_t k0,
                                      uint32_t k1, uint32_t w[4])
{
    uint32_t c0 = q, c1 = v_lo, c2 = v_hi, c3 = hr;
    philox4x32_10(c0, c1, c2, c3, k0, k1);
    w[0] = c0; w[1] = c1; w[2] = c2; w[3] = c3;
}

// Radix select, two bits per step.  With bits [s, 32) of the threshold key decided (P),
// a key "matches" when its bits [s, 32) equal P's; radix2_count packs, for this thread's
// keys, how many matching keys have digit (key >> (s-2)) & 3 equal to 0, 1, 2, 3 (bits
// 0-7, 8-15, 16-23, 24-31); sums of these over the item (<= 128 keys) do not overflow a
// field.  radix2_decide takes the summed counts and either finishes (every matching key
// is selected: their number == krem) or fixes the next digit.
__device__ __forceinline__ uint32_t radix2_count(uint32_t w, bool valid, uint32_t P, int s)
{
    // (w ^ P) >> s with the shift clamped at 32 (s == 32: nothing decided, all match)
    const bool match = valid && __funnelshift_rc(w ^ P, 0u, (uint32_t)s) == 0u;
    return match ? 1u << (((w >> (s - 2)) & 3u) << 3) : 0u;
}

__device__ __forceinline__ bool radix2_decide(uint32_t x, int &krem, uint32_t &P, int &s)
{
    const int n0 = (int)(x & 0xFFu), n1 = (int)((x >> 8) & 0xFFu), n2 = (int)((x >> 16) & 0xFFu);
    const int cm = n0 + n1 + n2 + (int)(x >> 24);
    if (cm == krem) return true;
    uint32_t dg;
    if (krem <= n0) {
        dg = 0;
    } else if (krem <= n0 + n1) {
        dg = 1;
        krem -= n0;
    } else if (krem <= n0 + n1 + n2) {
        dg = 2;
        krem -= n0 + n1;
    } else {
        dg = 3;
        krem -= n0 + n1 + n2;
    }
    s -= 2;
    P |= dg << s;
    return s == 0;
}

// Generic exact selection for any k < d: binary search of the k-th smallest key
// value T (33 counting passes over the d keys), then one ascending-j emission
// pass taking key < T and the first (k - #{key < T}) offsets with key == T.
__device__ __noinline__ void select_generic(const HopDev &hd, const Item &it, int64_t d, int k, uint32_t v_lo,
                                            uint32_t v_hi, uint32_t hr, uint32_t k0, uint32_t k1)
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

// Selection for d <= 128: every key fits in registers (4 consecutive offsets per lane,
// one Philox call), so the k-th smallest key is found by a radix select over them
// directly, ties broken by ascending j, and the selected offsets are emitted in
// ascending j (j = 4 lane + t).
__device__ __forceinline__ void select_small(const HopDev &hd, const Item &it, int64_t d, int k, uint32_t v_lo, uint32_t v_hi,
                             uint32_t hr, uint32_t k0, uint32_t k1)
{
    const int lane = lane_id();
    uint32_t w[4] = {0, 0, 0, 0};
    uint32_t vm = 0;                                  // valid offsets of this lane
    if (4 * lane < d) {
        keys4((uint32_t)lane, v_lo, v_hi, hr, k0, k1, w);
#pragma unroll
        for (int t = 0; t < 4; ++t) vm |= (uint32_t)(4 * lane + t < d) << t;
    }
    uint32_t P = 0;
    int krem = k, s = 32;
    while (true) {
        uint32_t x = 0;
#pragma unroll
        for (int t = 0; t < 4; ++t) x += radix2_count(w[t], vm >> t & 1, P, s);
        if (radix2_decide(__reduce_add_sync(0xffffffffu, x), krem, P, s)) break;
    }
    uint32_t ltm = 0, eqm = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const uint32_t hi = s == 32 ? 0u : (w[t] >> s), ph = s == 32 ? 0u : (P >> s);
        ltm |= (uint32_t)((vm >> t & 1) && hi < ph) << t;
        eqm |= (uint32_t)((vm >> t & 1) && hi == ph) << t;
    }
    const int ce = __popc(eqm);
    int er = warp_incl_scan(ce) - ce;                 // equal keys before this lane (ascending j)
    uint32_t sel = ltm;
#pragma unroll
    for (int t = 0; t < 4; ++t)
        if (eqm >> t & 1) {
            if (er < krem) sel |= 1u << t;
            ++er;
        }
    const int cs = __popc(sel);
    emit_run4(it, sel, warp_incl_scan(cs) - cs, 4 * lane);
}

// Fast selection for k <= kSelMaxK: one pass over the d keys keeps the candidates
// below a threshold T (expected 2k + 32 of them) in shared memory, in ascending j;
// the k smallest composites among them are found by a register radix select (m <= 128)
// or rank counting, and emitted in ascending j.  Falls back to select_generic if the candidate count is < k or
// exceeds the slots (both astronomically rare; the result is identical).
__device__ __forceinline__ void select_fast(const HopDev &hd, const Item &it, int64_t d, int k, uint32_t v_lo, uint32_t v_hi,
                            uint32_t hr, uint32_t k0, uint32_t k1, uint64_t *cand)
{
    // any threshold gives the same result (the selection below is exact; too few or too
    // many candidates fall back to select_generic), so T may be approximate: float math
    const uint64_t E = 2ull * (uint64_t)k + 32;
    const uint64_t T = (E >= (uint64_t)d) ? (1ull << 32)
                                          : (uint64_t)(__fdividef((float)E, (float)d) * 4294967296.0f);
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
    if (m <= 128) {
        // radix select of the k-th smallest key among the m candidates, held 4 per lane
        // (slot c = lane + 32 i); one warp reduction per two bits, early exit once every
        // candidate that still matches the decided bits is selected.
        uint32_t key[4];
        bool val[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int c = lane_id() + 32 * i;
            val[i] = c < m;
            key[i] = val[i] ? (uint32_t)(cand[c] >> 32) : 0u;
        }
        uint32_t P = 0;          // decided high bits of the threshold key
        int krem = k;            // selections still to make among keys matching P
        int s = 32;              // bits [s, 32) are decided
        while (true) {   // two bits per step; early exit once every matching key is selected
            uint32_t x = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) x += radix2_count(key[i], val[i], P, s);
            if (radix2_decide(__reduce_add_sync(0xffffffffu, x), krem, P, s)) break;
        }
        // selected: key below P on the decided bits, or matching them and among the first
        // krem such candidates in slot (= ascending j) order
        int eq_seen = 0;
        uint32_t selm = 0;
        int64_t jj[4];
        int32_t ss[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int c = lane_id() + 32 * i;
            const uint32_t hi = s == 32 ? 0u : (key[i] >> s), ph = s == 32 ? 0u : (P >> s);
            const bool lt = val[i] && hi < ph;
            const bool eq = val[i] && hi == ph;
            const uint32_t beq = __ballot_sync(0xffffffffu, eq);
            const bool sel = lt || (eq && eq_seen + __popc(beq & lanemask_lt()) < krem);
            eq_seen += __popc(beq);
            const uint32_t bs = __ballot_sync(0xffffffffu, sel);
            selm |= (uint32_t)sel << i;
            jj[i] = sel ? (int64_t)(uint32_t)cand[c] : 0;
            ss[i] = out + __popc(bs & lanemask_lt());
            out += __popc(bs);
        }
        emit_edges4(it, selm, jj, ss);
        __syncwarp();
        return;
    }
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

// One chunk of a heavy item (d > kHeavyD): keys of offsets [c * kHeavyChunk, ...) below
// the item's threshold go to the item's candidate buffer; the warp that finishes the
// item's last chunk selects the k smallest composites and emits them in ascending j.
__device__ __forceinline__ void heavy_task(const GraphDev &g, const HopDev &hd, uint32_t task, uint32_t seed_lo, uint32_t seed_hi,
                           uint64_t *cand)
{
    const int lane = lane_id();
    const uint32_t hs = task >> 16, c = task & 0xFFFFu;
    const QEntry e = hd.heavy_items[hs];
    const int r = e.r;
    const RelDev &R = g.rel[r];
    const int64_t ib = e.ib;
    const int64_t d = e.d;
    const int64_t v = e.v;
    const int k = hd.fanout[r];
    const uint32_t hr = ((uint32_t)hd.h << 16) | (uint32_t)r;
    const uint32_t v_lo = (uint32_t)v, v_hi = (uint32_t)((uint64_t)v >> 32);
    const uint64_t E = 2ull * (uint64_t)k + 32;
    const uint64_t T = (uint64_t)(__fdividef((float)E, (float)d) * 4294967296.0f);   // identical for every chunk
    uint32_t *cnt = hd.heavy_cnt + hs;
    uint64_t *buf = hd.heavy_cand + (int64_t)hs * kHeavyCap;
    const int64_t q_lo = (int64_t)c * (kHeavyChunk / 4), q_hi = min((d + 3) >> 2, q_lo + kHeavyChunk / 4);
    for (int64_t q0 = q_lo; q0 < q_hi; q0 += 32) {
        const int64_t q = q0 + lane;
        uint32_t w[4] = {0, 0, 0, 0};
        uint32_t f = 0;
        if (q < q_hi) {
            keys4((uint32_t)q, v_lo, v_hi, hr, seed_lo, seed_hi, w);
#pragma unroll
            for (int t = 0; t < 4; ++t) f |= (uint32_t)(4 * q + t < d && (uint64_t)w[t] < T) << t;
        }
        const int cf = __popc(f);
        const int ex = warp_incl_scan(cf) - cf;
        const int tot = __shfl_sync(0xffffffffu, ex + cf, 31);
        if (tot) {
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(cnt, (uint32_t)tot);
            base = __shfl_sync(0xffffffffu, base, 0) + ex;
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (f >> t & 1) {
                    if (base < (uint32_t)kHeavyCap) buf[base] = ((uint64_t)w[t] << 32) | (uint64_t)(4 * q + t);
                    ++base;
                }
        }
    }
    __threadfence();
    uint32_t done = 0;
    const uint32_t nch = (uint32_t)((d + kHeavyChunk - 1) / kHeavyChunk);
    if (lane == 0) done = atomicAdd(hd.heavy_done + hs, 1u);
    done = __shfl_sync(0xffffffffu, done, 0);
    if (done != nch - 1) return;
    // ---- last chunk: finalize the item
    __threadfence();
    const int32_t pos0 = e.pos0;
    const int p = (int)(ib >> 56);
    const int64_t base0 = ib & ((1ll << 56) - 1);
    Item itm;
    item_common(g, hd, R, itm);
    itm.ebase = R.edge_base[p] + base0;
    itm.ix = R.indices[p] + base0;
    itm.src_out = hd.src[r] + pos0;
    itm.eid_out = hd.eids[r] + pos0;
    const int m = (int)*(volatile uint32_t *)cnt;
    if (m < k || m > kHeavyCap) {   // astronomically rare: exact recomputation over all d keys
        select_generic(hd, itm, d, k, v_lo, v_hi, hr, seed_lo, seed_hi);
        return;
    }
    for (int slot = lane; slot < m; slot += 32) cand[slot] = __ldcg(buf + slot);
    __syncwarp();
    // selected flags of this lane's slots (slot = lane + 32 t): the k smallest composites
    uint32_t selm = 0;
    bool done_sel = false;
    if (m <= 128) {
        // radix select of the k-th smallest key over registers (as in select_small)
        uint32_t key[4];
        bool val[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int slot = lane + 32 * t;
            val[t] = slot < m;
            key[t] = val[t] ? (uint32_t)(cand[slot] >> 32) : 0u;
        }
        uint32_t P = 0;
        int krem = k, s = 32;
        while (true) {
            uint32_t x = 0;
#pragma unroll
            for (int t = 0; t < 4; ++t) x += radix2_count(key[t], val[t], P, s);
            if (radix2_decide(__reduce_add_sync(0xffffffffu, x), krem, P, s)) break;
        }
        uint32_t neq = 0;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const uint32_t hi = s == 32 ? 0u : (key[t] >> s), ph = s == 32 ? 0u : (P >> s);
            const bool lt = val[t] && hi < ph, eq = val[t] && hi == ph;
            neq += eq;
            if (lt || eq) selm |= 1u << t;
        }
        neq = __reduce_add_sync(0xffffffffu, neq);
        done_sel = (int)neq == krem;   // else a key tie straddles the boundary: composite ranks below
    }
    if (!done_sel) {
        selm = 0;
        for (int t = 0; lane + 32 * t < m; ++t) {
            const uint64_t mine = cand[lane + 32 * t];
            int rank = 0;
            for (int o = 0; o < m; ++o) rank += cand[o] < mine;   // composites are unique
            if (rank < k) selm |= 1u << t;
        }
    }
    // emit the k selected offsets in ascending j: rank among the selected by j
    __syncwarp();
    uint32_t *sel_j = reinterpret_cast<uint32_t *>(buf);   // the item's buffer is free now
    const int cs = __popc(selm);
    int w0 = warp_incl_scan(cs) - cs;
    for (int t = 0; t < 16; ++t)
        if (selm >> t & 1) sel_j[w0++] = (uint32_t)cand[lane + 32 * t];
    __threadfence_block();
    __syncwarp();
    for (int t = 0; t < 16; ++t)
        if (selm >> t & 1) {
            const uint32_t j = (uint32_t)cand[lane + 32 * t];
            int rank = 0;
            for (int o = 0; o < k; ++o) rank += ((volatile uint32_t *)sel_j)[o] < j;
            emit_edge(hd, itm, rank, (int64_t)j);
        }
    __syncwarp();
}

// Sampling of one hop, part 1: the selection items (d > k, queued by phase_count):
// heavy items as chunk tasks first (largest work first), then one warp per item;
// both fetched dynamically.  cand: kSelCap slots of this warp in shared memory.
__device__ __forceinline__ void phase_select(const GraphDev &g, const HopDev &hd, int bid, int nb, uint64_t *cand)
{
    const int lane = lane_id();
    const uint32_t seed_lo = (uint32_t)hd.dyn[0], seed_hi = (uint32_t)(hd.dyn[0] >> 32);
    const QEntry *const selq = hd.selq;
    (void)bid;
    // ---- heavy chunk tasks
    const uint32_t ntask = min(*(const volatile uint32_t *)(hd.meta + kMetaHeavyQ + hd.h), (uint32_t)hd.max_heavy_tasks);
    uint32_t *hnext = (uint32_t *)(hd.meta + kMetaHeavyNext + hd.h);
    for (;;) {
        uint32_t t = 0;
        if (lane == 0) t = atomicAdd(hnext, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= ntask) break;
        const uint32_t task = hd.heavyq[t];
        if (task != 0xFFFFFFFFu) heavy_task(g, hd, task, seed_lo, seed_hi, cand);
    }
    // ---- selections (d > k): warp per item, fetched kGrab at a time (lane q < kGrab
    // loads item q's data, so the fetch chain costs one round per kGrab items)
    // (kGrab = 1 when there are few items per warp: load balance first)
    const uint32_t nsel = *(const volatile uint32_t *)(hd.meta + kMetaSel + hd.h);
    const int kGrab = nsel >= 16u * (uint32_t)nb * (blockDim.x >> 5) ? 4 : 1;
    uint32_t *snext = (uint32_t *)(hd.meta + kMetaSelNext + hd.h);
    for (;;) {
        uint32_t w0 = 0;
        if (lane == 0) w0 = atomicAdd(snext, (uint32_t)kGrab);
        w0 = __shfl_sync(0xffffffffu, w0, 0);
        if (w0 >= nsel) break;
        uint32_t my_r = 0;
        int32_t my_pos0 = 0, my_d = 0;
        int64_t my_ib = 0, my_v = 0;
        if (lane < kGrab && w0 + lane < nsel) {
            const QEntry e = selq[w0 + lane];
            my_r = (uint32_t)e.r;
            my_pos0 = e.pos0;
            my_ib = e.ib;
            my_d = e.d;
            my_v = e.v;
        }
        const int cnt = (int)min((uint32_t)kGrab, nsel - w0);
        for (int q = 0; q < cnt; ++q) {
            const int r = (int)__shfl_sync(0xffffffffu, my_r, q);
            const int32_t pos0 = __shfl_sync(0xffffffffu, my_pos0, q);
            const int64_t ib = __shfl_sync(0xffffffffu, my_ib, q);
            const int64_t d = __shfl_sync(0xffffffffu, my_d, q);
            const int64_t v = __shfl_sync(0xffffffffu, my_v, q);
            const RelDev &R = g.rel[r];
            const int p = (int)(ib >> 56);
            const int64_t base = ib & ((1ll << 56) - 1);
            Item itm;
            item_common(g, hd, R, itm);
            itm.ebase = R.edge_base[p] + base;
            itm.ix = R.indices[p] + base;
            itm.src_out = hd.src[r] + pos0;
            itm.eid_out = hd.eids[r] + pos0;
            const int k = hd.fanout[r];
            const uint32_t hr = ((uint32_t)hd.h << 16) | (uint32_t)r;
            if (d <= 128)
                select_small(hd, itm, d, k, (uint32_t)v, (uint32_t)((uint64_t)v >> 32), hr, seed_lo, seed_hi);
            else if (k <= kSelMaxK)
                select_fast(hd, itm, d, k, (uint32_t)v, (uint32_t)((uint64_t)v >> 32), hr, seed_lo, seed_hi, cand);
            else
                select_generic(hd, itm, d, k, (uint32_t)v, (uint32_t)((uint64_t)v >> 32), hr, seed_lo, seed_hi);
        }
    }
}

// Selections of tiny items (k < d <= kTinyD = 64): 8 lanes per item, 4 items per warp;
// lane sl of an item holds the keys of offsets 4 sl .. 4 sl + 3 (one Philox call) and,
// when d > 32, of 32 + 4 sl .. 32 + 4 sl + 3 (a second call).  The same register radix
// select as select_small, with the sums taken over the 8 lanes of the item; all groups
// step together (finished groups idle).  Tiny items cost about the same, so they are
// strided statically over the warps, and the queue entry and item data of the next round
// are loaded while this round computes.  (Measured: items with 32 < d <= 64 took a whole
// warp each in select_small, with 3/4 of its 128 key slots empty.)
struct TinyItem {
    uint32_t r;
    int32_t pos0, d;
    int64_t ib, v;
};

__device__ __forceinline__ void tiny_load(const QEntry *e, bool ok, TinyItem &t)
{
    t.r = 0;
    t.pos0 = 0;
    t.d = 0;
    t.ib = 0;
    t.v = 0;
    if (ok) {
        const QEntry x = *e;
        t.r = (uint32_t)x.r;
        t.pos0 = x.pos0;
        t.ib = x.ib;
        t.d = x.d;
        t.v = x.v;
    }
}

// G lanes per item (G = 8: d <= 64, two key words per lane when d > 32; G = 4: d <= 16),
// 32 / G items per warp, static stride over the queue (item q at top[-q]).
template <int G>
__device__ __forceinline__ void tiny_items(const GraphDev &g, const HopDev &hd, const QEntry *top, int64_t ntiny,
                                           int bid, int nb)
{
    constexpr int IPW = 32 / G;   // items per warp
    const int lane = lane_id(), gi = lane / G, sl = lane % G;
    const uint32_t seed_lo = (uint32_t)hd.dyn[0], seed_hi = (uint32_t)(hd.dyn[0] >> 32);
    const int64_t nw = (int64_t)nb * (blockDim.x >> 5);
    int64_t q = ((int64_t)bid * (blockDim.x >> 5) + (threadIdx.x >> 5)) * IPW + gi;
    if (q - gi >= ntiny) return;   // warp-uniform
    TinyItem cur;
    tiny_load(top - q, q < ntiny, cur);
    const int64_t step = nw * IPW;
    // exclusive scan / total over the G lanes of the item
    auto group_excl = [&](int x, int &tot) {
        int y = x;
#pragma unroll
        for (int o = 1; o < G; o <<= 1) {
            const int z = __shfl_up_sync(0xffffffffu, y, o, G);
            if (sl >= o) y += z;
        }
        tot = __shfl_sync(0xffffffffu, y, G - 1, G);
        return y - x;
    };
    for (; q - gi < ntiny; q += step) {
        const bool act = q < ntiny;
        TinyItem nxt;
        tiny_load(top - (q + step), q + step < ntiny, nxt);   // next round's item in flight
        Item itm;
        int k = 0;
        const int32_t d = cur.d;
        uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0}, vm = 0;   // bit t < 4: j = 4 sl + t; t >= 4: j = 4 G + 4 sl + t - 4
        if (act) {
            const int r = (int)cur.r;
            const RelDev &R = g.rel[r];
            const int p = (int)(cur.ib >> 56);
            const int64_t base = cur.ib & ((1ll << 56) - 1);
            item_common(g, hd, R, itm);
            itm.ebase = R.edge_base[p] + base;
            itm.ix = R.indices[p] + base;
            itm.src_out = hd.src[r] + cur.pos0;
            itm.eid_out = hd.eids[r] + cur.pos0;
            k = hd.fanout[r];
            const uint32_t vlo = (uint32_t)cur.v, vhi = (uint32_t)((uint64_t)cur.v >> 32);
            const uint32_t hr = ((uint32_t)hd.h << 16) | (uint32_t)r;
            if (4 * sl < d) {
                keys4((uint32_t)sl, vlo, vhi, hr, seed_lo, seed_hi, w);
#pragma unroll
                for (int t = 0; t < 4; ++t) vm |= (uint32_t)(4 * sl + t < d) << t;
            }
            if (G == 8 && 32 + 4 * sl < d) {
                keys4((uint32_t)(8 + sl), vlo, vhi, hr, seed_lo, seed_hi, w + 4);
#pragma unroll
                for (int t = 0; t < 4; ++t) vm |= (uint32_t)(32 + 4 * sl + t < d) << (4 + t);
            }
        }
        const bool upper = G == 8 && __any_sync(0xffffffffu, (vm >> 4) != 0);   // warp-uniform: any d > 32
        uint32_t P = 0;
        int krem = k, s = 32;
        bool done = !act;
        while (__any_sync(0xffffffffu, !done)) {   // two bits per step
            uint32_t pk = 0;
            if (!done) {
#pragma unroll
                for (int t = 0; t < 4; ++t) pk += radix2_count(w[t], vm >> t & 1, P, s);
                if (upper) {
#pragma unroll
                    for (int t = 4; t < 8; ++t) pk += radix2_count(w[t], vm >> t & 1, P, s);
                }
            }
#pragma unroll
            for (int o = 1; o < G; o <<= 1) pk += __shfl_xor_sync(0xffffffffu, pk, o);
            if (!done) done = radix2_decide(pk, krem, P, s);
        }
        uint32_t ltm = 0, eqm = 0;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const uint32_t hi = s == 32 ? 0u : (w[t] >> s), ph = s == 32 ? 0u : (P >> s);
            ltm |= (uint32_t)((vm >> t & 1) && hi < ph) << t;
            eqm |= (uint32_t)((vm >> t & 1) && hi == ph) << t;
        }
        // ascending j: the lower halves of the item's lanes (j < 4 G), then the upper halves
        int te0, te1 = 0, tc0, tc1;
        int er0 = group_excl(__popc(eqm & 0xFu), te0);
        int er1 = G == 8 ? te0 + group_excl(__popc(eqm >> 4), te1) : 0;
        uint32_t sel = ltm;
#pragma unroll
        for (int t = 0; t < 4; ++t)
            if (eqm >> t & 1) {
                if (er0 < krem) sel |= 1u << t;
                ++er0;
            }
        if (G == 8) {
#pragma unroll
            for (int t = 4; t < 8; ++t)
                if (eqm >> t & 1) {
                    if (er1 < krem) sel |= 1u << t;
                    ++er1;
                }
        }
        const int slot0 = group_excl(__popc(sel & 0xFu), tc0);
        const int slot1 = G == 8 ? tc0 + group_excl(__popc(sel >> 4), tc1) : 0;
        if (act) {
            emit_run4(itm, sel & 0xFu, slot0, 4 * sl);
            if (G == 8 && (sel >> 4)) emit_run4(itm, sel >> 4, slot1, 32 + 4 * sl);
        }
        cur = nxt;
    }
}

// Selections of tiny items: k < d <= kTinyD16 with 4 lanes per item (their own queue), the
// rest of k < d <= kTinyD with 8 lanes (the top of the selection queue).
__device__ __forceinline__ void phase_tiny(const GraphDev &g, const HopDev &hd, int bid, int nb)
{
    static_assert(kTinyD == 64 && kTinyD16 == 16, "8 lanes x (4 + 4) keys, 4 lanes x 4 keys");
    const int64_t n16 = *(const volatile uint32_t *)(hd.meta + kMetaTiny16 + hd.h);
    tiny_items<4>(g, hd, hd.tinyq16 + (hd.selq_cap - 1), n16, bid, nb);
    const int64_t ntiny = *(const volatile uint32_t *)(hd.meta + kMetaTiny + hd.h);
    tiny_items<8>(g, hd, hd.selq + (hd.selq_cap - 1), ntiny, bid, nb);
}

// Sampling of one hop, part 2: the full-neighbourhood items (d <= k or k = -1) as
// segmented copies, 32 items per warp, 4 independent load chains per lane.
__device__ __forceinline__ void phase_copy(const GraphDev &g, const HopDev &hd, int bid, int nb)
{
    const int warps = blockDim.x >> 5;
    const int lane = lane_id();
    const int64_t gw = (int64_t)bid * warps + (threadIdx.x >> 5), nw = (int64_t)nb * warps;
    uint32_t *const kcnt = hd.cd.kcnt;
    const int32_t bshift = g.bshift;
    // ---- full neighbourhoods (copyq, queued by phase_count with their output slots):
    // segmented copy over groups of 32 items
    const int64_t total = *(const volatile uint32_t *)(hd.meta + kMetaCopy + hd.h);
    const QEntry *const copyq = hd.copyq;
    for (int64_t g0 = gw * 32; g0 < total; g0 += nw * 32) {
        const int64_t it = g0 + lane;
        int r = 0;
        int32_t c = 0;
        int64_t ib = 0;
        uint32_t *srcp = nullptr;
        int64_t *eidp = nullptr;
        if (it < total) {
            const QEntry e = copyq[it];
            r = e.r;
            c = e.d;
            ib = e.ib;
            srcp = hd.src[r] + e.pos0;
            eidp = hd.eids[r] + e.pos0;
        }
        const int32_t incl = warp_incl_scan(c);
        const int32_t tot = __shfl_sync(0xffffffffu, incl, 31);
        const int32_t excl = incl - c;
        constexpr int U = 4;   // slots per lane per round: U independent load chains in flight
        for (int32_t b0 = 0; b0 < tot; b0 += 32 * U) {
            uint32_t gid[U], goff[U];
            uint32_t *dsrc[U];
            int64_t *deid[U];
            int64_t eid[U], bb[U];
            const int32_t *ixp[U];
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const int32_t s = b0 + q * 32 + lane;
                int L = 0;   // the lane whose item holds output slot s: last lane with excl <= s
#pragma unroll
                for (int step = 16; step > 0; step >>= 1) {
                    const int cand_l = L + step;
                    const int32_t ex = __shfl_sync(0xffffffffu, excl, cand_l & 31);
                    if (cand_l < 32 && ex <= s) L = cand_l;
                }
                const int32_t exL = __shfl_sync(0xffffffffu, excl, L);
                const int64_t ibL = __shfl_sync(0xffffffffu, ib, L);
                const int rL = __shfl_sync(0xffffffffu, r, L);
                uint32_t *const srcL = (uint32_t *)__shfl_sync(0xffffffffu, (unsigned long long)srcp, L);
                int64_t *const eidL = (int64_t *)__shfl_sync(0xffffffffu, (unsigned long long)eidp, L);
                dsrc[q] = nullptr;
                if (s < tot) {
                    const int p = (int)(ibL >> 56);
                    const int64_t base = ibL & ((1ll << 56) - 1);
                    const int32_t j = s - exL;
                    const RelDev &R = g.rel[rL];
                    ixp[q] = R.indices[p] + base + j;
                    gid[q] = goff[q] = (uint32_t)g.off[R.src_vt];
                    bb[q] = g.bbase[R.src_vt];
                    eid[q] = R.edge_base[p] + base + j;
                    dsrc[q] = srcL + j;
                    deid[q] = eidL + j;
                }
            }
#pragma unroll
            for (int q = 0; q < U; ++q)
                if (dsrc[q]) gid[q] += (uint32_t)__ldg(ixp[q]);
#pragma unroll
            for (int q = 0; q < U; ++q)
                if (dsrc[q]) {
                    *dsrc[q] = gid[q];
                    *deid[q] = eid[q];
                    atomicAdd(kcnt + bb[q] + ((gid[q] - goff[q]) >> bshift), 1u);   // mark_src: RED
                }
        }
    }
}

// ============================================================================ link prediction

// Link-prediction targets (NEXT-3, DESIGN.md §3 L1-L4): per positive (src_i, dst_i) of
// relation r, n_neg corrupted dsts drawn uniformly from t(r)'s range; every endpoint is a
// key of the level-0 compaction (compact.cuh, kModeLp), which yields the distinct
// endpoints in ascending gid as the seeds F_0 and every pair in local ids.
__device__ __forceinline__ void phase_lp_mark(const GraphDev &g, const HopDev &hd, const LpDev &lp, int bid, int nb)
{
    const int64_t n = (int64_t)hd.dyn[1];
    const int64_t *__restrict__ src = hd.dyn[2] ? (const int64_t *)hd.dyn[2] : lp.src_stage;
    const int64_t *__restrict__ dst = hd.dyn[3] ? (const int64_t *)hd.dyn[3] : lp.dst_stage;
    const uint32_t k0 = (uint32_t)hd.dyn[4], k1 = (uint32_t)(hd.dyn[4] >> 32);
    const int r = (int)hd.dyn[5];
    const int sv = g.rel[r].src_vt, tv = g.rel[r].dst_vt;
    const int64_t s_lo = g.off[sv], s_hi = g.off[sv + 1], t_lo = g.off[tv], t_hi = g.off[tv + 1];
    const uint64_t n_t = (uint64_t)(t_hi - t_lo);
    const int n_neg = lp.n_neg;
    uint32_t *const kcnt = hd.cd.kcnt;
    int64_t *const neg = lp.neg;
    for (int64_t i = bid * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)nb * blockDim.x) {
        const int64_t a = src[i], b = dst[i];
        if (a < s_lo || a >= s_hi || b < t_lo || b >= t_hi) {
            atomicOr(hd.meta + kMetaErr, kErrSeedRange);
            continue;
        }
        atomicAdd(kcnt + bucket_of(g, sv, a), 1u);
        atomicAdd(kcnt + bucket_of(g, tv, b), 1u);
        for (int q = 0; q < n_neg; ++q) {
            uint32_t c0 = (uint32_t)i, c1 = (uint32_t)q, c2 = 0u, c3 = 0x4E454721u;   // 'NEG!'
            philox4x32_10(c0, c1, c2, c3, k0, k1);
            const int64_t x = t_lo + (int64_t)(((uint64_t)c0 * n_t) >> 32);
            neg[i * n_neg + q] = x;
            atomicAdd(kcnt + bucket_of(g, tv, x), 1u);
        }
    }
}

}  // namespace eg
