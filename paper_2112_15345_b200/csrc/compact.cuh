// compact.cuh -- frontier compaction and relabel of one level, batch-local.
//
// The method (DESIGN.md §3 readings 6-7): after hop h, the new sources of each
// type u are new_h[u] = sorted(unique{sampled src gids of type u} \ S_{h-1}[u]), appended
// after the dst prefix: S_h[u] = F_h[u] ++ new_h[u] ("compute the frontier (i.e., the unique
// set of vertices)" P:698-700; "graph compaction to remove empty vertices and relabel
// vertices and edges" P:566-568); every sampled edge's source is relabelled to
// its index in S_h[s(r)].
//
// B200 form.  Nothing here is sized by the graph: the keys of a level (its sampled sources,
// or the seeds / link-prediction endpoints at level 0) are bucketed by gid into fine buckets
// of 2^bshift gids (bucket_of), and every structure is sized by the batch:
//
//   mark     (fused into the kernels that produce the keys)  kcnt[bucket]++  (RED, L2)
//   kscan    one CTA per batch: prefixes kofs / mofs of the key and member counts, and the
//            compaction TASKS: runs of consecutive buckets of one type holding < 256
//            elements, or a single bucket with more ("big")
//   scatter  each key -> elems[--kcur[b]] with its payload (edge / seed slot); each member
//            of the previous level -> its bucket's member run
//   count    a warp per task:
//              sort path (runs): the task's keys and members (the batch's vertices so far,
//              kept sorted by gid with their positions) go to shared memory, each element is
//              ranked (inside its bucket among the keys, by binary search among the members),
//              duplicates collapse to group heads; the sorted elements go to a scratch;
//              bitmap path (big buckets): a 2^bshift-bit bitmap per warp in shared memory;
//            -> the task's count of new vertices
//   tscan    exclusive prefix of the task counts (tiles + a one-warp look-back over tiles)
//   emit     a warp per task: new vertices appended to their type's node array (in gid
//            order), the merged member list of the next level written, every key relabelled.
//
// Every step reads and writes batch-sized arrays that stay in L2; the old form (a gid ->
// position map and bitmaps over all N vertices per batch in flight) paid a 32-B DRAM sector
// per random access (ncu r02: 1.8 GB of DRAM traffic per C4 launch of 16 batches).
#pragma once
#include "common.cuh"

namespace eg {

#ifndef EG_TASK_ELEMS
#define EG_TASK_ELEMS 224
#endif
#ifndef EG_BIG_BUCKET
#define EG_BIG_BUCKET 32
#endif
constexpr int kTaskElems = EG_TASK_ELEMS;   // T: a run of small buckets closes once its elements cross a multiple of T
constexpr int kBigBucket = EG_BIG_BUCKET;   // buckets with more elements are tasks of their own (bitmap path)
constexpr int kSortCap = 256;      // elements of a sort-path task: 8 per lane
static_assert(kTaskElems + kBigBucket <= kSortCap, "a run holds < T + kBigBucket elements");
constexpr int kMaxWordsPerLane = 1 << (kMaxBucketShift - 10);   // bitmap words of a bucket per lane

// Warp-private shared memory of the compaction (the two paths never run at once).
struct CompactSmem {
    union {
        struct {
            unsigned long long e[kSortCap];      // elements in bucket order
            unsigned long long srt[kSortCap];    // sorted
            int32_t pos[kSortCap];               // position of group heads (by sorted index)
        } s;
        struct {
            uint32_t a[32 * kMaxWordsPerLane];   // keys
            uint32_t m[32 * kMaxWordsPerLane];   // members
            uint16_t pa[32 * kMaxWordsPerLane];  // exclusive prefix of popc(a | m) per word
            uint16_t pn[32 * kMaxWordsPerLane];  // exclusive prefix of popc(a & ~m) per word
        } b;
    };
};

// Composite element: gid (bits 63..32), flag (bit 31: 0 member / seed-with-position, 1 key),
// payload (bits 30..0: a member's position or a key's slot).  Sorting composites orders by
// gid, a vertex's member entry before its keys, keys by slot.
__device__ __forceinline__ unsigned long long comp(uint32_t gid, uint32_t flag, uint32_t pay)
{
    return ((unsigned long long)gid << 32) | ((unsigned long long)flag << 31) | (pay & 0x7FFFFFFFu);
}

__device__ __forceinline__ int type_of_bucket_gid(const GraphDev &g, int64_t gid)
{
    int u = 0;
    while (u + 1 < g.n_vt && gid >= g.off[u + 1]) ++u;
    return u;
}

__device__ __forceinline__ int type_of_bucket(const GraphDev &g, int64_t b)
{
    int u = 0;
    while (u + 1 < g.n_vt && b >= g.bbase[u + 1]) ++u;
    return u;
}

// |F_h[u]| before the level's new vertices (the link-prediction seeds: none).
__device__ __forceinline__ int32_t level_nodes_before(const HopDev &hd, int u)
{
    return hd.h < 0 ? 0 : meta_nodes(hd.meta, hd.h)[u];
}

// ============================================================================ kscan

// Tiles of kScanTile buckets, one CTA of 512 threads each (8 buckets per thread, 16-B
// loads), tiles taken by ticket; each tile publishes its totals (keys, members, tasks) and
// adds those of all earlier tiles (<= 32: one warp reads them at once).  Outputs: kofs /
// mofs = exclusive prefixes of the key / member counts per bucket; the compaction TASKS:
// bucket b starts a task if it is its tile's or its type's first bucket, if it or its
// predecessor is big (> kBigBucket elements), or if the tile's elements before it crossed a
// multiple of kTaskElems since its predecessor.  Clears mcnt (the compaction counts the
// next level's members into it); records each type's first task (ftask).
constexpr int kScanThreads = 512;
constexpr int kScanPer = kScanTile / kScanThreads;   // 8
static_assert(kScanPer == 8, "two 16-B loads per array and thread");

__device__ __forceinline__ unsigned long long tlb_word(uint32_t hi, uint32_t lo)
{
    return (1ull << 63) | ((unsigned long long)(hi & 0x7FFFFFFFu) << 32) | lo;
}

__device__ __forceinline__ void phase_kscan(const GraphDev &g, const HopDev &hd)
{
    __shared__ unsigned long long sh64[kScanThreads / 32 + 1];
    __shared__ int32_t sh32[kScanThreads / 32 + 1];
    __shared__ uint32_t last_e[kScanThreads];
    __shared__ int32_t s_tile;
    __shared__ unsigned long long s_base;   // keys << 32 | members before this tile
    __shared__ uint32_t s_tbase;            // tasks before this tile
    const CompactDev &cd = hd.cd;
    const int level = hd.h + 1;
    const int64_t NB = g.nb;
    const int ntiles = (int)((NB + kScanTile - 1) / kScanTile);
    if (threadIdx.x == 0) s_tile = (int32_t)atomicAdd((uint32_t *)(hd.meta + kMetaKTicket + level), 1u);
    __syncthreads();
    const int tile = s_tile;
    if (tile >= ntiles) return;
    const int64_t b0 = (int64_t)tile * kScanTile + (int64_t)threadIdx.x * kScanPer;
    EG_DCHECK(b0 + kScanPer <= cd.nb_pad);
    uint32_t kc[kScanPer], mc[kScanPer];
    {
        const uint4 *kp = reinterpret_cast<const uint4 *>(cd.kcnt + b0);
        const uint4 *mp = reinterpret_cast<const uint4 *>(cd.mcnt + b0);
        const uint4 k0 = __ldcg(kp), k1 = __ldcg(kp + 1), m0 = __ldcg(mp), m1 = __ldcg(mp + 1);
        kc[0] = k0.x; kc[1] = k0.y; kc[2] = k0.z; kc[3] = k0.w; kc[4] = k1.x; kc[5] = k1.y; kc[6] = k1.z; kc[7] = k1.w;
        mc[0] = m0.x; mc[1] = m0.y; mc[2] = m0.z; mc[3] = m0.w; mc[4] = m1.x; mc[5] = m1.y; mc[6] = m1.z; mc[7] = m1.w;
    }
    // padded buckets (b >= NB) are zero (the launch memset covers the padding)
    unsigned long long loc = 0;   // keys << 32 | members
    uint32_t eloc = 0;
#pragma unroll
    for (int q = 0; q < kScanPer; ++q) {
        loc += ((unsigned long long)kc[q] << 32) | mc[q];
        eloc += kc[q] + mc[q];
    }
    last_e[threadIdx.x] = kc[kScanPer - 1] + mc[kScanPer - 1];
    unsigned long long ttot;
    const unsigned long long lbase = block_excl_scan(loc, sh64, &ttot);   // syncs: last_e visible
    const uint32_t E0 = (uint32_t)(lbase >> 32) + (uint32_t)lbase;        // tile-local elements before b0
    // task flags
    uint32_t flags = 0;
    {
        uint32_t E = E0, e_prev = threadIdx.x ? last_e[threadIdx.x - 1] : 0u;
#pragma unroll
        for (int q = 0; q < kScanPer; ++q) {
            const int64_t b = b0 + q;
            const uint32_t eb = kc[q] + mc[q];
            bool f = false;
            if (b < NB) {
                f = (threadIdx.x == 0 && q == 0) || eb > kBigBucket || e_prev > kBigBucket ||
                    (E / kTaskElems) != ((E - e_prev) / kTaskElems) || g.compact_bitmap;
                for (int u = 1; u < g.n_vt; ++u) f |= b == g.bbase[u];
            }
            flags |= (uint32_t)f << q;
            E += eb;
            e_prev = eb;
        }
    }
    int32_t tflags;
    const int32_t tl = block_excl_scan((int32_t)__popc(flags), sh32, &tflags);
    // tile look-back: publish this tile's totals, add every earlier tile's
    unsigned long long *tlb = cd.tlb + (size_t)level * 3 * kMaxScanTiles;
    if (threadIdx.x < 32) {
        if (threadIdx.x == 0) {
            volatile unsigned long long *v = tlb;
            v[kMaxScanTiles + tile] = tlb_word(0, (uint32_t)tflags);
            __threadfence();
            v[tile] = tlb_word((uint32_t)(ttot >> 32), (uint32_t)ttot);
        }
        __syncwarp();
        unsigned long long kb = 0;
        uint32_t tb = 0;
        const int p = threadIdx.x;
        if (p < tile) {
            volatile unsigned long long *v = tlb;
            unsigned long long w;
            SpinGuard sg;
            do {
                w = v[p];
                sg.step();
            } while (!(w >> 63));
            __threadfence();
            const unsigned long long wt = v[kMaxScanTiles + p];
            kb = (((w >> 32) & 0x7FFFFFFFull) << 32) | (w & 0xFFFFFFFFull);
            tb = (uint32_t)wt;
        }
        kb = warp_sum(kb);
        tb = warp_sum(tb);
        if (threadIdx.x == 0) {
            s_base = kb;
            s_tbase = tb;
        }
    }
    __syncthreads();
    const unsigned long long base = s_base + lbase;
    uint32_t ko = (uint32_t)(base >> 32), mo = (uint32_t)base;
    uint32_t t = s_tbase + (uint32_t)tl;
    uint32_t kv[kScanPer], mv[kScanPer], cv[kScanPer];
#pragma unroll
    for (int q = 0; q < kScanPer; ++q) {
        kv[q] = ko;
        mv[q] = mo;
        ko += kc[q];
        mo += mc[q];
        cv[q] = ko + mo;   // end of bucket b's keys in the element array: the scatter's cursor
        if (flags >> q & 1) {
            EG_DCHECK(t < (uint32_t)NB);
            for (int u = 0; u < g.n_vt; ++u)
                if (b0 + q == g.bbase[u]) cd.ftask[u] = (int32_t)t;   // the type's first task
            cd.tstart[t++] = (uint32_t)(b0 + q);
        }
    }
    uint4 *ko4 = reinterpret_cast<uint4 *>(cd.kofs + b0);
    uint4 *mo4 = reinterpret_cast<uint4 *>(cd.mofs + b0);
    uint4 *mz4 = reinterpret_cast<uint4 *>(cd.mcnt + b0);
    uint4 *kz4 = reinterpret_cast<uint4 *>(cd.kcnt + b0);
    uint4 *cu4 = reinterpret_cast<uint4 *>(cd.kcur + b0);
    ko4[0] = make_uint4(kv[0], kv[1], kv[2], kv[3]);
    ko4[1] = make_uint4(kv[4], kv[5], kv[6], kv[7]);
    mo4[0] = make_uint4(mv[0], mv[1], mv[2], mv[3]);
    mo4[1] = make_uint4(mv[4], mv[5], mv[6], mv[7]);
    cu4[0] = make_uint4(cv[0], cv[1], cv[2], cv[3]);
    cu4[1] = make_uint4(cv[4], cv[5], cv[6], cv[7]);
    mz4[0] = make_uint4(0u, 0u, 0u, 0u);   // counted again by the compaction (next level's members)
    mz4[1] = make_uint4(0u, 0u, 0u, 0u);
    kz4[0] = make_uint4(0u, 0u, 0u, 0u);   // counted again by the next hop's sampling
    kz4[1] = make_uint4(0u, 0u, 0u, 0u);
    if (tile == ntiles - 1 && threadIdx.x == 0) {
        const unsigned long long all = s_base + ttot;
        const uint32_t ntask = s_tbase + (uint32_t)tflags;
        cd.tstart[ntask] = (uint32_t)NB;
        cd.kofs[NB] = (uint32_t)(all >> 32);
        cd.mofs[NB] = (uint32_t)all;
        hd.meta[kMetaTasks + level] = (int32_t)ntask;
        // |S_level[u]| defaults to |F_h[u]| (a type without new vertices); the last task of
        // each type overwrites it
        if (level > 0)
            for (int u = 0; u < g.n_vt; ++u) meta_nodes(hd.meta, level)[u] = meta_nodes(hd.meta, level - 1)[u];
    }
}

// ============================================================================ scatter

// Key i of the level -> (gid, payload, type), or false if it is not a key (an out-of-range
// link-prediction endpoint, skipped by the marking kernel too).  cum: level_keys' prefix
// over relations (hop), types (seeds) or {0, n_pos} (link prediction).

__device__ __forceinline__ bool key_at(const GraphDev &g, const HopDev &hd, const LpDev &lp, const int64_t *cum,
                                       int64_t i, uint32_t &gid, uint32_t &pay, int &u)
{
    if (hd.mode == kModeHop) {
        int r = 0;
        while (i >= cum[r + 1]) ++r;
        gid = __ldcs(hd.src[r] + (i - cum[r]));
        pay = (uint32_t)i;
        u = g.rel[r].src_vt;
        return true;
    }
    if (hd.mode == kModeSeeds) {
        int t = 0;
        while (i >= cum[t + 1]) ++t;
        const int64_t p = i - cum[t];
        gid = (uint32_t)hd.nodes[t][p];
        pay = (uint32_t)p;
        u = t;
        return true;
    }
    // link prediction: i < n: src_i, < 2n: dst_i, else negative k = i - 2n of positive k / n_neg
    const int64_t n = cum[1];
    const int64_t *src = hd.dyn[2] ? (const int64_t *)hd.dyn[2] : lp.src_stage;
    const int64_t *dst = hd.dyn[3] ? (const int64_t *)hd.dyn[3] : lp.dst_stage;
    const int r = (int)hd.dyn[5];
    const int sv = g.rel[r].src_vt, tv = g.rel[r].dst_vt;
    const int64_t j = i < n ? i : (i < 2 * n ? i - n : (i - 2 * n) / max(1, lp.n_neg));
    const int64_t a = src[j], d = dst[j];
    if (a < g.off[sv] || a >= g.off[sv + 1] || d < g.off[tv] || d >= g.off[tv + 1]) return false;   // as phase_lp_mark
    if (i < n) {
        gid = (uint32_t)a;
        u = sv;
        pay = (uint32_t)i;
    } else if (i < 2 * n) {
        gid = (uint32_t)d;
        u = tv;
        pay = (uint32_t)(lp.cap_pos + j);
    } else {
        const int64_t k = i - 2 * n;
        gid = (uint32_t)lp.neg[k];
        u = tv;
        pay = (uint32_t)(2 * lp.cap_pos + lp.cap_pos * lp.n_neg + k);
    }
    return true;
}

// Number of keys of the level and the prefix used by key_at.
__device__ __forceinline__ int64_t level_keys(const GraphDev &g, const HopDev &hd, const LpDev &lp, int64_t *cum)
{
    cum[0] = 0;
    if (hd.mode == kModeHop) {
        for (int r = 0; r < g.n_rel; ++r) cum[r + 1] = cum[r] + meta_nnz(hd.meta, hd.h)[r];
        return cum[g.n_rel];
    }
    if (hd.mode == kModeSeeds) {
        for (int t = 0; t < g.n_vt; ++t) cum[t + 1] = cum[t] + meta_nodes(hd.meta, 0)[t];
        return cum[g.n_vt];
    }
    const int64_t n = (int64_t)hd.dyn[1];
    cum[1] = n;
    return n * (2 + lp.n_neg);
}

// The level's elements in ONE array, bucket by bucket: for bucket b, its members (sorted,
// copied in order) at [kofs[b] + mofs[b], kofs[b] + mofs[b + 1]), then its keys (any order)
// up to kofs[b + 1] + mofs[b + 1].  Composite elements (comp): gid, flag (0 member or seed,
// 1 key), payload (a member's position, a key's slot).
__device__ __forceinline__ void phase_scatter(const GraphDev &g, const HopDev &hd, const LpDev &lp, int bid, int nb)
{
    int64_t cum[EG_MAX_REL + 1];
    const int64_t n = level_keys(g, hd, lp, cum);
    const CompactDev &cd = hd.cd;
    const int64_t stride = (int64_t)nb * blockDim.x;
    constexpr int U = 4;   // independent element -> slot chains per thread
    // pointers hoisted into registers (HopDev lives in global memory; the stores below could
    // alias it as far as the compiler knows)
    const uint32_t *const kofs = cd.kofs;
    const uint32_t *const mofs = cd.mofs;
    uint32_t *const kcur = cd.kcur;   // per bucket: the end of its keys, counted down (kscan)
    unsigned long long *const el = cd.elems;
    const uint32_t cap = (uint32_t)cd.cap_elems;
    const uint32_t kflag = hd.mode == kModeSeeds ? 0u : 1u;   // seeds: keys that carry their position
    const int level = hd.h + 1;
    // members of the previous level (sorted by gid): member j of bucket b -> kofs[b] + j
    if (level > 0) {
        const uint32_t nm = __ldcg(mofs + g.nb);
        const uint32_t *const mg = cd.mg[(level - 1) & 1];
        const int32_t *const mp = cd.mp[(level - 1) & 1];
        for (int64_t j0 = (int64_t)bid * blockDim.x + threadIdx.x; j0 < nm; j0 += U * stride) {
            uint32_t gid[U];
            int32_t pos[U];
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const int64_t j = j0 + q * stride;
                gid[q] = j < nm ? __ldcs(mg + j) : 0u;
                pos[q] = j < nm ? __ldcs(mp + j) : 0;
            }
            uint32_t slot[U];
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const int64_t j = j0 + q * stride;
                if (j < nm) slot[q] = __ldcg(kofs + bucket_of(g, type_of_bucket_gid(g, gid[q]), gid[q])) + (uint32_t)j;
            }
#pragma unroll
            for (int q = 0; q < U; ++q)
                if (j0 + q * stride < nm) {
                    EG_DCHECK(slot[q] < cap);
                    el[slot[q]] = comp(gid[q], 0u, (uint32_t)pos[q]);
                }
        }
    }
    if (hd.mode == kModeHop && g.n_rel == 1) {   // homogeneous hop (C3, C4): no relation lookup
        const uint32_t *const src = hd.src[0];
        const int64_t bb = g.bbase[g.rel[0].src_vt];
        const uint32_t goff = (uint32_t)g.off[g.rel[0].src_vt];
        const int sh = g.bshift;
        for (int64_t i0 = (int64_t)bid * blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
            uint32_t gid[U], slot[U];
            int64_t b[U];
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const int64_t i = i0 + q * stride;
                gid[q] = i < n ? __ldcs(src + i) : goff;
                b[q] = bb + ((gid[q] - goff) >> sh);
            }
#pragma unroll
            for (int q = 0; q < U; ++q)
                if (i0 + q * stride < n) slot[q] = atomicSub(kcur + b[q], 1u) - 1u;
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const int64_t i = i0 + q * stride;
                if (i < n) {
                    if (slot[q] < cap) el[slot[q]] = comp(gid[q], kflag, (uint32_t)i);
                    else atomicOr(hd.meta + kMetaErr, kErrCapacity);
                }
            }
        }
        return;
    }
    for (int64_t i0 = (int64_t)bid * blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
        uint32_t gid[U], pay[U];
        int64_t b[U];
        bool ok[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
            const int64_t i = i0 + q * stride;
            int u = 0;
            ok[q] = i < n && key_at(g, hd, lp, cum, i, gid[q], pay[q], u);
            b[q] = ok[q] ? bucket_of(g, u, gid[q]) : 0;
        }
        uint32_t slot[U];
#pragma unroll
        for (int q = 0; q < U; ++q)
            if (ok[q]) slot[q] = atomicSub(kcur + b[q], 1u) - 1u;
#pragma unroll
        for (int q = 0; q < U; ++q)
            if (ok[q]) {
                if (slot[q] < cap) el[slot[q]] = comp(gid[q], kflag, pay[q]);
                else atomicOr(hd.meta + kMetaErr, kErrCapacity);
            }
    }
}

// ============================================================================ compact

// Two passes over the tasks with a scan of their counts in between (no task waits for
// another: a decoupled look-back over thousands of tiny concurrent tasks walked back over
// every task in flight, measured 121 us for C4's level 3).
//   compact_count  per task: its elements sorted in place (sort path) or put in a bitmap
//                  (big buckets) -> tnew[t] = entries of the next level's member list that
//                  are not members yet (new vertices; at the seeds' level every distinct seed)
//   tscan          tnew -> exclusive prefix G (in place), per batch
//   compact_emit   per task: new vertices at before[u] + G(t) - G(first task of u) + rank,
//                  the merged member list at m0 + G(t) + rank, every key relabelled

// Relabelled output of key (slot pay) at position pos.
__device__ __forceinline__ void key_out(const GraphDev &g, const HopDev &hd, const LpDev &lp, const int64_t *cum,
                                        uint32_t pay, int32_t pos)
{
    if (hd.mode == kModeHop) {
        int r = 0;
        while (r + 1 < g.n_rel && (int64_t)pay >= cum[r + 1]) ++r;
        EG_DCHECK((int64_t)pay < cum[r + 1] && pos >= 0);
        hd.indices[r][pay - cum[r]] = pos;
    } else if (hd.mode == kModeLp) {
        lp.pairs[pay] = pos;
        if ((int64_t)pay < lp.cap_pos)   // a positive's src is also the src of its n_neg negatives
            for (int q = 0; q < lp.n_neg; ++q) lp.pairs[2 * lp.cap_pos + (int64_t)pay * lp.n_neg + q] = pos;
    }
}

// A new vertex of type u at position pos of its node array (capacity-checked).
__device__ __forceinline__ void emit_node(const HopDev &hd, int u, int32_t pos, uint32_t gid)
{
    if (pos < hd.cap_nodes[u])
        hd.nodes[u][pos] = gid;
    else
        atomicOr(hd.meta + kMetaErr, kErrCapacity);
}

struct TaskRange {
    int64_t b0, b1;
    uint32_t e0, n;          // the task's elements: elems[e0, e0 + n)
    uint32_t m0;             // members before the task (= its first slot of the member list - G)
    uint32_t km, nm, nk;     // bitmap path (single bucket): members at [e0, e0 + nm), keys after
    int u;
    bool bitmap;
};

__device__ __forceinline__ TaskRange task_range(const GraphDev &g, const CompactDev &cd, int32_t t)
{
    TaskRange r;
    r.b0 = __ldcg(cd.tstart + t);
    r.b1 = __ldcg(cd.tstart + t + 1);
    const uint32_t k0 = __ldcg(cd.kofs + r.b0), k1 = __ldcg(cd.kofs + r.b1);
    r.m0 = __ldcg(cd.mofs + r.b0);
    const uint32_t m1 = __ldcg(cd.mofs + r.b1);
    r.e0 = k0 + r.m0;
    r.n = (k1 - k0) + (m1 - r.m0);
    r.nm = m1 - r.m0;
    r.nk = k1 - k0;
    r.u = type_of_bucket(g, r.b0);
    r.bitmap = r.b1 - r.b0 == 1 && (r.n > (uint32_t)kBigBucket || g.compact_bitmap);
    EG_DCHECK(r.b0 < r.b1 && r.b1 <= g.nb && (int64_t)r.e0 + r.n <= cd.cap_elems);
    EG_DCHECK(r.bitmap || r.n <= (uint32_t)kSortCap);
    return r;
}

// ---------------------------------------------------------------------------- sort path

// A run of buckets with n <= kSortCap elements (bucket by bucket: members sorted, then keys)
// -> sm.s.srt sorted by composite.  Blocked layout: lane owns elements [R lane, R lane + R);
// an element's bucket segment comes from segmented scans over the lanes (no search), its
// rank from the elements of its segment (<= kBigBucket of them).
__device__ __forceinline__ void sort_build(const GraphDev &g, const HopDev &hd, CompactSmem &sm, const TaskRange &T)
{
    const int lane = lane_id();
    const int n = (int)T.n;
    const unsigned long long *const el = hd.cd.elems + T.e0;
    const int R = (n + 31) >> 5;
    const int64_t goff = g.off[T.u];
    const int sh = g.bshift;
    unsigned long long c[kSortCap / 32];
#pragma unroll
    for (int j = 0; j < kSortCap / 32; ++j) {
        const int i = lane * R + j;
        c[j] = j < R && i < n ? __ldcg(el + i) : ~0ull;
    }
#pragma unroll
    for (int j = 0; j < kSortCap / 32; ++j) {
        const int i = lane * R + j;
        if (j < R && i < n) sm.s.e[i] = c[j];
    }
    // the bucket of the element before the lane's first one (segment starts)
    uint32_t bprev = 0xFFFFFFFFu;
    if (lane * R > 0 && lane * R < n) bprev = (uint32_t)((__ldcg(el + lane * R - 1) >> 32) - goff) >> sh;
    __syncwarp();
    // segment start (first element of the bucket) of each of the lane's elements: running
    // within the lane + the last start of the lanes before (max-scan)
    constexpr int RM = kSortCap / 32;
    uint32_t startm = 0;   // bit j: element R lane + j starts a bucket segment
#pragma unroll
    for (int j = 0; j < RM; ++j) {
        const int i = lane * R + j;
        if (j < R && i < n) {
            const uint32_t bk = (uint32_t)(((c[j] >> 32) - goff) >> sh);
            if (bk != bprev) startm |= 1u << j;
            bprev = bk;
        }
    }
    const int last = startm ? lane * R + 31 - __clz(startm) : -1;
    int lo_run = -1;
    int ls = last;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, ls, o);
        if (lane >= o) ls = max(ls, x);
    }
    lo_run = __shfl_up_sync(0xffffffffu, ls, 1);
    if (lane == 0) lo_run = -1;
    // segment end: the first start after the lane's elements (min-scan from the right)
    int fs = startm ? lane * R + __ffs(startm) - 1 : n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int x = __shfl_down_sync(0xffffffffu, fs, o);
        if (lane + o < 32) fs = min(fs, x);
    }
    int hi_run = __shfl_down_sync(0xffffffffu, fs, 1);
    if (lane == 31) hi_run = n;
    // the lane's elements: segment [lo, hi): lo = the last start at or before it, hi = the
    // first start after it (inside the lane, else from the lanes before / after)
    int lo = lo_run;
#pragma unroll
    for (int j = 0; j < RM; ++j) {
        const int i = lane * R + j;
        if (j < R && i < n) {
            if (startm >> j & 1) lo = i;
            const uint32_t after = startm & ~((2u << j) - 1u);
            const int hi = after ? lane * R + __ffs(after) - 1 : hi_run;
            const unsigned long long x = c[j];
            int r = lo;
            for (int k = lo; k < hi; ++k) r += sm.s.e[k] < x;
            EG_DCHECK(lo >= 0 && hi <= n && r < hi);
            sm.s.srt[r] = x;
        }
    }
    __syncwarp();
}

// Group heads of sorted elements [0, n) in the blocked layout (lane owns [R lane, R lane + R)):
// bit j of headm / newm / keym for element R lane + j.
struct Heads {
    int R;
    uint32_t headm, newm, keym;
    int last_head;   // sorted index of the last head among this lane's elements, or -1
};

__device__ __forceinline__ Heads sort_heads(const CompactSmem &sm, int n)
{
    const int lane = lane_id();
    Heads H;
    H.R = (n + 31) >> 5;
    H.headm = H.newm = H.keym = 0;
    H.last_head = -1;
    for (int j = 0; j < H.R; ++j) {
        const int i = lane * H.R + j;
        if (i >= n) break;
        const unsigned long long c = sm.s.srt[i];
        const bool head = i == 0 || (uint32_t)(sm.s.srt[i - 1] >> 32) != (uint32_t)(c >> 32);
        const bool key = (c >> 31) & 1;
        if (head) {
            H.headm |= 1u << j;
            H.last_head = i;
            if (key) H.newm |= 1u << j;
        }
        if (key) H.keym |= 1u << j;
    }
    return H;
}

// ---------------------------------------------------------------------------- bitmap path

// One big bucket -> sm.b: key bits a, member bits m, per-word exclusive prefixes of
// popc(a | m) (pa) and popc(a & ~m) (pn); returns (distinct << 16) | new.
__device__ __forceinline__ uint32_t bitmap_build(const GraphDev &g, const HopDev &hd, CompactSmem &sm, const TaskRange &T,
                                 bool check_dup)
{
    const int lane = lane_id();
    const int WL = 1 << (g.bshift - 10);   // words per lane (blocked: lane owns [WL lane, WL lane + WL))
    const uint32_t gid0 = (uint32_t)(g.off[T.u] + ((T.b0 - g.bbase[T.u]) << g.bshift));
    const unsigned long long *const el = hd.cd.elems + T.e0;
    for (int q = 0; q < WL; ++q) {
        sm.b.a[lane * WL + q] = 0u;
        sm.b.m[lane * WL + q] = 0u;
    }
    __syncwarp();
    // four loads in flight per lane before their shared-memory atomics; members first in el
    for (uint32_t i0 = lane; i0 < T.n; i0 += 128) {
        unsigned long long x[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) x[q] = i0 + 32 * q < T.n ? __ldcg(el + i0 + 32 * q) : 0ull;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t i = i0 + 32 * q;
            if (i >= T.n) continue;
            const uint32_t b = (uint32_t)(x[q] >> 32) - gid0;
            EG_DCHECK(b < (1u << g.bshift));
            if (i < T.nm) {
                atomicOr(sm.b.m + (b >> 5), 1u << (b & 31));
            } else {
                const uint32_t old = atomicOr(sm.b.a + (b >> 5), 1u << (b & 31));
                if (check_dup && (old >> (b & 31) & 1)) atomicOr(hd.meta + kMetaErr, kErrSeedDup);
            }
        }
    }
    __syncwarp();
    uint32_t ca = 0, cn = 0;
    for (int q = 0; q < WL; ++q) {
        const uint32_t a = sm.b.a[lane * WL + q], m = sm.b.m[lane * WL + q];
        ca += __popc(a | m);
        cn += __popc(a & ~m);
    }
    const uint32_t cnt = (ca << 16) | cn;   // <= 2^14 per bucket
    const uint32_t incl = warp_incl_scan(cnt);
    uint32_t pa = (incl - cnt) >> 16, pn = (incl - cnt) & 0xFFFFu;
    for (int q = 0; q < WL; ++q) {
        const uint32_t a = sm.b.a[lane * WL + q], m = sm.b.m[lane * WL + q];
        sm.b.pa[lane * WL + q] = (uint16_t)pa;
        sm.b.pn[lane * WL + q] = (uint16_t)pn;
        pa += __popc(a | m);
        pn += __popc(a & ~m);
    }
    __syncwarp();
    return __shfl_sync(0xffffffffu, incl, 31);
}

// ---------------------------------------------------------------------------- one task

// Pass A of a task: its elements deduplicated -> the task's count of entries of the next
// level's member list that are not members yet (new vertices; at the seeds' level every
// distinct seed).  Sort-path tasks leave their elements sorted in place (elems).
__device__ __forceinline__ uint32_t count_task(const GraphDev &g, const HopDev &hd, CompactSmem &sm,
                                               const TaskRange &T)
{
    const int lane = lane_id();
    const bool seeds = hd.mode == kModeSeeds;
    if (T.bitmap) return bitmap_build(g, hd, sm, T, seeds) & 0xFFFFu;   // a & ~m (seeds: m = 0)
    sort_build(g, hd, sm, T);
    const int n = (int)T.n;
    const Heads H = sort_heads(sm, n);
    // seeds: every distinct seed counts (they are all new to the member list); a repeated
    // gid is a duplicate seed
    if (seeds && __popc(H.headm) != min(H.R, max(0, n - lane * H.R))) atomicOr(hd.meta + kMetaErr, kErrSeedDup);
    unsigned long long *const el = hd.cd.elems + T.e0;   // sorted, in place
    for (int i = lane; i < n; i += 32) el[i] = sm.s.srt[i];
    __syncwarp();
    return warp_sum((uint32_t)__popc(seeds ? H.headm : H.newm));
}

// Pass B of a task: G = new entries of the earlier tasks (all types), Gu = those before its
// type's first task: new vertices at before[u] + G - Gu + rank, the merged member list at
// m0 + G + rank, every key relabelled.  Returns the task's new vertices.
__device__ __forceinline__ uint32_t emit_task(const GraphDev &g, const HopDev &hd, const LpDev &lp,
                                              const int64_t *cum, CompactSmem &sm, const TaskRange &T, uint32_t G,
                                              uint32_t Gu)
{
    const CompactDev &cd = hd.cd;
    const int lane = lane_id();
    const int level = hd.h + 1;
    const int32_t *mp_in = level > 0 ? cd.mp[(level - 1) & 1] : nullptr;
    uint32_t *const mg_out = cd.mg[level & 1];
    int32_t *const mp_out = cd.mp[level & 1];
    const bool seeds = hd.mode == kModeSeeds;
        const int32_t before = level_nodes_before(hd, T.u);
        const int32_t tbase = before + (int32_t)(G - Gu);              // position of the task's first new vertex
        const uint32_t mo = T.m0 + G;                                  // its first entry of the member list
        const unsigned long long *const el = cd.elems + T.e0;
        uint32_t tot_new;
        if (T.bitmap) {
            const uint32_t tot = bitmap_build(g, hd, sm, T, false);
            tot_new = tot & 0xFFFFu;
            const int WL = 1 << (g.bshift - 10);
            const uint32_t gid0 = (uint32_t)(g.off[T.u] + ((T.b0 - g.bbase[T.u]) << g.bshift));
            if (seeds) {   // positions given by the keys
                if (!hd.last)
                    for (uint32_t i = lane; i < T.n; i += 32) {
                        const unsigned long long c = __ldcg(el + i);
                        const uint32_t gid = (uint32_t)(c >> 32), x = gid - gid0;
                        const uint32_t w = x >> 5, low = (1u << (x & 31)) - 1u;
                        const uint32_t r = sm.b.pa[w] + __popc((sm.b.a[w] | sm.b.m[w]) & low);
                        mg_out[mo + r] = gid;
                        mp_out[mo + r] = (int32_t)(c & 0x7FFFFFFFu);
                    }
            } else {
                // new vertices: the bits of a & ~m, in gid order
                for (int q = 0; q < WL; ++q) {
                    const int w = lane * WL + q;
                    const uint32_t a = sm.b.a[w], m = sm.b.m[w];
                    uint32_t nwd = a & ~m;
                    while (nwd) {
                        const int bit = __ffs(nwd) - 1;
                        nwd &= nwd - 1;
                        const uint32_t low = (1u << bit) - 1u;
                        const uint32_t gid = gid0 + (uint32_t)(32 * w + bit);
                        const int32_t pos = tbase + (int32_t)(sm.b.pn[w] + __popc(a & ~m & low));
                        emit_node(hd, T.u, pos, gid);
                        if (!hd.last) {
                            const uint32_t r = sm.b.pa[w] + __popc((a | m) & low);
                            mg_out[mo + r] = gid;
                            mp_out[mo + r] = pos;
                        }
                    }
                }
                // members (el[0, nm), sorted): copied to their merged slots
                if (!hd.last)
                    for (uint32_t i0 = lane; i0 < T.nm; i0 += 128) {
                        unsigned long long cm[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) cm[q] = i0 + 32 * q < T.nm ? __ldcg(el + i0 + 32 * q) : 0ull;
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            if (i0 + 32 * q < T.nm) {
                                const uint32_t gid = (uint32_t)(cm[q] >> 32);
                                const uint32_t x = gid - gid0, w = x >> 5, low = (1u << (x & 31)) - 1u;
                                const uint32_t r = sm.b.pa[w] + __popc((sm.b.a[w] | sm.b.m[w]) & low);
                                mg_out[mo + r] = gid;
                                mp_out[mo + r] = (int32_t)(cm[q] & 0x7FFFFFFFu);
                            }
                    }
            }
            if (!hd.last && lane == 0 && (tot >> 16)) atomicAdd(cd.mcnt + T.b0, tot >> 16);
            if (!seeds)
                for (uint32_t i0 = T.nm + lane; i0 < T.n; i0 += 128) {   // relabel every key, 4 in flight per lane
                    unsigned long long ck[4];
                    int32_t pos[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) ck[q] = i0 + 32 * q < T.n ? __ldcg(el + i0 + 32 * q) : ((unsigned long long)gid0 << 32);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint32_t x = (uint32_t)(ck[q] >> 32) - gid0;
                        const uint32_t w = x >> 5, bit = x & 31, low = (1u << bit) - 1u;
                        const uint32_t a = sm.b.a[w], m = sm.b.m[w];
                        if (m >> bit & 1)
                            pos[q] = __ldcg(mp_in + T.m0 + (sm.b.pa[w] - sm.b.pn[w]) + __popc(m & low));
                        else
                            pos[q] = tbase + (int32_t)(sm.b.pn[w] + __popc((a & ~m) & low));
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (i0 + 32 * q < T.n) key_out(g, hd, lp, cum, (uint32_t)(ck[q] & 0x7FFFFFFFu), pos[q]);
                }
        } else {
            const int n = (int)T.n;
            unsigned long long v[kSortCap / 32];
#pragma unroll
            for (int j = 0; j < kSortCap / 32; ++j) v[j] = lane + 32 * j < n ? __ldcg(el + lane + 32 * j) : 0ull;
#pragma unroll
            for (int j = 0; j < kSortCap / 32; ++j)
                if (lane + 32 * j < n) sm.s.srt[lane + 32 * j] = v[j];
            __syncwarp();
            const Heads H = sort_heads(sm, n);
            const uint32_t cnt = ((uint32_t)__popc(H.headm) << 16) | (uint32_t)__popc(H.newm);   // n <= 256
            const uint32_t incl = warp_incl_scan(cnt);
            tot_new = __shfl_sync(0xffffffffu, incl, 31) & 0xFFFFu;
            uint32_t d_rank = (incl - cnt) >> 16, n_rank = (incl - cnt) & 0xFFFFu;
            for (int j = 0; j < H.R; ++j) {   // heads: positions, new vertices, the next member list
                if (!(H.headm >> j & 1)) continue;
                const int i = lane * H.R + j;
                const unsigned long long c = sm.s.srt[i];
                const uint32_t gid = (uint32_t)(c >> 32);
                int32_t pos;
                if (H.newm >> j & 1) {
                    pos = tbase + (int32_t)n_rank;
                    emit_node(hd, T.u, pos, gid);
                    ++n_rank;
                } else {
                    pos = (int32_t)(c & 0x7FFFFFFFu);   // a member's position, or a seed's own
                }
                sm.s.pos[i] = pos;
                if (!hd.last) {
                    mg_out[mo + d_rank] = gid;
                    mp_out[mo + d_rank] = pos;
                    atomicAdd(cd.mcnt + bucket_of(g, T.u, gid), 1u);
                }
                ++d_rank;
            }
            // the last head before each lane's first element: exclusive max-scan over lanes
            int lh = H.last_head;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int x = __shfl_up_sync(0xffffffffu, lh, o);
                if (lane >= o) lh = max(lh, x);
            }
            int hidx = __shfl_up_sync(0xffffffffu, lh, 1);
            if (lane == 0) hidx = -1;
            __syncwarp();
            if (!seeds)
                for (int j = 0; j < H.R; ++j) {   // relabel every key with its group head's position
                    const int i = lane * H.R + j;
                    if (i >= n) break;
                    if (H.headm >> j & 1) hidx = i;
                    if (H.keym >> j & 1)
                        key_out(g, hd, lp, cum, (uint32_t)(sm.s.srt[i] & 0x7FFFFFFFu), sm.s.pos[hidx]);
                }
        }
    return tot_new;
}

// ---------------------------------------------------------------------------- the kernels

// Pass A: a warp per task (static stride over the batch's tasks) -> tnew[t].
__device__ __forceinline__ void phase_compact_count(const GraphDev &g, const HopDev &hd, CompactSmem *smem, int bid,
                                                    int nb)
{
    const CompactDev &cd = hd.cd;
    const int level = hd.h + 1;
    CompactSmem &sm = smem[threadIdx.x >> 5];
    const int32_t ntask = *(volatile int32_t *)(hd.meta + kMetaTasks + level);
    const int32_t nw = nb * (blockDim.x >> 5);
    for (int32_t t = bid * (blockDim.x >> 5) + (threadIdx.x >> 5); t < ntask; t += nw) {
        const TaskRange T = task_range(g, cd, t);
        const uint32_t cnt = count_task(g, hd, sm, T);
        if (lane_id() == 0) cd.tnew[t] = cnt;
        __syncwarp();
    }
}

// tnew -> exclusive prefix, in place (tiles of kScanTile tasks, one CTA of 512 threads
// each, taken by ticket; one warp adds the totals of every earlier tile).
__device__ __forceinline__ void phase_tscan(const GraphDev &g, const HopDev &hd)
{
    __shared__ uint32_t sh[kScanThreads / 32 + 1];
    __shared__ int32_t s_tile;
    __shared__ uint32_t s_base;
    const CompactDev &cd = hd.cd;
    const int level = hd.h + 1;
    const int32_t ntask = *(volatile int32_t *)(hd.meta + kMetaTasks + level);
    const int ntiles = (ntask + kScanTile - 1) / kScanTile;
    if (threadIdx.x == 0) s_tile = (int32_t)atomicAdd((uint32_t *)(hd.meta + kMetaTicket + level), 1u);
    __syncthreads();
    const int tile = s_tile;
    if (tile >= ntiles) return;
    const int64_t t0 = (int64_t)tile * kScanTile + (int64_t)threadIdx.x * kScanPer;
    uint32_t v[kScanPer], loc = 0;
#pragma unroll
    for (int q = 0; q < kScanPer; ++q) {
        v[q] = t0 + q < ntask ? __ldcg(cd.tnew + t0 + q) : 0u;
        loc += v[q];
    }
    uint32_t ttot;
    const uint32_t lbase = block_excl_scan(loc, sh, &ttot);
    unsigned long long *tlb = cd.tlb + (size_t)level * 3 * kMaxScanTiles + 2 * kMaxScanTiles;
    if (threadIdx.x < 32) {
        volatile unsigned long long *w = tlb;
        if (threadIdx.x == 0) w[tile] = (1ull << 63) | ttot;
        uint32_t b = 0;
        const int p = threadIdx.x;
        if (p < tile) {
            unsigned long long x;
            SpinGuard sg;
            do {
                x = w[p];
                sg.step();
            } while (!(x >> 63));
            b = (uint32_t)x;
        }
        b = warp_sum(b);
        if (threadIdx.x == 0) s_base = b;
    }
    __syncthreads();
    uint32_t run = s_base + lbase;
#pragma unroll
    for (int q = 0; q < kScanPer; ++q) {
        if (t0 + q < ntask) cd.tnew[t0 + q] = run;
        run += v[q];
    }
}

// Pass B: a warp per task; the last task of each type records |S_level[u]|.
__device__ __forceinline__ void phase_compact_emit(const GraphDev &g, const HopDev &hd, const LpDev &lp,
                                                   CompactSmem *smem, int bid, int nb)
{
    const CompactDev &cd = hd.cd;
    const int level = hd.h + 1;
    CompactSmem &sm = smem[threadIdx.x >> 5];
    int64_t cum[EG_MAX_REL + 1];
    level_keys(g, hd, lp, cum);
    const int32_t ntask = *(volatile int32_t *)(hd.meta + kMetaTasks + level);
    const int32_t nw = nb * (blockDim.x >> 5);
    const bool seeds = hd.mode == kModeSeeds;
    for (int32_t t = bid * (blockDim.x >> 5) + (threadIdx.x >> 5); t < ntask; t += nw) {
        const TaskRange T = task_range(g, cd, t);
        const uint32_t G = __ldcg(cd.tnew + t);                                    // earlier tasks' new entries
        const uint32_t Gu = seeds ? 0u : __ldcg(cd.tnew + __ldcg(cd.ftask + T.u));  // ... before the type's first task
        const uint32_t tot_new = emit_task(g, hd, lp, cum, sm, T, G, Gu);
        // the last task of its type: |S_level[u]| = |F[u]| + the type's new vertices (the
        // seeds' sizes come from the seed split)
        if (lane_id() == 0 && T.b1 == g.bbase[T.u + 1] && !seeds)
            meta_nodes(hd.meta, level)[T.u] = level_nodes_before(hd, T.u) + (int32_t)(G - Gu + tot_new);
        __syncwarp();
    }
}

}  // namespace eg
