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
//   scatter  each key -> keys[kofs[b] + (--kcnt[b])], with its payload (edge / seed slot)
//   compact  a warp per task (dynamic tickets, in task order):
//              sort path (runs): the task's keys and members (the batch's vertices so far,
//              kept sorted by gid with their positions) go to shared memory in bucket order,
//              each element is ranked inside its bucket, duplicates collapse to group heads;
//              bitmap path (big buckets): a 2^bshift-bit bitmap per warp in shared memory;
//            the number of new vertices of the task -> decoupled look-back over the tasks
//            (global and per-type prefixes in one word) -> the new vertices' positions; then
//            new vertices are appended to their type's node array (in gid order), the merged
//            member list of the next level is written, and every key is relabelled.
//
// Every step reads and writes batch-sized arrays that stay in L2; the old form (a gid ->
// position map and bitmaps over all N vertices per batch in flight) paid a 32-B DRAM sector
// per random access (ncu r02: 1.8 GB of DRAM traffic per C4 launch of 16 batches).
#pragma once
#include "common.cuh"

namespace eg {

constexpr int kTaskElems = 224;    // T: a run of small buckets closes once its elements cross a multiple of T
constexpr int kBigBucket = 32;     // buckets with more elements are tasks of their own (bitmap path)
constexpr int kSortCap = 256;      // elements of a sort-path task: 8 per lane
static_assert(kTaskElems + kBigBucket <= kSortCap, "a run holds < T + kBigBucket elements");
constexpr int kMaxWordsPerLane = 1 << (kMaxBucketShift - 10);   // bitmap words of a bucket per lane

// Warp-private shared memory of the compaction (the two paths never run at once).
struct CompactSmem {
    union {
        struct {
            unsigned long long e[kSortCap];      // elements in bucket order
            unsigned long long srt[kSortCap];    // sorted
            uint32_t bk[kSortCap];               // bucket of e[i], relative to the task's first
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

// One CTA per batch.  kofs / mofs = exclusive prefixes of the key / member counts per
// bucket; tasks: bucket b starts a task if it is its type's first bucket, if it or its
// predecessor is big (> kBigBucket elements), or if the elements before it crossed a
// multiple of kTaskElems since its predecessor.  Clears mcnt (the compaction counts the
// next level's members into it) and the tasks' look-back words.
__device__ void phase_kscan(const GraphDev &g, const HopDev &hd)
{
    __shared__ unsigned long long sh64[33];
    __shared__ int32_t sh32[33];
    const CompactDev &cd = hd.cd;
    const int level = hd.h + 1;
    const int64_t NB = g.nb;
    const int64_t per = (NB + blockDim.x - 1) / blockDim.x;
    const int64_t a = min(NB, (int64_t)threadIdx.x * per), e = min(NB, a + per);
    // pass 1: sums of this thread's buckets
    unsigned long long loc = 0;   // keys << 32 | members
    for (int64_t b = a; b < e; ++b) loc += ((unsigned long long)__ldcg(cd.kcnt + b) << 32) | __ldcg(cd.mcnt + b);
    unsigned long long tot;
    unsigned long long base = block_excl_scan(loc, sh64, &tot);
    // pass 2: offsets and task flags
    uint32_t ko = (uint32_t)(base >> 32), mo = (uint32_t)base;
    int32_t nflag = 0;
    uint32_t e_prev = 0;          // elements of bucket b - 1
    if (a > 0 && a < e) e_prev = __ldcg(cd.kcnt + a - 1) + __ldcg(cd.mcnt + a - 1);
    const int u_first = a < e ? type_of_bucket(g, a) : 0;
    int u = u_first;
    for (int64_t b = a; b < e; ++b) {
        while (u + 1 < g.n_vt && b >= g.bbase[u + 1]) ++u;
        const uint32_t kc = __ldcg(cd.kcnt + b), mc = __ldcg(cd.mcnt + b);
        const uint32_t eb = kc + mc;
        const uint32_t E = ko + mo;                       // elements before b
        const bool flag = b == g.bbase[u] || eb > kBigBucket || e_prev > kBigBucket ||
                          (E / kTaskElems) != ((E - e_prev) / kTaskElems) || g.compact_bitmap;
        nflag += flag;
        cd.kofs[b] = ko;
        cd.mofs[b] = mo;
        ko += kc;
        mo += mc;
        e_prev = eb;
    }
    int32_t ntask;
    int32_t t = block_excl_scan(nflag, sh32, &ntask);
    // pass 3: task starts (re-derive the flags), clear the member counts
    e_prev = 0;
    if (a > 0 && a < e) e_prev = __ldcg(cd.kcnt + a - 1) + __ldcg(cd.mcnt + a - 1);
    u = u_first;
    __syncthreads();   // kcnt of a - 1 read above before anyone clears mcnt (kcnt is not cleared here)
    for (int64_t b = a; b < e; ++b) {
        while (u + 1 < g.n_vt && b >= g.bbase[u + 1]) ++u;
        const uint32_t eb = __ldcg(cd.kcnt + b) + __ldcg(cd.mcnt + b);
        const uint32_t E = cd.kofs[b] + cd.mofs[b];
        const bool flag = b == g.bbase[u] || eb > kBigBucket || e_prev > kBigBucket ||
                          (E / kTaskElems) != ((E - e_prev) / kTaskElems) || g.compact_bitmap;
        if (flag) cd.tstart[t++] = (uint32_t)b;
        e_prev = eb;
    }
    __syncthreads();
    for (int64_t b = a; b < e; ++b) cd.mcnt[b] = 0u;
    for (int i = threadIdx.x; i < ntask; i += blockDim.x) cd.lb[i] = 0ull;
    if (threadIdx.x == 0) {
        cd.tstart[ntask] = (uint32_t)NB;
        cd.kofs[NB] = (uint32_t)(tot >> 32);
        cd.mofs[NB] = (uint32_t)tot;
        hd.meta[kMetaTasks + level] = ntask;
    }
    // |S_level[u]| defaults to |F_h[u]| (a type without new vertices); the last task of each
    // type overwrites it
    if (level > 0 && threadIdx.x < g.n_vt)
        meta_nodes(hd.meta, level)[threadIdx.x] = meta_nodes(hd.meta, level - 1)[threadIdx.x];
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

__device__ void phase_scatter(const GraphDev &g, const HopDev &hd, const LpDev &lp, int bid, int nb)
{
    int64_t cum[EG_MAX_REL + 1];
    const int64_t n = level_keys(g, hd, lp, cum);
    const CompactDev &cd = hd.cd;
    const int64_t stride = (int64_t)nb * blockDim.x;
    constexpr int U = 4;   // independent key -> slot chains per thread
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
            if (ok[q]) slot[q] = __ldcg(cd.kofs + b[q]) + atomicSub(cd.kcnt + b[q], 1u) - 1u;
#pragma unroll
        for (int q = 0; q < U; ++q)
            if (ok[q]) {
                if (slot[q] < (uint32_t)cd.cap_keys) {
                    cd.keys[slot[q]] = gid[q];
                    cd.kidx[slot[q]] = pay[q];
                } else {
                    atomicOr(hd.meta + kMetaErr, kErrCapacity);
                }
            }
    }
}

// ============================================================================ compact

// Decoupled look-back word: status (bits 63..62: 1 aggregate, 2 inclusive prefix), the
// count over all earlier tasks (bits 61..31) and over the earlier tasks of the same type
// (bits 30..0).
__device__ __forceinline__ unsigned long long lb_word(unsigned long long st, uint32_t glob, uint32_t typ)
{
    return (st << 62) | ((unsigned long long)(glob & 0x7FFFFFFFu) << 31) | (typ & 0x7FFFFFFFu);
}

// Lane 0: publish task t's counts and find the exclusive prefixes.  glob = the task's
// entries of the next level's member list that are not members yet (its new vertices; at
// the seeds' level every distinct seed), counted over all earlier tasks; typ = its new
// vertices to append to the type's node array, counted over the earlier tasks of the
// same type.  Tasks are processed in ticket order, so every earlier task is held by a
// running warp and publishes its aggregate before it waits itself.
__device__ __forceinline__ void lookback(const GraphDev &g, const CompactDev &cd, int32_t t, int u, uint32_t glob,
                                         uint32_t typ, uint32_t &g_excl, uint32_t &t_excl)
{
    volatile unsigned long long *lb = cd.lb;
    lb[t] = lb_word(1, glob, typ);
    uint32_t gs = 0, ts = 0;
    bool same = true;
    const uint32_t first_b = (uint32_t)g.bbase[u];
    for (int32_t p = t - 1; p >= 0; --p) {
        if (same && __ldcg(cd.tstart + p) < first_b) same = false;   // p belongs to an earlier type
        unsigned long long w;
        uint64_t t0 = 0;
        for (uint32_t it = 0;; ++it) {   // bounded: a publication that never comes traps after ~2 s
            w = lb[p];
            if ((w >> 62) != 0) break;
            if ((it & 1023) == 1023) {
                uint64_t tn;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
                if (!t0) t0 = tn;
                else if (tn - t0 > 2000000000ull) __trap();
            }
        }
        gs += (uint32_t)(w >> 31) & 0x7FFFFFFFu;
        if (same) ts += (uint32_t)w & 0x7FFFFFFFu;
        if ((w >> 62) == 2) break;
    }
    __threadfence();
    lb[t] = lb_word(2, gs + glob, ts + typ);
    g_excl = gs;
    t_excl = ts;
}

// Relabelled output of key (slot pay) at position pos.
__device__ __forceinline__ void key_out(const GraphDev &g, const HopDev &hd, const LpDev &lp, const int64_t *cum,
                                        uint32_t pay, int32_t pos)
{
    if (hd.mode == kModeHop) {
        int r = 0;
        while ((int64_t)pay >= cum[r + 1]) ++r;
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

// Sort path: a run of buckets [b0, b1) with n = nk + nm <= kSortCap elements.
__device__ void compact_sort(const GraphDev &g, const HopDev &hd, const LpDev &lp, const int64_t *cum, CompactSmem &sm,
                             int32_t t, int u, int64_t b0, uint32_t k0, uint32_t nk, uint32_t m0, uint32_t nm)
{
    const CompactDev &cd = hd.cd;
    const int lane = lane_id();
    const int level = hd.h + 1;
    const uint32_t *mg_in = level > 0 ? cd.mg[(level - 1) & 1] : nullptr;
    const int32_t *mp_in = level > 0 ? cd.mp[(level - 1) & 1] : nullptr;
    const int n = (int)(nk + nm);
    // 1. elements in bucket order (per bucket: members, then keys)
    for (int i = lane; i < n; i += 32) {
        uint32_t gid, flag, pay;
        int64_t b;
        int idx;
        if (i < (int)nk) {
            gid = __ldcg(cd.keys + k0 + i);
            pay = __ldcg(cd.kidx + k0 + i);
            flag = hd.mode == kModeSeeds ? 0u : 1u;   // seeds: keys that carry their position
            b = bucket_of(g, u, gid);
            idx = i + (int)(__ldcg(cd.mofs + b + 1) - m0);
        } else {
            const int j = i - (int)nk;
            gid = __ldcg(mg_in + m0 + j);
            pay = (uint32_t)__ldcg(mp_in + m0 + j);
            flag = 0u;
            b = bucket_of(g, u, gid);
            idx = j + (int)(__ldcg(cd.kofs + b) - k0);
        }
        sm.s.e[idx] = comp(gid, flag, pay);
        sm.s.bk[idx] = (uint32_t)(b - b0);
    }
    __syncwarp();
    // 2. rank inside the bucket (elements of a bucket are contiguous) -> sorted order
    for (int i = lane; i < n; i += 32) {
        const unsigned long long c = sm.s.e[i];
        const uint32_t bk = sm.s.bk[i];
        int lo = i, hi = i + 1;
        while (lo > 0 && sm.s.bk[lo - 1] == bk) --lo;   // buckets of runs hold <= kBigBucket elements
        while (hi < n && sm.s.bk[hi] == bk) ++hi;
        int r = lo;
        for (int j = lo; j < hi; ++j) r += sm.s.e[j] < c;
        sm.s.srt[r] = c;
    }
    __syncwarp();
    // 3. group heads; blocked layout: lane owns sorted elements [R lane, R lane + R)
    const int R = (n + 31) >> 5;
    uint32_t newm = 0, headm = 0, keym = 0;
    int last_head = -1;   // sorted index of the last head at or before this lane's elements
    for (int j = 0; j < R; ++j) {
        const int i = lane * R + j;
        if (i >= n) break;
        const unsigned long long c = sm.s.srt[i];
        const bool head = i == 0 || (uint32_t)(sm.s.srt[i - 1] >> 32) != (uint32_t)(c >> 32);
        const bool key = (c >> 31) & 1;
        if (head) {
            headm |= 1u << j;
            last_head = i;
            if (key) newm |= 1u << j;
        }
        if (key) keym |= 1u << j;
        if (hd.mode == kModeSeeds && !head) atomicOr(hd.meta + kMetaErr, kErrSeedDup);
    }
    const uint32_t cnt = ((uint32_t)__popc(headm) << 16) | (uint32_t)__popc(newm);   // n <= 256: 16-bit fields
    const uint32_t incl = warp_incl_scan(cnt);
    const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
    uint32_t d_rank = (incl - cnt) >> 16, n_rank = (incl - cnt) & 0xFFFFu;
    const uint32_t tot_new = tot & 0xFFFFu, tot_dist = tot >> 16;
    uint32_t g_excl = 0, t_excl = 0;
    // seeds: every distinct seed is new to the member list, none is appended (positions given)
    if (lane == 0)
        lookback(g, cd, t, u, hd.mode == kModeSeeds ? tot_dist : tot_new, tot_new, g_excl, t_excl);
    g_excl = __shfl_sync(0xffffffffu, g_excl, 0);
    t_excl = __shfl_sync(0xffffffffu, t_excl, 0);
    const int32_t before = level_nodes_before(hd, u);
    // 4. heads: positions, new vertices, the merged member list of the next level
    for (int j = 0; j < R; ++j) {
        if (!(headm >> j & 1)) continue;
        const int i = lane * R + j;
        const unsigned long long c = sm.s.srt[i];
        const uint32_t gid = (uint32_t)(c >> 32);
        int32_t pos;
        if (newm >> j & 1) {
            pos = before + (int32_t)(t_excl + n_rank);
            emit_node(hd, u, pos, gid);
            ++n_rank;
        } else {
            pos = (int32_t)(c & 0x7FFFFFFFu);   // a member's position, or a seed's own
        }
        sm.s.pos[i] = pos;
        if (!hd.last) {
            const uint32_t o = m0 + g_excl + d_rank;
            cd.mg[level & 1][o] = gid;
            cd.mp[level & 1][o] = pos;
            atomicAdd(cd.mcnt + bucket_of(g, u, gid), 1u);
        }
        ++d_rank;
    }
    // the last head before each lane's first element: exclusive max-scan of last_head over
    // the lanes (segmented broadcast of the group heads' positions)
    int lh = last_head;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, lh, o);
        if (lane >= o) lh = max(lh, x);
    }
    int carry = __shfl_up_sync(0xffffffffu, lh, 1);
    if (lane == 0) carry = -1;
    __syncwarp();
    if (hd.mode == kModeSeeds) return;   // seeds carry their positions: nothing to relabel
    // 5. relabel every key with its group head's position
    int hidx = carry;
    for (int j = 0; j < R; ++j) {
        const int i = lane * R + j;
        if (i >= n) break;
        if (headm >> j & 1) hidx = i;
        if (keym >> j & 1) {
            const unsigned long long c = sm.s.srt[i];
            key_out(g, hd, lp, cum, (uint32_t)(c & 0x7FFFFFFFu), sm.s.pos[hidx]);
        }
    }
    __syncwarp();
}

// Bitmap path: one bucket b (2^bshift gids from gid0) with any number of elements.
__device__ void compact_bitmap(const GraphDev &g, const HopDev &hd, const LpDev &lp, const int64_t *cum,
                               CompactSmem &sm, int32_t t, int u, int64_t b, uint32_t k0, uint32_t nk, uint32_t m0,
                               uint32_t nm)
{
    const CompactDev &cd = hd.cd;
    const int lane = lane_id();
    const int level = hd.h + 1;
    const uint32_t *mg_in = level > 0 ? cd.mg[(level - 1) & 1] : nullptr;
    const int32_t *mp_in = level > 0 ? cd.mp[(level - 1) & 1] : nullptr;
    const int WL = 1 << (g.bshift - 10);   // words per lane (blocked: lane owns [WL lane, WL lane + WL))
    const int64_t gid0 = g.off[u] + ((b - g.bbase[u]) << g.bshift);
    for (int q = 0; q < WL; ++q) {
        sm.b.a[lane * WL + q] = 0u;
        sm.b.m[lane * WL + q] = 0u;
    }
    __syncwarp();
    for (uint32_t i = lane; i < nm; i += 32) {
        const uint32_t x = __ldcg(mg_in + m0 + i) - (uint32_t)gid0;
        atomicOr(sm.b.m + (x >> 5), 1u << (x & 31));
    }
    for (uint32_t i = lane; i < nk; i += 32) {
        const uint32_t x = __ldcg(cd.keys + k0 + i) - (uint32_t)gid0;
        const uint32_t old = atomicOr(sm.b.a + (x >> 5), 1u << (x & 31));
        if (hd.mode == kModeSeeds && (old >> (x & 31) & 1)) atomicOr(hd.meta + kMetaErr, kErrSeedDup);
    }
    __syncwarp();
    uint32_t ca = 0, cn = 0;
    for (int q = 0; q < WL; ++q) {
        const uint32_t a = sm.b.a[lane * WL + q], m = sm.b.m[lane * WL + q];
        ca += __popc(a | m);
        cn += __popc(a & ~m);
    }
    const uint32_t cnt = (ca << 16) | cn;   // <= 4096 per bucket
    const uint32_t incl = warp_incl_scan(cnt);
    const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
    uint32_t pa = (incl - cnt) >> 16, pn = (incl - cnt) & 0xFFFFu;
    for (int q = 0; q < WL; ++q) {
        const uint32_t a = sm.b.a[lane * WL + q], m = sm.b.m[lane * WL + q];
        sm.b.pa[lane * WL + q] = (uint16_t)pa;
        sm.b.pn[lane * WL + q] = (uint16_t)pn;
        pa += __popc(a | m);
        pn += __popc(a & ~m);
    }
    const uint32_t tot_new = tot & 0xFFFFu, tot_all = tot >> 16;
    uint32_t g_excl = 0, t_excl = 0;
    if (lane == 0) lookback(g, cd, t, u, tot_new, hd.mode == kModeSeeds ? 0u : tot_new, g_excl, t_excl);
    g_excl = __shfl_sync(0xffffffffu, g_excl, 0);
    t_excl = __shfl_sync(0xffffffffu, t_excl, 0);
    __syncwarp();
    const int32_t before = level_nodes_before(hd, u);
    const uint32_t mo = m0 + g_excl;   // merged member list of the next level: this bucket's first slot
    if (hd.mode == kModeSeeds) {
        // the seeds carry their positions: each (unique) key writes its merged entry
        if (!hd.last)
            for (uint32_t i = lane; i < nk; i += 32) {
                const uint32_t gid = __ldcg(cd.keys + k0 + i);
                const uint32_t x = gid - (uint32_t)gid0;
                const uint32_t w = x >> 5, low = (1u << (x & 31)) - 1u;
                const uint32_t r = sm.b.pa[w] + __popc((sm.b.a[w] | sm.b.m[w]) & low);
                cd.mg[level & 1][mo + r] = gid;
                cd.mp[level & 1][mo + r] = (int32_t)__ldcg(cd.kidx + k0 + i);
            }
    } else {
        for (int q = 0; q < WL; ++q) {
            const int w = lane * WL + q;
            const uint32_t a = sm.b.a[w], m = sm.b.m[w];
            uint32_t all = a | m;
            const uint32_t nw = a & ~m;
            uint32_t r = sm.b.pa[w];
            while (all) {
                const int bit = __ffs(all) - 1;
                all &= all - 1;
                const uint32_t gid = (uint32_t)gid0 + (uint32_t)(32 * w + bit);
                const uint32_t low = (1u << bit) - 1u;
                int32_t pos;
                if (nw >> bit & 1) {
                    pos = before + (int32_t)(t_excl + sm.b.pn[w] + __popc(nw & low));
                    emit_node(hd, u, pos, gid);
                } else {
                    pos = __ldcg(mp_in + m0 + (r - sm.b.pn[w] - __popc(nw & low)));
                }
                if (!hd.last) {
                    cd.mg[level & 1][mo + r] = gid;
                    cd.mp[level & 1][mo + r] = pos;
                }
                ++r;
            }
        }
    }
    if (!hd.last && lane == 0 && tot_all) atomicAdd(cd.mcnt + b, tot_all);
    if (hd.mode == kModeSeeds) return;
    // relabel every key
    for (uint32_t i = lane; i < nk; i += 32) {
        const uint32_t gid = __ldcg(cd.keys + k0 + i);
        const uint32_t pay = __ldcg(cd.kidx + k0 + i);
        const uint32_t x = gid - (uint32_t)gid0;
        const uint32_t w = x >> 5, bit = x & 31, low = (1u << bit) - 1u;
        const uint32_t a = sm.b.a[w], m = sm.b.m[w];
        int32_t pos;
        if (m >> bit & 1) {
            const uint32_t mem_rank = (sm.b.pa[w] - sm.b.pn[w]) + __popc(m & low);
            pos = __ldcg(mp_in + m0 + mem_rank);
        } else {
            pos = before + (int32_t)(t_excl + sm.b.pn[w] + __popc((a & ~m) & low));
        }
        key_out(g, hd, lp, cum, pay, pos);
    }
    __syncwarp();
}

// A warp per task, in ticket order.  The last task of each type records |S_level[u]|.
__device__ void phase_compact(const GraphDev &g, const HopDev &hd, const LpDev &lp, CompactSmem *smem)
{
    const CompactDev &cd = hd.cd;
    const int lane = lane_id();
    const int level = hd.h + 1;
    CompactSmem &sm = smem[threadIdx.x >> 5];
    int64_t cum[EG_MAX_REL + 1];
    level_keys(g, hd, lp, cum);
    const int32_t ntask = *(volatile int32_t *)(hd.meta + kMetaTasks + level);
    uint32_t *ticket = (uint32_t *)(hd.meta + kMetaTicket + level);
    for (;;) {
        int32_t t = 0;
        if (lane == 0) t = (int32_t)atomicAdd(ticket, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= ntask) break;
        const int64_t b0 = __ldcg(cd.tstart + t), b1 = __ldcg(cd.tstart + t + 1);
        const uint32_t k0 = __ldcg(cd.kofs + b0), k1 = __ldcg(cd.kofs + b1);
        const uint32_t m0 = __ldcg(cd.mofs + b0), m1 = __ldcg(cd.mofs + b1);
        const int u = type_of_bucket(g, b0);
        const uint32_t nk = k1 - k0, nm = m1 - m0;
        if (b1 - b0 == 1 && (nk + nm > (uint32_t)kBigBucket || g.compact_bitmap))
            compact_bitmap(g, hd, lp, cum, sm, t, u, b0, k0, nk, m0, nm);
        else
            compact_sort(g, hd, lp, cum, sm, t, u, b0, k0, nk, m0, nm);
        // the last task of its type: |S_level[u]| = |F[u]| + new vertices of the type (its own
        // inclusive look-back word; the seeds' sizes come from the seed split)
        if (lane == 0 && b1 == g.bbase[u + 1] && hd.mode != kModeSeeds) {
            const unsigned long long w = ((volatile unsigned long long *)cd.lb)[t];
            meta_nodes(hd.meta, level)[u] = level_nodes_before(hd, u) + (int32_t)((uint32_t)w & 0x7FFFFFFFu);
        }
    }
}

}  // namespace eg
