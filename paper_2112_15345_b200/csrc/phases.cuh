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
//   bitcount / emit   new sources of the hop in gid order after the dst prefix
//   relabel           local src ids = positions in src_nodes
#pragma once
#include "common.cuh"

namespace eg {

__device__ __forceinline__ uint32_t lanemask_lt() { return (1u << lane_id()) - 1u; }

// ============================================================================ seed split

// Seeds (caller order, mixed types) -> F_0[u] (stable per type) + pos[] for the
// dst-prefix relabel; flags out-of-range and duplicate seeds.  One block.
__device__ void phase_seed_split(const GraphDev &g, const HopDev &hd, const int64_t *__restrict__ slot_seeds)
{
    // the caller's buffer when it is device-accessible, else the slot's staged copy
    const int64_t *__restrict__ seeds = hd.dyn[2] ? (const int64_t *)hd.dyn[2] : slot_seeds;
    __shared__ int32_t wcnt[32][EG_MAX_VT];   // per warp, per type: count, then exclusive offset
    __shared__ int32_t base[EG_MAX_VT];
    // pointers hoisted into registers: HopDev lives in global memory and every store
    // below could alias it, so reading fields inside the loops would reload them
    int32_t *const pos = hd.pos;
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
        if (vt >= 0) {
            const int32_t p = wcnt[w][vt] + rank;
            if (p < hd.cap_nodes[vt]) {
                hd.nodes[vt][p] = gid;
                if (atomicCAS(pos + gid, -1, p) != -1) atomicOr(meta + kMetaErr, kErrSeedDup);
                const int64_t bit = g.boff[vt] + (gid - g.off[vt]);
                atomicOr(hd.members + (bit >> 5), 1u << (bit & 31));
            } else {
                atomicOr(meta + kMetaErr, kErrCapacity);
            }
        }
        __syncthreads();
    }
    if (threadIdx.x < g.n_vt)
        meta_nodes(meta, 0)[threadIdx.x] = min(base[threadIdx.x], hd.cap_nodes[threadIdx.x]);
    __syncthreads();
}

// ============================================================================ count + scan

// Virtual blocks (r, b), b < kScanBlocks: count c for the dst items of chunk b of
// F_h[t(r)] into the block indptr slots, record (owner, CSC row start) and d for
// the sampler, enqueue the items that need a selection; per-chunk sums -> partial.
__device__ void phase_count(const GraphDev &g, const HopDev &hd, int bid, int nb)
{
    __shared__ int32_t sh[33];
    const int32_t *nF = meta_nodes(hd.meta, hd.h);
    if (bid == 0 && threadIdx.x < g.n_vt)   // S_h starts as F_h; emit adds the new ones
        meta_nodes(hd.meta, hd.h + 1)[threadIdx.x] = nF[threadIdx.x];
    for (int vb = bid; vb < kScanBlocks * g.n_rel; vb += nb) {
        const int r = vb / kScanBlocks, b = vb % kScanBlocks;
        const RelDev &R = g.rel[r];
        const int t = R.dst_vt;
        const int k = hd.fanout[r];
        const int64_t n = nF[t];
        const int64_t chunk = (n + kScanBlocks - 1) / kScanBlocks;
        const int64_t lo = b * chunk, hi = min(n, lo + chunk);
        const int64_t *const nodes = hd.nodes[t];
        int64_t *const ibase = hd.ibase[r];
        int32_t *const ideg = hd.ideg[r];
        int32_t *const bip = hd.indptr[r];
        uint64_t *const selq = hd.selq;
        uint32_t *const selc = (uint32_t *)(hd.meta + kMetaSel + hd.h);
        int32_t sum = 0;
        for (int64_t t0 = lo; t0 < hi; t0 += blockDim.x) {   // block-uniform trip count
            const int64_t i = t0 + threadIdx.x;
            bool sel = false;
            if (i < hi) {
                int32_t c = 0;
                if (k != 0) {
                    const int64_t tid = nodes[i] - g.off[t];
                    const int p = owner_of(g, t, tid);
                    const int64_t x = tid - g.bounds[t][p];
                    const int64_t *ip = R.indptr[p];
                    const int64_t b0 = ip[x], d = ip[x + 1] - b0;
                    const bool all = (k < 0 || d <= k);
                    c = (int32_t)(all ? d : k);
                    sel = !all;
                    ibase[i] = ((int64_t)p << 56) | b0;
                    ideg[i] = (int32_t)d;
                }
                bip[i] = c;
                sum += c;
            }
            // heavy items (d > kHeavyD): split into tasks of kHeavyChunk keys for several warps
            if (sel && k <= kHeavyMaxK && ideg[i] > kHeavyD) {
                const int64_t d = ideg[i];
                const uint32_t nch = (uint32_t)((d + kHeavyChunk - 1) / kHeavyChunk);
                const uint32_t hs = atomicAdd((uint32_t *)(hd.meta + kMetaHeavy + hd.h), 1u);
                if (hs < (uint32_t)kMaxHeavy) {
                    const uint32_t t0 = atomicAdd((uint32_t *)(hd.meta + kMetaHeavyQ + hd.h), nch);
                    if (t0 + nch <= (uint32_t)kMaxHeavyTasks) {
                        hd.heavy_items[hs] = ((uint64_t)r << 32) | (uint64_t)i;
                        hd.heavy_cnt[hs] = 0;
                        hd.heavy_done[hs] = 0;
                        for (uint32_t c = 0; c < nch; ++c) hd.heavyq[t0 + c] = (hs << 16) | c;
                        sel = false;
                    } else {   // task list full: mark the reserved entries void, item goes to the normal queue
                        for (uint32_t c = 0; c < nch && t0 + c < (uint32_t)kMaxHeavyTasks; ++c)
                            hd.heavyq[t0 + c] = 0xFFFFFFFFu;
                    }
                }
            }
            const uint32_t m = __ballot_sync(0xffffffffu, sel);
            if (m) {
                uint32_t q = 0;
                if (lane_id() == 0) q = atomicAdd(selc, (uint32_t)__popc(m));
                q = __shfl_sync(0xffffffffu, q, 0);
                if (sel) selq[q + __popc(m & lanemask_lt())] = ((uint64_t)r << 32) | (uint64_t)i;
            }
        }
        sum = block_sum(sum, sh);
        if (threadIdx.x == 0) hd.partial[r * kScanBlocks + b] = sum;
    }
}

// Exclusive scan of the counts in place -> block indptr; nnz(h, r).  Also clears the
// chunk-group sums used by this hop's compaction.
__device__ void phase_scan(const GraphDev &g, const HopDev &hd, int bid, int nb, int32_t n_groups)
{
    __shared__ int32_t sh[33];
    if (bid == 0)
        for (int i = threadIdx.x; i < n_groups; i += blockDim.x) hd.chunk_pre[i] = 0;
    for (int vb = bid; vb < kScanBlocks * g.n_rel; vb += nb) {
        const int r = vb / kScanBlocks, b = vb % kScanBlocks;
        const int t = g.rel[r].dst_vt;
        const int64_t n = meta_nodes(hd.meta, hd.h)[t];
        const int64_t chunk = (n + kScanBlocks - 1) / kScanBlocks;
        const int64_t lo = b * chunk, hi = min(n, lo + chunk);
        int32_t s = 0;
        const int32_t *const partial = hd.partial + r * kScanBlocks;
        for (int j = threadIdx.x; j < b; j += blockDim.x) s += partial[j];
        int32_t carry = block_sum(s, sh);
        int32_t *const ip = hd.indptr[r];
        for (int64_t t0 = lo; t0 < hi; t0 += blockDim.x) {
            const int64_t i = t0 + threadIdx.x;
            const int32_t v = i < hi ? ip[i] : 0;
            int32_t tot;
            const int32_t ex = block_excl_scan(v, sh, &tot);
            if (i < hi) ip[i] = carry + ex;
            carry += tot;
        }
        if (b == kScanBlocks - 1 && threadIdx.x == 0) {
            ip[n] = carry;
            meta_nnz(hd.meta, hd.h)[r] = carry;
        }
    }
}

// ============================================================================ sampling

struct Item {
    const int32_t *pos;     // the batch's gid -> position map (read only here)
    uint32_t *bitmap;       // the batch's new-vertex bitmap
    int64_t bit_base;       // boff[s(r)] - off[s(r)]: bitmap bit of gid = bit_base + gid
    uint32_t soff;          // off[s(r)]
    int64_t ebase;          // global CSC position of this dst's first edge
    const int32_t *ix;      // src tids of this dst's in-edges
    uint32_t *src_out;      // this item's output slots
    int64_t *eid_out;
};

// Mark the source in the hop's bitmap (the first step of the compaction, fused into
// sampling).  Fire-and-forget RED.OR, no load: sources already in the batch are
// cleared from the bitmap by phase_bitcount (one check per unique source instead of
// a dependent pos[] load per sampled edge).
__device__ __forceinline__ void mark_src(uint32_t *bitmap, uint32_t gid, int64_t bit_base)
{
    const int64_t bit = bit_base + gid;
    atomicOr(bitmap + (bit >> 5), 1u << (bit & 31));   // result unused: RED
}

__device__ __forceinline__ void emit_edge(const HopDev &, const Item &it, int32_t slot, int64_t j)
{
    const uint32_t gid = it.soff + (uint32_t)__ldg(it.ix + j);
    it.src_out[slot] = gid;
    it.eid_out[slot] = it.ebase + j;
    mark_src(it.bitmap, gid, it.bit_base);
}

// Four keys key32(seed, h, r, v, 4q .. 4q+3) from one Philox call.
__device__ __forceinline__ void keys4(uint32_t q, uint32_t v_lo, uint32_t v_hi, uint32_t hr, uint32_t k0,
                                      uint32_t k1, uint32_t w[4])
{
    uint32_t c0 = q, c1 = v_lo, c2 = v_hi, c3 = hr;
    philox4x32_10(c0, c1, c2, c3, k0, k1);
    w[0] = c0; w[1] = c1; w[2] = c2; w[3] = c3;
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
__device__ void select_small(const HopDev &hd, const Item &it, int64_t d, int k, uint32_t v_lo, uint32_t v_hi,
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
    while (s > 0) {
        const int b = s - 1;
        uint32_t c0 = 0, cm = 0;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const bool match = (vm >> t & 1) && (s == 32 || (w[t] >> s) == (P >> s));
            cm += match;
            c0 += match && !((w[t] >> b) & 1u);
        }
        cm = __reduce_add_sync(0xffffffffu, cm);
        if ((int)cm == krem) break;
        c0 = __reduce_add_sync(0xffffffffu, c0);
        if (krem > (int)c0) {
            krem -= (int)c0;
            P |= 1u << b;
        }
        s = b;
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
    int slot = warp_incl_scan(cs) - cs;
#pragma unroll
    for (int t = 0; t < 4; ++t)
        if (sel >> t & 1) emit_edge(hd, it, slot++, 4 * lane + t);
}

// Fast selection for k <= kSelMaxK: one pass over the d keys keeps the candidates
// below a threshold T (expected 2k + 32 of them) in shared memory, in ascending j;
// the k smallest composites among them are found by a register radix select (m <= 128)
// or rank counting, and emitted in ascending j.  Falls back to select_generic if the candidate count is < k or
// exceeds the slots (both astronomically rare; the result is identical).
__device__ void select_fast(const HopDev &hd, const Item &it, int64_t d, int k, uint32_t v_lo, uint32_t v_hi,
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
        // (slot c = lane + 32 i); two warp reductions per bit, early exit once every
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
        while (s > 0) {
            const int b = s - 1;
            uint32_t c0 = 0, cm = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const bool match = val[i] && (s == 32 || (key[i] >> s) == (P >> s));
                cm += match;
                c0 += match && !((key[i] >> b) & 1u);
            }
            cm = __reduce_add_sync(0xffffffffu, cm);
            if ((int)cm == krem) break;                 // all matching keys are selected
            c0 = __reduce_add_sync(0xffffffffu, c0);
            if (krem > (int)c0) {
                krem -= (int)c0;
                P |= 1u << b;
            }
            s = b;
        }
        // selected: key below P on the decided bits, or matching them and among the first
        // krem such candidates in slot (= ascending j) order
        int eq_seen = 0;
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
            if (sel) emit_edge(hd, it, out + __popc(bs & lanemask_lt()), (int64_t)(uint32_t)cand[c]);
            out += __popc(bs);
        }
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
__device__ void heavy_task(const GraphDev &g, const HopDev &hd, uint32_t task, uint32_t seed_lo, uint32_t seed_hi,
                           uint64_t *cand)
{
    const int lane = lane_id();
    const uint32_t hs = task >> 16, c = task & 0xFFFFu;
    const uint64_t e = hd.heavy_items[hs];
    const int r = (int)(e >> 32);
    const int64_t i = (int64_t)(e & 0xFFFFFFFFu);
    const RelDev &R = g.rel[r];
    const int64_t ib = hd.ibase[r][i];
    const int64_t d = hd.ideg[r][i];
    const int64_t v = hd.nodes[R.dst_vt][i];
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
    const int32_t pos0 = hd.indptr[r][i];
    const int p = (int)(ib >> 56);
    const int64_t base0 = ib & ((1ll << 56) - 1);
    Item itm;
    itm.pos = hd.pos;
    itm.bitmap = hd.bitmap;
    itm.bit_base = g.boff[R.src_vt] - g.off[R.src_vt];
    itm.soff = (uint32_t)g.off[R.src_vt];
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
        while (s > 0) {
            const int b = s - 1;
            uint32_t c0 = 0, cm = 0;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const bool match = val[t] && (s == 32 || (key[t] >> s) == (P >> s));
                cm += match;
                c0 += match && !((key[t] >> b) & 1u);
            }
            cm = __reduce_add_sync(0xffffffffu, cm);
            if ((int)cm == krem) break;
            c0 = __reduce_add_sync(0xffffffffu, c0);
            if (krem > (int)c0) {
                krem -= (int)c0;
                P |= 1u << b;
            }
            s = b;
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
__device__ void phase_select(const GraphDev &g, const HopDev &hd, int bid, int nb, uint64_t *cand)
{
    const int lane = lane_id();
    const uint32_t seed_lo = (uint32_t)hd.dyn[0], seed_hi = (uint32_t)(hd.dyn[0] >> 32);
    const int32_t *const pos = hd.pos;
    uint32_t *const bitmap = hd.bitmap;
    const uint64_t *const selq = hd.selq;
    (void)bid;
    (void)nb;
    // ---- heavy chunk tasks
    const uint32_t ntask = min(*(const volatile uint32_t *)(hd.meta + kMetaHeavyQ + hd.h), (uint32_t)kMaxHeavyTasks);
    uint32_t *hnext = (uint32_t *)(hd.meta + kMetaHeavyNext + hd.h);
    for (;;) {
        uint32_t t = 0;
        if (lane == 0) t = atomicAdd(hnext, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= ntask) break;
        const uint32_t task = hd.heavyq[t];
        if (task != 0xFFFFFFFFu) heavy_task(g, hd, task, seed_lo, seed_hi, cand);
    }
    // ---- selections (d > k): warp per item
    const int64_t nsel = *(const volatile uint32_t *)(hd.meta + kMetaSel + hd.h);
    uint32_t *snext = (uint32_t *)(hd.meta + kMetaSelNext + hd.h);
    for (;;) {
        uint32_t wi = 0;
        if (lane == 0) wi = atomicAdd(snext, 1u);
        wi = __shfl_sync(0xffffffffu, wi, 0);
        if ((int64_t)wi >= nsel) break;
        const int64_t w = wi;
        const uint64_t e = selq[w];
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
        itm.pos = pos;
        itm.bitmap = bitmap;
        itm.bit_base = g.boff[R.src_vt] - g.off[R.src_vt];
        itm.soff = (uint32_t)g.off[R.src_vt];
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

// Sampling of one hop, part 2: the full-neighbourhood items (d <= k or k = -1) as
// segmented copies, 32 items per warp, 4 independent load chains per lane.
__device__ void phase_copy(const GraphDev &g, const HopDev &hd, int bid, int nb)
{
    const int warps = blockDim.x >> 5;
    const int lane = lane_id();
    const int64_t gw = (int64_t)bid * warps + (threadIdx.x >> 5), nw = (int64_t)nb * warps;
    uint32_t *const bitmap = hd.bitmap;
    // ---- full neighbourhoods: segmented copy over groups of 32 items
    const int32_t *nF = meta_nodes(hd.meta, hd.h);
    int64_t cum[EG_MAX_REL + 1];
    cum[0] = 0;
    for (int r = 0; r < g.n_rel; ++r) cum[r + 1] = cum[r] + (hd.fanout[r] != 0 ? nF[g.rel[r].dst_vt] : 0);
    const int64_t total = cum[g.n_rel];
    for (int64_t g0 = gw * 32; g0 < total; g0 += nw * 32) {
        const int64_t it = g0 + lane;
        int r = 0;
        int32_t pos0 = 0, cnt = 0, d = 0;
        int64_t ib = 0;
        uint32_t *srcp = nullptr;
        int64_t *eidp = nullptr;
        if (it < total) {
            while (it >= cum[r + 1]) ++r;
            const int64_t i = it - cum[r];
            const int32_t *bip = hd.indptr[r];
            pos0 = bip[i];
            cnt = bip[i + 1] - pos0;
            if (cnt > 0) {
                ib = hd.ibase[r][i];
                d = hd.ideg[r][i];
            }
            srcp = hd.src[r] + pos0;
            eidp = hd.eids[r] + pos0;
        }
        const int k = hd.fanout[r];
        const bool copy = cnt > 0 && !(k >= 0 && d > k);
        const int32_t c = copy ? cnt : 0;
        const int32_t incl = warp_incl_scan(c);
        const int32_t tot = __shfl_sync(0xffffffffu, incl, 31);
        const int32_t excl = incl - c;
        constexpr int U = 4;   // slots per lane per round: U independent load chains in flight
        for (int32_t b0 = 0; b0 < tot; b0 += 32 * U) {
            uint32_t gid[U];
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
                    gid[q] = (uint32_t)g.off[R.src_vt];
                    bb[q] = g.boff[R.src_vt] - g.off[R.src_vt];
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
                    mark_src(bitmap, gid[q], bb[q]);
                }
        }
    }
}

// ============================================================================ compaction

// Popcount of each bitmap chunk (virtual block per chunk, one uint4 per thread) and
// the sums of groups of kGroupChunks chunks.
constexpr int kGroupChunks = 256;

__device__ void phase_bitcount(const GraphDev &, const HopDev &hd, int bid, int nb, int32_t n_chunks)
{
    static_assert(kChunkWords == 4 * 256, "one uint4 per thread");
    __shared__ int32_t sh[33];
    for (int c = bid; c < n_chunks; c += nb) {
        const int64_t wq = (int64_t)c * (kChunkWords / 4) + threadIdx.x;
        uint4 *ap = reinterpret_cast<uint4 *>(hd.bitmap) + wq;
        const uint4 a = __ldcg(ap);
        int32_t v = 0;
        if (a.x | a.y | a.z | a.w) {
            const uint4 m = __ldcg(reinterpret_cast<const uint4 *>(hd.members) + wq);
            v = __popc(a.x & ~m.x) + __popc(a.y & ~m.y) + __popc(a.z & ~m.z) + __popc(a.w & ~m.w);
            if (v == 0) *ap = make_uint4(0, 0, 0, 0);   // only members marked: consumed here, emit skips
        }
        v = block_sum(v, sh);
        if (threadIdx.x == 0) {
            hd.chunk_cnt[c] = v;
            if (v) atomicAdd(hd.chunk_pre + c / kGroupChunks, v);
        }
    }
}

// number of set bits in chunks [0, c): group sums + the chunks of c's group before it
__device__ __forceinline__ int32_t bits_before(const HopDev &hd, int c, int32_t *sh)
{
    const int gi = c / kGroupChunks;
    int32_t s = 0;
    for (int j = threadIdx.x; j < gi; j += blockDim.x) s += __ldcg(hd.chunk_pre + j);
    for (int j = gi * kGroupChunks + threadIdx.x; j < c; j += blockDim.x) s += __ldcg(hd.chunk_cnt + j);
    return block_sum(s, sh);
}

// New vertices of each chunk, in gid order: append to the node array of their type,
// set pos[], fold them into the members, clear the marks.  Virtual block per chunk,
// one word per thread (1024 threads).
__device__ void phase_emit(const GraphDev &g, const HopDev &hd, int bid, int nb, int32_t n_chunks)
{
    __shared__ int32_t sh[33];   // blockDim.x == kChunkWords == 1024
    for (int c = bid; c < n_chunks; c += nb) {
        const int32_t mine = __ldcg(hd.chunk_cnt + c);
        if (mine == 0) continue;   // block-uniform
        const int64_t bit0 = (int64_t)c * kChunkBits;
        int u = 0;
        while (bit0 >= g.boff[u + 1]) ++u;
        const int fc = (int)(g.boff[u] / kChunkBits);
        const int32_t prior = bits_before(hd, c, sh) - bits_before(hd, fc, sh);
        const int32_t nF = meta_nodes(hd.meta, hd.h)[u];
        // one bitmap word per thread (blockDim.x == kChunkWords)
        const int64_t wi = (int64_t)c * kChunkWords + threadIdx.x;
        uint32_t *wp = hd.bitmap + wi;
        uint32_t *mp = hd.members + wi;
        const uint32_t x = __ldcg(wp);
        const uint32_t mm = x ? __ldcg(mp) : 0u;
        uint32_t word = x & ~mm;
        const int32_t pc = __popc(word);
        int32_t tot;
        int32_t position = nF + prior + block_excl_scan(pc, sh, &tot);
        if (pc) {
            const int64_t gbase = (g.off[u] - g.boff[u]) + wi * 32;   // gid of bit 0 of word wi
            int64_t *const nodes = hd.nodes[u];
            int32_t *const pos = hd.pos;
            int32_t *const meta = hd.meta;
            const int32_t cap = hd.cap_nodes[u];
            *mp = mm | word;                                          // now members
            while (word) {
                const int b = __ffs(word) - 1;
                word &= word - 1;
                const int64_t gid = gbase + b;
                if (position < cap) {
                    nodes[position] = gid;
                    pos[gid] = position;
                } else {
                    atomicOr(meta + kMetaErr, kErrCapacity);
                }
                ++position;
            }
        }
        if (x) *wp = 0u;                                              // marks consumed
        if (threadIdx.x == 0) atomicAdd(meta_nodes(hd.meta, hd.h + 1) + u, mine);
    }
}

// indices = pos[src]: the local id of every sampled src in S_h[s(r)].
__device__ void phase_relabel(const GraphDev &g, const HopDev &hd, int bid, int nb)
{
    const int32_t *const pos = hd.pos;
    const int64_t stride = (int64_t)nb * blockDim.x;
    for (int r = 0; r < g.n_rel; ++r) {
        const int64_t n = meta_nnz(hd.meta, hd.h)[r];
        const uint32_t *const src = hd.src[r];
        int32_t *const idx = hd.indices[r];
        for (int64_t e = bid * (int64_t)blockDim.x + threadIdx.x; e < n; e += stride) idx[e] = __ldcg(pos + src[e]);
    }
}

// End of batch: pos[] back to -1 for every vertex of the batch.
__device__ void phase_reset(const GraphDev &g, const HopDev &hd, int32_t level, int bid, int nb)
{
    const int32_t *n = meta_nodes(hd.meta, level);
    int64_t cum[EG_MAX_VT + 1];
    cum[0] = 0;
    for (int u = 0; u < g.n_vt; ++u) cum[u + 1] = cum[u] + min(n[u], hd.cap_nodes[u]);
    int32_t *const pos = hd.pos;
    uint32_t *const members = hd.members;
    for (int u = 0; u < g.n_vt; ++u) {
        const int64_t *const nodes = hd.nodes[u];
        const int64_t n = cum[u + 1] - cum[u];
        for (int64_t i = bid * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)nb * blockDim.x) {
            const int64_t gid = nodes[i];
            if (gid >= g.off[u] && gid < g.off[u + 1]) {
                pos[gid] = -1;
                const int64_t bit = g.boff[u] + (gid - g.off[u]);
                atomicAnd(members + (bit >> 5), ~(1u << (bit & 31)));
            }
        }
    }
}

}  // namespace eg
