// egonet.cu -- the C ABI (include/egonet.h): context, store, per-batch orchestration.
//
// Per batch (eg_sample_blocks), all on the context's stream, no host sync until the
// end (sizes live on the device; buffers are sized by host-computed upper bounds):
//   seed_split                                  F_0 per type, pos[] of the seeds
//   for each hop h:
//     count -> scan                             block indptr (min(d,k) per dst)
//     sample                                    warp per (dst, relation), key32
//     mark -> bitcount -> emit -> relabel       frontier + compaction
//   finish                                      last relabel + member bits cleared
//   one D2H of the batch counters (+ error bits)
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "kernels.h"

using namespace eg;

namespace {

const char *kVersion = "egonet 0.1.0 (sm_100a)";

struct ShardRel {
    int32_t src_vt, dst_vt;
    int64_t n_local_dst, n_local_edges, edge_base, max_degree;
    cudaIpcMemHandle_t indptr_h, indices_h;
    int64_t indptr_off, indices_off;
};

struct ShardFeat {
    int64_t row_bytes, n_rows;
    cudaIpcMemHandle_t h;
    int64_t off;
    int32_t has;
};

struct ShardBlob {
    uint32_t magic, version;
    int32_t rank, world, n_vt, n_rel;
    int64_t vt_counts[EG_MAX_VT];
    int64_t bounds[EG_MAX_VT][EG_MAX_RANKS + 1];
    ShardRel rel[EG_MAX_REL];
    ShardFeat feat[EG_MAX_VT];
};
constexpr uint32_t kBlobMagic = 0x45474F4E;  // 'EGON'

struct TimedPair {
    cudaEvent_t a, b;
    int kind;  // 0 sample, 1 gather
};

}  // namespace

// A lane: one stream.  Launches on different lanes are independent and run concurrently
// (the asynchronous mini-batch pipeline); launches on one lane are ordered.  Every
// batch's state (incl. its compaction state) lives in its slot: batch-sized, not graph-sized.
struct Lane {
    cudaStream_t stream = nullptr;
    cudaEvent_t ready = nullptr;     // caller stream -> lane ordering
};

// per (batch, hop): heavy items, their counters, candidate buffers and chunk tasks
size_t heavy_bytes(int64_t mh, int64_t mt)
{
    return sizeof(QEntry) * mh + 2 * sizeof(uint32_t) * mh + sizeof(uint64_t) * mh * kHeavyCap +
           sizeof(uint32_t) * mt;
}

// A batch "plan": everything fixed by (hops, fanouts, seed capacity, features, bundle
// size B): upper bounds, the memory layout of one batch (repeated B times), its slots.
struct Slot;
struct Plan {
    int32_t n_hops = 0;
    int32_t fanouts[EG_MAX_HOPS * EG_MAX_REL] = {};
    int64_t n_cap = 0;
    bool features = false;
    int32_t B = 1;
    int64_t capF[EG_MAX_HOPS + 1][EG_MAX_VT] = {};
    int64_t capE[EG_MAX_HOPS][EG_MAX_REL] = {};
    // per-batch layout (offsets inside a batch region of `stride` bytes)
    size_t o_meta = 0, o_dyn = 0, o_seeds = 0, stride = 0;
    size_t o_nodes[EG_MAX_VT] = {}, o_feat[EG_MAX_VT] = {};
    size_t o_ip[EG_MAX_HOPS][EG_MAX_REL] = {}, o_ix[EG_MAX_HOPS][EG_MAX_REL] = {}, o_ei[EG_MAX_HOPS][EG_MAX_REL] = {},
           o_src[EG_MAX_HOPS][EG_MAX_REL] = {},
           o_selq[EG_MAX_HOPS] = {}, o_copyq[EG_MAX_HOPS] = {}, o_tiny16[EG_MAX_HOPS] = {}, o_heavy[EG_MAX_HOPS] = {};
    int64_t selq_items[EG_MAX_HOPS] = {};
    int32_t max_heavy[EG_MAX_HOPS] = {}, max_heavy_tasks[EG_MAX_HOPS] = {};
    // batch-local compaction state (compact.cuh): meta | kcnt | mcnt contiguous (one memset)
    size_t o_elems = 0, o_tnew = 0, o_ftask = 0, o_kcur = 0;
    size_t o_clb[EG_MAX_HOPS] = {};
    int32_t count_tiles[EG_MAX_HOPS] = {};
    size_t o_kcnt = 0, o_mcnt = 0, o_tlb = 0, o_kofs = 0, o_mofs = 0, o_tstart = 0, o_mg[2] = {}, o_mp[2] = {}, zero_bytes = 0;
    int64_t cap_keys = 0, cap_members = 0;
    // link prediction (NEXT-3): n_cap = positives capacity; seeds <= n_cap * (2 + n_neg)
    bool lp = false;
    int32_t n_neg = 0;
    size_t o_lp_src = 0, o_lp_dst = 0, o_lp_neg = 0, o_lp_pairs = 0;
    size_t o_bd = 0, total = 0;      // BatchDev header, then B batch regions
    int32_t n_kernels = 0;
    std::vector<Slot *> slots;
    char *batch_base(char *mem, int b) const { return mem + o_bd + align_bd() + (size_t)b * stride; }
    static size_t align_bd() { return (sizeof(BatchDev) + 255) / 256 * 256; }
};

// One launch's worth of device memory (B batches) with its captured CUDA graph:
//   H2D {rng_seed, n_seeds} x B -> memset counters -> seed split -> per hop (count, scan,
//   sample, bitcount, emit) -> relabel -> reset -> [gather] -> D2H counters.
struct Slot {
    Plan *plan = nullptr;
    char *mem = nullptr;
    int32_t *h_meta = nullptr;   // pinned, B x kMetaSize
    uint64_t *h_dyn = nullptr;   // pinned, B x kDyn launch parameters (common.cuh)
    cudaGraphExec_t exec = nullptr;
    cudaEvent_t done = nullptr, s0 = nullptr, s1 = nullptr, g0 = nullptr, g1 = nullptr;
    int refs = 0;                // live eg_blocks handles of the last launch
    bool used = false, timed = false, finished = false;
    int lane = 0;
    int32_t gather_path = -1;    // kernel the captured gather node uses (eg_gather_path)
    std::vector<cudaEvent_t> tev;        // EG_TRACE: one event after each stage of the graph
    std::vector<std::string> tlab;
};

struct eg_ctx {
    int32_t rank = 0, world = 1, device = 0;
    cudaStream_t stream = nullptr;
    bool broken = false, loaded = false, peers_ready = false;
    std::string err = "ok";
    GraphDev g{};
    FeatDev f{};
    int64_t vt_counts[EG_MAX_VT] = {};
    int64_t rel_edges_total[EG_MAX_REL] = {};
    int64_t rel_max_degree[EG_MAX_REL] = {};
    int64_t n_total = 0;
    // own shard (for export)
    eg_relation own_rel[EG_MAX_REL] = {};
    eg_features own_feat[EG_MAX_VT] = {};
    bool host_feat[EG_MAX_VT] = {};                  // feature rows in pinned host memory (PCIe)
    GatherMaps gmaps{};                              // gather4 tensor maps of the local tables
    int32_t gather_path = -1;                        // kernel of the last gather enqueued (eg_gather_path)
    // pipeline: `depth` lanes, each carrying bundles of up to `bundle` batches
    std::vector<Lane> lanes;
    int next_lane = 0;
    int depth = 1, bundle = 1;
    std::vector<void *> ipc_bases;
    uint32_t attached = 0;                          // bit p: rank p's shard is mapped
    eg_shard_meta metas[EG_MAX_RANKS] = {};          // every rank's published shard metadata
    // instrumentation
    bool prof = false;
    std::vector<TimedPair> timed;
    double prof_ms[2] = {0, 0};
    int64_t prof_n[2] = {0, 0};
    int64_t launches = 0;
    // batch plans (CUDA graphs)
    std::vector<Plan *> plans;
    cudaStream_t cap_stream = nullptr;
    Fork fork{};                          // capture side stream + events (graph branches)
    bool trace = false;                   // EG_TRACE=1 at create: per-stage events in every graph
    int compact = 0;                      // EG_COMPACT at create: 0 default, 1 bitmap path for every bucket
    int prio = 1;                         // EG_PRIO at create: 0 none, 1 gather first, 2 sampling first
    int gather_mode = 2;                  // EG_GATHER at create: 0 tma, 1 ldg, 2 auto (gather.cu)
    bool peer_maps = true;                // EG_PEER_MAPS=0 at create: no gather4 maps over peer shards (A/B)
    std::vector<std::string> trace_names;
    std::vector<double> trace_ms;
    std::vector<int64_t> trace_n;
    std::set<eg_blocks *> live;           // handles not yet freed (orphaned by eg_destroy)
};

struct eg_blocks {
    eg_ctx *ctx = nullptr;
    Slot *slot = nullptr;
    int32_t bidx = 0;            // batch index within the slot's bundle
    int32_t n_hops = 0, n_vt = 0, n_rel = 0;
    bool ready = false;
    eg_status status = EG_OK;
    int64_t *nodes[EG_MAX_VT] = {};
    uint8_t *feat[EG_MAX_VT] = {};
    int32_t *indptr[EG_MAX_HOPS][EG_MAX_REL] = {};
    int32_t *indices[EG_MAX_HOPS][EG_MAX_REL] = {};
    int64_t *eids[EG_MAX_HOPS][EG_MAX_REL] = {};
    int32_t *meta = nullptr;  // device
    int64_t n_nodes[EG_MAX_HOPS + 1][EG_MAX_VT] = {};
    int64_t nnz[EG_MAX_HOPS][EG_MAX_REL] = {};
    // link prediction
    bool lp = false;
    int32_t lp_rel = 0, n_neg = 0;
    int64_t n_pos = 0, cap_pos = 0;
    int32_t *pairs = nullptr;
    int64_t *neg = nullptr;
};



namespace {

eg_status fail(eg_ctx *c, eg_status s, const std::string &msg)
{
    if (c) {
        c->err = msg;
        if (s == EG_ECUDA) c->broken = true;
    }
    return s;
}

#define EG_CUDA(ctx, call)                                                                        \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            return fail(ctx, EG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));       \
    } while (0)

eg_status enter(eg_ctx *c)
{
    if (!c) return EG_EINVAL;
    if (c->broken) return fail(c, EG_ESTATE, "context unusable after an earlier CUDA error: " + c->err);
    cudaError_t e = cudaSetDevice(c->device);
    if (e != cudaSuccess) return fail(c, EG_ECUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    return EG_OK;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

bool is_device_ptr(const void *p)
{
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

typedef CUresult (*PFN_addr_range)(CUdeviceptr *, size_t *, CUdeviceptr);

eg_status ipc_export(eg_ctx *c, const void *p, cudaIpcMemHandle_t *h, int64_t *off)
{
    static PFN_addr_range fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *sym = nullptr;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &sym, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !sym)
            return fail(c, EG_ECUDA, "cuMemGetAddressRange entry point unavailable");
        fn = (PFN_addr_range)sym;
    }
    CUdeviceptr base = 0;
    size_t sz = 0;
    if (fn(&base, &sz, (CUdeviceptr)p) != CUDA_SUCCESS) return fail(c, EG_ECUDA, "cuMemGetAddressRange failed");
    EG_CUDA(c, cudaIpcGetMemHandle(h, (void *)base));
    *off = (int64_t)((const char *)p - (const char *)base);
    return EG_OK;
}

void record_start(eg_ctx *c, TimedPair *tp, int kind)
{
    if (!c->prof) return;
    cudaEventCreate(&tp->a);
    cudaEventCreate(&tp->b);
    tp->kind = kind;
    cudaEventRecord(tp->a, c->stream);
}

void record_end(eg_ctx *c, TimedPair *tp)
{
    if (!c->prof) return;
    cudaEventRecord(tp->b, c->stream);
    c->timed.push_back(*tp);
}

void drain_timing(eg_ctx *c)
{
    for (auto &tp : c->timed) {
        cudaEventSynchronize(tp.b);
        float ms = 0;
        cudaEventElapsedTime(&ms, tp.a, tp.b);
        c->prof_ms[tp.kind] += ms;
        c->prof_n[tp.kind] += 1;
        cudaEventDestroy(tp.a);
        cudaEventDestroy(tp.b);
    }
    c->timed.clear();
}

// Upper bounds of a batch (host arithmetic shared with eg_batch_caps).
eg_status compute_caps(int32_t n_vt, const int64_t *vt_counts, int32_t n_rel, const int32_t *src_vt,
                       const int32_t *dst_vt, const int64_t *n_edges, const int64_t *maxdeg, int64_t n_seeds,
                       int32_t n_hops, const int32_t *fanouts, int64_t capF[][EG_MAX_VT],
                       int64_t capE[][EG_MAX_REL])
{
    for (int u = 0; u < n_vt; ++u) capF[0][u] = std::min(vt_counts[u], n_seeds);
    for (int h = 0; h < n_hops; ++h) {
        for (int u = 0; u < n_vt; ++u) capF[h + 1][u] = capF[h][u];
        for (int r = 0; r < n_rel; ++r) {
            const int64_t k = fanouts[h * n_rel + r];
            const int64_t kc = k < 0 ? maxdeg[r] : std::min(k, maxdeg[r]);
            const int64_t t = capF[h][dst_vt[r]];
            capE[h][r] = (kc > 0 && t > 0) ? std::min(n_edges[r], (t > INT64_MAX / kc) ? INT64_MAX : t * kc) : 0;
            capF[h + 1][src_vt[r]] += capE[h][r];
        }
        for (int u = 0; u < n_vt; ++u) capF[h + 1][u] = std::min(capF[h + 1][u], vt_counts[u]);
    }
    return EG_OK;
}


// Metadata part of a shard blob (no IPC handles).
void fill_meta(const eg_ctx *c, ShardBlob *b)
{
    memset(b, 0, sizeof(*b));
    b->magic = kBlobMagic;
    b->version = 1;
    b->rank = c->rank;
    b->world = c->world;
    b->n_vt = c->g.n_vt;
    b->n_rel = c->g.n_rel;
    for (int t = 0; t < b->n_vt; ++t) {
        b->vt_counts[t] = c->vt_counts[t];
        for (int p = 0; p <= c->world; ++p) b->bounds[t][p] = c->g.bounds[t][p];
        const eg_features &F = c->own_feat[t];
        b->feat[t].row_bytes = F.row_bytes;
        b->feat[t].n_rows = c->g.bounds[t][c->rank + 1] - c->g.bounds[t][c->rank];
        b->feat[t].has = F.rows != nullptr && b->feat[t].n_rows > 0;
    }
    for (int r = 0; r < b->n_rel; ++r) {
        const eg_relation &R = c->own_rel[r];
        ShardRel &sr = b->rel[r];
        sr.src_vt = R.src_vt;
        sr.dst_vt = R.dst_vt;
        sr.n_local_dst = c->g.bounds[R.dst_vt][c->rank + 1] - c->g.bounds[R.dst_vt][c->rank];
        sr.n_local_edges = R.n_local_edges;
        sr.edge_base = R.edge_base;
        sr.max_degree = c->rel_max_degree[r];
    }
}

// At least `depth` lanes.
eg_status ensure_lanes(eg_ctx *c, int depth)
{
    while ((int)c->lanes.size() < depth) {
        Lane ln;
        EG_CUDA(c, cudaStreamCreateWithFlags(&ln.stream, cudaStreamNonBlocking));
        EG_CUDA(c, cudaEventCreateWithFlags(&ln.ready, cudaEventDisableTiming));
        c->lanes.push_back(ln);
    }
    return EG_OK;
}

void to_meta(const ShardBlob &b, eg_shard_meta *m)
{
    memset(m, 0, sizeof(*m));
    m->rank = b.rank;
    m->world = b.world;
    m->n_vt = b.n_vt;
    m->n_rel = b.n_rel;
    for (int t = 0; t < EG_MAX_VT; ++t) {
        m->vt_counts[t] = b.vt_counts[t];
        for (int q = 0; q <= EG_MAX_RANKS; ++q) m->bounds[t][q] = b.bounds[t][q];
        m->row_bytes[t] = b.feat[t].row_bytes;
    }
    for (int r = 0; r < EG_MAX_REL; ++r) {
        m->rel_src_vt[r] = b.rel[r].src_vt;
        m->rel_dst_vt[r] = b.rel[r].dst_vt;
        m->rel_n_local_edges[r] = b.rel[r].n_local_edges;
        m->rel_edge_base[r] = b.rel[r].edge_base;
        m->rel_max_degree[r] = b.rel[r].max_degree;
    }
}

// The one consistency check of a partition's published metadata.
bool check_metas(int world, const eg_shard_meta *m, int64_t *edges, int64_t *maxdeg, std::string *why)
{
    if (world < 1 || world > EG_MAX_RANKS) return *why = "world out of range", false;
    const eg_shard_meta &a = m[0];
    if (a.n_vt < 1 || a.n_vt > EG_MAX_VT || a.n_rel < 1 || a.n_rel > EG_MAX_REL)
        return *why = "schema size out of range", false;
    for (int p = 0; p < world; ++p) {
        const eg_shard_meta &b = m[p];
        const std::string who = "rank " + std::to_string(p) + ": ";
        if (b.rank != p || b.world != world) return *why = who + "rank / world mismatch", false;
        if (b.n_vt != a.n_vt || b.n_rel != a.n_rel) return *why = who + "schema differs", false;
        for (int t = 0; t < a.n_vt; ++t) {
            if (b.vt_counts[t] != a.vt_counts[t]) return *why = who + "vertex counts differ", false;
            if (b.row_bytes[t] != a.row_bytes[t]) return *why = who + "feature row size differs", false;
            if (b.bounds[t][0] != 0 || b.bounds[t][world] != b.vt_counts[t])
                return *why = who + "bounds must span [0, N_t]", false;
            for (int q = 0; q <= world; ++q) {
                if (b.bounds[t][q] != a.bounds[t][q]) return *why = who + "partition bounds differ", false;
                if (q < world && b.bounds[t][q + 1] < b.bounds[t][q]) return *why = who + "bounds decrease", false;
            }
        }
        for (int r = 0; r < a.n_rel; ++r)
            if (b.rel_src_vt[r] != a.rel_src_vt[r] || b.rel_dst_vt[r] != a.rel_dst_vt[r])
                return *why = who + "relation types differ", false;
    }
    for (int r = 0; r < a.n_rel; ++r) {
        int64_t total = 0, mx = 0;
        for (int p = 0; p < world; ++p) {
            if (m[p].rel_edge_base[r] != total || m[p].rel_n_local_edges[r] < 0)
                return *why = "relation " + std::to_string(r) + ": edge bases not contiguous at rank " +
                              std::to_string(p), false;
            total += m[p].rel_n_local_edges[r];
            mx = std::max(mx, m[p].rel_max_degree[r]);
        }
        if (edges) edges[r] = total;
        if (maxdeg) maxdeg[r] = mx;
    }
    return true;
}

eg_status check_peer(eg_ctx *c, const ShardBlob &b, int p)
{
    if (b.magic != kBlobMagic || b.version != 1 || b.rank != p || b.world != c->world)
        return fail(c, EG_EPEER, "peer blob " + std::to_string(p) + ": header mismatch");
    to_meta(b, &c->metas[p]);
    return EG_OK;
}

// All ranks mapped: validate the partition, global edge counts / max degrees.
void build_gather_maps(eg_ctx *c);

eg_status finalize_peers(eg_ctx *c)
{
    std::string why;
    if (!check_metas(c->world, c->metas, c->rel_edges_total, c->rel_max_degree, &why))
        return fail(c, EG_EPEER, why);
    c->peers_ready = true;
    build_gather_maps(c);   // per-owner maps over the peer shards, now mapped
    return EG_OK;
}
}  // namespace

// =============================================================================== ABI

namespace {

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled()
{
    static EncodeTiledFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
        cudaGetLastError();
    }
    return fn;
}

// gather4 tensor maps (kernels.h GatherMaps): a type whose full table is on this GPU (world
// 1, or a replica) gets one map over it; otherwise, once every peer is mapped, one map per
// owner shard (own and peers').  Rows must be <= 1 KB (box <= 256 elements) and a multiple
// of 16 B; the kernel places each 4-row group at a 128-B aligned stage offset.  A type
// without maps is gathered by the other paths (same bytes).
bool encode_map(EncodeTiledFn fn, CUtensorMap *m, const void *base, int64_t rb, int64_t n)
{
    if (!base || rb <= 0 || rb > 1024 || rb % 16 || n < 1 || n > INT32_MAX || ((uintptr_t)base & 15)) return false;
    cuuint64_t dims[2] = {(cuuint64_t)(rb / 4), (cuuint64_t)n};
    cuuint64_t strides[1] = {(cuuint64_t)rb};
    cuuint32_t box[2] = {(cuuint32_t)(rb / 4), 1u};
    cuuint32_t es[2] = {1u, 1u};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void *>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void build_gather_maps(eg_ctx *c)
{
    EncodeTiledFn fn = encode_tiled();
    for (int u = 0; u < EG_MAX_VT; ++u) c->gmaps.grp[u] = c->gmaps.whole[u] = 0;
    if (!fn) return;
    for (int u = 0; u < c->g.n_vt; ++u) {
        const int64_t rb = c->f.row_bytes[u];
        if (c->host_feat[u] || !rb) continue;
        const void *whole = c->f.replica[u];
        if (!whole && c->world == 1) whole = c->f.rows[u][c->rank];
        if (whole) {
            if (encode_map(fn, &c->gmaps.map[u][0], whole, rb, c->vt_counts[u])) c->gmaps.grp[u] = c->gmaps.whole[u] = 1;
            continue;
        }
        if (!c->peer_maps || c->attached != (1u << c->world) - 1) continue;   // peers not mapped yet
        bool all = true;
        for (int p = 0; p < c->world && all; ++p) {
            const int64_t n = c->g.bounds[u][p + 1] - c->g.bounds[u][p];
            all = n == 0 || encode_map(fn, &c->gmaps.map[u][p], c->f.rows[u][p], rb, n);
        }
        c->gmaps.grp[u] = all ? 1 : 0;
    }
}

}  // namespace

extern "C" {

const char *eg_version(void) { return kVersion; }

int64_t eg_counter_bytes(void) { return (int64_t)sizeof(int32_t) * kMetaSize; }

const char *eg_last_error(const eg_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int64_t eg_kernel_launches(const eg_ctx *ctx) { return ctx ? ctx->launches : 0; }

eg_status eg_range_bounds(int64_t n, int32_t world, int64_t *bounds)
{
    if (n < 0 || world < 1 || !bounds) return EG_EINVAL;
    for (int p = 0; p <= world; ++p) bounds[p] = (int64_t)((__int128)p * n / world);
    return EG_OK;
}

eg_status eg_check_shard_metas(int32_t world, const eg_shard_meta *metas, int64_t *rel_edges,
                               int64_t *rel_max_degree, char *msg, size_t msg_len)
{
    if (!metas) return EG_EINVAL;
    std::string why;
    const bool ok = check_metas(world, metas, rel_edges, rel_max_degree, &why);
    if (msg && msg_len) {
        strncpy(msg, ok ? "ok" : why.c_str(), msg_len - 1);
        msg[msg_len - 1] = 0;
    }
    return ok ? EG_OK : EG_EPEER;
}

eg_status eg_batch_caps(int32_t n_vt, const int64_t *vt_counts, int32_t n_rel, const int32_t *rel_src_vt,
                        const int32_t *rel_dst_vt, const int64_t *rel_n_edges, const int64_t *rel_max_degree,
                        int64_t n_seeds, int32_t n_hops, const int32_t *fanouts, int64_t *caps_nodes,
                        int64_t *caps_edges)
{
    if (n_vt < 1 || n_vt > EG_MAX_VT || n_rel < 1 || n_rel > EG_MAX_REL || n_hops < 1 || n_hops > EG_MAX_HOPS ||
        n_seeds < 0)
        return EG_EINVAL;
    int64_t capF[EG_MAX_HOPS + 1][EG_MAX_VT], capE[EG_MAX_HOPS][EG_MAX_REL];
    compute_caps(n_vt, vt_counts, n_rel, rel_src_vt, rel_dst_vt, rel_n_edges, rel_max_degree, n_seeds, n_hops,
                 fanouts, capF, capE);
    for (int u = 0; u < n_vt; ++u) caps_nodes[u] = capF[n_hops][u];
    for (int h = 0; h < n_hops; ++h)
        for (int r = 0; r < n_rel; ++r) caps_edges[h * n_rel + r] = capE[h][r];
    return EG_OK;
}

eg_status eg_create(int32_t rank, int32_t world, int32_t device, void *stream, eg_ctx **out)
{
    if (!out) return EG_EINVAL;
    *out = nullptr;
    if (world < 1 || world > EG_MAX_RANKS || rank < 0 || rank >= world || device < 0) return EG_EINVAL;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device >= n) {
        cudaGetLastError();
        return EG_ECUDA;
    }
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major != 10) return EG_ECUDA;
    if (cudaSetDevice(device) != cudaSuccess) return EG_ECUDA;
    eg_ctx *c = new eg_ctx();
    c->rank = rank;
    c->world = world;
    c->device = device;
    c->stream = (cudaStream_t)stream;
    {
        const char *tr = getenv("EG_TRACE");
        c->trace = tr && tr[0] == '1';
        // EG_COMPACT=bitmap: every compaction bucket is a task of its own, on the bitmap path
        // (tests: both paths on the same inputs); default: runs of small buckets are sorted
        const char *cm = getenv("EG_COMPACT");
        c->compact = cm && cm[0] == 'b' ? 1 : 0;
        // EG_PRIO=gather|sample|none: per-node scheduling priority inside the batch graphs.
        // Default gather: measured (profiles/prio_sweep.sh) it shortens the gather's
        // duration in the pipelined run by 8-20 % at unchanged throughput (C2, C4).
        const char *pr = getenv("EG_PRIO");
        c->prio = !pr ? 1 : (pr[0] == 'g' ? 1 : (pr[0] == 's' ? 2 : 0));
        const char *pm = getenv("EG_PEER_MAPS");
        c->peer_maps = !(pm && pm[0] == '0');
        const char *ga = getenv("EG_GATHER");
        c->gather_mode = !ga ? 2 : (!strcmp(ga, "tma") ? 0 : (!strcmp(ga, "ldg") ? 1 : 2));
    }
    if (cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->fork.side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->fork.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->fork.join, cudaEventDisableTiming) != cudaSuccess) {
        delete c;
        return EG_ECUDA;
    }
    // stream-ordered allocations (host-output staging): keep freed blocks cached in the pool
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    *out = c;
    return EG_OK;
}

eg_status eg_set_stream(eg_ctx *ctx, void *stream)
{
    if (!ctx) return EG_EINVAL;
    ctx->stream = (cudaStream_t)stream;
    return EG_OK;
}

eg_status eg_load_partition(eg_ctx *c, int32_t n_vt, const int64_t *vt_counts, const int64_t *bounds,
                            int32_t n_rel, const eg_relation *rels, const eg_features *feats)
{
    eg_status st = enter(c);
    if (st) return st;
    if (c->loaded) return fail(c, EG_EINVAL, "partition already loaded");
    if (n_vt < 1 || n_vt > EG_MAX_VT || n_rel < 1 || n_rel > EG_MAX_REL || !vt_counts || !rels)
        return fail(c, EG_EINVAL, "n_vt / n_rel out of range or null arrays");
    GraphDev &g = c->g;
    g = GraphDev{};
    g.n_vt = n_vt;
    g.n_rel = n_rel;
    g.world = c->world;
    g.rank = c->rank;
    g.off[0] = 0;
    for (int t = 0; t < n_vt; ++t) {
        if (vt_counts[t] < 0) return fail(c, EG_EINVAL, "negative vertex count");
        c->vt_counts[t] = vt_counts[t];
        g.off[t + 1] = g.off[t] + vt_counts[t];
    }
    c->n_total = g.off[n_vt];
    if (c->n_total >= (int64_t)1 << 31) return fail(c, EG_EINVAL, "total vertex count must be < 2^31");
    for (int t = 0; t < n_vt; ++t) {
        for (int p = 0; p <= c->world; ++p)
            g.bounds[t][p] = bounds ? bounds[t * (c->world + 1) + p] : (int64_t)((__int128)p * vt_counts[t] / c->world);
        if (g.bounds[t][0] != 0 || g.bounds[t][c->world] != vt_counts[t])
            return fail(c, EG_EINVAL, "bounds must start at 0 and end at N_t");
        for (int p = 0; p < c->world; ++p)
            if (g.bounds[t][p + 1] < g.bounds[t][p]) return fail(c, EG_EINVAL, "bounds must be non-decreasing");
    }
    // compaction buckets (compact.cuh): type-aligned ranges of 2^bshift gids, bshift the
    // smallest in [12, kMaxBucketShift] (graphs under 2^20 vertices: from kMinBucketShift) that
    // keeps the graph's buckets <= 2^14 (C4: 2^13 gids per bucket, 13.6k buckets; C2 / C3:
    // 2^12; C1: 2^10).  Measured against the first rule (<= 2^16 buckets from 2^10: C4 2^11,
    // C2 / C3 2^10): the bucket scans halve, C4 +4.7 %, C2 +3.0 %, C3 +1.2 %; C1 prefers 2^10
    // (profiles/r02/bshift/).  EG_BSHIFT (A/B runs) sets it in [kMinBucketShift,
    // kMaxBucketShift]; results never depend on it.
    g.bshift = c->n_total >= (1ll << 20) ? 12 : kMinBucketShift;
    while (g.bshift < kMaxBucketShift && (c->n_total >> g.bshift) > (1 << 14)) ++g.bshift;
    if (const char *e = getenv("EG_BSHIFT")) {
        const int v = atoi(e);
        if (v >= kMinBucketShift && v <= kMaxBucketShift) g.bshift = v;
    }
    g.bbase[0] = 0;
    for (int t = 0; t < n_vt; ++t) g.bbase[t + 1] = g.bbase[t] + ((vt_counts[t] + (1ll << g.bshift) - 1) >> g.bshift);
    if (g.bbase[n_vt] > kMaxBuckets) return fail(c, EG_EINVAL, "too many vertices for the compaction buckets");
    g.nb = (int32_t)g.bbase[n_vt];
    g.compact_bitmap = c->compact;

    unsigned long long *d_max = nullptr;
    EG_CUDA(c, cudaMalloc(&d_max, sizeof(unsigned long long) * EG_MAX_REL));
    EG_CUDA(c, cudaMemsetAsync(d_max, 0, sizeof(unsigned long long) * EG_MAX_REL, c->stream));
    for (int r = 0; r < n_rel; ++r) {
        const eg_relation &R = rels[r];
        if (R.src_vt < 0 || R.src_vt >= n_vt || R.dst_vt < 0 || R.dst_vt >= n_vt)
            return fail(c, EG_EINVAL, "relation vertex type out of range");
        const int64_t n_local_dst = g.bounds[R.dst_vt][c->rank + 1] - g.bounds[R.dst_vt][c->rank];
        if (!R.indptr || (R.n_local_edges > 0 && !R.indices) || R.n_local_edges < 0 || R.edge_base < 0)
            return fail(c, EG_EINVAL, "relation shard pointers / sizes invalid");
        if (vt_counts[R.src_vt] == 0 && R.n_local_edges > 0)
            return fail(c, EG_EINVAL, "edges into an empty source type");
        g.rel[r].src_vt = R.src_vt;
        g.rel[r].dst_vt = R.dst_vt;
        g.rel[r].indptr[c->rank] = R.indptr;
        g.rel[r].indices[c->rank] = R.indices;
        g.rel[r].edge_base[c->rank] = R.edge_base;
        c->own_rel[r] = R;
        c->rel_edges_total[r] = R.n_local_edges;
        launch_max_degree(R.indptr, n_local_dst, d_max + r, c->stream);
        ++c->launches;
    }
    c->f = FeatDev{};
    for (int t = 0; t < n_vt; ++t) {
        eg_features F = feats ? feats[t] : eg_features{nullptr, 0};
        const int64_t n_rows = g.bounds[t][c->rank + 1] - g.bounds[t][c->rank];
        if (F.row_bytes < 0 || F.row_bytes % 16 || (F.rows && F.row_bytes == 0))
            return fail(c, EG_EINVAL, "row_bytes must be a positive multiple of 16");
        if (!F.rows && F.row_bytes > 0 && n_rows > 0)
            return fail(c, EG_EINVAL, "feature rows missing for a non-empty local range");
        const void *rows_dev = F.rows;
        c->host_feat[t] = false;
        if (F.rows) {
            // device memory, or pinned / registered host memory read zero-copy over PCIe by
            // the gather kernel (the paper's placement of graph data in CPU memory)
            cudaPointerAttributes at;
            if (cudaPointerGetAttributes(&at, F.rows) != cudaSuccess) {
                cudaGetLastError();
                return fail(c, EG_EINVAL, "feature rows: not device, pinned or registered host memory");
            }
            if (at.type == cudaMemoryTypeHost) {
                if (!at.devicePointer) return fail(c, EG_EINVAL, "feature rows: host memory not mapped for the device");
                if (c->world > 1)
                    return fail(c, EG_EINVAL, "host-memory feature rows are supported at world 1 only");
                rows_dev = at.devicePointer;
                c->host_feat[t] = true;
            } else if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged) {
                return fail(c, EG_EINVAL, "feature rows: pageable host memory (pin or register it)");
            }
        }
        c->f.rows[t][c->rank] = (const uint8_t *)rows_dev;
        c->f.row_bytes[t] = F.row_bytes;
        c->own_feat[t] = F;
    }
    unsigned long long h_max[EG_MAX_REL] = {};
    EG_CUDA(c, cudaMemcpyAsync(h_max, d_max, sizeof(h_max), cudaMemcpyDeviceToHost, c->stream));
    EG_CUDA(c, cudaStreamSynchronize(c->stream));
    EG_CUDA(c, cudaFree(d_max));
    for (int r = 0; r < n_rel; ++r) {
        c->rel_max_degree[r] = (int64_t)h_max[r];
        // heavy items are split into tasks (item << 16 | chunk of kHeavyChunk keys) and
        // degrees are int32 in the batch: in-degrees above kMaxInDegree would wrap
        if (c->rel_max_degree[r] > kMaxInDegree)
            return fail(c, EG_EINVAL, "relation " + std::to_string(r) + ": in-degree " +
                                          std::to_string(c->rel_max_degree[r]) + " exceeds 2^26");
    }

    if ((st = ensure_lanes(c, 1))) return st;
    EG_CUDA(c, cudaStreamSynchronize(c->stream));
    c->loaded = true;
    build_gather_maps(c);
    {
        ShardBlob self_meta;
        fill_meta(c, &self_meta);
        if ((st = check_peer(c, self_meta, c->rank))) return st;
    }
    c->attached = 1u << c->rank;
    c->peers_ready = false;
    if (c->world == 1) return finalize_peers(c);
    return EG_OK;
}

eg_status eg_export_shard(const eg_ctx *cc, void *buf, size_t *len)
{
    eg_ctx *c = const_cast<eg_ctx *>(cc);
    if (!c || !len) return EG_EINVAL;
    if (!buf) {
        *len = sizeof(ShardBlob);
        return EG_OK;
    }
    if (*len < sizeof(ShardBlob)) return fail(c, EG_EINVAL, "export buffer too small");
    eg_status st = enter(c);
    if (st) return st;
    if (!c->loaded) return fail(c, EG_EINVAL, "load the partition first");
    ShardBlob b;
    fill_meta(c, &b);
    for (int t = 0; t < b.n_vt; ++t)
        if (b.feat[t].has && (st = ipc_export(c, c->own_feat[t].rows, &b.feat[t].h, &b.feat[t].off))) return st;
    for (int r = 0; r < b.n_rel; ++r) {
        const eg_relation &R = c->own_rel[r];
        ShardRel &sr = b.rel[r];
        if ((st = ipc_export(c, R.indptr, &sr.indptr_h, &sr.indptr_off))) return st;
        if (R.n_local_edges > 0 && (st = ipc_export(c, R.indices, &sr.indices_h, &sr.indices_off))) return st;
    }
    memcpy(buf, &b, sizeof(b));
    *len = sizeof(b);
    return EG_OK;
}

eg_status eg_import_shards(eg_ctx *c, const void *blobs, size_t stride)
{
    eg_status st = enter(c);
    if (st) return st;
    if (!c->loaded) return fail(c, EG_EINVAL, "load the partition first");
    if (!blobs || stride < sizeof(ShardBlob)) return fail(c, EG_EINVAL, "blob stride too small");
    std::vector<ShardBlob> all(c->world);
    for (int p = 0; p < c->world; ++p) memcpy(&all[p], (const char *)blobs + p * stride, sizeof(ShardBlob));
    for (int p = 0; p < c->world; ++p)
        if ((st = check_peer(c, all[p], p))) return st;
    // map the peers' shards (deduplicate allocations shared by several buffers)
    for (int p = 0; p < c->world; ++p) {
        if (p == c->rank) continue;
        std::map<std::string, char *> opened;
        auto open = [&](const cudaIpcMemHandle_t &h, int64_t off, const void **outp) -> eg_status {
            std::string key((const char *)&h, sizeof(h));
            auto it = opened.find(key);
            char *base = nullptr;
            if (it == opened.end()) {
                void *bp = nullptr;
                cudaError_t e = cudaIpcOpenMemHandle(&bp, h, cudaIpcMemLazyEnablePeerAccess);
                if (e != cudaSuccess)
                    return fail(c, EG_ECUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
                c->ipc_bases.push_back(bp);
                base = (char *)bp;
                opened[key] = base;
            } else {
                base = it->second;
            }
            *outp = base + off;
            return EG_OK;
        };
        const ShardBlob &b = all[p];
        for (int r = 0; r < b.n_rel; ++r) {
            const void *ip = nullptr, *ix = nullptr;
            if ((st = open(b.rel[r].indptr_h, b.rel[r].indptr_off, &ip))) return st;
            if (b.rel[r].n_local_edges > 0 && (st = open(b.rel[r].indices_h, b.rel[r].indices_off, &ix))) return st;
            c->g.rel[r].indptr[p] = (const int64_t *)ip;
            c->g.rel[r].indices[p] = (const int32_t *)ix;
            c->g.rel[r].edge_base[p] = b.rel[r].edge_base;
        }
        for (int t = 0; t < b.n_vt; ++t) {
            if (!b.feat[t].has) continue;
            const void *rp = nullptr;
            if ((st = open(b.feat[t].h, b.feat[t].off, &rp))) return st;
            c->f.rows[t][p] = (const uint8_t *)rp;
        }
    }
    c->attached = (1u << c->world) - 1;
    return finalize_peers(c);
}

eg_status eg_attach_peer(eg_ctx *c, const eg_ctx *peer)
{
    eg_status st = enter(c);
    if (st) return st;
    if (!peer || !c->loaded || !peer->loaded) return fail(c, EG_EINVAL, "both contexts must be loaded");
    const int p = peer->rank;
    if (peer->world != c->world || p == c->rank) return fail(c, EG_EINVAL, "peer must be another rank of the same world");
    ShardBlob b;
    fill_meta(peer, &b);
    if ((st = check_peer(c, b, p))) return st;
    if (peer->device != c->device) {
        cudaError_t e = cudaDeviceEnablePeerAccess(peer->device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
            return fail(c, EG_ECUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
        cudaGetLastError();
    }
    for (int r = 0; r < c->g.n_rel; ++r) {
        c->g.rel[r].indptr[p] = peer->own_rel[r].indptr;
        c->g.rel[r].indices[p] = peer->own_rel[r].indices;
        c->g.rel[r].edge_base[p] = peer->own_rel[r].edge_base;
    }
    for (int t = 0; t < c->g.n_vt; ++t) c->f.rows[t][p] = (const uint8_t *)peer->own_feat[t].rows;
    c->attached |= 1u << p;
    if (c->attached == (1u << c->world) - 1) return finalize_peers(c);
    return EG_OK;
}

int32_t eg_gather_path(const eg_ctx *c) { return c ? c->gather_path : -1; }

eg_status eg_set_feature_replica(eg_ctx *c, int32_t vt, const void *rows, int64_t n_rows)
{
    eg_status st = enter(c);
    if (st) return st;
    if (!c->loaded) return fail(c, EG_ESTATE, "eg_set_feature_replica before eg_load_partition");
    if (!c->plans.empty()) return fail(c, EG_ESTATE, "eg_set_feature_replica after the first sampling call");
    if (vt < 0 || vt >= c->g.n_vt) return fail(c, EG_EINVAL, "vertex type out of range");
    if (!rows) {
        c->f.replica[vt] = nullptr;
        build_gather_maps(c);
        return EG_OK;
    }
    if (!c->f.row_bytes[vt]) return fail(c, EG_EINVAL, "vertex type has no features");
    if (n_rows != c->vt_counts[vt]) return fail(c, EG_EINVAL, "replica must hold all N_t rows of the type");
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, rows) != cudaSuccess || at.type != cudaMemoryTypeDevice ||
        at.device != c->device) {
        cudaGetLastError();
        return fail(c, EG_EINVAL, "replica rows must be device memory of this context's GPU");
    }
    c->f.replica[vt] = (const uint8_t *)rows;
    build_gather_maps(c);
    return EG_OK;
}

}  // extern "C"

namespace {

eg_status get_plan(eg_ctx *c, int32_t L, const int32_t *fanouts, int64_t n_cap, bool features, int32_t B,
                   Plan **out, bool lp = false, int32_t n_neg = 0)
{
    const GraphDev &g = c->g;
    const int V = g.n_vt, R = g.n_rel;
    for (Plan *p : c->plans)
        if (p->n_hops == L && p->n_cap == n_cap && p->features == features && p->B == B && p->lp == lp &&
            p->n_neg == n_neg && !memcmp(p->fanouts, fanouts, sizeof(int32_t) * L * R)) {
            *out = p;
            return EG_OK;
        }
    Plan *p = new Plan();
    p->n_hops = L;
    memcpy(p->fanouts, fanouts, sizeof(int32_t) * L * R);
    p->n_cap = n_cap;
    p->features = features;
    p->B = B;
    p->lp = lp;
    p->n_neg = n_neg;
    const int64_t seed_cap = lp ? n_cap * (2 + (int64_t)n_neg) : n_cap;   // distinct endpoints (LP)
    int32_t src_vt[EG_MAX_REL], dst_vt[EG_MAX_REL];
    for (int r = 0; r < R; ++r) {
        src_vt[r] = g.rel[r].src_vt;
        dst_vt[r] = g.rel[r].dst_vt;
    }
    compute_caps(V, c->vt_counts, R, src_vt, dst_vt, c->rel_edges_total, c->rel_max_degree, seed_cap, L, fanouts,
                 p->capF, p->capE);
    for (int h = 0; h <= L; ++h)
        for (int u = 0; u < V; ++u)
            if (p->capF[h][u] >= INT32_MAX) {
                delete p;
                return fail(c, EG_EINVAL, "batch exceeds 2^31 vertices of one type");
            }
    for (int h = 0; h < L; ++h)
        for (int r = 0; r < R; ++r)
            if (p->capE[h][r] >= INT32_MAX) {
                delete p;
                return fail(c, EG_EINVAL, "batch exceeds 2^31 edges of one relation");
            }
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off = align_up(off + std::max<size_t>(bytes, 1), 256);
        return o;
    };
    // meta, kcnt, mcnt, the kscan tile look-back words are contiguous: one memset per batch
    // and launch clears them.  Bucket arrays are padded to whole kscan tiles (16-B accesses).
    const int64_t NB = c->g.nb;
    const int64_t NBp = (NB + kScanTile - 1) / kScanTile * kScanTile;
    p->o_meta = off;
    off += align_up(sizeof(int32_t) * kMetaSize, 16);
    p->o_kcnt = off;
    off += sizeof(uint32_t) * NBp;
    p->o_mcnt = off;
    off += sizeof(uint32_t) * NBp;
    p->o_tlb = off;
    off += sizeof(unsigned long long) * 3 * kMaxScanTiles * (L + 1);
    for (int h = 0; h < L; ++h) {   // count tiles' look-back words
        int64_t tiles = 0;
        for (int r = 0; r < R; ++r) tiles += (p->capF[h][dst_vt[r]] + kCountTile - 1) / kCountTile;
        p->count_tiles[h] = (int32_t)std::max<int64_t>(1, tiles);
        p->o_clb[h] = off;
        off += sizeof(unsigned long long) * p->count_tiles[h];
    }
    p->zero_bytes = off - p->o_meta;
    off = align_up(off, 256);
    p->o_dyn = take(sizeof(uint64_t) * kDyn);
    p->o_kofs = take(sizeof(uint32_t) * (NBp + 1));
    p->o_mofs = take(sizeof(uint32_t) * (NBp + 1));
    p->o_kcur = take(sizeof(uint32_t) * NBp);
    p->o_tstart = take(sizeof(uint32_t) * (NB + 1));
    p->o_tnew = take(sizeof(uint32_t) * (NB + 1));
    p->o_ftask = take(sizeof(int32_t) * EG_MAX_VT);
    p->o_seeds = take(sizeof(int64_t) * (lp ? 1 : n_cap));
    if (lp) {
        p->o_lp_src = take(sizeof(int64_t) * n_cap);
        p->o_lp_dst = take(sizeof(int64_t) * n_cap);
        p->o_lp_neg = take(sizeof(int64_t) * n_cap * n_neg);
        p->o_lp_pairs = take(sizeof(int32_t) * n_cap * (2 + 2 * (int64_t)n_neg));
    }
    // keys of a level: its seeds / endpoints (level 0) or its hop's sampled edges; members:
    // every vertex of the batch
    p->cap_keys = seed_cap;
    for (int h = 0; h < L; ++h) {
        int64_t e = 0;
        for (int r = 0; r < R; ++r) e += p->capE[h][r];
        p->cap_keys = std::max(p->cap_keys, e);
    }
    for (int u = 0; u < V; ++u) p->cap_members += p->capF[L][u];
    if (p->cap_keys + p->cap_members >= INT32_MAX) {
        delete p;
        return fail(c, EG_EINVAL, "batch exceeds 2^31 keys / vertices");
    }
    p->o_elems = take(sizeof(unsigned long long) * (p->cap_keys + p->cap_members));
    for (int i = 0; i < 2; ++i) {
        p->o_mg[i] = take(sizeof(uint32_t) * p->cap_members);
        p->o_mp[i] = take(sizeof(int32_t) * p->cap_members);
    }
    for (int u = 0; u < V; ++u) p->o_nodes[u] = take(sizeof(int64_t) * p->capF[L][u]);
    for (int h = 0; h < L; ++h)
        for (int r = 0; r < R; ++r) {
            const int64_t nd = p->capF[h][dst_vt[r]] + 1;
            p->o_ip[h][r] = take(sizeof(int32_t) * nd);
            p->o_ix[h][r] = take(sizeof(int32_t) * p->capE[h][r]);
            p->o_ei[h][r] = take(sizeof(int64_t) * p->capE[h][r]);
            p->o_src[h][r] = take(sizeof(uint32_t) * p->capE[h][r]);
        }
    for (int h = 0; h < L; ++h) {
        int64_t items = 0;
        for (int r = 0; r < R; ++r) items += p->capF[h][dst_vt[r]];
        p->selq_items[h] = items;
        p->o_selq[h] = take(sizeof(QEntry) * items);
        p->o_copyq[h] = take(sizeof(QEntry) * items);
        p->o_tiny16[h] = take(sizeof(QEntry) * items);
        // heavy slots: one per 2048 frontier items beyond the first kMinHeavy
        p->max_heavy[h] = (int32_t)std::min<int64_t>(65535, kMinHeavy + items / 2048);
        p->max_heavy_tasks[h] = (int32_t)std::min<int64_t>(INT32_MAX / 2, (int64_t)p->max_heavy[h] * kHeavyTasksPerItem);
        p->o_heavy[h] = take(heavy_bytes(p->max_heavy[h], p->max_heavy_tasks[h]));
    }
    if (features)
        for (int u = 0; u < V; ++u)
            if (c->f.row_bytes[u]) p->o_feat[u] = take((size_t)(p->capF[L][u] * c->f.row_bytes[u]));
    p->stride = off;
    p->o_bd = 0;
    p->total = Plan::align_bd() + (size_t)B * p->stride;
    c->plans.push_back(p);
    *out = p;
    return EG_OK;
}

void fill_views(const Plan *p, char *base, eg_blocks *b)
{
    b->meta = (int32_t *)(base + p->o_meta);
    for (int u = 0; u < b->n_vt; ++u) {
        b->nodes[u] = (int64_t *)(base + p->o_nodes[u]);
        b->feat[u] = p->o_feat[u] ? (uint8_t *)(base + p->o_feat[u]) : nullptr;
    }
    for (int h = 0; h < p->n_hops; ++h)
        for (int r = 0; r < b->n_rel; ++r) {
            b->indptr[h][r] = (int32_t *)(base + p->o_ip[h][r]);
            b->indices[h][r] = (int32_t *)(base + p->o_ix[h][r]);
            b->eids[h][r] = (int64_t *)(base + p->o_ei[h][r]);
        }
}

// Record one launch of the slot's bundle into a CUDA graph (once per slot).
eg_status capture_slot(eg_ctx *c, Plan *p, Slot *sl)
{
    const GraphDev &g = c->g;
    const int V = g.n_vt, R = g.n_rel, L = p->n_hops, B = p->B;
    cudaStream_t cs = c->cap_stream;
    BatchDev *bd = new BatchDev();
    memset(bd, 0, sizeof(BatchDev));
    bd->n_hops = L;
    bd->trace = c->trace ? 1 : 0;
    bd->B = B;
    bd->lp = p->lp ? 1 : 0;
    bd->seed_sort = (!p->lp && p->n_cap <= 1024) ? 1 : 0;
    GatherSet gs{};
    gs.nb = B;
    for (int b = 0; b < B; ++b) {
        char *base = p->batch_base(sl->mem, b);
        HopDev hd{};
        hd.dyn = (const uint64_t *)(base + p->o_dyn);
        hd.meta = (int32_t *)(base + p->o_meta);
        CompactDev &cd = hd.cd;
        cd.kcnt = (uint32_t *)(base + p->o_kcnt);
        cd.mcnt = (uint32_t *)(base + p->o_mcnt);
        cd.tlb = (unsigned long long *)(base + p->o_tlb);
        cd.elems = (unsigned long long *)(base + p->o_elems);
        cd.tnew = (uint32_t *)(base + p->o_tnew);
        cd.ftask = (int32_t *)(base + p->o_ftask);
        cd.kofs = (uint32_t *)(base + p->o_kofs);
        cd.mofs = (uint32_t *)(base + p->o_mofs);
        cd.kcur = (uint32_t *)(base + p->o_kcur);
        cd.tstart = (uint32_t *)(base + p->o_tstart);
        for (int i = 0; i < 2; ++i) {
            cd.mg[i] = (uint32_t *)(base + p->o_mg[i]);
            cd.mp[i] = (int32_t *)(base + p->o_mp[i]);
        }
        cd.cap_elems = (int32_t)(p->cap_keys + p->cap_members);
        cd.cap_members = (int32_t)p->cap_members;
        cd.nb_pad = (int32_t)((g.nb + kScanTile - 1) / kScanTile * kScanTile);
        for (int u = 0; u < V; ++u) {
            hd.nodes[u] = (int64_t *)(base + p->o_nodes[u]);
            hd.cap_nodes[u] = (int32_t)p->capF[L][u];
        }
        bd->seeds[b] = (const int64_t *)(base + p->o_seeds);
        {   // the seeds' level: seed split / link-prediction targets + the level-0 compaction
            HopDev x = hd;
            x.h = -1;
            x.mode = p->lp ? kModeLp : kModeSeeds;
            x.last = 0;
            bd->seedh[b] = x;
        }
        if (p->lp) {
            LpDev &lp = bd->lpd[b];
            lp.n_neg = p->n_neg;
            lp.cap_pos = p->n_cap;
            lp.src_stage = (const int64_t *)(base + p->o_lp_src);
            lp.dst_stage = (const int64_t *)(base + p->o_lp_dst);
            lp.neg = (int64_t *)(base + p->o_lp_neg);
            lp.pairs = (int32_t *)(base + p->o_lp_pairs);
        }
        for (int h = 0; h < L; ++h) {
            HopDev x = hd;
            x.h = h;
            for (int r = 0; r < R; ++r) {
                x.fanout[r] = p->fanouts[h * R + r];
                x.indptr[r] = (int32_t *)(base + p->o_ip[h][r]);
                x.indices[r] = (int32_t *)(base + p->o_ix[h][r]);
                x.eids[r] = (int64_t *)(base + p->o_ei[h][r]);
                x.src[r] = (uint32_t *)(base + p->o_src[h][r]);
            }
            x.mode = kModeHop;
            x.last = h == L - 1;
            x.selq = (QEntry *)(base + p->o_selq[h]);
            x.copyq = (QEntry *)(base + p->o_copyq[h]);
            x.tinyq16 = (QEntry *)(base + p->o_tiny16[h]);
            x.selq_cap = (int32_t)p->selq_items[h];
            x.clb = (unsigned long long *)(base + p->o_clb[h]);
            char *hv = base + p->o_heavy[h];
            x.heavy_items = (QEntry *)hv;
            const int64_t mh = p->max_heavy[h];
            x.max_heavy = p->max_heavy[h];
            x.max_heavy_tasks = p->max_heavy_tasks[h];
            x.heavy_cnt = (uint32_t *)(hv + sizeof(QEntry) * mh);
            x.heavy_done = x.heavy_cnt + mh;
            x.heavy_cand = (uint64_t *)(hv + sizeof(QEntry) * mh + 2 * sizeof(uint32_t) * mh);
            x.heavyq = (uint32_t *)(x.heavy_cand + (size_t)mh * kHeavyCap);
            bd->hop[b][h] = x;
        }
        GatherDev &gd = gs.b[b];
        gd.meta = hd.meta;
        gd.level = L;
        for (int u = 0; u < V; ++u) {
            gd.nodes[u] = hd.nodes[u];
            gd.out[u] = p->o_feat[u] ? (uint8_t *)(base + p->o_feat[u]) : nullptr;
        }
    }
    cudaError_t e0 = cudaMemcpy(sl->mem + p->o_bd, bd, sizeof(BatchDev), cudaMemcpyHostToDevice);
    delete bd;
    if (e0 != cudaSuccess) return fail(c, EG_ECUDA, std::string("BatchDev upload: ") + cudaGetErrorString(e0));
    int nk = 0;
    auto mark = [&](const std::string &label) {
        if (!c->trace) return;
        cudaEvent_t ev;
        cudaEventCreate(&ev);
        cudaEventRecordWithFlags(ev, cs, cudaEventRecordExternal);
        sl->tev.push_back(ev);
        sl->tlab.push_back(label);
    };
    cudaGraphNode_t gather_node = nullptr;
    EG_CUDA(c, cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
    for (int b = 0; b < B; ++b) {
        char *base = p->batch_base(sl->mem, b);
        cudaMemcpyAsync(base + p->o_dyn, sl->h_dyn + kDyn * b, sizeof(uint64_t) * kDyn, cudaMemcpyHostToDevice, cs);
    }
    // counters + the compaction's bucket counts of every batch: one 2-D memset
    cudaMemset2DAsync(p->batch_base(sl->mem, 0) + p->o_meta, p->stride, 0, p->zero_bytes, B, cs);
    cudaEventRecordWithFlags(sl->s0, cs, cudaEventRecordExternal);
    mark("start");
    nk += launch_batch(g, (const BatchDev *)(sl->mem + p->o_bd), L, p->count_tiles, B, cs, c->fork, c->trace, p->lp,
                       !p->lp && p->n_cap <= 1024);
    mark("sample");
    cudaEventRecordWithFlags(sl->s1, cs, cudaEventRecordExternal);
    if (p->features) {
        bool any = false;
        for (int u = 0; u < V; ++u) any |= p->o_feat[u] != 0;
        cudaEventRecordWithFlags(sl->g0, cs, cudaEventRecordExternal);
        if (any) {
            sl->gather_path = launch_gather(g, c->f, gs, c->gmaps, cs, c->gather_mode);
            c->gather_path = sl->gather_path;
            ++nk;
            if (c->prio) {
                cudaStreamCaptureStatus st;
                const cudaGraphNode_t *deps = nullptr;
                size_t nd = 0;
                if (cudaStreamGetCaptureInfo(cs, &st, nullptr, nullptr, &deps, &nd) == cudaSuccess && nd == 1)
                    gather_node = deps[0];
            }
        }
        cudaEventRecordWithFlags(sl->g1, cs, cudaEventRecordExternal);
        mark("gather");
    }
    for (int b = 0; b < B; ++b)
        cudaMemcpyAsync(sl->h_meta + (size_t)b * kMetaSize, p->batch_base(sl->mem, b) + p->o_meta,
                        sizeof(int32_t) * kMetaSize, cudaMemcpyDeviceToHost, cs);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(cs, &graph);
    if (e != cudaSuccess) return fail(c, EG_ECUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    unsigned long long iflags = 0;
    if (c->prio) {
        // the favoured side (the gather, or the latency-bound sampling chain) gets the
        // greatest priority: the block scheduler places its CTAs first when several
        // lanes' kernels compete for SMs
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        size_t n = 0;
        cudaGraphGetNodes(graph, nullptr, &n);
        std::vector<cudaGraphNode_t> nodes(n);
        cudaGraphGetNodes(graph, nodes.data(), &n);
        for (cudaGraphNode_t nd : nodes) {
            cudaGraphNodeType ty;
            if (cudaGraphNodeGetType(nd, &ty) != cudaSuccess || ty != cudaGraphNodeTypeKernel) continue;
            const bool is_g = nd == gather_node;
            cudaKernelNodeAttrValue v{};
            v.priority = (is_g == (c->prio == 1)) ? hi : lo;
            cudaGraphKernelNodeSetAttribute(nd, cudaLaunchAttributePriority, &v);
        }
        iflags = cudaGraphInstantiateFlagUseNodePriority;
    }
    e = cudaGraphInstantiateWithFlags(&sl->exec, graph, iflags);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return fail(c, EG_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    p->n_kernels = nk;
    return EG_OK;
}

eg_status make_slot(eg_ctx *c, Plan *p, int lane, Slot **out);

eg_status acquire_slot(eg_ctx *c, Plan *p, Slot **out)
{
    const int lane = c->next_lane;
    c->next_lane = (c->next_lane + 1) % c->depth;
    for (Slot *sl : p->slots)
        if (sl->refs == 0 && sl->lane == lane) {
            if (sl->used) EG_CUDA(c, cudaEventSynchronize(sl->done));   // its last run has retired
            *out = sl;
            return EG_OK;
        }
    eg_status st = make_slot(c, p, lane, out);
    if (st) return st;
    // First use of this plan: capture a slot for every other lane now, so that no graph
    // capture or slot allocation happens later while batches are in flight (measured: a
    // capture inside a pipelined run stalled it, e.g. C2 at depth 6, 15k vs 57k batches/s).
    for (int l = 0; l < c->depth; ++l) {
        bool has = false;
        for (Slot *sl : p->slots) has |= sl->lane == l;
        Slot *extra = nullptr;
        if (!has && (st = make_slot(c, p, l, &extra))) return st;
    }
    return EG_OK;
}

eg_status make_slot(eg_ctx *c, Plan *p, int lane, Slot **out)
{
    Slot *sl = new Slot();
    sl->plan = p;
    sl->lane = lane;
    cudaError_t e = cudaMalloc(&sl->mem, p->total);
    if (e != cudaSuccess) {
        cudaGetLastError();
        delete sl;
        return fail(c, EG_ENOMEM, std::string("batch slot cudaMalloc: ") + cudaGetErrorString(e));
    }
    EG_CUDA(c, cudaMallocHost(&sl->h_meta, sizeof(int32_t) * kMetaSize * p->B));
    EG_CUDA(c, cudaMallocHost(&sl->h_dyn, sizeof(uint64_t) * kDyn * p->B));
    EG_CUDA(c, cudaEventCreateWithFlags(&sl->done, cudaEventDisableTiming));
    EG_CUDA(c, cudaEventCreate(&sl->s0));
    EG_CUDA(c, cudaEventCreate(&sl->s1));
    EG_CUDA(c, cudaEventCreate(&sl->g0));
    EG_CUDA(c, cudaEventCreate(&sl->g1));
    p->slots.push_back(sl);
    eg_status st = capture_slot(c, p, sl);
    if (st) return st;
    *out = sl;
    return EG_OK;
}

void destroy_plans(eg_ctx *c)
{
    for (Plan *p : c->plans) {
        for (Slot *sl : p->slots) {
            if (sl->exec) cudaGraphExecDestroy(sl->exec);
            cudaFree(sl->mem);
            cudaFreeHost(sl->h_meta);
            cudaFreeHost(sl->h_dyn);
            for (cudaEvent_t ev : {sl->done, sl->s0, sl->s1, sl->g0, sl->g1})
                if (ev) cudaEventDestroy(ev);
            for (cudaEvent_t ev : sl->tev) cudaEventDestroy(ev);
            delete sl;
        }
        delete p;
    }
    c->plans.clear();
}

void trace_add(eg_ctx *c, const std::string &name, double ms)
{
    size_t idx = 0;
    while (idx < c->trace_names.size() && c->trace_names[idx] != name) ++idx;
    if (idx == c->trace_names.size()) {
        c->trace_names.push_back(name);
        c->trace_ms.push_back(0);
        c->trace_n.push_back(0);
    }
    c->trace_ms[idx] += ms;
    c->trace_n[idx] += 1;
}

// The slot's last launch has completed (host waited): per-launch timing, once.
void slot_finished(eg_ctx *c, Slot *sl)
{
    if (sl->finished) return;
    sl->finished = true;
    if (!sl->timed) return;
    sl->timed = false;
    float ms = 0;
    if (cudaEventElapsedTime(&ms, sl->s0, sl->s1) == cudaSuccess) {
        c->prof_ms[0] += ms;
        c->prof_n[0] += 1;
    }
    if (sl->plan->features && cudaEventElapsedTime(&ms, sl->g0, sl->g1) == cudaSuccess) {
        c->prof_ms[1] += ms;
        c->prof_n[1] += 1;
    }
    if (c->trace) {
        // in-kernel phase stamps of batch 0 (batch.cu stamp indices): seed, level-0 compaction
        // (kscan, scatter, compact), per hop count/scan/select/copy/tiny + its level's compaction
        const uint64_t *st = reinterpret_cast<const uint64_t *>(sl->h_meta + kMetaStamps);
        std::vector<std::string> names = {"k.seed", "k.l0.kscan", "k.l0.scatter", "k.l0.compact"};
        for (int h = 0; h < sl->plan->n_hops; ++h)
            for (const char *x : {"count", "(unused)", "select", "copy", "tiny", "kscan", "scatter", "compact"})
                names.push_back("k.h" + std::to_string(h) + "." + x);
        for (size_t k = 0; k < names.size() && k < (size_t)kMaxStamps; ++k) {   // a stage runs until the next stamp
            if (!st[k]) continue;
            size_t k2 = k + 1;
            while (k2 < names.size() && k2 < (size_t)kMaxStamps && !st[k2]) ++k2;
            if (k2 >= names.size() || k2 >= (size_t)kMaxStamps) break;
            trace_add(c, names[k], (double)(st[k2] - st[k]) * 1e-6);
        }
        for (size_t k = 1; k < sl->tev.size(); ++k) {
            float e = 0;
            cudaEventElapsedTime(&e, sl->tev[k - 1], sl->tev[k]);
            trace_add(c, sl->tlab[k], e);
        }
    }
}

// Resolve a pending batch: wait for its launch, read sizes and error bits.
eg_status finish(eg_blocks *b)
{
    if (b->ready) return b->status;
    eg_ctx *c = b->ctx;
    if (!c) return EG_ESTATE;   // orphaned by eg_destroy
    Slot *sl = b->slot;
    cudaError_t e = cudaEventSynchronize(sl->done);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c->stream, sl->done, 0);
    b->ready = true;
    if (e != cudaSuccess) return b->status = fail(c, EG_ECUDA, std::string("batch: ") + cudaGetErrorString(e));
    slot_finished(c, sl);
    const int32_t *m = sl->h_meta + (size_t)b->bidx * kMetaSize;
    for (int l = 0; l <= b->n_hops; ++l)
        for (int u = 0; u < b->n_vt; ++u) b->n_nodes[l][u] = m[kMetaNodes + l * EG_MAX_VT + u];
    for (int h = 0; h < b->n_hops; ++h)
        for (int r = 0; r < b->n_rel; ++r) b->nnz[h][r] = m[kMetaNnz + h * EG_MAX_REL + r];
    const int32_t errbits = m[kMetaErr];
    if (errbits & kErrSeedRange)
        return b->status = fail(c, EG_ERANGE, b->lp ? "link-prediction endpoint outside its relation's vertex type"
                                                    : "seed gid outside [0, N_total)");
    if (errbits & kErrSeedDup) return b->status = fail(c, EG_EINVAL, "duplicate seeds");
    if (errbits) {   // cannot happen with true upper bounds; the batch state is not trustworthy
        c->broken = true;
        return b->status = fail(c, EG_ESTATE, "internal capacity overflow");
    }
    return b->status = EG_OK;
}

int64_t round_cap(int64_t n)
{
    int64_t c = 64;
    while (c < n) c <<= 1;
    return c;
}

// Link-prediction inputs of a bundle (NEXT-3).
struct LpArgs {
    const int64_t *const *src;
    const int64_t *const *dst;
    int32_t rel, n_neg;
    const uint64_t *neg_seeds;
};

// A device pointer the kernels can read for host or device memory `p`, or 0 when `p`
// is pageable host memory (then staged into the slot).
uint64_t device_view(const void *p)
{
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) == cudaSuccess &&
        (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged ||
         (at.type == cudaMemoryTypeHost && at.devicePointer)))
        return (uint64_t)(uintptr_t)(at.type == cudaMemoryTypeHost ? at.devicePointer : p);
    cudaGetLastError();
    return 0;
}

// One launch for nb batches (nb <= the context's bundle size).  n_seeds[b] = seeds of
// batch b, or its positives for link prediction (lp != null: seeds unused).
eg_status enqueue_bundle(eg_ctx *c, int32_t nb, const int64_t *const *seeds, const int64_t *n_seeds,
                         int32_t n_hops, const int32_t *fanouts, const uint64_t *rng_seeds, bool features,
                         eg_blocks **out, const LpArgs *lp = nullptr)
{
    eg_status st = enter(c);
    if (st) return st;
    if (!out) return fail(c, EG_EINVAL, "out is null");
    if (!c->loaded || !c->peers_ready) return fail(c, EG_EINVAL, "partition not loaded / peers not mapped");
    if (nb < 1 || nb > kMaxBundle) return fail(c, EG_EINVAL, "bundle size out of [1, kMaxBundle]");
    if (nb > c->bundle) return fail(c, EG_EINVAL, "bundle larger than eg_set_pipeline's bundle size");
    if (n_hops < 1 || n_hops > EG_MAX_HOPS) return fail(c, EG_EINVAL, "n_hops out of [1, EG_MAX_HOPS]");
    if (!fanouts || !n_seeds || !rng_seeds || (!lp && !seeds)) return fail(c, EG_EINVAL, "null argument");
    if (lp) {
        if (!lp->src || !lp->dst || !lp->neg_seeds) return fail(c, EG_EINVAL, "null argument");
        if (lp->rel < 0 || lp->rel >= c->g.n_rel) return fail(c, EG_EINVAL, "relation out of range");
        if (lp->n_neg < 0 || lp->n_neg > EG_MAX_NEG) return fail(c, EG_EINVAL, "n_neg out of [0, EG_MAX_NEG]");
    }
    int64_t nmax = 0;
    for (int b = 0; b < nb; ++b) {
        out[b] = nullptr;
        const bool bad = lp ? (n_seeds[b] > 0 && (!lp->src[b] || !lp->dst[b])) : (n_seeds[b] > 0 && !seeds[b]);
        if (n_seeds[b] < 0 || bad) return fail(c, EG_EINVAL, lp ? "bad positives" : "bad seeds");
        if (lp && n_seeds[b] >= ((int64_t)1 << 31)) return fail(c, EG_EINVAL, "more than 2^31 positives");
        nmax = std::max(nmax, n_seeds[b]);
    }
    for (int i = 0; i < n_hops * c->g.n_rel; ++i)
        if (fanouts[i] < -1) return fail(c, EG_EINVAL, "fanout must be >= -1");
    // a single batch uses a 1-batch plan; bundles use the context's bundle size
    const int32_t B = nb == 1 ? 1 : c->bundle;
    Plan *p = nullptr;
    if ((st = get_plan(c, n_hops, fanouts, round_cap(nmax), features, B, &p, lp != nullptr, lp ? lp->n_neg : 0)))
        return st;
    Slot *sl = nullptr;
    if ((st = acquire_slot(c, p, &sl))) return st;
    Lane &ln = c->lanes[sl->lane];
    EG_CUDA(c, cudaEventRecord(ln.ready, c->stream));          // inputs produced on the caller's stream
    EG_CUDA(c, cudaStreamWaitEvent(ln.stream, ln.ready, 0));
    for (int b = 0; b < B; ++b) {
        const int64_t n = b < nb ? n_seeds[b] : 0;
        uint64_t *dyn = sl->h_dyn + (size_t)kDyn * b;
        for (int k = 0; k < kDyn; ++k) dyn[k] = 0;
        dyn[0] = b < nb ? rng_seeds[b] : 0;
        dyn[1] = (uint64_t)n;
        // device memory (or pinned host memory, read over PCIe): the kernels read the
        // caller's buffer in place; pageable host memory is staged into the slot
        char *base = p->batch_base(sl->mem, b);
        auto place = [&](const int64_t *src, size_t off, uint64_t *slot) -> eg_status {
            if (n <= 0) return EG_OK;
            *slot = device_view(src);
            if (!*slot)
                EG_CUDA(c, cudaMemcpyAsync(base + off, src, sizeof(int64_t) * n, cudaMemcpyDefault, ln.stream));
            return EG_OK;
        };
        if (!lp) {
            if ((st = place(b < nb ? seeds[b] : nullptr, p->o_seeds, &dyn[2]))) return st;
        } else {
            if ((st = place(b < nb ? lp->src[b] : nullptr, p->o_lp_src, &dyn[2]))) return st;
            if ((st = place(b < nb ? lp->dst[b] : nullptr, p->o_lp_dst, &dyn[3]))) return st;
            dyn[4] = b < nb ? lp->neg_seeds[b] : 0;
            dyn[5] = (uint64_t)lp->rel;
        }
    }
    sl->timed = c->prof;
    sl->finished = false;
    if (p->features) c->gather_path = sl->gather_path;
    EG_CUDA(c, cudaGraphLaunch(sl->exec, ln.stream));
    EG_CUDA(c, cudaEventRecord(sl->done, ln.stream));
    sl->used = true;
    sl->refs = nb;
    c->launches += p->n_kernels;
    for (int b = 0; b < nb; ++b) {
        eg_blocks *h = new eg_blocks();
        h->ctx = c;
        h->slot = sl;
        h->bidx = b;
        h->n_hops = n_hops;
        h->n_vt = c->g.n_vt;
        h->n_rel = c->g.n_rel;
        fill_views(p, p->batch_base(sl->mem, b), h);
        if (lp) {
            h->lp = true;
            h->lp_rel = lp->rel;
            h->n_neg = lp->n_neg;
            h->n_pos = n_seeds[b];
            h->cap_pos = p->n_cap;
            h->pairs = (int32_t *)(p->batch_base(sl->mem, b) + p->o_lp_pairs);
            h->neg = (int64_t *)(p->batch_base(sl->mem, b) + p->o_lp_neg);
        }
        c->live.insert(h);
        out[b] = h;
    }
    return EG_OK;
}

}  // namespace

extern "C" {

eg_status eg_sample_blocks(eg_ctx *c, const int64_t *seeds, int64_t n_seeds, int32_t n_hops,
                           const int32_t *fanouts, uint64_t rng_seed, eg_blocks **out)
{
    return eg_sample_minibatch(c, seeds, n_seeds, n_hops, fanouts, rng_seed, 0, out);
}

eg_status eg_sample_minibatch(eg_ctx *c, const int64_t *seeds, int64_t n_seeds, int32_t n_hops,
                              const int32_t *fanouts, uint64_t rng_seed, int32_t flags, eg_blocks **out)
{
    return eg_sample_bundle(c, 1, &seeds, &n_seeds, n_hops, fanouts, &rng_seed, flags, out);
}

eg_status eg_sample_bundle(eg_ctx *c, int32_t n_batches, const int64_t *const *seeds, const int64_t *n_seeds,
                           int32_t n_hops, const int32_t *fanouts, const uint64_t *rng_seeds, int32_t flags,
                           eg_blocks **out)
{
    eg_status st = enqueue_bundle(c, n_batches, seeds, n_seeds, n_hops, fanouts, rng_seeds,
                                  (flags & EG_FEATURES) != 0, out);
    if (st) return st;
    if (!(flags & EG_ASYNC)) {
        eg_status first = EG_OK;
        for (int b = 0; b < n_batches; ++b) {
            st = finish(out[b]);
            if (st && !first) first = st;
        }
        if (first) {
            for (int b = 0; b < n_batches; ++b) {
                eg_blocks_free(out[b]);
                out[b] = nullptr;
            }
            return first;
        }
    }
    return EG_OK;
}

eg_status eg_sample_lp_bundle(eg_ctx *c, int32_t n_batches, const int64_t *const *src, const int64_t *const *dst,
                              const int64_t *n_pos, int32_t rel, int32_t n_neg, const uint64_t *neg_seeds,
                              int32_t n_hops, const int32_t *fanouts, const uint64_t *rng_seeds, int32_t flags,
                              eg_blocks **out)
{
    LpArgs lp{src, dst, rel, n_neg, neg_seeds};
    eg_status st = enqueue_bundle(c, n_batches, nullptr, n_pos, n_hops, fanouts, rng_seeds,
                                  (flags & EG_FEATURES) != 0, out, &lp);
    if (st) return st;
    if (!(flags & EG_ASYNC)) {
        eg_status first = EG_OK;
        for (int b = 0; b < n_batches; ++b) {
            st = finish(out[b]);
            if (st && !first) first = st;
        }
        if (first) {
            for (int b = 0; b < n_batches; ++b) {
                eg_blocks_free(out[b]);
                out[b] = nullptr;
            }
            return first;
        }
    }
    return EG_OK;
}

eg_status eg_lp_view_get(const eg_blocks *cb, eg_lp_view *out)
{
    if (!cb || !out) return EG_EINVAL;
    eg_blocks *b = const_cast<eg_blocks *>(cb);
    if (!b->lp) return EG_EINVAL;
    eg_status st = finish(b);
    if (st) return st;
    const int64_t cap = b->cap_pos, m = (int64_t)b->n_neg;
    out->n_pos = b->n_pos;
    out->n_neg = b->n_neg;
    out->rel = b->lp_rel;
    out->pos_src = b->pairs;
    out->pos_dst = b->pairs + cap;
    out->neg_src = b->pairs + 2 * cap;
    out->neg_dst = b->pairs + 2 * cap + cap * m;
    out->neg_dst_gid = b->neg;
    return EG_OK;
}

eg_status eg_sage_mean_layer(eg_ctx *c, const eg_blocks *cb, int32_t hop, int32_t rel, const void *x_src,
                             int32_t x_dtype, int64_t ld_src, const void *x_dst, int64_t ld_dst, int32_t F,
                             const void *w, int32_t H, float *out, int64_t ld_out, int32_t flags)
{
    eg_status st = enter(c);
    if (st) return st;
    if (!cb) return fail(c, EG_EINVAL, "blocks is null");
    eg_blocks *b = const_cast<eg_blocks *>(cb);
    if ((st = finish(b))) return st;
    if (hop < 0 || hop >= b->n_hops || rel < 0 || rel >= b->n_rel) return fail(c, EG_EINVAL, "hop / rel out of range");
    if (F < 1 || F > 256) return fail(c, EG_EINVAL, "F must be in [1, 256]");
    if (H < 16 || H > 256 || H % 16) return fail(c, EG_EINVAL, "H must be a multiple of 16 in [16, 256]");
    if (x_dtype < 0 || x_dtype > 2) return fail(c, EG_EINVAL, "x_dtype must be 0 (f32), 1 (f16) or 2 (bf16)");
    if (!x_src || !w || !out) return fail(c, EG_EINVAL, "null operand");
    const int esz = x_dtype == 0 ? 4 : 2;
    auto aligned = [&](const void *p, int64_t ld) {
        return ((uintptr_t)p % 16) == 0 && (ld * esz) % 16 == 0 && ld >= F;
    };
    if (!aligned(x_src, ld_src) || (x_dst && !aligned(x_dst, ld_dst)))
        return fail(c, EG_EINVAL, "input rows must be 16-byte aligned with ld >= F");
    if (((uintptr_t)out % 16) || ld_out % 4 || ld_out < H) return fail(c, EG_EINVAL, "out rows must be 16-byte aligned");
    if (sage_smem_bytes(F, H, x_dst != nullptr) > 200 * 1024)
        return fail(c, EG_EINVAL, "shared-memory budget exceeded: (128 + H) * padded K * 2 > 200 KB");
    const int t = c->g.rel[rel].dst_vt;
    SageArgs a{};
    a.indptr = b->indptr[hop][rel];
    a.indices = b->indices[hop][rel];
    a.x_src = x_src;
    a.x_dst = x_dst;
    a.ld_src = ld_src;
    a.ld_dst = ld_dst;
    a.w = w;
    a.out = out;
    a.ld_out = ld_out;
    a.n_dst = (int32_t)b->n_nodes[hop][t];
    a.F = F;
    a.H = H;
    a.accumulate = (flags & EG_ACCUMULATE) ? 1 : 0;
    uint32_t cols = 32;
    while ((int)cols < H) cols <<= 1;
    a.tmem_cols = cols;
    // W by the TMA when its [H][parts][F] view has 16-B strides (EG_SAGE_W_TMA=0: by the warps)
    static const bool w_tma_env = !getenv("EG_SAGE_W_TMA") || atoi(getenv("EG_SAGE_W_TMA")) != 0;
    a.w_tma = 0;
    if (w_tma_env && F % 8 == 0 && ((uintptr_t)w % 16) == 0) {
        if (EncodeTiledFn fn = encode_tiled()) {
            const int parts = x_dst ? 2 : 1;
            cuuint64_t dims[3] = {(cuuint64_t)F, (cuuint64_t)parts, (cuuint64_t)H};
            cuuint64_t strides[2] = {(cuuint64_t)F * 2, (cuuint64_t)parts * F * 2};
            cuuint32_t box[3] = {64u, 1u, (cuuint32_t)H};
            cuuint32_t es[3] = {1u, 1u, 1u};
            a.w_tma = fn(&a.wmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(w), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
        }
    }
    EG_CUDA(c, launch_sage(a, x_dtype, c->stream));
    ++c->launches;
    return EG_OK;
}

eg_status eg_blocks_stats(const eg_blocks *cb, int64_t *total_edges, int64_t *n_inputs)
{
    if (!cb) return EG_EINVAL;
    eg_blocks *b = const_cast<eg_blocks *>(cb);
    eg_status st = finish(b);
    if (st) return st;
    if (total_edges) {
        int64_t e = 0;
        for (int h = 0; h < b->n_hops; ++h)
            for (int r = 0; r < b->n_rel; ++r) e += b->nnz[h][r];
        *total_edges = e;
    }
    if (n_inputs)
        for (int u = 0; u < b->n_vt; ++u) n_inputs[u] = b->n_nodes[b->n_hops][u];
    return EG_OK;
}

eg_status eg_blocks_wait(eg_blocks *b)
{
    if (!b) return EG_EINVAL;
    if (!b->ctx) return EG_ESTATE;
    cudaSetDevice(b->ctx->device);
    return finish(b);
}

int32_t eg_blocks_n_hops(const eg_blocks *b) { return b ? b->n_hops : 0; }

int64_t eg_blocks_n_inputs(const eg_blocks *b, int32_t u)
{
    if (!b || u < 0 || u >= b->n_vt) return -1;
    if (finish(const_cast<eg_blocks *>(b))) return -1;
    return b->n_nodes[b->n_hops][u];
}

eg_status eg_block_view_get(const eg_blocks *cb, int32_t hop, eg_block_view *v)
{
    if (!cb || !v || hop < 0 || hop >= cb->n_hops) return EG_EINVAL;
    eg_blocks *b = const_cast<eg_blocks *>(cb);
    eg_status st = finish(b);
    if (st) return st;
    memset(v, 0, sizeof(*v));
    v->hop = hop;
    v->n_vt = b->n_vt;
    v->n_rel = b->n_rel;
    for (int u = 0; u < b->n_vt; ++u) {
        v->dst_nodes[u] = b->nodes[u];
        v->n_dst[u] = b->n_nodes[hop][u];
        v->src_nodes[u] = b->nodes[u];
        v->n_src[u] = b->n_nodes[hop + 1][u];
    }
    for (int r = 0; r < b->n_rel; ++r) {
        v->indptr[r] = b->indptr[hop][r];
        v->indices[r] = b->indices[hop][r];
        v->eids[r] = b->eids[hop][r];
        v->nnz[r] = b->nnz[hop][r];
    }
    return EG_OK;
}

eg_status eg_blocks_features(const eg_blocks *cb, int32_t u, const void **rows, int64_t *n_rows, int64_t *row_bytes)
{
    if (!cb || u < 0 || u >= cb->n_vt || !rows || !n_rows || !row_bytes) return EG_EINVAL;
    eg_blocks *b = const_cast<eg_blocks *>(cb);
    eg_status st = finish(b);
    if (st) return st;
    *rows = b->feat[u];
    *n_rows = b->feat[u] ? b->n_nodes[b->n_hops][u] : 0;
    *row_bytes = b->feat[u] ? b->ctx->f.row_bytes[u] : 0;
    return EG_OK;
}

eg_status eg_blocks_copy_features(const eg_blocks *cb, void *const *host, int32_t flags)
{
    if (!cb || !host) return EG_EINVAL;
    eg_blocks *b = const_cast<eg_blocks *>(cb);
    if (!b->ctx) return EG_ESTATE;
    eg_ctx *c = b->ctx;
    eg_status st = enter(c);
    if (st) return st;
    if ((st = finish(b))) return st;   // sizes (the launch has completed on its lane)
    for (int u = 0; u < b->n_vt; ++u) {
        if (!host[u]) continue;
        if (!b->feat[u]) return fail(c, EG_EINVAL, "vertex type " + std::to_string(u) + " has no gathered rows");
        const int64_t bytes = b->n_nodes[b->n_hops][u] * c->f.row_bytes[u];
        if (bytes) EG_CUDA(c, cudaMemcpyAsync(host[u], b->feat[u], (size_t)bytes, cudaMemcpyDeviceToHost, c->stream));
    }
    if (!(flags & EG_ASYNC)) EG_CUDA(c, cudaStreamSynchronize(c->stream));
    return EG_OK;
}

eg_status eg_gather_features(eg_ctx *c, const eg_blocks *cb, void *const *out)
{
    eg_status st = enter(c);
    if (st) return st;
    if (!cb || !out || cb->ctx != c) return fail(c, EG_EINVAL, "bad blocks / out");
    eg_blocks *b = const_cast<eg_blocks *>(cb);
    if ((st = finish(b))) return st;
    GatherSet gs{};
    gs.nb = 1;
    GatherDev &gd = gs.b[0];
    gd.meta = b->meta;
    gd.level = b->n_hops;
    void *staging[EG_MAX_VT] = {};
    bool any = false;
    for (int u = 0; u < b->n_vt; ++u) {
        gd.nodes[u] = b->nodes[u];
        if (!out[u]) continue;
        if (!c->f.row_bytes[u]) return fail(c, EG_EINVAL, "vertex type " + std::to_string(u) + " has no features");
        const int64_t bytes = b->n_nodes[b->n_hops][u] * c->f.row_bytes[u];
        if (bytes == 0) continue;
        if (is_device_ptr(out[u])) {
            gd.out[u] = (uint8_t *)out[u];
        } else {
            EG_CUDA(c, cudaMallocAsync(&staging[u], bytes, c->stream));
            gd.out[u] = (uint8_t *)staging[u];
        }
        any = true;
    }
    if (!any) return EG_OK;
    TimedPair tp;
    record_start(c, &tp, 1);
    c->gather_path = launch_gather(c->g, c->f, gs, c->gmaps, c->stream, c->gather_mode);
    c->launches += 1;
    EG_CUDA(c, cudaGetLastError());
    record_end(c, &tp);
    bool staged = false;
    for (int u = 0; u < b->n_vt; ++u)
        if (staging[u]) {
            EG_CUDA(c, cudaMemcpyAsync(out[u], staging[u], b->n_nodes[b->n_hops][u] * c->f.row_bytes[u],
                                       cudaMemcpyDeviceToHost, c->stream));
            EG_CUDA(c, cudaFreeAsync(staging[u], c->stream));
            staged = true;
        }
    if (staged) EG_CUDA(c, cudaStreamSynchronize(c->stream));
    return EG_OK;
}

eg_status eg_blocks_free(eg_blocks *b)
{
    if (!b) return EG_OK;
    if (b->ctx) {   // else orphaned: its context (and slot) are gone, only the handle remains
        b->ctx->live.erase(b);
        if (b->slot && b->slot->refs > 0) b->slot->refs -= 1;   // reuse waits for the slot's last run
    }
    delete b;
    return EG_OK;
}

eg_status eg_set_pipeline(eg_ctx *c, int32_t depth, int32_t bundle)
{
    eg_status st = enter(c);
    if (st) return st;
    if (!c->loaded) return fail(c, EG_EINVAL, "load the partition first");
    if (depth < 1 || depth > 16) return fail(c, EG_EINVAL, "pipeline depth must be in [1, 16]");
    if (bundle < 1 || bundle > kMaxBundle) return fail(c, EG_EINVAL, "bundle size must be in [1, kMaxBundle]");
    if ((st = ensure_lanes(c, depth))) return st;
    c->next_lane = 0;
    c->depth = depth;
    c->bundle = bundle;
    return EG_OK;
}

int32_t eg_trace_get(const eg_ctx *c, int32_t i, char *name, size_t name_len, double *total_ms, int64_t *count)
{
    if (!c) return 0;
    const int32_t n = (int32_t)c->trace_names.size();
    if (i >= 0 && i < n) {
        if (name && name_len) {
            strncpy(name, c->trace_names[i].c_str(), name_len - 1);
            name[name_len - 1] = 0;
        }
        if (total_ms) *total_ms = c->trace_ms[i];
        if (count) *count = c->trace_n[i];
    }
    return n;
}

eg_status eg_set_profiling(eg_ctx *c, int32_t enable)
{
    if (!c) return EG_EINVAL;
    c->prof = enable != 0;
    return EG_OK;
}

eg_status eg_get_profile(eg_ctx *c, double out[4])
{
    eg_status st = enter(c);
    if (st) return st;
    drain_timing(c);
    out[0] = c->prof_ms[0];
    out[1] = c->prof_ms[1];
    out[2] = (double)c->prof_n[0];
    out[3] = (double)c->prof_n[1];
    c->prof_ms[0] = c->prof_ms[1] = 0;
    c->prof_n[0] = c->prof_n[1] = 0;
    return EG_OK;
}

eg_status eg_destroy(eg_ctx *c)
{
    if (!c) return EG_OK;
    cudaSetDevice(c->device);
    // every launch still in flight (async batches never resolved) reads slot memory and
    // the peer mappings: wait for all lanes before anything is released
    cudaStreamSynchronize(c->stream);
    for (Lane &ln : c->lanes)
        if (ln.stream) cudaStreamSynchronize(ln.stream);
    cudaDeviceSynchronize();
    drain_timing(c);
    // handles the caller has not freed: orphan them, so that a later eg_blocks_free only
    // deletes the handle and every other call on it returns EG_ESTATE
    for (eg_blocks *b : c->live) {
        b->ctx = nullptr;
        b->slot = nullptr;
        b->ready = true;
        b->status = EG_ESTATE;
    }
    c->live.clear();
    destroy_plans(c);
    if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
    if (c->fork.side) cudaStreamDestroy(c->fork.side);
    if (c->fork.fork) cudaEventDestroy(c->fork.fork);
    if (c->fork.join) cudaEventDestroy(c->fork.join);
    for (void *p : c->ipc_bases) cudaIpcCloseMemHandle(p);
    for (Lane &ln : c->lanes) {
        if (ln.stream) cudaStreamSynchronize(ln.stream);
        if (ln.ready) cudaEventDestroy(ln.ready);
        if (ln.stream) cudaStreamDestroy(ln.stream);
    }
    c->lanes.clear();
    delete c;
    return EG_OK;
}

}  // extern "C"
