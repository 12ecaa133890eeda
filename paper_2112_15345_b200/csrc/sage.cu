// sage.cu -- the consumer step of a mini-batch (SURVEY §8f NEXT-4 i): one GraphSAGE-mean
// layer over a block relation, pre-activation (DESIGN.md §3 readings C1-C2):
//
//   z_v = W_self h_v + W_neigh mean_{u in N_block(v)} h_u        (Eq. 1)
//
// as ONE fused kernel on the 5th-generation tensor cores: z = [X_dst | M] [W_self | W_neigh]^T
// where the mean-aggregated rows M are never written to HBM.  Persistent CTAs (one per SM,
// 16 warps):
//   * W (H x K, bf16) is staged once per CTA into shared memory in the canonical 128-byte-
//     swizzled K-major layout the MMA reads -- by the TMA (3-D boxes of a [H][parts][F]
//     view, SWIZZLE_128B, zero-filled padding) while the warps build the first A tile, or
//     by the warps when F % 8 != 0;
//   * per tile of 128 dst rows each warp builds 8 consecutive rows of the A operand in the
//     same layout: the self rows (bf16) and the neighbour means (fp32 sums of coalesced
//     warp-wide row reads, up to 32 / NW of them in flight per warp, then bf16);
//   * one thread issues K/16 tcgen05.mma.cta_group::1.kind::f16 (M = 128, N = H) into a
//     TMEM accumulator and commits them to an mbarrier;
//   * the epilogue drains the accumulator with tcgen05.ld (warp w: TMEM lanes 32 (w % 4)
//     .. +31 = tile rows), stages it through A's shared memory and stores full fp32 row
//     segments.
// Measured per C4 tile (globaltimer stamps, EG_SAGE_TRACE): A build ~8 us, MMA ~1.4 us,
// epilogue ~3 us (profiles/r02/sage/).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "kernels.h"

namespace eg {

namespace {

__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// UMMA shared-memory matrix descriptor: K-major, 128-byte swizzle, 8-row atoms of 1024 B
// (start address, LBO = 16 B (unused for this layout), SBO = 1024 B, version 1, layout 2).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr)
{
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// Instruction descriptor of kind::f16: D fp32, A / B bf16, both K-major, M = 128, N = n.
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int n)
{
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ void mbar_init1(uint64_t *bar)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_wait_parity(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "SAGE_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra SAGE_WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

// Byte offset of (row, k) in a K-major SW128 operand of `rows` rows: 64-column blocks of
// rows x 128 B, 16-B chunk index XOR (row mod 8) inside each 8-row atom.
__device__ __forceinline__ uint32_t sw128_off(int rows, int row, int k)
{
    return (uint32_t)((k >> 6) * rows * 128 + row * 128 + ((((k & 63) >> 3) ^ (row & 7)) << 4) + ((k & 7) << 1));
}

template <typename T> __device__ __forceinline__ float to_f(T x);
template <> __device__ __forceinline__ float to_f<float>(float x) { return x; }
template <> __device__ __forceinline__ float to_f<__half>(__half x) { return __half2float(x); }
template <> __device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

// CPL consecutive elements of a row from column c (c + CPL <= F: one vector load; the
// host checks 16-byte aligned rows), converted to fp32; columns >= F read as 0.
template <typename T, int CPL>
__device__ __forceinline__ void load_cols(const T *row, int c, int F, float (&v)[CPL])
{
    if (c + CPL <= F) {
        constexpr int B = CPL * (int)sizeof(T);
        if constexpr (B == 32) {
            const uint4 a = __ldg(reinterpret_cast<const uint4 *>(row + c));
            const uint4 b = __ldg(reinterpret_cast<const uint4 *>(row + c) + 1);
            const T *ea = reinterpret_cast<const T *>(&a), *eb = reinterpret_cast<const T *>(&b);
#pragma unroll
            for (int e = 0; e < CPL / 2; ++e) {
                v[e] = to_f(ea[e]);
                v[CPL / 2 + e] = to_f(eb[e]);
            }
        } else if constexpr (B == 16) {
            const uint4 a = __ldg(reinterpret_cast<const uint4 *>(row + c));
            const T *ea = reinterpret_cast<const T *>(&a);
#pragma unroll
            for (int e = 0; e < CPL; ++e) v[e] = to_f(ea[e]);
        } else if constexpr (B == 8) {
            const uint2 a = __ldg(reinterpret_cast<const uint2 *>(row + c));
            const T *ea = reinterpret_cast<const T *>(&a);
#pragma unroll
            for (int e = 0; e < CPL; ++e) v[e] = to_f(ea[e]);
        } else {
#pragma unroll
            for (int e = 0; e < CPL; ++e) v[e] = to_f(row[c + e]);
        }
    } else {
#pragma unroll
        for (int e = 0; e < CPL; ++e) v[e] = c + e < F ? to_f(row[c + e]) : 0.f;
    }
}

// CPL fp32 values -> bf16 into the A / B operand at (row, k..k+CPL-1) (one 16-B chunk).
template <int CPL>
__device__ __forceinline__ void store_bf16(uint8_t *base, int rows, int row, int k, const float (&v)[CPL])
{
    uint32_t p[CPL / 2];
#pragma unroll
    for (int e = 0; e < CPL / 2; ++e) {
        const __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
        p[e] = *reinterpret_cast<const uint32_t *>(&h);
    }
    uint8_t *dst = base + sw128_off(rows, row, k);
    if constexpr (CPL == 8) *reinterpret_cast<uint4 *>(dst) = make_uint4(p[0], p[1], p[2], p[3]);
    else if constexpr (CPL == 4) *reinterpret_cast<uint2 *>(dst) = make_uint2(p[0], p[1]);
    else *reinterpret_cast<uint32_t *>(dst) = p[0];
}

// Raw row slice for the A build: the CPL elements of columns c .. c+CPL-1 as NW 32-bit
// words (vector loads when the slice is inside the row; columns >= F read as 0).  The
// loads of a whole group of edges are issued before any is converted, so a warp keeps
// 32 / NW row reads in flight.
template <typename T, int CPL> constexpr int raw_words() { return CPL * (int)sizeof(T) / 4; }

template <typename T, int CPL>
__device__ __forceinline__ void load_raw(const T *row, int c, int F, uint32_t (&u)[raw_words<T, CPL>()])
{
    constexpr int NW = raw_words<T, CPL>();
    if (c + CPL <= F) {
        const uint32_t *p = reinterpret_cast<const uint32_t *>(row + c);
        if constexpr (NW == 1) {
            u[0] = __ldg(p);
        } else if constexpr (NW == 2) {
            const uint2 x = __ldg(reinterpret_cast<const uint2 *>(p));
            u[0] = x.x; u[1] = x.y;
        } else {
#pragma unroll
            for (int q = 0; q < NW / 4; ++q) {
                const uint4 x = __ldg(reinterpret_cast<const uint4 *>(p) + q);
                u[4 * q] = x.x; u[4 * q + 1] = x.y; u[4 * q + 2] = x.z; u[4 * q + 3] = x.w;
            }
        }
    } else {
#pragma unroll
        for (int q = 0; q < NW; ++q) u[q] = 0u;   // zero bits = 0.0 in every input type
        T *e = reinterpret_cast<T *>(u);
#pragma unroll
        for (int i = 0; i < CPL; ++i)
            if (c + i < F) e[i] = row[c + i];
    }
}

template <typename T, int CPL>
__device__ __forceinline__ void raw_add(float (&acc)[CPL], const uint32_t (&u)[raw_words<T, CPL>()])
{
    const T *e = reinterpret_cast<const T *>(u);
#pragma unroll
    for (int i = 0; i < CPL; ++i) acc[i] += to_f(e[i]);
}

#ifdef EG_SAGE_TRACE
// phase timing (A/B builds only): thread 0 of CTAs 0 and 100 keeps globaltimer stamps
// (0 entry, 1 W staged, then per tile 2 A built, 3 MMA done, 4 epilogue done; 9 exit) and
// writes them as raw u64 into output rows 0 / 1 at exit (the outputs are then wrong).
#define SAGE_STAMP(k)                                                                                  \
    do {                                                                                               \
        if (threadIdx.x == 0) {                                                                        \
            uint64_t t_;                                                                               \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                     \
            const int i_ = (k) <= 1 ? (k) : (k) == 5 ? 9 : 2 + 3 * (tile_no < 2 ? tile_no : 1) + (k) - 2; \
            stamps[i_] = t_;                                                                           \
        }                                                                                              \
    } while (0)
#else
#define SAGE_STAMP(k) do {} while (0)
#endif
constexpr int kTileM = 128;
// warps per CTA (A-operand builders; TMEM lane group = warp % 4): 16, so that each lane
// can hold a group of raw row slices in flight (128 registers); measured against 32 warps
// x 4 rows with 4 rows in flight per warp (round 1): C4 45.6 vs 70.3 us, C2 28.6 vs 42.0
// us cold, C3 +1 % (profiles/r02/sage/)
template <int CPL> __host__ __device__ constexpr int warps_for() { return 16; }

// Epilogue of one tile: warp w drains TMEM lanes 32 (w % 4) .. +31 (= tile rows), CW
// columns at a time (column groups w / 4), into its 32 x CW fp32 slice of the staging area
// (float4 slots XOR-swizzled by row: conflict-free both ways), then writes the slice back
// row by row: each store instruction covers 32 / (CW / 4) rows x CW * 4 contiguous bytes
// (round 2; a lane-per-row store touched 32 lines per instruction and, with the MMA,
// took ~40 % of the kernel: ncu, profiles/r02/sage/).
// Epilogue without staging (A smaller than the staging slices: K = 64 without the self
// term): lane = row, 8 fp32 per TMEM load stored as two float4.
template <int kWarps>
__device__ __forceinline__ void epilogue_rows(const SageArgs &a, uint32_t tmem, int row0, int warp, int lane)
{
    const int lg = warp & 3;
    const int row = row0 + lg * 32 + lane;
    float *orow = a.out + (int64_t)row * a.ld_out;
    for (int col = (warp >> 2) * 8; col < a.H; col += 2 * kWarps) {
        uint32_t r[8];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
            : "r"(tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)col));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (row < a.n_dst) {
            float4 x0 = make_float4(__uint_as_float(r[0]), __uint_as_float(r[1]), __uint_as_float(r[2]),
                                    __uint_as_float(r[3]));
            float4 x1 = make_float4(__uint_as_float(r[4]), __uint_as_float(r[5]), __uint_as_float(r[6]),
                                    __uint_as_float(r[7]));
            float4 *o = reinterpret_cast<float4 *>(orow + col);
            if (a.accumulate) {
                const float4 p0 = o[0], p1 = o[1];
                x0.x += p0.x; x0.y += p0.y; x0.z += p0.z; x0.w += p0.w;
                x1.x += p1.x; x1.y += p1.y; x1.z += p1.z; x1.w += p1.w;
            }
            o[0] = x0;
            o[1] = x1;
        }
    }
}

template <int CW, int kWarps>
__device__ __forceinline__ void epilogue(const SageArgs &a, uint32_t tmem, float *stage_all, int row0, int warp, int lane)
{
    constexpr int F4 = CW / 4;          // float4 slots per staged row
    constexpr int RPI = 32 / F4;        // rows per store instruction
    constexpr int SW = 8 / F4;          // rows sharing a swizzle phase
    float *stage = stage_all + warp * (32 * CW);
    const int lg = warp & 3;
    for (int col0 = (warp >> 2) * CW; col0 < a.H; col0 += (kWarps / 4) * CW) {
        const int nc = min(CW, a.H - col0);   // a multiple of 8 (H % 16 == 0)
        uint32_t r[CW];
#pragma unroll
        for (int q = 0; q < CW / 8; ++q) {
            if (8 * q < nc)
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                    : "=r"(r[8 * q]), "=r"(r[8 * q + 1]), "=r"(r[8 * q + 2]), "=r"(r[8 * q + 3]), "=r"(r[8 * q + 4]),
                      "=r"(r[8 * q + 5]), "=r"(r[8 * q + 6]), "=r"(r[8 * q + 7])
                    : "r"(tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(col0 + 8 * q)));
            else
#pragma unroll
                for (int e = 0; e < 8; ++e) r[8 * q + e] = 0u;
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int c4 = 0; c4 < F4; ++c4) {
            const int ph = c4 ^ ((lane / SW) % F4);
            *reinterpret_cast<float4 *>(stage + lane * CW + 4 * ph) =
                make_float4(__uint_as_float(r[4 * c4]), __uint_as_float(r[4 * c4 + 1]), __uint_as_float(r[4 * c4 + 2]),
                            __uint_as_float(r[4 * c4 + 3]));
        }
        __syncwarp();
        const int c4 = lane % F4;
#pragma unroll
        for (int it = 0; it < F4; ++it) {
            const int rr = it * RPI + lane / F4;
            const int ph = c4 ^ ((rr / SW) % F4);
            float4 x = *reinterpret_cast<const float4 *>(stage + rr * CW + 4 * ph);
            const int row = row0 + lg * 32 + rr;
            if (row < a.n_dst && 4 * c4 < nc) {
                float4 *o = reinterpret_cast<float4 *>(a.out + (int64_t)row * a.ld_out + col0 + 4 * c4);
                if (a.accumulate) {
                    const float4 p = *o;
                    x.x += p.x; x.y += p.y; x.z += p.z; x.w += p.w;
                }
                *o = x;
            }
        }
        __syncwarp();
    }
}

// CPL = Fp / 32 columns per lane (Fp = F rounded up to 64).
template <typename T, int CPL>
__global__ void __launch_bounds__(warps_for<CPL>() * 32, 1) sage_kernel(const __grid_constant__ SageArgs a)
{
    constexpr int kWarps = warps_for<CPL>();
    constexpr int R = kTileM / kWarps;            // rows per warp
    constexpr int NW = raw_words<T, CPL>();       // words per lane per row slice
    constexpr int S = 32 / NW;                    // edges whose row loads are in flight together
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    constexpr int Fp = CPL * 32;
    const int parts = a.x_dst ? 2 : 1;                // [self | neigh] or [neigh]
    const int Kp = parts * Fp;
    uint8_t *sB = smem;                               // H x Kp
    uint8_t *sA = smem + (size_t)a.H * Kp * 2;        // 128 x Kp
    uint64_t *mbar = reinterpret_cast<uint64_t *>(sA + (size_t)kTileM * Kp * 2);   // MMA done
    uint64_t *mbar_w = mbar + 1;                                                     // W staged (TMA)
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(mbar + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int tile_no = -1;
    (void)tile_no;
#ifdef EG_SAGE_TRACE
    uint64_t stamps[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#endif
    SAGE_STAMP(0);

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_slot)),
                     "r"(a.tmem_cols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x == 32) {
        mbar_init1(mbar);
        mbar_init1(mbar_w);
    }
    if (!a.w_tma) {
        // W -> sB by the warps: padded column kp of part p maps to W column p * F + (kp - p * Fp)
        const int K = parts * a.F;
        const __nv_bfloat16 *wt = static_cast<const __nv_bfloat16 *>(a.w);
        const bool wvec = (a.F % 8) == 0 && ((uintptr_t)a.w % 16) == 0;   // 16-B chunks of W rows
        for (int i = threadIdx.x; i < a.H * (Kp / 8); i += blockDim.x) {
            const int n = i / (Kp / 8), kp = (i % (Kp / 8)) * 8;
            const int p = kp / Fp, c = kp - p * Fp;
            uint8_t *dst = sB + sw128_off(a.H, n, kp);
            if (wvec) {   // bf16 bits copied as they are
                const uint4 v = c < a.F ? __ldg(reinterpret_cast<const uint4 *>(wt + (int64_t)n * K + p * a.F + c))
                                        : make_uint4(0, 0, 0, 0);
                *reinterpret_cast<uint4 *>(dst) = v;
            } else {
                float v[8];
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    v[e] = c + e < a.F ? __bfloat162float(wt[(int64_t)n * K + p * a.F + c + e]) : 0.f;
                store_bf16<8>(sB, a.H, n, kp, v);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (a.w_tma && threadIdx.x == 0) {
        // W -> sB by the TMA while the warps build the first A tile: per part and 64-column
        // block one 3-D box {64, 1, H} of the [H][parts][F] view of W; SWIZZLE_128B writes the
        // canonical K-major layout and zero-fills the padding columns F .. Fp-1
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(mbar_w)),
                     "r"(a.H * Kp * 2)
                     : "memory");
        for (int p = 0; p < parts; ++p)
            for (int j = 0; j < Fp / 64; ++j)
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_addr(sB + (size_t)(p * (Fp / 64) + j) * a.H * 128)),
                    "l"(&a.wmap), "r"(64 * j), "r"(p), "r"(0), "r"(smem_addr(mbar_w))
                    : "memory");
    }
    SAGE_STAMP(1);
    const uint32_t tmem = *tmem_slot;
    const uint32_t idesc = idesc_bf16_f32(a.H);
    const T *xs = static_cast<const T *>(a.x_src);
    const T *xd = static_cast<const T *>(a.x_dst);
    uint32_t phase = 0;

    // the row bounds and the first 32 edge indices of this warp's rows in the NEXT tile are
    // loaded while the current tile finishes (its MMA and epilogue), which takes two of the
    // A build's dependent memory round trips off every tile but the first
    const int c = lane * CPL;
    const int rbase = warp * R;
    auto load_bounds = [&](int t) {
        int v = 0;
        if (lane <= R && t * kTileM < a.n_dst) v = __ldg(a.indptr + min(t * kTileM + rbase + lane, a.n_dst));
        return v;
    };
    auto load_first_idx = [&](int bounds) {
        const int b0 = __shfl_sync(0xffffffffu, bounds, 0), b1 = __shfl_sync(0xffffffffu, bounds, R);
        return lane < min(32, b1 - b0) ? __ldg(a.indices + b0 + lane) : 0;
    };
    int pv_next = load_bounds(blockIdx.x);
    int idx_next = load_first_idx(pv_next);
    for (int tile = blockIdx.x; tile * kTileM < a.n_dst; tile += gridDim.x) {
        const int row0 = tile * kTileM;
        ++tile_no;
        // ---- A operand: warp w builds the R consecutive rows rbase .. rbase + R - 1, whose
        // sampled edges are one contiguous CSC range [e0, e1): the row bounds (one load per
        // lane), then per 32 edges one index load per lane, then the source rows in groups
        // of S = 32 / NW edges with every load of a group in flight before the first is
        // summed (round 2: the round-1 build issued index -> row chains for 4 rows at a time,
        // ~14 dependent memory round trips per tile; this one needs ~4).
        const int pv = pv_next, idx0 = idx_next;
        pv_next = load_bounds(tile + gridDim.x);
        const int e0 = __shfl_sync(0xffffffffu, pv, 0), e1 = __shfl_sync(0xffffffffu, pv, R);
        if (xd) {
            uint32_t sr[R][NW];
#pragma unroll
            for (int i = 0; i < R; ++i) {
                if (row0 + rbase + i < a.n_dst) load_raw<T, CPL>(xd + (int64_t)(row0 + rbase + i) * a.ld_dst, c, a.F, sr[i]);
                else
#pragma unroll
                    for (int q = 0; q < NW; ++q) sr[i][q] = 0u;
            }
#pragma unroll
            for (int i = 0; i < R; ++i) {
                float f[CPL];
#pragma unroll
                for (int e = 0; e < CPL; ++e) f[e] = 0.f;
                raw_add<T, CPL>(f, sr[i]);
                store_bf16<CPL>(sA, kTileM, rbase + i, c, f);
            }
        }
        {
            float acc[CPL];
#pragma unroll
            for (int e = 0; e < CPL; ++e) acc[e] = 0.f;
            int cur = 0;                                  // row (of the warp's R) of the next edge
            int nxt = __shfl_sync(0xffffffffu, pv, 1);    // its end offset
            // mean of row `cur` into A, then the next row (warp-uniform)
            auto flush = [&]() {
                const int d = nxt - __shfl_sync(0xffffffffu, pv, cur);
                const float inv = d > 0 ? 1.f / (float)d : 0.f;
#pragma unroll
                for (int e = 0; e < CPL; ++e) acc[e] *= inv;
                store_bf16<CPL>(sA, kTileM, rbase + cur, (parts - 1) * Fp + c, acc);
#pragma unroll
                for (int e = 0; e < CPL; ++e) acc[e] = 0.f;
                ++cur;
                nxt = __shfl_sync(0xffffffffu, pv, cur + 1 <= R ? cur + 1 : R);
            };
            for (int base = e0; base < e1; base += 32) {
                const int ne = min(32, e1 - base);
                const int myidx = base == e0 ? idx0 : (lane < ne ? __ldg(a.indices + base + lane) : 0);
                for (int s0 = 0; s0 < ne; s0 += S) {
                    uint32_t raw[S][NW];
#pragma unroll
                    for (int q = 0; q < S; ++q) {
                        const int src = __shfl_sync(0xffffffffu, myidx, s0 + q);
                        if (s0 + q < ne) load_raw<T, CPL>(xs + (int64_t)src * a.ld_src, c, a.F, raw[q]);
                    }
#pragma unroll
                    for (int q = 0; q < S; ++q) {
                        if (s0 + q < ne) {
                            const int e = base + s0 + q;
                            while (e >= nxt) flush();
                            raw_add<T, CPL>(acc, raw[q]);
                        }
                    }
                }
            }
            while (cur < R) flush();
        }
        idx_next = load_first_idx(pv_next);
        // generic-proxy smem writes -> visible to the tensor core (async proxy)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        SAGE_STAMP(2);
        if (threadIdx.x == 0) {
            if (a.w_tma && tile_no == 0) mbar_wait_parity(mbar_w, 0);   // W landed
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t a0 = smem_addr(sA), b0 = smem_addr(sB);
            for (int s = 0; s < Kp / 16; ++s) {
                const int k = s * 16;
                const uint64_t da = sw128_desc(a0 + (k >> 6) * kTileM * 128 + (k & 63) * 2);
                const uint64_t db = sw128_desc(b0 + (k >> 6) * a.H * 128 + (k & 63) * 2);
                const uint32_t acc_flag = s > 0 ? 1u : 0u;
                asm volatile(
                    "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                    "l"(da), "l"(db), "r"(idesc), "r"(acc_flag)
                    : "memory");
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_addr(mbar))
                         : "memory");
        }
        mbar_wait_parity(mbar, phase);
        phase ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        SAGE_STAMP(3);
        // ---- epilogue (A is free once the MMAs completed): staged through A's shared memory
        // so that the fp32 rows leave as full row segments
        const int cw = 2 * Kp / kWarps;   // staging columns per warp that fit A's bytes
        if (cw >= 32) epilogue<32, kWarps>(a, tmem, reinterpret_cast<float *>(sA), row0, warp, lane);
        else if (cw >= 16) epilogue<16, kWarps>(a, tmem, reinterpret_cast<float *>(sA), row0, warp, lane);
        else if (cw >= 8) epilogue<8, kWarps>(a, tmem, reinterpret_cast<float *>(sA), row0, warp, lane);
        else epilogue_rows<kWarps>(a, tmem, row0, warp, lane);
        SAGE_STAMP(4);
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();   // A and the accumulator are free for the next tile
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    __syncthreads();
    SAGE_STAMP(5);
#ifdef EG_SAGE_TRACE
    if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == 100))
        for (int i = 0; i < 10; ++i)
            reinterpret_cast<uint64_t *>(a.out + (blockIdx.x == 0 ? 0 : a.ld_out))[i] = stamps[i];
#endif
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols)
                     : "memory");
}

template <typename T, int CPL>
cudaError_t launch_typed(const SageArgs &a, cudaStream_t s)
{
    const int Fp = CPL * 32, Kp = (a.x_dst ? 2 : 1) * Fp;
    const size_t smem = (size_t)(a.H + kTileM) * Kp * 2 + 1024 + 64;
    cudaError_t e = cudaFuncSetAttribute(sage_kernel<T, CPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int tiles = (a.n_dst + kTileM - 1) / kTileM;
    if (tiles == 0) return cudaSuccess;
    sage_kernel<T, CPL><<<tiles < kSMs ? tiles : kSMs, warps_for<CPL>() * 32, smem, s>>>(a);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_cpl(const SageArgs &a, cudaStream_t s)
{
    const int Fp = (a.F + 63) / 64 * 64;
    if (Fp == 64) return launch_typed<T, 2>(a, s);
    if (Fp == 128) return launch_typed<T, 4>(a, s);
    return launch_typed<T, 8>(a, s);
}

}  // namespace

size_t sage_smem_bytes(int F, int H, bool self_term)
{
    const int Fp = (F + 63) / 64 * 64;
    return (size_t)(H + kTileM) * (self_term ? 2 : 1) * Fp * 2 + 1024 + 64;
}

cudaError_t launch_sage(const SageArgs &a, int x_dtype, cudaStream_t s)
{
    if (x_dtype == 0) return launch_cpl<float>(a, s);
    if (x_dtype == 1) return launch_cpl<__half>(a, s);
    return launch_cpl<__nv_bfloat16>(a, s);
}

}  // namespace eg
