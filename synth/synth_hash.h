/*
 * synth/synth_hash.h -- the counter-based hash of the SYNTHETIC INPUT GENERATOR.
 *
 * Shared by the host generator (synth.c) and the device generator
 * (synth_dev.cu) so that a shard generated on a GPU is byte-identical to the
 * host copy the oracle reads.  It is input generation only: none of the
 * sampling method's arithmetic (Philox key32, selection, compaction, gather)
 * lives here, and neither the oracle nor the product kernels include it.
 *
 * mix64 is the splitmix64 finaliser (Steele, Lea, Flood; "variant 13" constants).
 */
#ifndef SYNTH_HASH_H
#define SYNTH_HASH_H
#include <stdint.h>

#ifdef __CUDACC__
#define SY_FN __host__ __device__ __forceinline__
#else
#define SY_FN static inline
#endif

#define SY_TAG_DEG  (0x4445475FULL << 32)   /* 'DEG_' */
#define SY_TAG_SRC  (0x5352435FULL << 32)   /* 'SRC_' */
#define SY_TAG_FEAT (0x46454154ULL << 32)   /* 'FEAT' */
#define SY_TAG_TRN  (0x54524E5FULL << 32)   /* 'TRN_' */
#define SY_TAG_PERM (0x5045524DULL << 32)   /* 'PERM' */

SY_FN uint64_t sy_mix64(uint64_t z)
{
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

/* hash of (generator seed G, tag, a, b) */
SY_FN uint64_t sy_hash(uint64_t G, uint64_t tag, uint64_t a, uint64_t b)
{
    uint64_t h = sy_mix64(G + tag * 0x9E3779B97F4A7C15ULL);
    h = sy_mix64(h ^ a);
    return sy_mix64(h + b);
}

/* src tid of global CSC position e of relation r; uniform over [0, n_src) */
SY_FN int32_t sy_src_tid(uint64_t G, int32_t r, int64_t e, int64_t n_src)
{
    uint64_t w = sy_hash(G, SY_TAG_SRC + (uint64_t)r, (uint64_t)e, 0) >> 32;
    return (int32_t)((w * (uint64_t)n_src) >> 32);
}

/* Planted communities: each vertex type is split into n_comm
 * contiguous blocks; the source of an edge whose dst lies in block c is drawn from the
 * src type's block c with probability q_thr / 2^32, else uniformly (the same hash word
 * as sy_src_tid for the uniform draw, the low word for the coin). */
SY_FN int32_t sy_src_tid_loc(uint64_t G, int32_t r, int64_t e, int64_t n_src, int64_t dst_tid, int64_t n_dst,
                             uint32_t q_thr, int32_t n_comm)
{
    uint64_t h = sy_hash(G, SY_TAG_SRC + (uint64_t)r, (uint64_t)e, 0);
    uint64_t w = h >> 32;
    if ((uint32_t)h < q_thr && n_dst > 0) {
        int64_t c = dst_tid * n_comm / n_dst;
        int64_t lo = c * n_src / n_comm, hi = (c + 1) * n_src / n_comm;
        if (hi > lo) return (int32_t)(lo + (int64_t)((w * (uint64_t)(hi - lo)) >> 32));
    }
    return (int32_t)((w * (uint64_t)n_src) >> 32);
}

/* feature element c of row (u, tid): dtype 0 = fp32 bits in [1,2), 1 = fp16 bits in [1,2).
 * One 64-bit hash yields two 32-bit words (columns 2m and 2m+1). */
SY_FN uint32_t sy_feat_word(uint64_t G, int32_t u, int64_t tid, int64_t c)
{
    uint64_t h = sy_hash(G, SY_TAG_FEAT + (uint64_t)u, (uint64_t)tid, (uint64_t)(c >> 1));
    return (c & 1) ? (uint32_t)(h >> 32) : (uint32_t)h;
}

SY_FN uint32_t sy_feat_f32(uint64_t G, int32_t u, int64_t tid, int64_t c)
{
    return 0x3F800000u | (sy_feat_word(G, u, tid, c) >> 9);
}

SY_FN uint16_t sy_feat_f16(uint64_t G, int32_t u, int64_t tid, int64_t c)
{
    return (uint16_t)(0x3C00u | (sy_feat_word(G, u, tid, c) & 0x3FFu));
}
#endif
