/*
 * ngemm ORACLE — CPU restatement of the reference algorithm for the u8 x i8 -> i32 path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library, and only as the checker
 * or the reported CPU baseline.  The product path (libngemm_cuda.so) never links or
 * calls it; there is no CPU fallback.
 *
 * Every function cites the reference file:line (under /root/reference/proj/include/ngemm)
 * whose behaviour it restates.  Parity is pinned: tests/test_oracle.py checks this
 * restatement against the reference's own golden vectors (test_matrix.cpp:37-59,
 * test_gemm.cpp:44-52, test_layout.cpp:61-146, test_lanes.cpp:31-40) and against
 * fixtures produced by the reference itself (oracle/_ref, tests/golden/make_golden.py).
 */
#ifndef NGEMM_ORACLE_H
#define NGEMM_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* --- PRNG: xorshift64* seeded through one splitmix64 step (prng.hpp:13-43) --- */
typedef struct { uint64_t state; } ngo_rng;
void ngo_rng_seed(ngo_rng* r, uint64_t seed);
uint64_t ngo_rng_next(ngo_rng* r);
/* Uniform draw in [lo, hi] by plain modulo (prng.hpp:33-38). */
int64_t ngo_rng_next_in(ngo_rng* r, int64_t lo, int64_t hi);

/* mat_random (matrix.hpp:131-143): row-major fill from one stream; elem_size 1 (u8/i8).
 * Values are stored as their low byte, exactly like MatrixBuf::set (matrix.hpp:61-77). */
void ngo_mat_random_u8(uint8_t* out, int64_t rows, int64_t cols, uint64_t seed, int64_t lo, int64_t hi);
void ngo_mat_random_i8(int8_t* out, int64_t rows, int64_t cols, uint64_t seed, int64_t lo, int64_t hi);

/* Config-2 input generator (NOT in the reference; defined and frozen by SURVEY.md 8(d)):
 * Box-Muller over XorShift64Star(seed) 53-bit uniforms, lround(sigma*z), clipped to
 * [-128, 127], row-major fill, one draw pair per element (the cosine branch). */
void ngo_mat_random_i16(int16_t* out, int64_t rows, int64_t cols, uint64_t seed, int64_t lo, int64_t hi);
void ngo_mat_normal_i8(int8_t* out, int64_t rows, int64_t cols, uint64_t seed, double sigma);

/* --- GEMM oracles.  A [M x K] u8 row-major (stride lda), B [N x K] i8 row-major (ldb),
 * C [M x N] i32 row-major (ldc).  Rows [m0, m1) only, so callers can shard. --- */
/* gemm_ref (gemm.hpp:36-52): C = sum_k a*b accumulated in uint32 (wraps mod 2^32). */
void ngo_gemm_ref_rows(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb,
                       int32_t* c, int64_t ldc, int64_t m0, int64_t m1, int64_t n, int64_t k);
/* gemm_sat_oracle (gemm.hpp:83-104): adjacent even-aligned K pairs summed and clamped
 * to int16 (madd_pair_u8i8_sat, lanes.hpp:28-33), odd tail paired with 0 (gemm.hpp:95-96),
 * then wrap-added in int32 (wrap_add_i32, common.hpp:132-135). */
void ngo_gemm_sat_rows(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb,
                       int32_t* c, int64_t ldc, int64_t m0, int64_t m1, int64_t n, int64_t k);
/* Whole-matrix convenience with `threads` worker threads (row shards); mode 0 = sat
 * (HardwareSaturating), 1 = exact (WideningExact) — the reference SatMode order (lanes.hpp:18). */
void ngo_gemm(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb, int32_t* c, int64_t ldc,
              int64_t m, int64_t n, int64_t k, int mode, int threads);

/* gemm_ref on i16 x i16 operands (gemm.hpp:36-52 is kind-generic; gemm_sat_oracle defers to
 * it for i16, gemm.hpp:85): C = sum_k a*b in uint32.  The reference's i16 kernels (pmaddwd
 * pairs wrap-added, gemm.hpp:161-190) give the same value mod 2^32.  A [M x K], B [N x K]. */
void ngo_gemm_i16(const int16_t* a, int64_t lda, const int16_t* b, int64_t ldb, int32_t* c, int64_t ldc,
                  int64_t m, int64_t n, int64_t k);

/* Pair primitive (lanes.hpp:28-38); mode as above. */
int32_t ngo_madd_pair(uint8_t a0, uint8_t a1, int8_t b0, int8_t b1, int mode);

/* --- PackedWeight addressing (layout.hpp:120-182). --- */
typedef struct {
    int32_t w, h, v;           /* KernelShape (layout.hpp:21-27) */
    int64_t tm, tn, tk;        /* TileConfig (layout.hpp:84-88) */
    int32_t perm;              /* Perm tag 0..5 = MNK MKN NMK NKM KMN KNM (layout.hpp:54) */
    int64_t m_orig, k_orig;
    int64_t m_pad, k_pad;      /* round_up(m_orig, tm), round_up(k_orig, tk) (layout.hpp:125) */
} ngo_packed_meta;

/* Fills m_pad/k_pad; returns 0, or -1 for a tile TileConfig::validate rejects
 * (layout.hpp:92-102), -2 for a shape pack_weights rejects for 8-bit (layout.hpp:258-262). */
int ngo_packed_init(ngo_packed_meta* p, int32_t w, int32_t h, int32_t v, int64_t tm, int64_t tn,
                    int64_t tk, int32_t perm, int64_t m_orig, int64_t k_orig);
/* PackedWeight::block_offset / elem_offset (layout.hpp:152-171). */
int64_t ngo_packed_block_offset(const ngo_packed_meta* p, int64_t m_blk, int64_t k_blk);
int64_t ngo_packed_elem_offset(const ngo_packed_meta* p, int64_t gm, int64_t gk);
/* pack_weights for 8-bit (layout.hpp:221-229, 252-270): dst has m_pad*k_pad bytes, zeroed here. */
void ngo_pack_u8(const ngo_packed_meta* p, const uint8_t* a, int64_t lda, uint8_t* dst);
/* unpack_weights (layout.hpp:231-248): returns 0, or 1 + flat padded index of the first
 * nonzero padding byte (CorruptionError). */
int64_t ngo_unpack_u8(const ngo_packed_meta* p, const uint8_t* src, uint8_t* a, int64_t lda);

/* --- digests --- */
/* FNV-1a 64 over bytes (test_matrix.cpp:20-27). */
uint64_t ngo_fnv1a(const void* data, size_t n);
/* MatrixBuf::checksum for i32 (matrix.hpp:85-90): sum widened to int64. */
int64_t ngo_checksum_i32(const int32_t* c, int64_t rows, int64_t cols, int64_t ldc);

#ifdef __cplusplus
}
#endif
#endif
