/*
 * ngemm ORACLE — CPU restatement of the reference u8 x i8 -> i32 path.
 * TEST INFRASTRUCTURE ONLY (see oracle.h): the checker and the reported CPU baseline,
 * never the product.  Plain C11 + pthreads.
 */
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* prng.hpp:14-20 — splitmix64 step; a zero state is replaced by the golden gamma. */
void ngo_rng_seed(ngo_rng* r, uint64_t seed) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    r->state = z ^ (z >> 31);
    if (r->state == 0) r->state = 0x9E3779B97F4A7C15ull;
}

/* prng.hpp:22-29 — xorshift64* output step. */
uint64_t ngo_rng_next(ngo_rng* r) {
    uint64_t x = r->state;
    x ^= x >> 12;
    x ^= x << 25;
    x ^= x >> 27;
    r->state = x;
    return x * 0x2545F4914F6CDD1Dull;
}

/* prng.hpp:33-38 — plain modulo range mapping (callers guarantee lo <= hi). */
int64_t ngo_rng_next_in(ngo_rng* r, int64_t lo, int64_t hi) {
    uint64_t span = (uint64_t)(hi - lo) + 1u;
    if (span == 0) return (int64_t)ngo_rng_next(r);
    return lo + (int64_t)(ngo_rng_next(r) % span);
}

/* matrix.hpp:131-143 — one stream, row-major order; MatrixBuf::set truncates to the byte. */
void ngo_mat_random_u8(uint8_t* out, int64_t rows, int64_t cols, uint64_t seed, int64_t lo, int64_t hi) {
    ngo_rng r;
    ngo_rng_seed(&r, seed);
    int64_t n = rows * cols;
    for (int64_t i = 0; i < n; ++i) out[i] = (uint8_t)ngo_rng_next_in(&r, lo, hi);
}

void ngo_mat_random_i8(int8_t* out, int64_t rows, int64_t cols, uint64_t seed, int64_t lo, int64_t hi) {
    ngo_rng r;
    ngo_rng_seed(&r, seed);
    int64_t n = rows * cols;
    for (int64_t i = 0; i < n; ++i) out[i] = (int8_t)ngo_rng_next_in(&r, lo, hi);
}

/* mat_random for ElemKind::I16 (matrix.hpp:146-158): same stream, value cast to int16. */
void ngo_mat_random_i16(int16_t* out, int64_t rows, int64_t cols, uint64_t seed, int64_t lo, int64_t hi) {
    ngo_rng r;
    ngo_rng_seed(&r, seed);
    int64_t n = rows * cols;
    for (int64_t i = 0; i < n; ++i) out[i] = (int16_t)ngo_rng_next_in(&r, lo, hi);
}

/* SURVEY.md 8(d) c2 generator (ours; the reference has no normal generator). */
void ngo_mat_normal_i8(int8_t* out, int64_t rows, int64_t cols, uint64_t seed, double sigma) {
    ngo_rng r;
    ngo_rng_seed(&r, seed);
    const double two_pi = 6.283185307179586476925286766559;
    const double inv53 = 1.0 / 9007199254740992.0; /* 2^-53 */
    int64_t n = rows * cols;
    for (int64_t i = 0; i < n; ++i) {
        double u1 = (double)((ngo_rng_next(&r) >> 11) + 1u) * inv53; /* (0, 1] */
        double u2 = (double)(ngo_rng_next(&r) >> 11) * inv53;        /* [0, 1) */
        double z = sqrt(-2.0 * log(u1)) * cos(two_pi * u2);
        long v = lround(sigma * z);
        if (v < -128) v = -128;
        if (v > 127) v = 127;
        out[i] = (int8_t)v;
    }
}

/* lanes.hpp:28-38 with sat_i16 (common.hpp:141-145). */
int32_t ngo_madd_pair(uint8_t a0, uint8_t a1, int8_t b0, int8_t b1, int mode) {
    int32_t s = (int32_t)a0 * b0 + (int32_t)a1 * b1;
    if (mode == 0) {
        if (s > 32767) s = 32767;
        if (s < -32768) s = -32768;
    }
    return s;
}

/* gemm.hpp:40-52: exact, uint32 accumulator (wrapping). */
void ngo_gemm_ref_rows(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb,
                       int32_t* c, int64_t ldc, int64_t m0, int64_t m1, int64_t n, int64_t k) {
    for (int64_t mi = m0; mi < m1; ++mi) {
        const uint8_t* arow = a + mi * lda;
        int32_t* crow = c + mi * ldc;
        for (int64_t ni = 0; ni < n; ++ni) {
            const int8_t* brow = b + ni * ldb;
            uint32_t acc = 0;
            for (int64_t ki = 0; ki < k; ++ki) acc += (uint32_t)((int32_t)arow[ki] * brow[ki]);
            crow[ni] = (int32_t)acc;
        }
    }
}

/* gemm.hpp:36-52 on i16 operands: every product fits int32; sum in uint32 (wraps). */
void ngo_gemm_i16(const int16_t* a, int64_t lda, const int16_t* b, int64_t ldb, int32_t* c, int64_t ldc,
                  int64_t m, int64_t n, int64_t k) {
    for (int64_t mi = 0; mi < m; ++mi) {
        const int16_t* arow = a + mi * lda;
        for (int64_t ni = 0; ni < n; ++ni) {
            const int16_t* brow = b + ni * ldb;
            uint32_t acc = 0;
            for (int64_t ki = 0; ki < k; ++ki) acc += (uint32_t)((int32_t)arow[ki] * (int32_t)brow[ki]);
            c[mi * ldc + ni] = (int32_t)acc;
        }
    }
}

/* gemm.hpp:86-102: pairs (k0, k0+1) for even k0, odd tail paired with zero, wrap-add. */
void ngo_gemm_sat_rows(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb,
                       int32_t* c, int64_t ldc, int64_t m0, int64_t m1, int64_t n, int64_t k) {
    for (int64_t mi = m0; mi < m1; ++mi) {
        const uint8_t* arow = a + mi * lda;
        int32_t* crow = c + mi * ldc;
        for (int64_t ni = 0; ni < n; ++ni) {
            const int8_t* brow = b + ni * ldb;
            uint32_t acc = 0;
            for (int64_t k0 = 0; k0 < k; k0 += 2) {
                uint8_t a1 = k0 + 1 < k ? arow[k0 + 1] : 0;
                int8_t b1 = k0 + 1 < k ? brow[k0 + 1] : 0;
                int32_t s = (int32_t)arow[k0] * brow[k0] + (int32_t)a1 * b1;
                if (s > 32767) s = 32767;
                if (s < -32768) s = -32768;
                acc += (uint32_t)s;
            }
            crow[ni] = (int32_t)acc;
        }
    }
}

typedef struct {
    const uint8_t* a; int64_t lda;
    const int8_t* b; int64_t ldb;
    int32_t* c; int64_t ldc;
    int64_t m0, m1, n, k;
    int mode;
} ngo_job;

static void* ngo_worker(void* p) {
    ngo_job* j = (ngo_job*)p;
    if (j->mode == 0)
        ngo_gemm_sat_rows(j->a, j->lda, j->b, j->ldb, j->c, j->ldc, j->m0, j->m1, j->n, j->k);
    else
        ngo_gemm_ref_rows(j->a, j->lda, j->b, j->ldb, j->c, j->ldc, j->m0, j->m1, j->n, j->k);
    return NULL;
}

void ngo_gemm(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb, int32_t* c, int64_t ldc,
              int64_t m, int64_t n, int64_t k, int mode, int threads) {
    if (threads < 1) threads = 1;
    if (threads > m) threads = (int)m;
    if (threads <= 1) {
        ngo_job j = {a, lda, b, ldb, c, ldc, 0, m, n, k, mode};
        ngo_worker(&j);
        return;
    }
    pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    ngo_job* jobs = (ngo_job*)malloc(sizeof(ngo_job) * (size_t)threads);
    for (int t = 0; t < threads; ++t) {
        int64_t r0 = m * t / threads, r1 = m * (t + 1) / threads;
        ngo_job j = {a, lda, b, ldb, c, ldc, r0, r1, n, k, mode};
        jobs[t] = j;
        pthread_create(&tid[t], NULL, ngo_worker, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
    free(jobs);
    free(tid);
}

/* --- PackedWeight (layout.hpp) --- */

static int ngo_m_before_k(int32_t perm) { return perm == 0 || perm == 1 || perm == 2; } /* layout.hpp:77-79 */

static int64_t ngo_round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; } /* common.hpp:147-149 */

int ngo_packed_init(ngo_packed_meta* p, int32_t w, int32_t h, int32_t v, int64_t tm, int64_t tn,
                    int64_t tk, int32_t perm, int64_t m_orig, int64_t k_orig) {
    memset(p, 0, sizeof *p);
    if (v * h != w || h != 4) return -2;                        /* layout.hpp:258-262 */
    if (tm < v || tm % v != 0) return -1;                       /* layout.hpp:93-96 */
    if (tk < h || tk % h != 0) return -1;                       /* layout.hpp:97-100 */
    if (tn < 1) return -1;                                      /* layout.hpp:101 */
    if (perm < 0 || perm > 5) return -1;
    p->w = w; p->h = h; p->v = v;
    p->tm = tm; p->tn = tn; p->tk = tk; p->perm = perm;
    p->m_orig = m_orig; p->k_orig = k_orig;
    p->m_pad = ngo_round_up(m_orig, tm);
    p->k_pad = ngo_round_up(k_orig, tk);
    return 0;
}

/* layout.hpp:152-165 */
int64_t ngo_packed_block_offset(const ngo_packed_meta* p, int64_t m_blk, int64_t k_blk) {
    int64_t tile_m = m_blk * p->v / p->tm;
    int64_t tile_k = k_blk * p->h / p->tk;
    int64_t bm = m_blk - tile_m * (p->tm / p->v);
    int64_t bk = k_blk - tile_k * (p->tk / p->h);
    int64_t tiles_m = p->m_pad / p->tm;
    int64_t tiles_k = p->k_pad / p->tk;
    int64_t tile_lin = ngo_m_before_k(p->perm) ? tile_m * tiles_k + tile_k : tile_k * tiles_m + tile_m;
    int64_t blocks_per_tile = (p->tm / p->v) * (p->tk / p->h);
    int64_t blk_lin = bm * (p->tk / p->h) + bk;
    return (tile_lin * blocks_per_tile + blk_lin) * p->w;
}

/* layout.hpp:167-171 with inner_offset (layout.hpp:44-52): m_in_block * h + k_in_block. */
int64_t ngo_packed_elem_offset(const ngo_packed_meta* p, int64_t gm, int64_t gk) {
    return ngo_packed_block_offset(p, gm / p->v, gk / p->h) + (gm % p->v) * p->h + (gk % p->h);
}

/* layout.hpp:221-229 (constructor zero fill: layout.hpp:122-126) */
void ngo_pack_u8(const ngo_packed_meta* p, const uint8_t* a, int64_t lda, uint8_t* dst) {
    memset(dst, 0, (size_t)(p->m_pad * p->k_pad));
    for (int64_t gm = 0; gm < p->m_orig; ++gm)
        for (int64_t gk = 0; gk < p->k_orig; ++gk)
            dst[ngo_packed_elem_offset(p, gm, gk)] = a[gm * lda + gk];
}

/* layout.hpp:231-248 */
int64_t ngo_unpack_u8(const ngo_packed_meta* p, const uint8_t* src, uint8_t* a, int64_t lda) {
    for (int64_t gm = 0; gm < p->m_pad; ++gm)
        for (int64_t gk = 0; gk < p->k_pad; ++gk) {
            uint8_t v = src[ngo_packed_elem_offset(p, gm, gk)];
            if (gm < p->m_orig && gk < p->k_orig) a[gm * lda + gk] = v;
            else if (v != 0) return 1 + gm * p->k_pad + gk;
        }
    return 0;
}

uint64_t ngo_fnv1a(const void* data, size_t n) {
    const uint8_t* d = (const uint8_t*)data;
    uint64_t h = 1469598103934665603ull;
    for (size_t i = 0; i < n; ++i) {
        h ^= d[i];
        h *= 1099511628211ull;
    }
    return h;
}

int64_t ngo_checksum_i32(const int32_t* c, int64_t rows, int64_t cols, int64_t ldc) {
    int64_t s = 0;
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t j = 0; j < cols; ++j) s += c[r * ldc + j];
    return s;
}
