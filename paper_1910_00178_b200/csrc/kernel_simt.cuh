// kernel_simt.cuh — CUDA-core (IDP.4A) tiled GEMM, both SatMode semantics.
//
// This is the path for HardwareSaturating mode on inputs that can saturate (the pairwise
// int16 clamp of VPMADDUBSW has no tensor-core formulation) and the
// Engine::Emulated path of the drop-in API.  It reproduces the reference arithmetic exactly:
//   exact: C = sum_k a*b mod 2^32                        (gemm_ref, gemm.hpp:36-52)
//   sat  : C = sum_j sat16(a[2j]b[2j] + a[2j+1]b[2j+1])  (gemm_sat_oracle, gemm.hpp:83-104)
// K is consumed in 4-byte words starting at k = 0, so every pair is even-aligned exactly as
// in the reference kernels (simd_native.hpp:157); K tails are zero-padded, which pairs an odd
// last element with 0 (gemm.hpp:95-96).  All int32 adds wrap, so the summation order is
// immaterial (common.hpp:129-135).
//
// Tiling: 128x128 (8x8 outputs per thread) or 64x64 (4x4) output tiles per 256-thread CTA,
// K staged through shared memory 32 bytes (8 words) at a time, transposed to word-major so the
// inner loop is LDS.128 per 4 operand words; next-stage global loads are prefetched into
// registers.  Small problems add K splits (atomic wrap-add into a zeroed C) to fill 148 SMs.
// The saturating inner step (sat_word_add, ptx.cuh) is 2 IDP.4A on the masked A halves, one
// I2IP.S16.S32.SAT packing both pair sums with int16 saturation and one IDP.2A wrap-adding
// them: 4 instructions per 4 MACs, CUDA-core (IDP pipe) bound — which is why the pairs that
// provably cannot saturate go to the tensor cores for large shapes (kernel_satfix.cuh).
#pragma once

#include "ptx.cuh"

namespace ngemm_dev {

namespace simt {
constexpr int BKW = 8;  // BK = 32 bytes (8 K-words) per smem stage
constexpr int THREADS = 256;
}  // namespace simt

// Loads 16 bytes (4 K-words) of row `r` starting at byte `k0`; zero outside [0,rows)x[0,K).
// WORDS: rows with an unaligned pitch are read as 5 aligned words realigned by funnel shifts
// instead of 16 byte loads (the prep kernels; the tiled kernel keeps the lighter byte path,
// which costs it no registers in its prefetch stage).
template <bool WORDS = false>
__device__ __forceinline__ uint4 simt_load16(const uint8_t* __restrict__ base, int64_t ld, int64_t r,
                                             int64_t rows, int64_t k0, int64_t K, bool vec_ok) {
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r >= rows || k0 >= K) return v;
    const uint8_t* p = base + r * ld + k0;
    if (vec_ok && k0 + 16 <= K) return __ldg(reinterpret_cast<const uint4*>(p));
    const uintptr_t addr = reinterpret_cast<uintptr_t>(p);
    if (WORDS && k0 + 20 <= K && (k0 >= 4 || (addr & 3) == 0)) {
        // unaligned row pitch: 5 aligned words, realigned by funnel shifts (the 20 bytes read
        // stay inside the row)
        const uint32_t* q = reinterpret_cast<const uint32_t*>(addr & ~uintptr_t(3));
        const uint32_t sh = static_cast<uint32_t>(addr & 3) * 8;
        uint32_t x[5];
#pragma unroll
        for (int i = 0; i < 5; ++i) x[i] = __ldg(q + i);
        return make_uint4(__funnelshift_r(x[0], x[1], sh), __funnelshift_r(x[1], x[2], sh),
                          __funnelshift_r(x[2], x[3], sh), __funnelshift_r(x[3], x[4], sh));
    }
    uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 16; ++i)
        if (k0 + i < K) w[i >> 2] |= static_cast<uint32_t>(__ldg(p + i)) << (8 * (i & 3));
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// MODE: 1 = WideningExact, 0 = HardwareSaturating (u8 x s8 words of 4 K-elements);
//       2 = the 16-bit path, i16 x i16 words of 2 K-elements (madd_pair_i16, lanes.hpp:42-47:
//           no saturation stage, everything mod 2^32).  K, lda, ldb are in BYTES here.
// TILE: 128 (8x8 outputs per thread) or 64 (4x4, for small shapes).  blockIdx.z selects a
// K split of k_split bytes (a multiple of 32, so pairs stay even-aligned); with split > 1
// the partials are wrap-added into a zeroed C.
template <int MODE, int TILE>
__global__ void __launch_bounds__(simt::THREADS, 2)
    simt_gemm_kernel(const uint8_t* __restrict__ A, int64_t lda, const int8_t* __restrict__ B, int64_t ldb,
                     int32_t* __restrict__ C, int64_t ldc, int64_t M, int64_t N, int64_t K, int vec_ok,
                     int c_vec_ok, int64_t k_split, int accumulate) {
    using namespace simt;
    constexpr int TT = TILE / 16;     // outputs per thread per dimension
    constexpr int LDS = TILE + 4;     // padded word stride (bank-conflict free stores)
    constexpr int LOADS = (TILE * 2 + THREADS - 1) / THREADS;  // uint4 loads per operand per thread
    pdl_launch_dependents();
    pdl_wait();
    __shared__ __align__(16) uint32_t As[BKW][LDS];
    __shared__ __align__(16) uint32_t Bs[BKW][LDS];

    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    const int64_t m0 = static_cast<int64_t>(blockIdx.y) * TILE;
    const int64_t n0 = static_cast<int64_t>(blockIdx.x) * TILE;
    const int64_t kb = static_cast<int64_t>(blockIdx.z) * k_split;
    const int64_t ke = min(K, kb + k_split);
    const uint8_t* Bu = reinterpret_cast<const uint8_t*>(B);

    int32_t acc[TT][TT];
#pragma unroll
    for (int i = 0; i < TT; ++i)
#pragma unroll
        for (int j = 0; j < TT; ++j) acc[i][j] = 0;

    const int64_t nk = (ke - kb + 31) / 32;
    uint4 ra[LOADS], rb[LOADS];
#pragma unroll
    for (int l = 0; l < LOADS; ++l) {
        const int li = tid + l * THREADS, lr = li >> 1, lh = li & 1;
        ra[l] = li < TILE * 2 ? simt_load16(A, lda, m0 + lr, M, kb + lh * 16, ke, vec_ok) : make_uint4(0, 0, 0, 0);
        rb[l] = li < TILE * 2 ? simt_load16(Bu, ldb, n0 + lr, N, kb + lh * 16, ke, vec_ok) : make_uint4(0, 0, 0, 0);
    }

    for (int64_t kt = 0; kt < nk; ++kt) {
        __syncthreads();
#pragma unroll
        for (int l = 0; l < LOADS; ++l) {
            const int li = tid + l * THREADS, lr = li >> 1, lh = li & 1;
            if (li < TILE * 2) {
                As[lh * 4 + 0][lr] = ra[l].x;
                As[lh * 4 + 1][lr] = ra[l].y;
                As[lh * 4 + 2][lr] = ra[l].z;
                As[lh * 4 + 3][lr] = ra[l].w;
                Bs[lh * 4 + 0][lr] = rb[l].x;
                Bs[lh * 4 + 1][lr] = rb[l].y;
                Bs[lh * 4 + 2][lr] = rb[l].z;
                Bs[lh * 4 + 3][lr] = rb[l].w;
            }
        }
        __syncthreads();
        if (kt + 1 < nk) {
#pragma unroll
            for (int l = 0; l < LOADS; ++l) {
                const int li = tid + l * THREADS, lr = li >> 1, lh = li & 1;
                if (li < TILE * 2) {
                    const int64_t kn = kb + (kt + 1) * 32 + lh * 16;
                    ra[l] = simt_load16(A, lda, m0 + lr, M, kn, ke, vec_ok);
                    rb[l] = simt_load16(Bu, ldb, n0 + lr, N, kn, ke, vec_ok);
                }
            }
        }
#pragma unroll
        for (int kw = 0; kw < BKW; ++kw) {
            uint32_t a[TT], b[TT];
#pragma unroll
            for (int h = 0; h < TT / 4; ++h) {
                const uint4 av = *reinterpret_cast<const uint4*>(&As[kw][h * (TILE / 2) + ty * 4]);
                const uint4 bv = *reinterpret_cast<const uint4*>(&Bs[kw][h * (TILE / 2) + tx * 4]);
                a[h * 4 + 0] = av.x; a[h * 4 + 1] = av.y; a[h * 4 + 2] = av.z; a[h * 4 + 3] = av.w;
                b[h * 4 + 0] = bv.x; b[h * 4 + 1] = bv.y; b[h * 4 + 2] = bv.z; b[h * 4 + 3] = bv.w;
            }
            if constexpr (MODE == 1) {
#pragma unroll
                for (int i = 0; i < TT; ++i)
#pragma unroll
                    for (int j = 0; j < TT; ++j) acc[i][j] = dp4a_us(a[i], b[j], acc[i][j]);
            } else if constexpr (MODE == 2) {
#pragma unroll
                for (int i = 0; i < TT; ++i) {
                    const int32_t alo = static_cast<int16_t>(a[i] & 0xFFFFu), ahi = static_cast<int32_t>(a[i]) >> 16;
#pragma unroll
                    for (int j = 0; j < TT; ++j) {
                        const int32_t blo = static_cast<int16_t>(b[j] & 0xFFFFu), bhi = static_cast<int32_t>(b[j]) >> 16;
                        acc[i][j] = static_cast<int32_t>(static_cast<uint32_t>(acc[i][j]) +
                                                         static_cast<uint32_t>(alo * blo) +
                                                         static_cast<uint32_t>(ahi * bhi));
                    }
                }
            } else {
#pragma unroll
                for (int i = 0; i < TT; ++i) {
                    const uint32_t alo = a[i] & 0x0000FFFFu, ahi = a[i] & 0xFFFF0000u;
#pragma unroll
                    for (int j = 0; j < TT; ++j) acc[i][j] = sat_word_add(alo, ahi, b[j], acc[i][j]);
                }
            }
        }
    }

#pragma unroll
    for (int i = 0; i < TT; ++i) {
        const int64_t row = m0 + (i / 4) * (TILE / 2) + ty * 4 + (i % 4);
        if (row >= M) continue;
        int32_t* crow = C + row * ldc;
#pragma unroll
        for (int h = 0; h < TT / 4; ++h) {
            const int64_t col = n0 + h * (TILE / 2) + tx * 4;
            if (accumulate) {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (col + j < N) atomicAdd(reinterpret_cast<unsigned int*>(crow + col + j),
                                               static_cast<unsigned int>(acc[i][h * 4 + j]));
            } else if (c_vec_ok && col + 4 <= N) {
                *reinterpret_cast<int4*>(crow + col) =
                    make_int4(acc[i][h * 4 + 0], acc[i][h * 4 + 1], acc[i][h * 4 + 2], acc[i][h * 4 + 3]);
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (col + j < N) crow[col + j] = acc[i][h * 4 + j];
            }
        }
    }
}

}  // namespace ngemm_dev
