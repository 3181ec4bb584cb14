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
// Tiling: 128x128 output tile per 256-thread CTA, 8x8 outputs per thread, K staged through
// shared memory 32 bytes (8 words) at a time, transposed to word-major so the inner loop is
// two LDS.128 per operand; next-tile global loads are prefetched into registers.
#pragma once

#include "ptx.cuh"

namespace ngemm_dev {

namespace simt {
constexpr int BM = 128, BN = 128, BKW = 8;  // BK = 32 bytes
constexpr int LDS = BM + 4;                  // padded word stride (bank-conflict free stores)
constexpr int THREADS = 256;
}  // namespace simt

// Loads 16 bytes (4 K-words) of row `r` starting at byte `k0`; zero outside [0,rows)x[0,K).
__device__ __forceinline__ uint4 simt_load16(const uint8_t* __restrict__ base, int64_t ld, int64_t r,
                                             int64_t rows, int64_t k0, int64_t K, bool vec_ok) {
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r >= rows || k0 >= K) return v;
    const uint8_t* p = base + r * ld + k0;
    if (vec_ok && k0 + 16 <= K) return __ldg(reinterpret_cast<const uint4*>(p));
    uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 16; ++i)
        if (k0 + i < K) w[i >> 2] |= static_cast<uint32_t>(__ldg(p + i)) << (8 * (i & 3));
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// MODE: 1 = WideningExact, 0 = HardwareSaturating (u8 x s8 words of 4 K-elements);
//       2 = the 16-bit path, i16 x i16 words of 2 K-elements (madd_pair_i16, lanes.hpp:42-47:
//           no saturation stage, everything mod 2^32).  K, lda, ldb are in BYTES here.
template <int MODE>
__global__ void __launch_bounds__(simt::THREADS, 2)
    simt_gemm_kernel(const uint8_t* __restrict__ A, int64_t lda, const int8_t* __restrict__ B, int64_t ldb,
                     int32_t* __restrict__ C, int64_t ldc, int64_t M, int64_t N, int64_t K, int vec_ok,
                     int c_vec_ok, const int32_t* __restrict__ guard) {
    using namespace simt;
    pdl_launch_dependents();
    pdl_wait();
    if (guard != nullptr && sat_safe(guard)) return;  // the tensor-core kernel took this call
    __shared__ __align__(16) uint32_t As[BKW][LDS];
    __shared__ __align__(16) uint32_t Bs[BKW][LDS];

    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    const int64_t m0 = static_cast<int64_t>(blockIdx.y) * BM;
    const int64_t n0 = static_cast<int64_t>(blockIdx.x) * BN;
    const uint8_t* Bu = reinterpret_cast<const uint8_t*>(B);

    // loader mapping: row lr, 16-byte half lh of the 32-byte K slice
    const int lr = tid >> 1, lh = tid & 1;

    int32_t acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0;

    const int64_t nk = (K + 31) / 32;
    uint4 ra = simt_load16(A, lda, m0 + lr, M, lh * 16, K, vec_ok);
    uint4 rb = simt_load16(Bu, ldb, n0 + lr, N, lh * 16, K, vec_ok);

    for (int64_t kt = 0; kt < nk; ++kt) {
        __syncthreads();
        As[lh * 4 + 0][lr] = ra.x;
        As[lh * 4 + 1][lr] = ra.y;
        As[lh * 4 + 2][lr] = ra.z;
        As[lh * 4 + 3][lr] = ra.w;
        Bs[lh * 4 + 0][lr] = rb.x;
        Bs[lh * 4 + 1][lr] = rb.y;
        Bs[lh * 4 + 2][lr] = rb.z;
        Bs[lh * 4 + 3][lr] = rb.w;
        __syncthreads();
        if (kt + 1 < nk) {
            const int64_t kn = (kt + 1) * 32 + lh * 16;
            ra = simt_load16(A, lda, m0 + lr, M, kn, K, vec_ok);
            rb = simt_load16(Bu, ldb, n0 + lr, N, kn, K, vec_ok);
        }
#pragma unroll
        for (int kw = 0; kw < BKW; ++kw) {
            uint32_t a[8], b[8];
            const uint4 a0 = *reinterpret_cast<const uint4*>(&As[kw][ty * 4]);
            const uint4 a1 = *reinterpret_cast<const uint4*>(&As[kw][64 + ty * 4]);
            const uint4 b0 = *reinterpret_cast<const uint4*>(&Bs[kw][tx * 4]);
            const uint4 b1 = *reinterpret_cast<const uint4*>(&Bs[kw][64 + tx * 4]);
            a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
            a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
            b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
            b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
            if constexpr (MODE == 1) {
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[i][j] = dp4a_us(a[i], b[j], acc[i][j]);
            } else if constexpr (MODE == 2) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int32_t alo = static_cast<int16_t>(a[i] & 0xFFFFu), ahi = static_cast<int32_t>(a[i]) >> 16;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int32_t blo = static_cast<int16_t>(b[j] & 0xFFFFu), bhi = static_cast<int32_t>(b[j]) >> 16;
                        acc[i][j] = static_cast<int32_t>(static_cast<uint32_t>(acc[i][j]) +
                                                         static_cast<uint32_t>(alo * blo) +
                                                         static_cast<uint32_t>(ahi * bhi));
                    }
                }
            } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const uint32_t alo = a[i] & 0x0000FFFFu, ahi = a[i] & 0xFFFF0000u;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int32_t p0 = clamp_i16(dp4a_us(alo, b[j], 0));
                        const int32_t p1 = clamp_i16(dp4a_us(ahi, b[j], 0));
                        acc[i][j] = static_cast<int32_t>(static_cast<uint32_t>(acc[i][j]) +
                                                         static_cast<uint32_t>(p0) + static_cast<uint32_t>(p1));
                    }
                }
            }
        }
    }

#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t row = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
        if (row >= M) continue;
        int32_t* crow = C + row * ldc;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t col = n0 + h * 64 + tx * 4;
            if (c_vec_ok && col + 4 <= N) {
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
