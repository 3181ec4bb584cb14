// kernel_skinny.cuh — memory-bound path for skinny inference GEMMs (M <= 16).
//
// C[M x N] = A[M x K] * B[N x K]^T with M tiny: every byte of B is used by at most 16 MACs,
// so the kernel is an HBM stream over B (read exactly once with 128-bit coalesced loads)
// while the whole of A sits in shared memory.  Each warp owns NR consecutive B rows at a
// time; lane l multiplies the 16-byte K chunks l, l+32, ... of those rows against the same
// chunks of every A row (IDP.4A, mixed signedness), then the warp folds its M*NR partial
// sums with a transposing butterfly (each level halves the live values per lane, so the
// whole fold costs ~M*NR shuffles instead of 5*M*NR).  This is the GPU analogue of the
// reference's tree reduction phase (lanes.hpp:147-159); int32 wrap-add makes the order
// immaterial.  K chunks start at multiples of 16 bytes, so saturating pairs stay
// even-aligned (gemm.hpp:94-99).
#pragma once

#include "ptx.cuh"

namespace ngemm_dev {

namespace skinny {
constexpr int THREADS = 256;
constexpr int WARPS = THREADS / 32;
}  // namespace skinny

template <int V, int OFF>
__device__ __forceinline__ void butterfly_fold(int32_t (&v)[V], int& base, int lane) {
    if constexpr (V > 1 && OFF > 0) {
        const bool up = (lane & OFF) != 0;
#pragma unroll
        for (int i = 0; i < V / 2; ++i) {
            const int32_t keep = up ? v[i + V / 2] : v[i];
            const int32_t send = up ? v[i] : v[i + V / 2];
            v[i] = static_cast<int32_t>(static_cast<uint32_t>(keep) +
                                        static_cast<uint32_t>(__shfl_xor_sync(0xffffffffu, send, OFF)));
        }
        if (up) base += V / 2;
        int32_t (&w)[V / 2 > 0 ? V / 2 : 1] = reinterpret_cast<int32_t (&)[V / 2 > 0 ? V / 2 : 1]>(v);
        butterfly_fold<V / 2, OFF / 2>(w, base, lane);
    } else if constexpr (OFF > 0) {
        // one value left per lane: plain xor-reduction over the remaining lane bits
#pragma unroll
        for (int o = OFF; o > 0; o >>= 1)
            v[0] = static_cast<int32_t>(static_cast<uint32_t>(v[0]) +
                                        static_cast<uint32_t>(__shfl_xor_sync(0xffffffffu, v[0], o)));
    }
}

template <int MT, int NR>
struct SkinnyFold {
    static constexpr int V = MT * NR;
    // values left per lane after halving at offsets 16, 8, ... (at most 5 levels)
    static constexpr int LEVELS = (V >= 32) ? 5 : (V >= 16 ? 4 : (V >= 8 ? 3 : (V >= 4 ? 2 : (V >= 2 ? 1 : 0))));
    static constexpr int LEFT = V >> LEVELS;
    static constexpr int LANE_MASK = (1 << (5 - LEVELS)) - 1;  // lanes whose low bits are 0 write
};

// MODE: 1 exact, 0 saturating.  MT: padded row count (1,2,4,8,16).  NR: B rows per warp pass.
template <int MODE, int MT, int NR>
__global__ void __launch_bounds__(skinny::THREADS)
    skinny_gemm_kernel(const uint8_t* __restrict__ A, int64_t lda, const int8_t* __restrict__ B, int64_t ldb,
                       int32_t* __restrict__ C, int64_t ldc, int M, int64_t N, int64_t K, int64_t kpad,
                       int b_vec_ok) {
    extern __shared__ __align__(16) uint8_t a_s[];  // [MT][kpad], zero padded
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    // stage A (rows >= M and bytes >= K are zero)
    for (int64_t i = tid; i < static_cast<int64_t>(MT) * kpad; i += skinny::THREADS) {
        const int64_t r = i / kpad, k = i - r * kpad;
        a_s[i] = (r < M && k < K) ? A[r * lda + k] : 0;
    }
    __syncthreads();

    const uint8_t* Bu = reinterpret_cast<const uint8_t*>(B);
    const int64_t nchunk = kpad / 16;
    const int64_t groups = (N + NR - 1) / NR;
    for (int64_t g = static_cast<int64_t>(blockIdx.x) * skinny::WARPS + warp; g < groups;
         g += static_cast<int64_t>(gridDim.x) * skinny::WARPS) {
        const int64_t n0 = g * NR;
        int32_t acc[MT * NR];
#pragma unroll
        for (int i = 0; i < MT * NR; ++i) acc[i] = 0;

        for (int64_t ch = lane; ch < nchunk; ch += 32) {
            const int64_t k0 = ch * 16;
            uint4 bv[NR];
#pragma unroll
            for (int r = 0; r < NR; ++r) {
                const int64_t n = n0 + r;
                if (n < N && b_vec_ok && k0 + 16 <= K) {
                    const uint4* p = reinterpret_cast<const uint4*>(Bu + n * ldb + k0);
                    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(bv[r].x), "=r"(bv[r].y), "=r"(bv[r].z), "=r"(bv[r].w)
                                 : "l"(p));
                } else {
                    uint32_t w[4] = {0, 0, 0, 0};
                    if (n < N) {
                        const uint8_t* p = Bu + n * ldb + k0;
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            if (k0 + i < K) w[i >> 2] |= static_cast<uint32_t>(__ldg(p + i)) << (8 * (i & 3));
                    }
                    bv[r] = make_uint4(w[0], w[1], w[2], w[3]);
                }
            }
#pragma unroll
            for (int m = 0; m < MT; ++m) {
                const uint4 av = *reinterpret_cast<const uint4*>(a_s + m * kpad + k0);
                const uint32_t aw[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
                for (int r = 0; r < NR; ++r) {
                    const uint32_t bw[4] = {bv[r].x, bv[r].y, bv[r].z, bv[r].w};
                    int32_t s = acc[m * NR + r];
                    if constexpr (MODE == 1) {
#pragma unroll
                        for (int q = 0; q < 4; ++q) s = dp4a_us(aw[q], bw[q], s);
                    } else {
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const int32_t p0 = clamp_i16(dp4a_us(aw[q] & 0x0000FFFFu, bw[q], 0));
                            const int32_t p1 = clamp_i16(dp4a_us(aw[q] & 0xFFFF0000u, bw[q], 0));
                            s = static_cast<int32_t>(static_cast<uint32_t>(s) + static_cast<uint32_t>(p0) +
                                                     static_cast<uint32_t>(p1));
                        }
                    }
                    acc[m * NR + r] = s;
                }
            }
        }

        int base = 0;
        butterfly_fold<MT * NR, 16>(acc, base, lane);
        using F = SkinnyFold<MT, NR>;
        if ((lane & F::LANE_MASK) == 0) {
#pragma unroll
            for (int i = 0; i < F::LEFT; ++i) {
                const int idx = base + i;
                const int m = idx / NR, r = idx - m * NR;
                const int64_t n = n0 + r;
                if (m < M && n < N) C[static_cast<int64_t>(m) * ldc + n] = acc[i];
            }
        }
    }
}

}  // namespace ngemm_dev
