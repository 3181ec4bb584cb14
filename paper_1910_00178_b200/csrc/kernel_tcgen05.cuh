// kernel_tcgen05.cuh — the exact-mode u8 x s8 -> s32 GEMM on 5th-generation tensor cores.
//
//   C[M x N] (int32, row-major) = A[M x K] (u8, K-major) * B[N x K]^T (s8, K-major)
//
// Both operands are K-major, which is the native UMMA operand layout, so no transpose or
// repack is needed for the reference's row-major A and [N x K] B (matrix.hpp:14-16).
// tcgen05.mma kind::i8 with A unsigned, B signed and saturate = 0 accumulates in int32
// modulo 2^32 exactly like gemm_ref / wrap_add_i32 (gemm.hpp:46-50, common.hpp:132-135).
//
// Structure (persistent, warp-specialised, one CTA per SM):
//   warp 0      : TMA producer — A and B tiles (128-byte K slabs, SWIZZLE_128B) into a
//                 STAGES-deep shared-memory ring guarded by full/empty mbarriers;
//   warp 1      : MMA issuer — one elected thread issues BK/32 tcgen05.mma per stage into a
//                 TMEM accumulator (double-buffered across tiles), tcgen05.commit frees stages;
//   warp 2      : TMEM allocator;
//   warps 4..7  : epilogue — tcgen05.ld (32 lanes x 32 columns per warp per step) -> registers
//                 -> 128-byte row segments of C, overlapped with the next tile's MMAs.
// Split-K (kSplit > 1) writes through red.global.add on a zeroed C; integer wrap-add is
// associative, so split-K is bit-exact.
#pragma once

#include "ptx.cuh"

namespace ngemm_dev {

namespace tc {
constexpr int BM = 128;       // UMMA M per CTA
constexpr int BK = 128;       // bytes of K per stage (one SWIZZLE_128B row)
constexpr int UMMA_K = 32;    // K per tcgen05.mma kind::i8
constexpr int THREADS = 256;  // 8 warps
constexpr int GROUP_M = 16;   // rasterisation group (L2 reuse of B across consecutive tiles)

template <int BN, int STAGES>
struct Smem {
    static constexpr int A_BYTES = BM * BK;
    static constexpr int B_BYTES = BN * BK;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                   : (2 * BN <= 256) ? 256 : 512;
    static constexpr int BAR_OFFSET = STAGES * STAGE_BYTES;
    static constexpr int BAR_BYTES = (2 * STAGES + 4) * 8 + 16;
    static constexpr int TOTAL = BAR_OFFSET + BAR_BYTES + 1024;  // +1024 for manual alignment
};
}  // namespace tc

struct TileMap {
    int tiles_m, tiles_n, splits;
    __device__ __forceinline__ void coords(int t, int& tm, int& tn, int& ks) const {
        const int per_split = tiles_m * tiles_n;
        ks = t / per_split;
        t -= ks * per_split;
        const int group_size = tc::GROUP_M * tiles_n;
        const int g = t / group_size;
        const int first_m = g * tc::GROUP_M;
        const int gm = min(tiles_m - first_m, tc::GROUP_M);
        const int r = t - g * group_size;
        tm = first_m + r % gm;
        tn = r / gm;
    }
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(tc::THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                   int32_t* __restrict__ C, int64_t ldc, int M, int N, int num_kb_total, TileMap map,
                   int c_vec_ok) {
    using S = tc::Smem<BN, STAGES>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::BAR_OFFSET);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int num_tiles = map.tiles_m * map.tiles_n * map.splits;
    const int kb_per_split = (num_kb_total + map.splits - 1) / map.splits;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tma_a);
        tma_prefetch(&tma_b);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], 128);
        }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc<1>(tmem_slot, S::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer
            const uint64_t pol_a = policy_evict_normal();
            const uint64_t pol_b = policy_evict_normal();
            int s = 0;
            uint32_t ph = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
                int tm, tn, ks;
                map.coords(t, tm, tn, ks);
                const int kb0 = ks * kb_per_split;
                const int kb1 = min(num_kb_total, kb0 + kb_per_split);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&empty[s], ph ^ 1);
                    mbar_arrive_expect_tx(&full[s], S::STAGE_BYTES);
                    uint8_t* sa = smem + s * S::A_BYTES;
                    uint8_t* sb = smem + STAGES * S::A_BYTES + s * S::B_BYTES;
                    tma_load_2d(sa, &tma_a, &full[s], kb * tc::BK, tm * tc::BM, pol_a);
                    tma_load_2d(sb, &tma_b, &full[s], kb * tc::BK, tn * BN, pol_b);
                    if (++s == STAGES) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer (single thread)
            constexpr uint32_t idesc = idesc_i8(tc::BM, BN, /*a_signed=*/false, /*b_signed=*/true);
            int s = 0;
            uint32_t ph = 0;
            int acc = 0;
            uint32_t acc_ph = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
                int tm, tn, ks;
                map.coords(t, tm, tn, ks);
                const int kb0 = ks * kb_per_split;
                const int kb1 = min(num_kb_total, kb0 + kb_per_split);
                mbar_wait(&tempty[acc], acc_ph ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + s * S::A_BYTES);
                    const uint32_t sb = smem_u32(smem + STAGES * S::A_BYTES + s * S::B_BYTES);
#pragma unroll
                    for (int k = 0; k < tc::BK / tc::UMMA_K; ++k) {
                        mma_i8<1>(d_tmem, sdesc_k_sw128(sa + k * tc::UMMA_K), sdesc_k_sw128(sb + k * tc::UMMA_K),
                                  idesc, (kb > kb0 || k > 0) ? 1u : 0u);
                    }
                    mma_commit(&empty[s]);
                    if (++s == STAGES) { s = 0; ph ^= 1; }
                }
                mma_commit(&tfull[acc]);
                acc ^= 1;
                if (acc == 0) acc_ph ^= 1;
            }
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: TMEM -> registers -> global
        const int ew = warp & 3;  // TMEM lane quadrant this warp may access
        int acc = 0;
        uint32_t acc_ph = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
            int tm, tn, ks;
            map.coords(t, tm, tn, ks);
            const int kb0 = ks * kb_per_split;
            const bool has_k = kb0 < num_kb_total;
            mbar_wait(&tfull[acc], acc_ph);
            tc_fence_after();
            const int64_t row = static_cast<int64_t>(tm) * tc::BM + ew * 32 + lane;
            const uint32_t taddr = tmem_base + acc * BN + (static_cast<uint32_t>(ew * 32) << 16);
            int32_t* crow = C + row * ldc;
#pragma unroll 1
            for (int c = 0; c < BN; c += 32) {
                uint32_t v[32];
                tmem_ld_32x32b_x32(taddr + c, v);
                tmem_wait_ld();
                if (!has_k || row >= M) continue;
                const int64_t col0 = static_cast<int64_t>(tn) * BN + c;
                if (map.splits == 1) {
                    if (c_vec_ok && col0 + 32 <= N) {
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            *reinterpret_cast<int4*>(crow + col0 + 4 * q) =
                                make_int4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                    } else {
#pragma unroll
                        for (int q = 0; q < 32; ++q)
                            if (col0 + q < N) crow[col0 + q] = static_cast<int32_t>(v[q]);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < 32; ++q)
                        if (col0 + q < N) atomicAdd(reinterpret_cast<unsigned int*>(crow + col0 + q), v[q]);
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty[acc]);
            acc ^= 1;
            if (acc == 0) acc_ph ^= 1;
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<1>(tmem_base, S::TMEM_COLS);
    }
}

}  // namespace ngemm_dev
