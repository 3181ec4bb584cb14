// kernel_tcgen05.cuh — the exact-mode u8 x s8 -> s32 GEMM on 5th-generation tensor cores.
//
//   C[M x N] (int32, row-major) = A[M x K] (u8, K-major) * B[N x K]^T (s8, K-major)
//
// Both operands are K-major, which is the native UMMA operand layout, so no transpose or
// repack is needed for the reference's row-major A and [N x K] B (matrix.hpp:14-16).
// tcgen05.mma kind::i8 with A unsigned, B signed and saturate = 0 accumulates in int32
// modulo 2^32 exactly like gemm_ref / wrap_add_i32 (gemm.hpp:46-50, common.hpp:132-135).
//
// Structure (persistent, warp-specialised, one CTA per SM; CG = 2 pairs the two SMs of a
// TPC into one cluster that computes a 256 x BN tile with cta_group::2 MMAs):
//   warp 0      : TMA producer — this CTA's 128 rows of A and BN/CG rows of B per 128-byte
//                 K slab (SWIZZLE_128B) into a STAGES-deep smem ring (full/empty mbarriers;
//                 with CG = 2 both CTAs' loads complete on the leader's full barrier);
//   warp 1      : MMA issuer (leader CTA only) — one thread issues BK/32 tcgen05.mma per
//                 stage into a double-buffered TMEM accumulator; tcgen05.commit (multicast
//                 to the pair) frees the stage in both CTAs and publishes finished tiles;
//   warp 2      : TMEM allocator (cta_group::CG);
//   warps 4..7  : epilogue — tcgen05.ld 32 lanes x 32 columns -> registers -> smem -> TMA,
//                 overlapped with the next tile's MMAs (double-buffered TMEM accumulator).
//   C leaves through swizzled smem staging and TMA tensor stores (full 128-byte lines);
//   split-K (splits > 1) uses the TMA unit's s32 reduce-add into a zeroed C — integer
//   wrap-add is associative, so split-K is bit-exact.
#pragma once

#include "ptx.cuh"

namespace ngemm_dev {

namespace tc {
constexpr int BM = 128;       // rows of A per CTA (UMMA M = 128 * CG)
constexpr int BK = 128;       // bytes of K per stage (one SWIZZLE_128B row)
constexpr int UMMA_K = 32;    // K per tcgen05.mma kind::i8
constexpr int THREADS = 256;  // 8 warps
constexpr int GROUP_M = 8;    // rasterisation group (measured best of 4..64 at 16384^3, profiles/groupm)

template <int BN, int STAGES, int CG>
struct Smem {
    static constexpr int A_BYTES = BM * BK;
    static constexpr int B_BYTES = (BN / CG) * BK;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                   : (2 * BN <= 256) ? 256 : 512;
    // epilogue staging: 4 warps x 2 buffers x (32 rows x 32 int32) in SWIZZLE_128B order
    static constexpr int STAGE_C_BYTES = 32 * 32 * 4;
    static constexpr int C_OFFSET = STAGES * STAGE_BYTES;
    static constexpr int BAR_OFFSET = C_OFFSET + 4 * 2 * STAGE_C_BYTES;
    static constexpr int BAR_BYTES = (2 * STAGES + 4) * 8 + 16;
    static constexpr int TOTAL = BAR_OFFSET + BAR_BYTES + 1024;  // +1024 for manual alignment
    static_assert(TOTAL <= 232448, "exceeds the 227 KB opt-in shared memory per CTA");
};
}  // namespace tc

struct TileMap {
    int tiles_m, tiles_n, splits;  // tiles_m counts 128*CG-row tiles
    int group_m;                   // rasterisation: group_m M-tiles walked down before moving along N
    __device__ __forceinline__ void coords(int t, int& tm, int& tn, int& ks) const {
        const int per_split = tiles_m * tiles_n;
        ks = t / per_split;
        t -= ks * per_split;
        const int group_size = group_m * tiles_n;
        const int g = t / group_size;
        const int first_m = g * group_m;
        const int gm = min(tiles_m - first_m, group_m);
        const int r = t - g * group_size;
        tm = first_m + r % gm;
        tn = r / gm;
    }
};

template <int BN, int STAGES, int CG>
__global__ void __launch_bounds__(tc::THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                   const __grid_constant__ CUtensorMap tma_c, int32_t* __restrict__ C, int64_t ldc, int M, int N,
                   int num_kb_total, TileMap map, int c_mode) {
    // c_mode: 0 = TMA tensor store of C (SWIZZLE_128B staging), 1 = TMA reduce-add into a
    // zeroed C (split-K), 2 = direct 128-byte row-segment stores (C not TMA-describable).
    using S = tc::Smem<BN, STAGES, CG>;
    constexpr int UMMA_M = tc::BM * CG;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::BAR_OFFSET);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = (CG == 2) ? cluster_ctarank() : 0;  // 0 = pair leader
    const int unit = (CG == 2) ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
    const int num_units = (CG == 2) ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);
    const int num_tiles = map.tiles_m * map.tiles_n * map.splits;
    const int kb_per_split = (num_kb_total + map.splits - 1) / map.splits;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tma_a);
        tma_prefetch(&tma_b);
        if (c_mode != 2) tma_prefetch(&tma_c);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], 4 * CG);  // one arrival per epilogue warp of every CTA
        }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc<CG>(tmem_slot, S::TMEM_COLS);
    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer (both CTAs)
            const uint64_t pol = policy_evict_normal();
            int s = 0;
            uint32_t ph = 0;
            for (int t = unit; t < num_tiles; t += num_units) {
                int tm, tn, ks;
                map.coords(t, tm, tn, ks);
                const int kb0 = ks * kb_per_split;
                const int kb1 = min(num_kb_total, kb0 + kb_per_split);
                const int row_a = tm * UMMA_M + static_cast<int>(rank) * tc::BM;
                const int row_b = tn * BN + static_cast<int>(rank) * (BN / CG);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&empty[s], ph ^ 1);
                    uint8_t* sa = smem + s * S::A_BYTES;
                    uint8_t* sb = smem + STAGES * S::A_BYTES + s * S::B_BYTES;
                    if constexpr (CG == 1) {
                        mbar_arrive_expect_tx(&full[s], S::STAGE_BYTES);
                        tma_load_2d(sa, &tma_a, &full[s], kb * tc::BK, row_a, pol);
                        tma_load_2d(sb, &tma_b, &full[s], kb * tc::BK, row_b, pol);
                    } else {
                        // both CTAs' bytes land on the leader's full barrier; the leader arms it
                        if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * S::STAGE_BYTES);
                        tma_load_2d_cg2(sa, &tma_a, &full[s], kb * tc::BK, row_a, pol);
                        tma_load_2d_cg2(sb, &tma_b, &full[s], kb * tc::BK, row_b, pol);
                    }
                    if (++s == STAGES) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {
            // ---------------- MMA issuer (single thread of the leader CTA)
            constexpr uint32_t idesc = idesc_i8(UMMA_M, BN, /*a_signed=*/false, /*b_signed=*/true);
            int s = 0;
            uint32_t ph = 0;
            int acc = 0;
            uint32_t acc_ph = 0;
            for (int t = unit; t < num_tiles; t += num_units) {
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
                        mma_i8<CG>(d_tmem, sdesc_k_sw128(sa + k * tc::UMMA_K), sdesc_k_sw128(sb + k * tc::UMMA_K),
                                   idesc, (kb > kb0 || k > 0) ? 1u : 0u);
                    }
                    if constexpr (CG == 1) mma_commit(&empty[s]);
                    else mma_commit_cg2_mc(&empty[s], 0x3);
                    if (++s == STAGES) { s = 0; ph ^= 1; }
                }
                if constexpr (CG == 1) mma_commit(&tfull[acc]);
                else mma_commit_cg2_mc(&tfull[acc], 0x3);
                acc ^= 1;
                if (acc == 0) acc_ph ^= 1;
            }
        }
    } else if (warp >= 4) {
        // ---------------- epilogue (both CTAs): TMEM -> registers -> swizzled smem -> TMA store
        const int ew = warp & 3;  // TMEM lane quadrant this warp may access
        uint8_t* stage_c = smem + S::C_OFFSET + ew * 2 * S::STAGE_C_BYTES;
        int acc = 0, cbuf = 0;
        uint32_t acc_ph = 0;
        for (int t = unit; t < num_tiles; t += num_units) {
            int tm, tn, ks;
            map.coords(t, tm, tn, ks);
            const int kb0 = ks * kb_per_split;
            const bool has_k = kb0 < num_kb_total;
            mbar_wait(&tfull[acc], acc_ph);
            tc_fence_after();
            const int row0 = tm * UMMA_M + static_cast<int>(rank) * tc::BM + ew * 32;
            const uint32_t taddr = tmem_base + acc * BN + (static_cast<uint32_t>(ew * 32) << 16);
#pragma unroll 1
            for (int c = 0; c < BN; c += 32) {
                uint32_t v[32];
                tmem_ld_32x32b_x32(taddr + c, v);
                tmem_wait_ld();
                if (!has_k || row0 >= M) continue;
                const int col0 = tn * BN + c;
                if (c_mode != 2) {
                    uint8_t* buf = stage_c + cbuf * S::STAGE_C_BYTES;
                    // the TMA store that last read this buffer must be done with it
                    if (lane == 0) tma_store_wait_read<1>();
                    __syncwarp();
                    const uint32_t rowp = smem_u32(buf) + lane * 128;
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        st_shared_v4(rowp + ((j ^ (lane & 7)) << 4), v[4 * j], v[4 * j + 1], v[4 * j + 2],
                                     v[4 * j + 3]);
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        if (c_mode == 0) tma_store_2d(&tma_c, buf, col0, row0);
                        else tma_reduce_add_2d(&tma_c, buf, col0, row0);
                        tma_store_commit();
                    }
                    cbuf ^= 1;
                } else {
                    const int64_t row = static_cast<int64_t>(row0) + lane;
                    if (row < M) {
                        int32_t* crow = C + row * ldc;
#pragma unroll
                        for (int q = 0; q < 32; ++q)
                            if (col0 + q < N) crow[col0 + q] = static_cast<int32_t>(v[q]);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (CG == 1) mbar_arrive(&tempty[acc]);
                else mbar_arrive_cluster(&tempty[acc], 0);
            }
            acc ^= 1;
            if (acc == 0) acc_ph ^= 1;
        }
        if (lane == 0) tma_store_wait<0>();
    }

    tc_fence_before();
    if constexpr (CG == 2) cluster_sync(); else __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<CG>(tmem_base, S::TMEM_COLS);
    }
}

}  // namespace ngemm_dev
