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

// Phase-trace hooks (scripts/probes/tc_trace.py; the library build compiles them out).
#ifndef TC_TRACE_NOW
#define TC_TRACE_NOW(p)
#define TC_TRACE_KEEP(p)
#define TC_TRACE_FLUSH()
#define TC_TRACE_END()
#endif

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
    // BN <= 256: two accumulators (the epilogue of one tile overlaps the next tile's MMAs);
    // BN = 512: one accumulator over all 512 TMEM columns (25 % less L2->SM operand traffic per
    // MAC than 256 x 256; the epilogue overlaps only the next tile's first loads)
    static constexpr int NACC = BN > 256 ? 1 : 2;
    static constexpr int MMA_N = BN > 256 ? 256 : BN;  // UMMA N <= 256: BN = 512 issues two per K step
    static constexpr int TMEM_COLS = (NACC * BN <= 32) ? 32 : (NACC * BN <= 64) ? 64 : (NACC * BN <= 128) ? 128
                                   : (NACC * BN <= 256) ? 256 : 512;
    static_assert(NACC * BN <= 512, "the accumulators must fit the 512 TMEM columns");
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
    int preissue;                  // 1-CTA tiles: issue the first STAGES loads before the block sync
    int l2hint;                    // L2 eviction hints: bit 0 A evict_last, bit 1 B evict_first, bit 2 C evict_first
    int prefetch;                  // warm L2 with the first operand slabs before the PDL wait
    int dbg;                       // probes only (NGEMM_TC_DBG): bit 0 skip C stores, bit 1 skip MMAs,
                                   // bit 2 skip operand loads (1-CTA configs)
    int trace_id;                  // trace build: launch index for the phase stamps (-1 otherwise)
    int a_signed, b_signed;        // operand formats (u8 x s8 for the NGEMM path; any mix for i16 planes)
    int shift;                     // epilogue: C (+)= acc << shift  (i16 byte-plane decomposition)
    // c_mode 4, fused requantisation: out[r][c] = clamp(rint(float(acc + bias[c]) * scale[c]) + zp)
    const float* rq_scale;
    const int32_t* rq_bias;        // may be null
    int8_t* rq_out;
    int64_t rq_ldo;
    int rq_zp;
    // Tail split: the first full_tiles tiles run whole; every later tile (the last, partial wave)
    // runs as two half-width tiles (BN/2 columns each), so a wave that would leave more than half
    // of the SMs idle becomes a wave of half-length work items on (nearly) all of them.
    int full_tiles;
    __device__ __forceinline__ int work_items(int num_tiles) const { return full_tiles + 2 * (num_tiles - full_tiles); }
    // work item u -> tile coordinates and half (-1 = whole tile, 0 / 1 = left / right half)
    __device__ __forceinline__ void item(int u, int& tm, int& tn, int& ks, int& half) const {
        if (u < full_tiles) {
            coords(u, tm, tn, ks);
            half = -1;
        } else {
            const int v = u - full_tiles;
            coords(full_tiles + (v >> 1), tm, tn, ks);
            half = v & 1;
        }
    }
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

// MC = 2 (CG = 2 only): a cluster of two CTA pairs computes two horizontally adjacent
// 256 x BN tiles that share the same A rows; each CTA loads half of its A slab and multicasts
// it to its counterpart in the other pair, halving A's L2->SM traffic.  The pairs run in
// lockstep: every CTA's empty barrier waits for both pairs' MMA commits.
template <int BN, int STAGES, int CG, int MC = 1>
__global__ void __launch_bounds__(tc::THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                   const __grid_constant__ CUtensorMap tma_b_half, const __grid_constant__ CUtensorMap tma_c, int32_t* __restrict__ C, int64_t ldc, int M, int N,
                   int num_kb_total, TileMap map, int c_mode) {
    // c_mode: 0 = TMA tensor store of C (SWIZZLE_128B staging), 1 = TMA reduce-add into a
    // zeroed C (split-K), 2 = direct scalar stores (C not TMA-describable), 3 = direct 16-byte
    // vector stores (aligned C, single-wave grids), 4 = fused requantisation to int8 (map.rq_*).
    TC_TRACE_KEEP(0);
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
    static_assert(MC == 1 || MC == 2, "A is multicast across at most two tiles");
    constexpr int CL = CG * MC;  // CTAs per cluster
    const uint32_t crank = (CL > 1) ? cluster_ctarank() : 0;
    const uint32_t rank = crank & (CG - 1);           // rank within the pair: 0 = pair leader
    const uint32_t pair = crank / CG;                 // which pair of the cluster (MC = 2)
    const uint32_t leader = pair * CG;                // cluster rank of this pair's leader
    const uint16_t pair_mask = static_cast<uint16_t>(((1u << CG) - 1u) << leader);
    const int unit = static_cast<int>(blockIdx.x) / CL;
    const int num_units = static_cast<int>(gridDim.x) / CL;
    const int num_tiles = map.work_items(map.tiles_m * map.tiles_n * map.splits);  // work items
    const int kb_per_split = (num_kb_total + map.splits - 1) / map.splits;

    pdl_launch_dependents();

    // ---------------- TMA producer state (warp 0, one thread; both CTAs of a pair)
    int p_t = unit, p_kb = 0, p_kb1 = 0, p_s = 0, p_row_a = 0, p_row_b = 0, p_half = -1;
    uint32_t p_ph = 0;
    bool p_open = false;
    auto produce = [&](int budget) {
        // L2 policy: the raster walks group_m M-tiles down while sweeping N, so an A slab is
        // re-read by every wave of its group (keep it: evict_last) while a B slab is dead once
        // the current wave has passed (stream it: evict_first).  map.l2hint bits select each.
        const uint64_t pol_a = (map.l2hint & 1) ? policy_evict_last() : policy_evict_normal();
        const uint64_t pol_b = (map.l2hint & 2) ? policy_evict_first() : policy_evict_normal();
        while (p_t < num_tiles && budget != 0) {
            if (!p_open) {
                int tm, tn, ks;
                map.item(p_t, tm, tn, ks, p_half);
                tn = tn * MC + static_cast<int>(pair);
                p_kb = ks * kb_per_split;
                p_kb1 = min(num_kb_total, p_kb + kb_per_split);
                p_row_a = tm * UMMA_M + static_cast<int>(rank) * tc::BM;
                p_row_b = p_half < 0 ? tn * BN + static_cast<int>(rank) * (BN / CG)
                                     : tn * BN + p_half * (BN / 2) + static_cast<int>(rank) * (BN / (2 * CG));
                p_open = true;
            }
            const CUtensorMap* tb = p_half < 0 ? &tma_b : &tma_b_half;
            const uint32_t stage_tx = S::A_BYTES + (p_half < 0 ? S::B_BYTES : S::B_BYTES / 2);
            if (p_kb >= p_kb1) {
                p_t += num_units;
                p_open = false;
                continue;
            }
            mbar_wait(&empty[p_s], p_ph ^ 1);  // returns at once for the first STAGES fills
            uint8_t* sa = smem + p_s * S::A_BYTES;
            uint8_t* sb = smem + STAGES * S::A_BYTES + p_s * S::B_BYTES;
            if (CG == 1 && (map.dbg & 4)) {
                mbar_arrive(&full[p_s]);  // probes only: no operand traffic
            } else if constexpr (CG == 1) {
                mbar_arrive_expect_tx(&full[p_s], MC == 1 ? stage_tx : S::STAGE_BYTES);
                if constexpr (MC == 1) {
                    tma_load_2d(sa, &tma_a, &full[p_s], p_kb * tc::BK, p_row_a, pol_a);
                } else {
                    // this CTA's half of the shared A slab, to itself and its neighbour in the cluster
                    tma_load_2d_mc(sa + pair * (S::A_BYTES / 2), &tma_a, &full[p_s], p_kb * tc::BK,
                                   p_row_a + static_cast<int>(pair) * (tc::BM / 2), static_cast<uint16_t>(0x3), pol_a);
                }
                tma_load_2d(sb, tb, &full[p_s], p_kb * tc::BK, p_row_b, pol_b);
            } else {
                // both CTAs' bytes land on the leader's full barrier; the leader arms it
                if (rank == 0) mbar_arrive_expect_tx(&full[p_s], 2 * (MC == 1 ? stage_tx : S::STAGE_BYTES));
                if constexpr (MC == 1) {
                    tma_load_2d_cg2(sa, &tma_a, &full[p_s], p_kb * tc::BK, p_row_a, pol_a);
                } else {
                    // this CTA's half of the shared A slab, to itself and its counterpart
                    const uint16_t mask = static_cast<uint16_t>((1u << rank) | (1u << (rank + CG)));
                    tma_load_2d_cg2_mc(sa + pair * (S::A_BYTES / 2), &tma_a, &full[p_s], p_kb * tc::BK,
                                       p_row_a + static_cast<int>(pair) * (tc::BM / 2), mask, pol_a);
                }
                tma_load_2d_cg2(sb, tb, &full[p_s], p_kb * tc::BK, p_row_b, pol_b);
            }
            ++p_kb;
            if (++p_s == STAGES) { p_s = 0; p_ph ^= 1; }
            --budget;
        }
    };

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tma_a);
        tma_prefetch(&tma_b);
        if (map.full_tiles < map.tiles_m * map.tiles_n * map.splits) tma_prefetch(&tma_b_half);
        if (c_mode <= 1) tma_prefetch(&tma_c);
        if (MC == 1 && map.prefetch && unit < map.full_tiles) {
            // warm L2 with this CTA's first STAGES operand slabs before the dependency wait
            // (tma_prefetch_tile_2d: prefetch only, re-read after pdl_wait), so the first HBM
            // round trips overlap the preceding grid's tail and this CTA's setup
            int tm, tn, ks;
            map.coords(unit, tm, tn, ks);
            const int kb0 = ks * kb_per_split;
            const int kb1 = min(num_kb_total, min(kb0 + kb_per_split, kb0 + STAGES));
            const int row_a = tm * UMMA_M + static_cast<int>(rank) * tc::BM;
            const int row_b = tn * BN + static_cast<int>(rank) * (BN / CG);
            for (int kb = kb0; kb < kb1; ++kb) {
                tma_prefetch_tile_2d(&tma_a, kb * tc::BK, row_a);
                tma_prefetch_tile_2d(&tma_b, kb * tc::BK, row_b);
            }
        }
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], MC);  // one commit per pair that reads this stage
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], 4 * CG);  // one arrival per epilogue warp of every CTA
        }
        fence_mbar_init();
        if (CL == 1 && map.preissue) {
            // single-CTA tiles: start the operand stream before the block-wide sync, so the first
            // DRAM round trips overlap TMEM allocation and the sync
            pdl_wait();
            produce(STAGES);
        }
    }
    if (warp == 2) tmem_alloc<CG>(tmem_slot, S::TMEM_COLS);
    tc_fence_before();
    if constexpr (CL > 1) cluster_sync(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    TC_TRACE_KEEP(1);
    pdl_wait();  // operands / C may belong to the preceding kernel in the stream
    TC_TRACE_FLUSH();

    if (warp == 0) {
        if (lane == 0) {
            TC_TRACE_NOW(3);
            produce(-1);
            TC_TRACE_NOW(4);
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {
            // ---------------- MMA issuer (single thread of the leader CTA)
            const uint32_t idesc_full = idesc_i8(UMMA_M, S::MMA_N, map.a_signed != 0, map.b_signed != 0);
            const uint32_t idesc_half = idesc_i8(UMMA_M, S::MMA_N / 2, map.a_signed != 0, map.b_signed != 0);
            int s = 0;
            uint32_t ph = 0;
            int acc = 0;
            uint32_t acc_ph = 0;
            for (int t = unit; t < num_tiles; t += num_units) {
                int tm, tn, ks, half;
                map.item(t, tm, tn, ks, half);
                const uint32_t idesc = half < 0 ? idesc_full : idesc_half;
                const int kb0 = ks * kb_per_split;
                const int kb1 = min(num_kb_total, kb0 + kb_per_split);
                mbar_wait(&tempty[acc], acc_ph ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    if (t == unit && kb == kb0) TC_TRACE_NOW(5);
                    const uint32_t sa = smem_u32(smem + s * S::A_BYTES);
                    const uint32_t sb = smem_u32(smem + STAGES * S::A_BYTES + s * S::B_BYTES);
#pragma unroll
                    for (int h = 0; h < BN / S::MMA_N; ++h) {
                        // BN = 512: MMA h reads rows [128h, 128h + 128) of each CTA's B slab (this
                        // CTA's 256 rows of B) and accumulates into TMEM columns [256h, 256h + 256).
                        // All K steps of a stage go into one accumulator before the other: issuing
                        // the two accumulators' MMAs alternately (so that they could share the A
                        // collector) measured 15 % slower (profiles/r2/collector_kmajor_ab_r2.log)
#pragma unroll
                        for (int k = 0; k < tc::BK / tc::UMMA_K; ++k) {
                            if (map.dbg & 2) break;
                            mma_i8<CG>(d_tmem + h * S::MMA_N, sdesc_k_sw128(sa + k * tc::UMMA_K),
                                       sdesc_k_sw128(sb + h * (S::MMA_N / CG) * tc::BK + k * tc::UMMA_K), idesc,
                                       (kb > kb0 || k > 0) ? 1u : 0u);
                        }
                    }
                    if constexpr (CG == 1 && MC == 1) mma_commit(&empty[s]);
                    else if constexpr (CG == 1) mma_commit_mc(&empty[s], static_cast<uint16_t>(0x3));  // both read A
                    else mma_commit_cg2_mc(&empty[s], MC == 1 ? pair_mask : static_cast<uint16_t>(0xF));
                    if (++s == STAGES) { s = 0; ph ^= 1; }
                }
                if constexpr (CG == 1) mma_commit(&tfull[acc]);
                else mma_commit_cg2_mc(&tfull[acc], pair_mask);
                if (++acc == S::NACC) { acc = 0; acc_ph ^= 1; }
            }
            TC_TRACE_NOW(6);
        }
    } else if (warp >= 4) {
        // ---------------- epilogue (both CTAs): TMEM -> registers -> swizzled smem -> TMA store
        const int ew = warp & 3;  // TMEM lane quadrant this warp may access
        // C is written once and never re-read by this kernel: map.l2hint bit 2 streams it through
        // L2 with evict_first so it does not push out the operand slabs the next waves re-read
        const uint64_t pol_c = policy_evict_first();
        uint8_t* stage_c = smem + S::C_OFFSET + ew * 2 * S::STAGE_C_BYTES;
        int acc = 0, cbuf = 0;
        uint32_t acc_ph = 0;
        for (int t = unit; t < num_tiles; t += num_units) {
            int tm, tn, ks, half;
            map.item(t, tm, tn, ks, half);
            tn = tn * MC + static_cast<int>(pair);
            const int ncols = half < 0 ? BN : BN / 2;
            const int col_base = tn * BN + (half < 0 ? 0 : half * (BN / 2));
            const int kb0 = ks * kb_per_split;
            const bool has_k = kb0 < num_kb_total;
            mbar_wait(&tfull[acc], acc_ph);
            tc_fence_after();
            if (t == unit && warp == 4 && lane == 0) TC_TRACE_NOW(7);
            const int row0 = tm * UMMA_M + static_cast<int>(rank) * tc::BM + ew * 32;
            const uint32_t taddr = tmem_base + acc * BN + (static_cast<uint32_t>(ew * 32) << 16);
            // one 32-column chunk of this warp's 32 accumulator rows: registers -> C
            auto emit = [&](uint32_t (&v)[32], const int c) {
                if (t == unit && c == 0 && warp == 4 && lane == 0) TC_TRACE_NOW(10);
                if (!has_k || row0 >= M) return;
                if (map.shift) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] <<= map.shift;  // mod 2^32, like the accumulator
                }
                // BN = 512 (pairs): TMEM columns [256h + 128r, 256h + 128r + 128) hold tile columns
                // [256r + 128h, +128) — CTA r's B slab is tile columns [256r, 256r + 256)
                const int col0 = col_base + (BN > 256 ? ((c >> 7) & 1) * 256 + (c >> 8) * 128 + (c & 127) : c);
                if (c_mode == 4) {
                    // fused requantisation to int8: each lane loads one column's scale / bias and
                    // the warp broadcasts them; lane = row, 32 int8 per row, two 16-byte stores
                    const int col = col0 + lane;
                    const float my_s = col < N ? __ldg(map.rq_scale + col) : 0.0f;
                    const int32_t my_b = (map.rq_bias != nullptr && col < N) ? __ldg(map.rq_bias + col) : 0;
                    uint32_t packed[8];
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float sj = __shfl_sync(0xffffffffu, my_s, j);
                        const int32_t bj = __shfl_sync(0xffffffffu, my_b, j);
                        const int8_t q = requant_s8(v[j], bj, sj, map.rq_zp);
                        if ((j & 3) == 0) packed[j >> 2] = 0;
                        packed[j >> 2] |= (static_cast<uint32_t>(static_cast<uint8_t>(q))) << (8 * (j & 3));
                    }
                    const int64_t row = static_cast<int64_t>(row0) + lane;
                    if (row < M) {
                        int8_t* orow = map.rq_out + row * map.rq_ldo + col0;
                        if (col0 + 32 <= N && (reinterpret_cast<uintptr_t>(orow) & 15) == 0) {
                            st_global_v4(orow, packed[0], packed[1], packed[2], packed[3]);
                            st_global_v4(orow + 16, packed[4], packed[5], packed[6], packed[7]);
                        } else {
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                if (col0 + j < N) orow[j] = static_cast<int8_t>((packed[j >> 2] >> (8 * (j & 3))) & 0xFFu);
                        }
                    }
                    return;
                }
                if (c_mode <= 1) {
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
                    if (lane == 0 && !(map.dbg & 1)) {
                        if (c_mode == 0 && (map.l2hint & 4)) tma_store_2d_hint(&tma_c, buf, col0, row0, pol_c);
                        else if (c_mode == 0) tma_store_2d(&tma_c, buf, col0, row0);
                        else tma_reduce_add_2d(&tma_c, buf, col0, row0);
                        tma_store_commit();
                    }
                    if (t == unit && c == 0 && warp == 4 && lane == 0) TC_TRACE_NOW(11);
                    cbuf ^= 1;
                } else {
                    // direct stores, lane = row: c_mode 3 (16-byte aligned C) writes each row's
                    // 128-byte segment with 8 vector stores and never waits on them — for
                    // single-wave grids, where the TMA store path's staging and drain sit on
                    // the critical path; c_mode 2 (C not TMA-describable) stores scalars
                    const int64_t row = static_cast<int64_t>(row0) + lane;
                    if (row < M) {
                        int32_t* crow = C + row * ldc + col0;
                        if (c_mode == 3 && col0 + 32 <= N) {
#pragma unroll
                            for (int j = 0; j < 8; ++j)
                                st_global_v4(crow + 4 * j, v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                        } else {
#pragma unroll
                            for (int q = 0; q < 32; ++q)
                                if (col0 + q < N) crow[q] = static_cast<int32_t>(v[q]);
                        }
                    }
                }
            };
            // two register sets: the tcgen05.ld of the next chunk is in flight while this one is
            // staged and stored (tcgen05.wait::ld waits for every outstanding load, so the next
            // load is issued right after the wait)
            uint32_t va[32], vb[32];
            tmem_ld_32x32b_x32(taddr, va);
#pragma unroll 1
            for (int c = 0; c < ncols; c += 64) {
                tmem_wait_ld();
                if (c + 32 < ncols) tmem_ld_32x32b_x32(taddr + c + 32, vb);
                emit(va, c);
                if (c + 32 < ncols) {
                    tmem_wait_ld();
                    if (c + 64 < ncols) tmem_ld_32x32b_x32(taddr + c + 64, va);
                    emit(vb, c + 32);
                }
            }
            if (t == unit && warp == 4 && lane == 0) TC_TRACE_NOW(12);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (CG == 1) mbar_arrive(&tempty[acc]);
                else mbar_arrive_cluster(&tempty[acc], leader);
            }
            if (++acc == S::NACC) { acc = 0; acc_ph ^= 1; }
        }
        // the staging smem must be read out before the CTA exits; the global writes themselves
        // complete before the grid does (and before a dependent grid's griddepcontrol.wait)
        if (lane == 0) tma_store_wait_read<0>();
        if (warp == 4 && lane == 0) TC_TRACE_NOW(8);
    }

    tc_fence_before();
    if constexpr (CL > 1) cluster_sync(); else __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<CG>(tmem_base, S::TMEM_COLS);
    }
    TC_TRACE_END();
}

}  // namespace ngemm_dev

namespace ngemm_dev {

// ---------------------------------------------------------------------------------------------
// tc_skinny_kernel — exact-mode skinny GEMM (M <= 16) on the tensor cores with the operands
// swapped: D^T[n, m] = B[n, :] . A[m, :].  B's rows fill the UMMA M = 128 dimension and the
// (zero-padded) A rows the UMMA N = 16 dimension, so no MMA work is wasted on padding M and
// the kernel is a pure TMA stream over B: each CTA owns 128 rows of B and one K slice and
// issues all of its TMA loads up front.  The KS CTAs that share a row tile form one thread-
// block cluster along K; their 128 x 16 partial tiles are summed through distributed shared
// memory (each rank reduces 128/KS columns and writes them to C), so split-K needs no
// workspace, no zeroing pass and no atomics.  Instruction descriptor: A operand (B tile)
// signed, B operand (A slice) unsigned; s32 accumulation mod 2^32.
// ---------------------------------------------------------------------------------------------
namespace tcs {
constexpr int BN_ROWS = 128;  // rows of B per CTA (UMMA M)
constexpr int MPAD = 16;      // A rows (UMMA N)
constexpr int BK = 128;
constexpr int THREADS = 256;
template <int STAGES>
struct Smem {
    static constexpr int B_BYTES = BN_ROWS * BK;  // 16 KB
    static constexpr int A_BYTES = MPAD * BK;     // 2 KB
    static constexpr int STAGE_BYTES = B_BYTES + A_BYTES;
    static constexpr int P_OFFSET = STAGES * STAGE_BYTES;
    static constexpr int P_BYTES = MPAD * BN_ROWS * 4;  // partial tile [16 m][128 n] int32
    static constexpr int BAR_OFFSET = P_OFFSET + P_BYTES;
    static constexpr int TOTAL = BAR_OFFSET + (2 * STAGES + 2) * 8 + 16 + 1024;
};
}  // namespace tcs

template <int STAGES>
__global__ void __launch_bounds__(tcs::THREADS, 1)
    tc_skinny_kernel(const __grid_constant__ CUtensorMap tma_b, const __grid_constant__ CUtensorMap tma_a,
                     int32_t* __restrict__ C, int64_t ldc, int M, int N, int num_kb, int kb_per_cta) {
    using S = tcs::Smem<STAGES>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::BAR_OFFSET);
    uint64_t* empty = full + STAGES;
    uint64_t* done = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 2);
    int32_t* part = reinterpret_cast<int32_t*>(smem + S::P_OFFSET);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nt = blockIdx.x;
    const int ks = blockIdx.y, nks = gridDim.y;  // cluster = the nks CTAs of this row tile
    const int kb0 = ks * kb_per_cta, kb1 = min(num_kb, kb0 + kb_per_cta);

    pdl_launch_dependents();
    // The producer initialises the barriers and issues the first STAGES loads BEFORE the
    // block-wide sync, so the DRAM latency overlaps TMEM allocation and the sync itself.
    const uint64_t pol_b = policy_evict_first();  // B is streamed exactly once
    const uint64_t pol_a = policy_evict_last();   // A is re-read by every CTA
    int p_s = 0, p_kb = kb0;
    uint32_t p_ph = 0;
    if (warp == 0 && lane == 0) {
        tma_prefetch(&tma_b);
        tma_prefetch(&tma_a);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(&done[0], 1);
        fence_mbar_init();
        pdl_wait();  // inputs may come from the preceding kernel
        for (; p_kb < kb1 && p_kb < kb0 + STAGES; ++p_kb) {
            mbar_arrive_expect_tx(&full[p_s], S::STAGE_BYTES);
            uint8_t* sb = smem + p_s * S::STAGE_BYTES;
            tma_load_2d(sb, &tma_b, &full[p_s], p_kb * tcs::BK, nt * tcs::BN_ROWS, pol_b);
            tma_load_2d(sb + S::B_BYTES, &tma_a, &full[p_s], p_kb * tcs::BK, 0, pol_a);
            if (++p_s == STAGES) { p_s = 0; p_ph ^= 1; }
        }
    }
    if (warp == 2) tmem_alloc<1>(tmem_slot, 32);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_wait();

    if (warp == 0 && lane == 0) {
        for (; p_kb < kb1; ++p_kb) {
            mbar_wait(&empty[p_s], p_ph ^ 1);
            mbar_arrive_expect_tx(&full[p_s], S::STAGE_BYTES);
            uint8_t* sb = smem + p_s * S::STAGE_BYTES;
            tma_load_2d(sb, &tma_b, &full[p_s], p_kb * tcs::BK, nt * tcs::BN_ROWS, pol_b);
            tma_load_2d(sb + S::B_BYTES, &tma_a, &full[p_s], p_kb * tcs::BK, 0, pol_a);
            if (++p_s == STAGES) { p_s = 0; p_ph ^= 1; }
        }
    } else if (warp == 1 && lane == 0) {
        constexpr uint32_t idesc = idesc_i8(tcs::BN_ROWS, tcs::MPAD, /*a_signed=*/true, /*b_signed=*/false);
        int s = 0;
        uint32_t ph = 0;
        for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(&full[s], ph);
            tc_fence_after();
            const uint32_t sb = smem_u32(smem + s * S::STAGE_BYTES);
#pragma unroll
            for (int k = 0; k < tcs::BK / 32; ++k)
                mma_i8<1>(tmem_base, sdesc_k_sw128(sb + k * 32), sdesc_k_sw128(sb + S::B_BYTES + k * 32), idesc,
                          (kb > kb0 || k > 0) ? 1u : 0u);
            mma_commit(&empty[s]);
            if (++s == STAGES) { s = 0; ph ^= 1; }
        }
        mma_commit(&done[0]);
    } else if (warp >= 4) {
        // partial tile TMEM -> smem [m][n]
        const int ew = warp & 3;
        const int nl = ew * 32 + lane;
        if (kb0 < kb1) {
            mbar_wait(&done[0], 0);
            tc_fence_after();
            uint32_t v[16];
            tmem_ld_32x32b_x16(tmem_base + (static_cast<uint32_t>(ew * 32) << 16), v);
            tmem_wait_ld();
#pragma unroll
            for (int m = 0; m < tcs::MPAD; ++m) part[m * tcs::BN_ROWS + nl] = static_cast<int32_t>(v[m]);
        } else {
#pragma unroll
            for (int m = 0; m < tcs::MPAD; ++m) part[m * tcs::BN_ROWS + nl] = 0;
        }
    }
    tc_fence_before();
    if (nks > 1) cluster_sync(); else __syncthreads();

    // rank ks reduces columns [ks*cw, (ks+1)*cw) of the tile over the cluster and writes C
    const int cw = tcs::BN_ROWS / nks;  // host keeps nks a power of two <= 8
    const uint32_t part_addr = smem_u32(part);
    for (int i = threadIdx.x; i < tcs::MPAD * cw; i += tcs::THREADS) {
        const int m = i / cw, nl = ks * cw + (i - m * cw);
        const int n = nt * tcs::BN_ROWS + nl;
        if (m >= M || n >= N) continue;
        const uint32_t off = part_addr + static_cast<uint32_t>((m * tcs::BN_ROWS + nl) * 4);
        uint32_t sum = static_cast<uint32_t>(part[m * tcs::BN_ROWS + nl]);
        if (nks > 1) {
            // issue all remote loads back to back, then add (latency overlaps)
            uint32_t r[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) r[q] = (q < nks && q != ks) ? dsmem_ld_u32(off, q) : 0u;
#pragma unroll
            for (int q = 0; q < 8; ++q) sum += r[q];
        }
        C[static_cast<int64_t>(m) * ldc + n] = static_cast<int32_t>(sum);
    }
    if (nks > 1) cluster_sync(); else __syncthreads();  // peers may still read our partial
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<1>(tmem_base, 32);
    }
}

}  // namespace ngemm_dev
