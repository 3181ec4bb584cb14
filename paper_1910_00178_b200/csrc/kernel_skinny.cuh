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

// Phase-trace hooks for scripts/probes/skinny_trace.cu (no code in the library build).
#ifndef SKINNY_TRACE_AT
#define SKINNY_TRACE_AT(phase)
#define SKINNY_TRACE_END()
#endif

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
    pdl_launch_dependents();
    pdl_wait();

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
                        for (int q = 0; q < 4; ++q)
                            s = sat_word_add(aw[q] & 0x0000FFFFu, aw[q] & 0xFFFF0000u, bw[q], s);
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

namespace ngemm_dev {

// ---------------------------------------------------------------------------------------------
// skinny_rows_kernel — the NGEMM broadcast idea on the GPU: every LANE owns one row of B (one
// output column n) and accumulates all M outputs C[0..M)[n] in registers, while the matching
// K-slice of A is BROADCAST to the warp from shared memory (one 16-byte wavefront serves all
// 32 lanes).  No cross-lane reduction at all (the paper's phase-3 tree reduction disappears,
// PAPER.md §3); the 8 warps of a CTA split the CTA's K range and meet once in shared memory.
// B is read exactly once, 32 contiguous bytes (one full DRAM sector) per lane per step.
// Grid: 32-row tiles of B x K splits; with K splits > 1 the partials are added into a zeroed C
// (int32 wrap-add is order independent).  K splits start at multiples of 32 bytes, so
// HardwareSaturating pairs stay even-aligned (gemm.hpp:94-99).
// ---------------------------------------------------------------------------------------------
namespace skinny_rows {
constexpr int THREADS = 256;
constexpr int WARPS = 8;
constexpr int STEP = 32;  // bytes of K per lane per step
}  // namespace skinny_rows

template <int MODE, int MT>
__global__ void __launch_bounds__(skinny_rows::THREADS)
    skinny_rows_kernel(const uint8_t* __restrict__ A, int64_t lda, const int8_t* __restrict__ B, int64_t ldb,
                       int32_t* __restrict__ C, int64_t ldc, int M, int64_t N, int64_t K, int64_t k_range,
                       int b_vec_ok, int accumulate) {
    extern __shared__ __align__(16) uint8_t sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    pdl_launch_dependents();
    pdl_wait();
    const int64_t n0 = static_cast<int64_t>(blockIdx.x) * 32;
    const int64_t kbeg = static_cast<int64_t>(blockIdx.y) * k_range;
    const int64_t kend = min(K, kbeg + k_range);
    const int64_t span = ((kend - kbeg) + skinny_rows::STEP - 1) / skinny_rows::STEP * skinny_rows::STEP;

    // A[0..MT) x [kbeg, kbeg+span) into smem, zero beyond M rows / K
    uint8_t* a_s = sm;
    for (int64_t i = tid; i < static_cast<int64_t>(MT) * span; i += skinny_rows::THREADS) {
        const int64_t r = i / span, k = kbeg + (i - r * span);
        a_s[i] = (r < M && k < kend) ? A[r * lda + k] : 0;
    }
    __syncthreads();

    const int64_t n = n0 + lane;
    const uint8_t* brow = reinterpret_cast<const uint8_t*>(B) + n * ldb;
    int32_t acc[MT];
#pragma unroll
    for (int m = 0; m < MT; ++m) acc[m] = 0;

    const int64_t steps = span / skinny_rows::STEP;
#pragma unroll 2
    for (int64_t s = warp; s < steps; s += skinny_rows::WARPS) {
        const int64_t off = s * skinny_rows::STEP;  // within the CTA's K range
        const int64_t k = kbeg + off;
        uint32_t bw[8];
        if (n < N && b_vec_ok && k + 32 <= kend) {
            const uint4* p = reinterpret_cast<const uint4*>(brow + k);
            uint4 v0, v1;
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v0.x), "=r"(v0.y), "=r"(v0.z), "=r"(v0.w) : "l"(p));
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v1.x), "=r"(v1.y), "=r"(v1.z), "=r"(v1.w) : "l"(p + 1));
            bw[0] = v0.x; bw[1] = v0.y; bw[2] = v0.z; bw[3] = v0.w;
            bw[4] = v1.x; bw[5] = v1.y; bw[6] = v1.z; bw[7] = v1.w;
        } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) bw[q] = 0;
            if (n < N) {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    if (k + i < kend) bw[i >> 2] |= static_cast<uint32_t>(__ldg(brow + k + i)) << (8 * (i & 3));
            }
        }
#pragma unroll
        for (int m = 0; m < MT; ++m) {
            const uint4 a0 = *reinterpret_cast<const uint4*>(a_s + m * span + off);       // broadcast
            const uint4 a1 = *reinterpret_cast<const uint4*>(a_s + m * span + off + 16);  // broadcast
            const uint32_t aw[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            int32_t sacc = acc[m];
            if constexpr (MODE == 1) {
#pragma unroll
                for (int q = 0; q < 8; ++q) sacc = dp4a_us(aw[q], bw[q], sacc);
            } else {
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    sacc = sat_word_add(aw[q] & 0x0000FFFFu, aw[q] & 0xFFFF0000u, bw[q], sacc);
            }
            acc[m] = sacc;
        }
    }

    // fold the 8 warps' partials: red[w][m][lane]
    __syncthreads();
    int32_t* red = reinterpret_cast<int32_t*>(sm);  // reuse the A staging area (>= 8*MT*32*4 bytes)
#pragma unroll
    for (int m = 0; m < MT; ++m) red[(warp * MT + m) * 32 + lane] = acc[m];
    __syncthreads();
    for (int i = tid; i < MT * 32; i += skinny_rows::THREADS) {
        const int m = i >> 5, l = i & 31;
        uint32_t s = 0;
#pragma unroll
        for (int w = 0; w < skinny_rows::WARPS; ++w) s += static_cast<uint32_t>(red[(w * MT + m) * 32 + l]);
        const int64_t nn = n0 + l;
        if (m < M && nn < N) {
            int32_t* dst = C + static_cast<int64_t>(m) * ldc + nn;
            if (accumulate) atomicAdd(reinterpret_cast<unsigned int*>(dst), s);
            else *dst = static_cast<int32_t>(s);
        }
    }
}

}  // namespace ngemm_dev

namespace ngemm_dev {

// ---------------------------------------------------------------------------------------------
// skinny_mma_kernel — exact-mode skinny GEMM (M <= 16) as a pure load stream.  Each warp owns 16
// rows of B and one K slice; every thread keeps 16-byte loads of B in flight and feeds warp-level
// integer MMAs (mma.sync m16n8k32 u8 x s8 -> s32: B rows as the MMA's M, the <= 16 rows of A,
// broadcast from shared memory, as its N).  No TMEM, TMA descriptors, mbarriers or clusters —
// for a 0.6-4.5 MB operand the kernel's latency chain, not the math, is the cost (see
// scripts/probes/floor.cu: a bare 4 MB load stream takes ~2 us).  Because the dot product is
// order independent mod 2^32, the K bytes of a 128-byte chunk are assigned to MMA k-groups by
// thread (t owns bytes [t*16, t*16+16) and [64 + t*16, 64 + t*16 + 16)) — the SAME mapping for
// A and B — so every B load is a full 16-byte vector.  The CTA's warps split K and meet once in
// shared memory; grid K splits (if any) wrap-add into a zeroed C.
// ---------------------------------------------------------------------------------------------
namespace skinny_mma {
constexpr int CHUNK = 128;  // bytes of K per warp step
}  // namespace skinny_mma

// Tail of a 16-byte operand read (fewer than 16 bytes left in the K range, or an operand that
// is not 16-byte aligned): byte loads, zero fill; a rolled loop keeps the kernels' code small.
__device__ __forceinline__ uint4 load16_tail(const uint8_t* p, int64_t avail) {
    uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll 1
    for (int i = 0; i < 16 && i < avail; ++i) w[i >> 2] |= static_cast<uint32_t>(__ldg(p + i)) << (8 * (i & 3));
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// 16 bytes of an operand row at p; avail = bytes of the row left in the K range (<= 0: zero).
// STREAM: B (read once, bypass L1); else A (re-read by every warp, via L1).
template <bool STREAM>
__device__ __forceinline__ uint4 load16_row(const uint8_t* p, int64_t avail, bool vec) {
    uint4 v = make_uint4(0, 0, 0, 0);
    if (avail <= 0) return v;
    if (vec && avail >= 16) {
        if constexpr (STREAM)
            asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"  // read-only for the kernel
                : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
        else
            v = __ldg(reinterpret_cast<const uint4*>(p));
        return v;
    }
    return load16_tail(p, avail);
}

__device__ __forceinline__ void mma_u8s8_m16n8k32(int32_t (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                                  uint32_t a3, uint32_t b0, uint32_t b1) {
    // A operand (row-major 16x32) signed: B's rows; B operand (col-major 32x8) unsigned: A's rows.
    // not volatile: lets the compiler hoist the next chunk's loads above these MMAs
    asm(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// WARPS per CTA (8/16/32); RG: 16-row groups per CTA; KS = WARPS / RG warps split the CTA's
// K range.  MT: 8 or 16.
// A (<= 16 rows) is read straight through L1 (every warp of the CTA re-reads the same few KB),
// so the kernel's first instructions are the B loads: no staging pass, no block barrier before
// the stream starts.
template <int MT, int RG, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    skinny_mma_kernel(const uint8_t* __restrict__ A, int64_t lda, const int8_t* __restrict__ B, int64_t ldb,
                      int32_t* __restrict__ C, int64_t ldc, int M, int64_t N, int64_t K, int64_t k_range,
                      int vec_ok, int accumulate, int64_t batch_sa, int64_t batch_sb, int64_t batch_sc, Requant rq) {
    constexpr int KS = WARPS / RG;
    constexpr int NB = MT / 8;  // n8 blocks of A rows
    __shared__ __align__(16) int32_t red[WARPS * 16 * MT];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    SKINNY_TRACE_AT(0);
    pdl_launch_dependents();
    // strided batch: blockIdx.z selects one of several independent GEMMs of the same shape
    A += blockIdx.z * batch_sa;
    B += blockIdx.z * batch_sb;
    C += blockIdx.z * batch_sc;
    const int64_t kbeg = static_cast<int64_t>(blockIdx.y) * k_range;
    const int64_t kend = min(K, kbeg + k_range);
    if (vec_ok & 2) {
        // warm L2 with this CTA's B rows (and A) while the preceding grid drains: the HBM fetch
        // overlaps its tail instead of starting after it (see prefetch_l2_bulk)
        const uint32_t span = static_cast<uint32_t>((kend - kbeg) & ~int64_t(15));
        const int64_t nrow = static_cast<int64_t>(blockIdx.x) * RG * 16 + tid;
        if (span != 0) {
            if (tid < RG * 16) {
                if (nrow < N) prefetch_l2_bulk(reinterpret_cast<const uint8_t*>(B) + nrow * ldb + kbeg, span);
            } else if (tid < RG * 16 + M) {
                prefetch_l2_bulk(A + (tid - RG * 16) * lda + kbeg, span);
            }
        }
    }
    pdl_wait();
    SKINNY_TRACE_AT(1);
    const int rg = warp / KS, ks = warp % KS;
    const int64_t n0 = (static_cast<int64_t>(blockIdx.x) * RG + rg) * 16;
    const uint8_t* Bu = reinterpret_cast<const uint8_t*>(B);

    // per-thread operand rows: B rows n0+g and n0+g+8, A rows nb*8+g; thread t reads bytes
    // [c*64 + t*16, +16) of each 128-byte chunk (rows outside the matrix read as zeros)
    const bool vec = vec_ok != 0;
    const int64_t kt = kbeg + t * 16;
    const int64_t rem = kend - kt;  // bytes of the K range left from this thread's first byte
    const uint8_t* pb = Bu + (n0 + g) * ldb + kt;
    const uint8_t* pa = A + g * lda + kt;
    const bool ok_b0 = n0 + g < N, ok_b1 = n0 + g + 8 < N;
    // B rows (g, g+8) x halves c; A rows (nb*8 + g) x halves c
    auto load_chunk = [&](int64_t ch, uint4 (&bv)[2][2], uint4 (&av)[NB][2]) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int64_t o = ch * skinny_mma::CHUNK + c * 64;
            bv[0][c] = load16_row<true>(pb + o, ok_b0 ? rem - o : 0, vec);
            bv[1][c] = load16_row<true>(pb + 8 * ldb + o, ok_b1 ? rem - o : 0, vec);
#pragma unroll
            for (int nb = 0; nb < NB; ++nb)
                av[nb][c] = load16_row<false>(pa + nb * 8 * lda + o, (nb * 8 + g < M) ? rem - o : 0, vec);
        }
    };

    int32_t d[NB][4];
#pragma unroll
    for (int j = 0; j < NB; ++j) d[j][0] = d[j][1] = d[j][2] = d[j][3] = 0;
    auto compute = [&](const uint4 (&bv)[2][2], const uint4 (&av)[NB][2]) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const uint32_t ba[4] = {bv[0][c].x, bv[0][c].y, bv[0][c].z, bv[0][c].w};
            const uint32_t bb[4] = {bv[1][c].x, bv[1][c].y, bv[1][c].z, bv[1][c].w};
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) {
                const uint32_t aa[4] = {av[nb][c].x, av[nb][c].y, av[nb][c].z, av[nb][c].w};
#pragma unroll
                for (int j = 0; j < 2; ++j)
                    mma_u8s8_m16n8k32(d[nb], ba[2 * j], bb[2 * j], ba[2 * j + 1], bb[2 * j + 1], aa[2 * j],
                                      aa[2 * j + 1]);
            }
        }
    };

    // whole chunks with both B rows in range (warp-uniform): unconditional 16-byte loads; A rows
    // past M read row 0 and are zeroed by a select (no branch)
    auto load_chunk_fast = [&](int64_t ch, uint4 (&bv)[2][2], uint4 (&av)[NB][2]) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int64_t o = ch * skinny_mma::CHUNK + c * 64;
            bv[0][c] = load16_row<true>(pb + o, 16, true);
            bv[1][c] = load16_row<true>(pb + 8 * ldb + o, 16, true);
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) {
                const bool ok = nb * 8 + g < M;
                const uint4 v = __ldg(reinterpret_cast<const uint4*>((ok ? pa + nb * 8 * lda : A + kt) + o));
                av[nb][c] = ok ? v : make_uint4(0, 0, 0, 0);
            }
        }
    };

    const int64_t chunks = (kend - kbeg + skinny_mma::CHUNK - 1) / skinny_mma::CHUNK;
    const int64_t fast_chunks = ((vec_ok & 4) && n0 + 16 <= N) ? (kend - kbeg) / skinny_mma::CHUNK : 0;
#pragma unroll 4
    for (int64_t ch = ks; ch < chunks; ch += KS) {
        uint4 bv[2][2], av[NB][2];
        if (ch < fast_chunks) load_chunk_fast(ch, bv, av);
        else load_chunk(ch, bv, av);
        compute(bv, av);
    }

    SKINNY_TRACE_AT(2);
    // meet the KS warps of this row group in smem: red[rg][ks][16 rows][MT cols]
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
        const int col = nb * 8 + t * 2;
        int32_t* r0 = red + ((rg * KS + ks) * 16 + g) * MT + col;
        int32_t* r8 = red + ((rg * KS + ks) * 16 + g + 8) * MT + col;
        r0[0] = d[nb][0];
        r0[1] = d[nb][1];
        r8[0] = d[nb][2];
        r8[1] = d[nb][3];
    }
    __syncthreads();
    SKINNY_TRACE_AT(3);
    // accumulate == 2 (RG = 1): the grid's K splits of a row group form one thread-block cluster
    // along y; every rank publishes its 16 x MT partial sums in shared memory and rank r adds up and
    // stores the outputs i with i % splits == r through DSMEM — no zeroing pass, no atomics
    __shared__ int32_t xsum[RG == 1 ? 16 * MT : 1];
    const bool xred = RG == 1 && accumulate == 2;
    const uint32_t nsplit = gridDim.y, xrank = blockIdx.y;
    if (xred) {
        for (int i = tid; i < 16 * MT; i += WARPS * 32) {
            const int m = i / 16, row = i % 16;
            uint32_t s = 0;
#pragma unroll
            for (int q = 0; q < KS; ++q) s += static_cast<uint32_t>(red[(q * 16 + row) * MT + m]);
            xsum[i] = static_cast<int32_t>(s);
        }
        cluster_sync();
    }
    for (int i = tid; i < RG * 16 * MT; i += WARPS * 32) {
        const int m = i / (RG * 16), rr = i % (RG * 16);  // consecutive threads -> consecutive n
        const int r_g = rr / 16, row = rr % 16;
        uint32_t s = 0;
        if (xred) {
            if (static_cast<uint32_t>(i) % nsplit != xrank) continue;
            for (uint32_t q = 0; q < nsplit; ++q) s += dsmem_ld_u32(smem_u32(&xsum[i]), q);
        } else {
#pragma unroll
            for (int q = 0; q < KS; ++q) s += static_cast<uint32_t>(red[((r_g * KS + q) * 16 + row) * MT + m]);
        }
        const int64_t n = (static_cast<int64_t>(blockIdx.x) * RG + r_g) * 16 + row;
        if (m < M && n < N) {
            if (rq.out != nullptr) {  // fused requantisation (single K split only)
                rq.out[static_cast<int64_t>(m) * rq.ldo + n] = requant_s8(s, rq.bias ? rq.bias[n] : 0, rq.scale[n], rq.zp);
                continue;
            }
            int32_t* dst = C + static_cast<int64_t>(m) * ldc + n;
            if (accumulate == 1) atomicAdd(reinterpret_cast<unsigned int*>(dst), s);
            else *dst = static_cast<int32_t>(s);
        }
    }
    if (xred) cluster_sync();  // peers may still be reading this CTA's partial sums
    SKINNY_TRACE_AT(4);
    SKINNY_TRACE_END();
}

}  // namespace ngemm_dev

namespace ngemm_dev {

// ---------------------------------------------------------------------------------------------
// skinny_sat_kernel — HardwareSaturating skinny GEMM (M <= 16) with the load-stream layout of
// skinny_mma_kernel: each warp owns 16 rows of B (lane g of each quad on rows g and g+8) and a K
// slice; thread t of a quad reads bytes [c*64 + t*16, +16) of each 128-byte chunk (c = 0, 1),
// so every load is a 16-byte vector and pair boundaries stay even-aligned.  A (<= 16 rows) comes
// through L1.  Per 4-byte K word: 2 IDP.4A on the masked A halves, each pair sum clamped to
// int16, wrap-added (accumulated on the FMA pipe).  The quad's four K phases fold with two
// shuffle levels (transposing, so each lane keeps 1/4 of the values), the CTA's warps meet in
// shared memory.
// ---------------------------------------------------------------------------------------------
// Register caps for the 8-warp CTAs: the B-mask form at <= 128 so two CTAs fit per SM (at 133
// registers one CTA per SM made 16x4096x1024 13.1 us instead of 7.9), the A-mask form at <= 85
// so three fit, <= 64 for MT <= 4 so four fit (batches are occupancy-bound: 95 registers / two
// CTAs cost 26 % at 16x4096x1024 x 128; profiles/r2/batched_ab_r2.log)
template <int MT, int WARPS, bool MSPLIT, bool BMASK>
__global__ void __launch_bounds__(WARPS * 32, WARPS == 8 ? (BMASK ? 2 : (MT <= 4 ? 4 : 3)) : 1)
    skinny_sat_kernel(const uint8_t* __restrict__ A, int64_t lda, const int8_t* __restrict__ B, int64_t ldb,
                      int32_t* __restrict__ C, int64_t ldc, int M, int64_t N, int64_t K, int64_t k_range, int vec_ok,
                      int accumulate, int64_t batch_sa, int64_t batch_sb, int64_t batch_sc) {
    // MSPLIT: the CTA's warps split A's rows (MS groups of MW <= 4 rows) as well as K (KS warps
    // per row group), so each warp keeps 2 x MW accumulators and a short unrolled body (its MS - 1
    // siblings re-read the same B bytes through L1).  It pays when N has few 16-row groups (one
    // warp per K slice leaves SMs idle and its ~1000-instruction body misses the instruction
    // cache: 35 % no_instruction stalls, profiles/r2/stalls_c2_sat_r2.txt); with many row groups
    // the 4x B reads cost more (profiles/r2/skinny_sat_r2.log).
    constexpr int MW = (MSPLIT && MT > 4) ? 4 : MT, MS = MT / MW, KS = WARPS / MS;
    static_assert(MT % MW == 0 && WARPS % MS == 0, "warps must split the row groups evenly");
    constexpr int V = 2 * MW;  // values per thread: rows {g, g+8} x MW
    __shared__ __align__(16) int32_t red[KS * 16 * MT];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int warp_m = warp % MS, warp_k = warp / MS, mb = warp_m * MW;
    pdl_launch_dependents();
    A += blockIdx.z * batch_sa;  // strided batch (blockIdx.z), as in skinny_mma_kernel
    B += blockIdx.z * batch_sb;
    C += blockIdx.z * batch_sc;
    const int64_t n0 = static_cast<int64_t>(blockIdx.x) * 16;
    if (vec_ok & 2) {  // warm L2 before the dependency wait, as in skinny_mma_kernel
        const int64_t kb = static_cast<int64_t>(blockIdx.y) * k_range;
        const uint32_t span = static_cast<uint32_t>((min(K, kb + k_range) - kb) & ~int64_t(15));
        if (span != 0 && kb < K) {
            if (tid < 16) {
                if (n0 + tid < N) prefetch_l2_bulk(reinterpret_cast<const uint8_t*>(B) + (n0 + tid) * ldb + kb, span);
            } else if (tid < 16 + M) {
                prefetch_l2_bulk(A + (tid - 16) * lda + kb, span);
            }
        }
    }
    pdl_wait();
    const uint8_t* Bu = reinterpret_cast<const uint8_t*>(B);

    int32_t acc[V];
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] = 0;
    // The pair masks go on B (once per chunk, shared by all M rows of A): for a K word with
    // bytes b0..b3, blo = b & 0xFFFF and bhi = b & 0xFFFF0000, so dp4a(a, blo) = a0 b0 + a1 b1 and
    // dp4a(a, bhi) = a2 b2 + a3 b3 — the same two pair sums as masking A, one LOP per B word
    // instead of one per (A word, B row).  Then one I2IP.SAT packs both clamped sums and one
    // IDP.2A wrap-adds them (sat_word_add's last two steps).
    auto sat_pairs_add = [](uint32_t a, uint32_t blo, uint32_t bhi, int32_t acc_in) {
        const int32_t p0 = dp4a_us(a, blo, 0);
        const int32_t p1 = dp4a_us(a, bhi, 0);
        uint32_t packed;
        asm("cvt.pack.sat.s16.s32 %0, %1, %2;" : "=r"(packed) : "r"(p1), "r"(p0));
        int32_t r;
        asm("dp2a.lo.s32.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(packed), "r"(0x0101), "r"(acc_in));
        return r;
    };

    const int64_t kbeg = static_cast<int64_t>(blockIdx.y) * k_range;
    const int64_t kend = min(K, kbeg + k_range);
    const int64_t chunks = (kend - kbeg + 127) / 128;
    const bool vec = vec_ok != 0, rows_full = n0 + 16 <= N;
    const uint8_t* pb = Bu + (n0 + g) * ldb + t * 16;  // thread t reads bytes [c*64 + t*16, +16) of a chunk
    const uint8_t* pa = A + t * 16;
    // one chunk: B words (2 rows x 2 halves x 4 words) masked once, then every A row against them;
    // `lb` / `la` load 16 bytes of B / A (unconditional on the fast path, bounded on the ragged one)
    auto chunk = [&](int64_t k0, auto lb, auto la) {
        if constexpr (!BMASK) {
            // mask A instead (two LOPs per A word, shared by the two B rows) and keep B raw: 16
            // fewer live registers — for one A row, 32-warp CTAs (64 registers), and batches, whose
            // throughput depends on occupancy more than on the instruction count
            // (profiles/r2/batched_ab_r2.log: 123 vs 80 registers cost 26 % at 16x4096x1024 x 128)
            uint4 bv[2][2];
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
                for (int r = 0; r < 2; ++r) bv[r][c] = lb(r, c);
#pragma unroll
            for (int mm = 0; mm < MW; ++mm) {
                if (mb + mm >= M) break;  // uniform
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const uint4 av = la(mb + mm, c);
                    const uint32_t aw[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
                    for (int r = 0; r < 2; ++r) {
                        const uint32_t bw[4] = {bv[r][c].x, bv[r][c].y, bv[r][c].z, bv[r][c].w};
                        int32_t sacc = acc[r * MW + mm];
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            sacc = sat_word_add(aw[q] & 0x0000FFFFu, aw[q] & 0xFFFF0000u, bw[q], sacc);
                        acc[r * MW + mm] = sacc;
                    }
                }
            }
        } else {
        uint32_t blo[2][2][4], bhi[2][2][4];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const uint4 bv = lb(r, c);
                const uint32_t w[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    blo[r][c][q] = w[q] & 0x0000FFFFu;
                    bhi[r][c][q] = w[q] & 0xFFFF0000u;
                }
            }
        }
#pragma unroll
        for (int mm = 0; mm < MW; ++mm) {
            if (mb + mm >= M) break;  // uniform
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const uint4 av = la(mb + mm, c);
                const uint32_t aw[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    int32_t sacc = acc[r * MW + mm];
#pragma unroll
                    for (int q = 0; q < 4; ++q) sacc = sat_pairs_add(aw[q], blo[r][c][q], bhi[r][c][q], sacc);
                    acc[r * MW + mm] = sacc;
                }
            }
        }
        }  // B-side masks
    };
#pragma unroll 1
    for (int64_t ch = warp_k; ch < chunks && mb < M; ch += KS) {
        const int64_t k0 = kbeg + ch * 128;  // k_range is a multiple of 128: pairs stay even-aligned
        if ((vec_ok & 4) && rows_full && k0 + 128 <= kend) {
            // whole chunk in range (warp-uniform): unconditional 16-byte loads (through L1 when
            // sibling warps of other row groups read the same B bytes)
            chunk(k0,
                  [&](int r, int c) { return load16_row<MS == 1>(pb + r * 8 * ldb + k0 + c * 64, 16, true); },
                  [&](int m, int c) { return __ldg(reinterpret_cast<const uint4*>(pa + m * lda + k0 + c * 64)); });
        } else {
            // ragged chunk (K tail, last row group, unaligned operands): bounded loads, zero fill
            chunk(k0,
                  [&](int r, int c) {
                      return load16_row<MS == 1>(pb + r * 8 * ldb + k0 + c * 64,
                                                 (n0 + g + 8 * r < N) ? kend - (k0 + c * 64 + t * 16) : 0, vec);
                  },
                  [&](int m, int c) {
                      return load16_row<false>(pa + m * lda + k0 + c * 64, kend - (k0 + c * 64 + t * 16), vec);
                  });
        }
    }
    // fold the quad's 4 K phases: after offsets 1 and 2 each lane holds V/4 totals
    int base = 0;
    {
        const bool up = (t & 1) != 0;
#pragma unroll
        for (int i = 0; i < V / 2; ++i) {
            const int32_t keep = up ? acc[i + V / 2] : acc[i], send = up ? acc[i] : acc[i + V / 2];
            acc[i] = static_cast<int32_t>(static_cast<uint32_t>(keep) +
                                          static_cast<uint32_t>(__shfl_xor_sync(0xffffffffu, send, 1)));
        }
        if (up) base += V / 2;
        if constexpr (V >= 4) {
            const bool up2 = (t & 2) != 0;
#pragma unroll
            for (int i = 0; i < V / 4; ++i) {
                const int32_t keep = up2 ? acc[i + V / 4] : acc[i], send = up2 ? acc[i] : acc[i + V / 4];
                acc[i] = static_cast<int32_t>(static_cast<uint32_t>(keep) +
                                              static_cast<uint32_t>(__shfl_xor_sync(0xffffffffu, send, 2)));
            }
            if (up2) base += V / 4;
        } else {
            acc[0] = static_cast<int32_t>(static_cast<uint32_t>(acc[0]) +
                                          static_cast<uint32_t>(__shfl_xor_sync(0xffffffffu, acc[0], 2)));
        }
    }
    // lane (g, t) now holds values base .. base + LEFT - 1 of the index space r * MW + mm
    constexpr int LEFT = V >= 4 ? V / 4 : 1;
    if (V >= 4 || (t & 2) == 0) {
#pragma unroll
        for (int i = 0; i < LEFT; ++i) {
            const int idx = base + i, r = idx / MW, m = mb + idx - r * MW;
            red[(warp_k * 16 + g + 8 * r) * MT + m] = acc[i];
        }
    }
    __syncthreads();
    for (int i = tid; i < 16 * MT; i += WARPS * 32) {
        const int m = i / 16, row = i % 16;
        uint32_t s = 0;
#pragma unroll
        for (int w = 0; w < KS; ++w) s += static_cast<uint32_t>(red[(w * 16 + row) * MT + m]);
        const int64_t n = n0 + row;
        if (m < M && n < N) {
            int32_t* dst = C + static_cast<int64_t>(m) * ldc + n;
            if (accumulate) atomicAdd(reinterpret_cast<unsigned int*>(dst), s);
            else *dst = static_cast<int32_t>(s);
        }
    }
}

}  // namespace ngemm_dev

namespace ngemm_dev {

// ---------------------------------------------------------------------------------------------
// skinny_sathyb_kernel — HardwareSaturating skinny GEMM (4 < M <= 16) on the warp-level tensor
// cores plus a sparse fix, the M <= 16 counterpart of kernel_satfix.cuh.
//
// A is unsigned (<= 255), so a pair (b0, b1) of B can only clamp when both bytes have the same
// sign and |b0 + b1| >= 129: with opposite signs (or a zero) the pair sum stays inside
// [255 * -128, 255 * 127]; with equal signs its extreme is 255 * (b0 + b1), and 255 * 128 = 32640
// still fits int16.  Every other pair contributes its exact product, so
//     C_sat = A . B (exact, mma.sync as in skinny_mma_kernel) + sum over listed pairs of (sat16(s) - s).
// The load stream and fragment mapping are skinny_mma_kernel's.  Per 128-byte chunk each lane
// tests its 16 B words (two dp4a against 0x0101 give b0 + b1 + 128 and b2 + b3 + 128; one unsigned
// compare each), the warp counts the listed words (redux) and takes one of two warp-uniform paths:
//   sparse (<= QCAP listed words; weight-like B, sigma = 32: ~4 of 512): the exact MMAs, then the
//       listed words go to a per-warp queue in shared memory and (word, A row) units are spread
//       over the lanes — each adds its correction to corr[row][m] (shared-memory atomic, only when
//       a pair really clamps);
//   dense (uniform int8 B: ~44 % of the words): no MMA; the chunk's saturating sums are computed
//       with the dp4a / cvt.pack.sat / dp2a step of skinny_sat_kernel, one A row at a time (rolled
//       loop), into this lane's private cells of part[warp][t][row][m].
// At the end every lane adds its MMA fragment into its own part cells as well, and the CTA sums
// part over warps and K phases plus corr.  All terms wrap mod 2^32, so the result is bit-exact.
// ---------------------------------------------------------------------------------------------
namespace skinny_sathyb {
constexpr int QCAP = 128;  // queue entries per warp; more listed words than this -> dense path
template <int MT, int WARPS>
struct Smem {
    static constexpr int PART = WARPS * 4 * 16 * MT * 4;  // [warp][t][row][m] int32
    static constexpr int QUEUE = WARPS * QCAP * 8;        // [warp][entry]{word, meta}
    static constexpr int CORR = 16 * MT * 4;              // [row][m]
    static constexpr int TOTAL = PART + QUEUE + CORR + 16;  // + the "a warp took the dense path" flag
};
}  // namespace skinny_sathyb

template <int MT, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, WARPS == 8 ? 2 : 1)
    skinny_sathyb_kernel(const uint8_t* __restrict__ A, int64_t lda, const int8_t* __restrict__ B, int64_t ldb,
                         int32_t* __restrict__ C, int64_t ldc, int M, int64_t N, int64_t K, int64_t k_range,
                         int vec_ok, int accumulate, int64_t batch_sa, int64_t batch_sb, int64_t batch_sc) {
    using S = skinny_sathyb::Smem<MT, WARPS>;
    constexpr int NB = MT / 8;
    constexpr int QCAP = skinny_sathyb::QCAP;
    extern __shared__ __align__(16) uint8_t sathyb_smem[];
    int32_t* part = reinterpret_cast<int32_t*>(sathyb_smem);
    uint2* queue = reinterpret_cast<uint2*>(sathyb_smem + S::PART);
    int32_t* corr = reinterpret_cast<int32_t*>(sathyb_smem + S::PART + S::QUEUE);
    // bit w set: warp w took the dense path and wrote all of its part cells (else only its MMA
    // fragment's cells are valid)
    unsigned* dense_mask = reinterpret_cast<unsigned*>(sathyb_smem + S::PART + S::QUEUE + S::CORR);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    pdl_launch_dependents();
    A += blockIdx.z * batch_sa;
    B += blockIdx.z * batch_sb;
    C += blockIdx.z * batch_sc;
    const int64_t kbeg = static_cast<int64_t>(blockIdx.y) * k_range;
    const int64_t kend = min(K, kbeg + k_range);
    const int64_t n0 = static_cast<int64_t>(blockIdx.x) * 16;
    if (vec_ok & 2) {  // warm L2 before the dependency wait, as in skinny_mma_kernel
        const uint32_t span = static_cast<uint32_t>((kend - kbeg) & ~int64_t(15));
        if (span != 0) {
            if (tid < 16) {
                if (n0 + tid < N) prefetch_l2_bulk(reinterpret_cast<const uint8_t*>(B) + (n0 + tid) * ldb + kbeg, span);
            } else if (tid < 16 + M) {
                prefetch_l2_bulk(A + (tid - 16) * lda + kbeg, span);
            }
        }
    }
    // this lane's private cells part[warp][t][g + 8r][m], and the shared corrections
    int32_t* my_part = part + ((warp * 4 + t) * 16 + g) * MT;
    for (int i = tid; i < 16 * MT; i += WARPS * 32) corr[i] = 0;
    if (tid == 0) *dense_mask = 0;
    __syncthreads();
    pdl_wait();
    const uint8_t* Bu = reinterpret_cast<const uint8_t*>(B);
    const bool vec = vec_ok != 0;
    const int64_t kt = kbeg + t * 16;
    const int64_t rem = kend - kt;
    const uint8_t* pb = Bu + (n0 + g) * ldb + kt;
    const uint8_t* pb8 = pb + 8 * ldb;
    const bool ok_b0 = n0 + g < N, ok_b1 = n0 + g + 8 < N;
    const uint8_t* pa_frag[NB];  // A rows nb*8 + g (row 0 stands in for rows past M; zeroed by a_ok)
    bool a_ok[NB];
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
        a_ok[nb] = nb * 8 + g < M;
        pa_frag[nb] = A + static_cast<int64_t>(a_ok[nb] ? nb * 8 + g : 0) * lda + kt;
    }
    // flush: lane l always handles A row l % 16 (units are entry * 16 + row, 32 lanes per step)
    const uint8_t* pa_fix = A + static_cast<int64_t>(lane & 15) * lda + kbeg;
    const bool fix_row_ok = (lane & 15) < M;
    uint2* my_queue = queue + warp * QCAP;

    int32_t d[NB][4];
#pragma unroll
    for (int j = 0; j < NB; ++j) d[j][0] = d[j][1] = d[j][2] = d[j][3] = 0;
    int32_t dacc[2][MT];  // dense path: rows {g, g+8} x A rows, this lane's K phase
#pragma unroll
    for (int m = 0; m < MT; ++m) dacc[0][m] = dacc[1][m] = 0;
    bool used_dense = false;

    // 16 bytes of A row m at this lane's K phase of chunk offset o (zero past the K range)
    auto load_a = [&](int m, int64_t o, bool fast) {
        const uint8_t* p = A + static_cast<int64_t>(m) * lda + kt + o;
        if (fast) return __ldg(reinterpret_cast<const uint4*>(p));
        return load16_row<false>(p, rem - o, vec);
    };

    const int64_t chunks = (kend - kbeg + skinny_mma::CHUNK - 1) / skinny_mma::CHUNK;
    const int64_t fast_chunks = ((vec_ok & 4) && n0 + 16 <= N) ? (kend - kbeg) / skinny_mma::CHUNK : 0;
#pragma unroll 1
    for (int64_t ch = warp; ch < chunks; ch += WARPS) {
        const bool fast = ch < fast_chunks;  // warp-uniform
        uint32_t bw[2][2][4];                // [row g / g+8][half c][word]
        uint4 av[NB][2];                     // the MMA's A-row fragments travel with the B loads
        const uint32_t o0 = static_cast<uint32_t>(ch) * skinny_mma::CHUNK;
        if (fast) {
            // whole chunk in range and 16-byte aligned: eight plain vector loads
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const uint4 v0 = load16_row<true>(pb + o0 + c * 64, 16, true);
                const uint4 v1 = load16_row<true>(pb8 + o0 + c * 64, 16, true);
                bw[0][c][0] = v0.x; bw[0][c][1] = v0.y; bw[0][c][2] = v0.z; bw[0][c][3] = v0.w;
                bw[1][c][0] = v1.x; bw[1][c][1] = v1.y; bw[1][c][2] = v1.z; bw[1][c][3] = v1.w;
#pragma unroll
                for (int nb = 0; nb < NB; ++nb) {
                    const uint4 v = __ldg(reinterpret_cast<const uint4*>(pa_frag[nb] + o0 + c * 64));
                    av[nb][c] = a_ok[nb] ? v : make_uint4(0, 0, 0, 0);
                }
            }
        } else {
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int64_t o = static_cast<int64_t>(o0) + c * 64;
                const uint4 v0 = load16_row<true>(pb + o, ok_b0 ? rem - o : 0, vec);
                const uint4 v1 = load16_row<true>(pb8 + o, ok_b1 ? rem - o : 0, vec);
                bw[0][c][0] = v0.x; bw[0][c][1] = v0.y; bw[0][c][2] = v0.z; bw[0][c][3] = v0.w;
                bw[1][c][0] = v1.x; bw[1][c][1] = v1.y; bw[1][c][2] = v1.z; bw[1][c][3] = v1.w;
#pragma unroll
                for (int nb = 0; nb < NB; ++nb)
                    av[nb][c] = load16_row<false>(pa_frag[nb] + o, a_ok[nb] ? rem - o : 0, vec);
            }
        }
        // listed words: a pair can clamp iff |b0 + b1| >= 129  <=>  unsigned(b0 + b1 + 128) > 256
        uint32_t listed = 0;
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t s0 = static_cast<uint32_t>(dp4a_ss(bw[r][c][q], 0x00000101u, 128));
                    const uint32_t s1 = static_cast<uint32_t>(dp4a_ss(bw[r][c][q], 0x01010000u, 128));
                    if (s0 > 256u || s1 > 256u) listed |= 1u << (r * 8 + c * 4 + q);
                }
        const int mine = __popc(listed);
        const int total = __reduce_add_sync(0xffffffffu, mine);
        if (total > QCAP) {
            // ---- dense: the chunk's saturating sums for every A row, accumulated in registers
            // (A-side pair masks: two LOPs per A word shared by both B rows, as in skinny_sat_kernel;
            // an out-of-line version kept the sparse path's registers lower but ran 1.6x slower)
            used_dense = true;
#pragma unroll
            for (int m = 0; m < MT; ++m) {
                if (m >= M) break;  // uniform
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const uint4 am = load_a(m, ch * skinny_mma::CHUNK + c * 64, fast);
                    const uint32_t aw[4] = {am.x, am.y, am.z, am.w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint32_t alo = aw[q] & 0x0000FFFFu, ahi = aw[q] & 0xFFFF0000u;
                        dacc[0][m] = sat_word_add(alo, ahi, bw[0][c][q], dacc[0][m]);
                        dacc[1][m] = sat_word_add(alo, ahi, bw[1][c][q], dacc[1][m]);
                    }
                }
            }
            continue;
        }
        // ---- sparse: exact MMAs on everything ...
#pragma unroll
        for (int c = 0; c < 2; ++c) {
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) {
                const uint32_t aa[4] = {av[nb][c].x, av[nb][c].y, av[nb][c].z, av[nb][c].w};
#pragma unroll
                for (int j = 0; j < 2; ++j)
                    mma_u8s8_m16n8k32(d[nb], bw[0][c][2 * j], bw[1][c][2 * j], bw[0][c][2 * j + 1], bw[1][c][2 * j + 1],
                                      aa[2 * j], aa[2 * j + 1]);
            }
        }
        if (total == 0) continue;
        // ... then the listed words: queue them (exclusive scan of the lanes' counts; a lane has
        // none or one or two, so a short loop over its set bits with the word picked by a select
        // tree beats sixteen predicated stores) ...
        int pos = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int up = __shfl_up_sync(0xffffffffu, pos, o);
            if (lane >= o) pos += up;
        }
        pos -= mine;
        for (uint32_t rest = listed; rest != 0; rest &= rest - 1) {
            const int i = __ffs(rest) - 1;  // (r * 8 + c * 4 + q)
            uint32_t w = bw[0][0][0];
#pragma unroll
            for (int j = 1; j < 16; ++j) w = (i == j) ? bw[j >> 3][(j >> 2) & 1][j & 3] : w;
            // meta: K offset of the word inside the CTA's K range, B row of the tile
            const uint32_t koff = o0 + static_cast<uint32_t>(((i >> 2) & 1) * 64 + t * 16 + (i & 3) * 4);
            my_queue[pos++] = make_uint2(w, (koff << 4) | static_cast<uint32_t>(g + (i & 8)));
        }
        __syncwarp();
        // ... and spread (word, A row) units over the lanes: lane l takes A row l % 16 of entries
        // (l / 16) + 2 i, four entries per pass (loads first)
        for (int base = lane >> 4; base < total; base += 8) {
            uint2 e[4];
            uint32_t aw[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int ei = base + 2 * i;
                const bool on = ei < total && fix_row_ok;
                e[i] = on ? my_queue[ei] : make_uint2(0, 0);
                const uint32_t ko = e[i].y >> 4;
                aw[i] = 0;
                if (on) {
                    if (vec && kbeg + ko + 4 <= kend) {
                        aw[i] = __ldg(reinterpret_cast<const uint32_t*>(pa_fix + ko));
                    } else {
                        for (int b4 = 0; b4 < 4; ++b4)
                            if (kbeg + ko + b4 < kend) aw[i] |= static_cast<uint32_t>(__ldg(pa_fix + ko + b4)) << (8 * b4);
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                // entries past the list carry a zero word: their correction is zero
                const int32_t p0 = dp4a_us(aw[i], e[i].x & 0x0000FFFFu, 0), p1 = dp4a_us(aw[i], e[i].x & 0xFFFF0000u, 0);
                const int32_t fix = sat2_add(p0, p1, 0) - (p0 + p1);
                if (fix != 0) atomicAdd(&corr[(e[i].y & 15u) * MT + (lane & 15)], fix);
            }
        }
        __syncwarp();
    }

    // this lane's cells of part: the MMA fragment d[nb] = rows {g, g+8} x A rows nb*8 + 2t, +1 (K-phase
    // plane t of this warp), plus, after a dense chunk, the dense sums of every A row
    if (used_dense) {  // warp-uniform
        if (lane == 0) atomicOr(dense_mask, 1u << warp);  // read after the block-wide barrier below
#pragma unroll
        for (int m = 0; m < MT; ++m) {
            my_part[m] = dacc[0][m];
            my_part[8 * MT + m] = dacc[1][m];
        }
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
            const int col = nb * 8 + t * 2;
            my_part[col] += d[nb][0];
            my_part[col + 1] += d[nb][1];
            my_part[8 * MT + col] += d[nb][2];
            my_part[8 * MT + col + 1] += d[nb][3];
        }
    } else {
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
            const int col = nb * 8 + t * 2;
            *reinterpret_cast<int2*>(my_part + col) = make_int2(d[nb][0], d[nb][1]);
            *reinterpret_cast<int2*>(my_part + 8 * MT + col) = make_int2(d[nb][2], d[nb][3]);
        }
    }
    __syncthreads();
    // accumulate == 2: K splits reduced across a thread-block cluster through DSMEM, as in
    // skinny_mma_kernel (xsum aliases the queue, which is no longer in use)
    int32_t* xsum = reinterpret_cast<int32_t*>(queue);
    const bool xred = accumulate == 2;
    const uint32_t nsplit = gridDim.y, xrank = blockIdx.y;
    for (int pass = 0; pass < (xred ? 2 : 1); ++pass) {
    if (xred && pass == 1) cluster_sync();
    for (int i = tid; i < 16 * MT; i += WARPS * 32) {
        const int m = i / 16, row = i % 16;
        if (xred && pass == 1) {
            if (static_cast<uint32_t>(i) % nsplit != xrank) continue;
            uint32_t t2 = 0;
            for (uint32_t q = 0; q < nsplit; ++q) t2 += dsmem_ld_u32(smem_u32(&xsum[i]), q);
            const int64_t n2 = n0 + row;
            if (m < M && n2 < N) C[static_cast<int64_t>(m) * ldc + n2] = static_cast<int32_t>(t2);
            continue;
        }
        uint32_t s = static_cast<uint32_t>(corr[row * MT + m]);
        const unsigned dm = *dense_mask;
        // a warp without dense chunks holds A row m only in K-phase plane (m % 8) / 2 (its MMA fragment)
#pragma unroll
        for (int w = 0; w < WARPS; ++w) {
            if (dm & (1u << w)) {
#pragma unroll
                for (int q = 0; q < 4; ++q) s += static_cast<uint32_t>(part[((w * 4 + q) * 16 + row) * MT + m]);
            } else {
                s += static_cast<uint32_t>(part[((w * 4 + ((m & 7) >> 1)) * 16 + row) * MT + m]);
            }
        }
        if (xred) {
            xsum[i] = static_cast<int32_t>(s);
            continue;
        }
        const int64_t n = n0 + row;
        if (m < M && n < N) {
            int32_t* dst = C + static_cast<int64_t>(m) * ldc + n;
            if (accumulate == 1) atomicAdd(reinterpret_cast<unsigned int*>(dst), s);
            else *dst = static_cast<int32_t>(s);
        }
    }
    }
    if (xred) cluster_sync();  // peers may still be reading this CTA's partial sums
}

}  // namespace ngemm_dev
