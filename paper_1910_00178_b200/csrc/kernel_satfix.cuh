// kernel_satfix.cuh — HardwareSaturating on the tensor cores plus a sparse CUDA-core fix.
//
// The reference's saturating result is C = sum_j sat16(a[2j]b[2j] + a[2j+1]b[2j+1])
// (gemm_sat_oracle, gemm.hpp:83-104; VPMADDUBSW, simd_native.hpp:144-178).  A is unsigned,
// so for a B pair (b0, b1) the pair sum over all a0, a1 in [0, amax] spans
// [amax*(min(b0,0)+min(b1,0)), amax*(max(b0,0)+max(b1,0))].  When that interval fits int16
// the pair can never clamp and its contribution is the exact a0*b0 + a1*b1 — tensor-core
// work.  Only the remaining "dangerous" pairs (for uniform int8 B about a quarter of them;
// for weight-like B with sigma = 32 about 0.4 %) need the clamp.  So:
//
//   C = A . B_safe          (tcgen05 kind::i8, exact; B_safe = B with dangerous pairs zeroed)
//     + sum over dangerous pairs of sat16(pair sum)   (sat_fix_kernel, CUDA cores)
//
// Both terms wrap mod 2^32 like wrap_add_i32 (common.hpp:132-135), so the split is bit-exact.
// Pairs stay even-aligned in absolute k (chunks of 256 bytes start at multiples of 256).
//
// Tiled operand layouts written by the two prep kernels (so the fix kernel streams whole
// tiles with 1-D bulk copies into a double-buffered shared-memory pipeline):
//   A_pm  [m-tile u][chunk c][pair j < 128][word p < 128]  u32 = (a[r0][2j], a[r0][2j+1],
//          a[r1][2j], a[r1][2j+1]) with p = 4 l + q, r0 = l + 64 q, r1 = r0 + 32: lane l of the
//          fix kernel owns tile rows l + 32 t (t < 8), so one LDS.128 gives a lane pair j of its
//          8 rows and one dp4a against (b0, b1, 0, 0) or (0, 0, b0, b1) is one row's pair sum
//   B_t   [n-tile t][chunk c][row r < 128][256 bytes]   B's bytes, tile by tile
//   L_t   [n-tile t][chunk c]{count[128] u8, list[128][128] u8}   per row, its dangerous pairs
//          in the chunk as B byte offsets 2j (the fix walks these lists)
//   flags [n-tile t][chunk c]                           dangerous pairs in the tile chunk
// Rows past M / N and bytes past K are zero.
#pragma once

#include "kernel_simt.cuh"
#include "ptx.cuh"

namespace ngemm_dev {

namespace satfix {
constexpr int CHUNK = 256;           // K bytes per chunk (128 pairs = 4 mask words per row)
constexpr int TM = 256;              // A rows per tile (32 lanes x 8 rows)
constexpr int NPW = 8;               // B rows per warp
constexpr int WARPS = 16;
constexpr int TN = NPW * WARPS;      // B rows per tile (128)
constexpr int THREADS = WARPS * 32;
constexpr int A_TILE = (CHUNK / 2) * (TM / 2) * 4;   // 64 KB
constexpr int B_TILE = TN * CHUNK;                   // 32 KB
constexpr int L_TILE = TN + TN * (CHUNK / 2);        // 16.1 KB: counts + index lists
constexpr int STAGE = A_TILE + B_TILE + L_TILE;
constexpr int MAX_LIST = 128;                        // chunks per CTA (host caps the split)
constexpr int SMEM = 1024 + 2 * STAGE + 64 + MAX_LIST * 4;  // + alignment slack for the 1024-B swizzle
static_assert(TM * TN * 4 <= 2 * STAGE, "C staging (32 x 32 swizzled boxes) reuses the stage buffers");
static_assert(SMEM <= 232448, "fits the opt-in shared memory of an SM");
}  // namespace satfix

// Pair sums of four signed bytes: the two 16-bit lanes {b0+b1, b2+b3} of the positive parts
// (pos) and of the magnitudes of the negative parts (neg).
__device__ __forceinline__ void pair_pos_neg(uint32_t w, uint32_t& pos, uint32_t& neg) {
    const uint32_t p = __vmaxs4(w, 0u);
    const uint32_t q = __vsub4(0u, __vmins4(w, 0u));  // -128 -> 0x80 = 128 (unsigned)
    pos = (p & 0x00FF00FFu) + ((p >> 8) & 0x00FF00FFu);
    neg = (q & 0x00FF00FFu) + ((q >> 8) & 0x00FF00FFu);
}

// A -> A_pm, and max(A) into guard[0].  Thread = (tile u, chunk c, 32-byte segment s, word
// rp) with rp fastest, so every store instruction of a warp writes 128 contiguous bytes.
__global__ void sat_prep_a_kernel(const uint8_t* __restrict__ a, int64_t lda, int64_t m, int64_t k, int vec_ok,
                                  int64_t chunks, uint32_t* __restrict__ apm, int32_t* __restrict__ guard) {
    using namespace satfix;
    pdl_launch_dependents();
    pdl_wait();
    const int64_t tiles = (m + TM - 1) / TM;
    const int64_t total = tiles * chunks * 8 * (TM / 2);
    uint32_t amax4 = 0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int rp = static_cast<int>(i & (TM / 2 - 1));
        const int s = static_cast<int>((i >> 7) & 7);
        const int64_t tc = i >> 10;  // u * chunks + c
        const int64_t u = tc / chunks, c = tc - u * chunks;
        // word rp = 4 l + q holds rows l + 64 q and l + 64 q + 32 of the tile
        const int64_t r0 = u * TM + (rp >> 2) + 64 * (rp & 3), r1 = r0 + 32, kb = c * CHUNK + s * 32;
        const uint4 x0 = simt_load16<true>(a, lda, r0, m, kb, k, vec_ok);
        const uint4 x1 = simt_load16<true>(a, lda, r0, m, kb + 16, k, vec_ok);
        const uint4 y0 = simt_load16<true>(a, lda, r1, m, kb, k, vec_ok);
        const uint4 y1 = simt_load16<true>(a, lda, r1, m, kb + 16, k, vec_ok);
        const uint32_t xa[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
        const uint32_t ya[8] = {y0.x, y0.y, y0.z, y0.w, y1.x, y1.y, y1.z, y1.w};
        uint32_t* dst = apm + tc * (A_TILE / 4) + (s * 16) * (TM / 2) + rp;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            amax4 = __vmaxu4(amax4, __vmaxu4(xa[e], ya[e]));
            dst[(2 * e) * (TM / 2)] = __byte_perm(xa[e], ya[e], 0x5410);
            dst[(2 * e + 1) * (TM / 2)] = __byte_perm(xa[e], ya[e], 0x7632);
        }
    }
    int32_t amax = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) amax = max(amax, static_cast<int32_t>((amax4 >> (8 * q)) & 0xFF));
    for (int o = 16; o > 0; o >>= 1) amax = max(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if ((threadIdx.x & 31) == 0 && amax) atomicMax(&guard[0], amax);
}

// B -> B_safe (row-major, pitch lds, dangerous pairs zeroed: the tensor-core operand), B_t,
// L_t, flags and the dangerous-pair count (guard[4..5]).  Thread = (tile t, chunk c, row r,
// 16-byte piece q) with q fastest: the 16 lanes of a half warp cover one row's 256-byte chunk
// (coalesced 256-byte loads and stores), a segmented scan over them places each lane's entries
// in the row's index list, and a block (16 rows of ONE tile chunk: 128 rows = 8 blocks) adds
// its count to the tile chunk's flag with one atomic.  One short item per thread (N K / 16
// threads), so the kernel is bandwidth- rather than latency-bound (the 64-byte-per-thread
// version took 21.7 us for a 4 MiB B: profiles/r2/launches_c4_satfix_ext_r2_final.csv).
__global__ void __launch_bounds__(256)
    sat_prep_b_kernel(const int8_t* __restrict__ b, int64_t ldb, int64_t n, int64_t k, int vec_ok, int64_t chunks,
                      uint8_t* __restrict__ bsafe, int64_t lds, uint8_t* __restrict__ bt, uint8_t* __restrict__ lt,
                      uint32_t* __restrict__ flags, int32_t* __restrict__ guard) {
    using namespace satfix;
    __shared__ uint32_t blk_cnt;
    pdl_launch_dependents();
    pdl_wait();
    const int64_t amax = guard[0];
    // dangerous iff amax * pos > 32767 or amax * neg > 32768
    const uint32_t pos_lim = amax ? static_cast<uint32_t>(32767 / amax) : 0xFFFFu;
    const uint32_t neg_lim = amax ? static_cast<uint32_t>(32768 / amax) : 0xFFFFu;
    const uint8_t* bu = reinterpret_cast<const uint8_t*>(b);
    const int64_t tiles = (n + TN - 1) / TN;
    const int64_t total = tiles * chunks * TN * 16;  // a multiple of 2048: whole blocks per tile chunk
    unsigned long long cnt_all = 0;  // thread 0 of the block only
    for (int64_t base = blockIdx.x * static_cast<int64_t>(blockDim.x); base < total;
         base += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = base + threadIdx.x;
        const int q = static_cast<int>(i & 15);
        const int r = static_cast<int>((i >> 4) & (TN - 1));
        const int64_t tc = i >> 11;  // t * chunks + c  (block-uniform: 256 threads = 16 rows of it)
        const int64_t t = tc / chunks, c = tc - t * chunks;
        const int64_t row = t * TN + r, c0 = c * CHUNK + q * 16;
        if (threadIdx.x == 0) blk_cnt = 0;
        __syncthreads();
        const uint4 orig = simt_load16<true>(bu, ldb, row, n, c0, k, vec_ok);
        uint32_t w[4] = {orig.x, orig.y, orig.z, orig.w};
        uint32_t mask = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            uint32_t pos, neg;
            pair_pos_neg(w[e], pos, neg);
            const bool d0 = (pos & 0xFFFFu) > pos_lim || (neg & 0xFFFFu) > neg_lim;
            const bool d1 = (pos >> 16) > pos_lim || (neg >> 16) > neg_lim;
            mask |= (d0 ? 1u : 0u) << (e * 2);
            mask |= (d1 ? 1u : 0u) << (e * 2 + 1);
            w[e] &= (d0 ? 0u : 0x0000FFFFu) | (d1 ? 0u : 0xFFFF0000u);
        }
        *reinterpret_cast<uint4*>(bt + tc * B_TILE + r * CHUNK + q * 16) = orig;
        if (row < n) *reinterpret_cast<uint4*>(bsafe + row * lds + c0) = make_uint4(w[0], w[1], w[2], w[3]);
        // the row's index list: inclusive scan of the popcounts over the row's 16 lanes
        const uint32_t mine = __popc(mask);
        uint32_t incl = mine;
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) {
            const uint32_t up = __shfl_up_sync(0xffffffffu, incl, o, 16);
            if (q >= o) incl += up;
        }
        const uint32_t row_total = __shfl_sync(0xffffffffu, incl, 15, 16);
        uint8_t* rec = lt + tc * L_TILE;
        if (q == 0) rec[r] = static_cast<uint8_t>(row_total);  // 0..128
        uint8_t* lst = rec + TN + r * (CHUNK / 2) + (incl - mine);
        // entries are B byte offsets 2j (<= 254): the fix kernel uses them unmasked — any byte,
        // even a stale one past the count, addresses inside the row and inside the A tile
        for (uint32_t mb = mask, e = 0; mb; mb &= mb - 1, ++e)
            lst[e] = static_cast<uint8_t>(2 * (q * 8 + __ffs(mb) - 1));
        // two rows per warp -> one shared-memory add per warp, one global atomic per block
        const uint32_t other = __shfl_sync(0xffffffffu, row_total, 16);
        if ((threadIdx.x & 31) == 0 && row_total + other) atomicAdd(&blk_cnt, row_total + other);
        __syncthreads();
        if (threadIdx.x == 0 && blk_cnt) {
            atomicAdd(&flags[tc], blk_cnt);
            cnt_all += blk_cnt;
        }
    }
    if (threadIdx.x == 0 && cnt_all) atomicAdd(reinterpret_cast<unsigned long long*>(guard + 4), cnt_all);
}

// The sparse fix: C[m][n] += sum over the dangerous pairs j of row n of
// sat16(A[m][2j] B[n][2j] + A[m][2j+1] B[n][2j+1]), after the tensor-core kernel stored
// C = A . B_safe.
//
// CTA = (n-tile, m-tile, K split): 16 warps, warp w owns B rows 8w..8w+7 of the tile, lane l
// owns A rows l + 32 t (t < 8).  The tile chunks that hold dangerous pairs (flags) are streamed
// through two shared-memory stages by 1-D bulk copies (A_pm 64 KB + B_t 32 KB + L_t 16 KB per
// chunk), the next chunk's copies in flight while the current one is computed.  Each warp
// walks its rows' index lists (warp-uniform: no divergence) two pairs at a time, so both pair
// sums of a row are clamped and added by one cvt.pack.sat + one dp2a.  Epilogue: the tile's
// sums are staged as 32 x 32 SWIZZLE_128B boxes (conflict-free: lane l writes row l of a box)
// and added to C by TMA reduce-add (wrapping s32 adds in L2, any number of K splits).
__global__ void __launch_bounds__(satfix::THREADS, 1)
    sat_fix_kernel(const __grid_constant__ CUtensorMap tma_c, const uint32_t* __restrict__ apm,
                   const uint8_t* __restrict__ bt, const uint8_t* __restrict__ lt, const uint32_t* __restrict__ flags,
                   int64_t chunks, int64_t tiles_n, int64_t total_units, int64_t total_pairs,
                   const int32_t* __restrict__ guard) {
    using namespace satfix;
    // no early launch_dependents: the next grid's CTAs would wait in SM slots this grid still
    // needs; they launch as this grid's CTAs exit
    pdl_wait();
    const unsigned long long listed = *reinterpret_cast<const volatile unsigned long long*>(guard + 4);
    if (listed == 0) return;  // nothing can clamp
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1024-aligned
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * STAGE);
    int* nlist_p = reinterpret_cast<int*>(smem + 2 * STAGE + 16);
    int* list = reinterpret_cast<int*>(smem + 2 * STAGE + 64);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        fence_mbar_init();
    }
    // Work split over (tile, chunk) units in tile-major order, CTA b taking units
    // [b * per, (b + 1) * per): whole tiles per CTA, or stream-K (per = total / CTAs: a CTA's
    // run may end one tile and start the next, each segment closing with its own TMA reduce-add,
    // and every SM stays busy whatever the tile count — whole tiles leave 20 of 148 SMs idle at
    // 2048^3).  The choice weighs the per-chunk work, which grows with the share of listed pairs
    // (read on the device from the prep kernel's count: no host round trip), against the
    // per-segment epilogue: measured ~1 us + 55 us x density per chunk, ~3 us per epilogue
    // (profiles/r2/satfix_streamk_r2.log).  `g` counts chunk stages across segments (parity).
    const int64_t tiles = total_units / chunks;
    const int64_t per_tiles = (tiles + gridDim.x - 1) / gridDim.x * chunks;
    const int64_t per_stream = (total_units + gridDim.x - 1) / gridDim.x;
    const float w = 1.0f + 55.0f * static_cast<float>(listed) / static_cast<float>(total_pairs), e = 3.0f;
    const float cost_tiles = static_cast<float>(per_tiles) * w + static_cast<float>(per_tiles / chunks) * e;
    const float cost_stream =
        static_cast<float>(per_stream) * w + static_cast<float>((per_stream + chunks - 1) / chunks + 1) * e;
    const int64_t units_per_cta = cost_stream < cost_tiles ? per_stream : per_tiles;
    const int64_t u_begin = static_cast<int64_t>(blockIdx.x) * units_per_cta;
    const int64_t u_end = min(total_units, u_begin + units_per_cta);
    uint32_t g = 0;
    for (int64_t pos = u_begin; pos < u_end;) {
        const int64_t tile = pos / chunks;
        const int64_t c_begin = pos - tile * chunks;
        const int64_t c_end = min(min(chunks, c_begin + (u_end - pos)), c_begin + static_cast<int64_t>(MAX_LIST));
        pos += c_end - c_begin;
        const int64_t t = tile % tiles_n, u = tile / tiles_n;
        __syncthreads();  // the previous segment's list and staging smem are done with
        if (warp == 0) {  // the chunks with dangerous pairs, compacted by ballots
            int cnt = 0;
            for (int64_t cb = c_begin; cb < c_end; cb += 32) {
                const int64_t c = cb + lane;
                const bool hit = c < c_end && flags[t * chunks + c] != 0u;
                const uint32_t bal = __ballot_sync(0xffffffffu, hit);
                if (hit) list[cnt + __popc(bal & ((1u << lane) - 1u))] = static_cast<int>(c);
                cnt += __popc(bal);
            }
            if (lane == 0) *nlist_p = cnt;
        }
        __syncthreads();
        const int nl_count = *nlist_p;
        if (nl_count == 0) continue;  // block-uniform: no dangerous pair in this segment

        auto issue = [&](int i) {
            const int s = (g + i) & 1;
            const int64_t c = list[i];
            uint8_t* st = smem + s * STAGE;
            mbar_arrive_expect_tx(&full[s], STAGE);
            bulk_load_1d(st, apm + (u * chunks + c) * (A_TILE / 4), A_TILE, &full[s]);
            bulk_load_1d(st + A_TILE, bt + (t * chunks + c) * B_TILE, B_TILE, &full[s]);
            bulk_load_1d(st + A_TILE + B_TILE, lt + (t * chunks + c) * L_TILE, L_TILE, &full[s]);
        };
        if (tid == 0) issue(0);

        int32_t acc[NPW][8];  // [row of B][t]: A row l + 32 t
#pragma unroll
        for (int i = 0; i < NPW; ++i)
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[i][e] = 0;

        for (int i = 0; i < nl_count; ++i) {
            // the other stage was released by the __syncthreads that ended iteration i - 1
            if (tid == 0 && i + 1 < nl_count) issue(i + 1);
            mbar_wait(&full[(g + i) & 1], ((g + i) >> 1) & 1);
            // shared-window addresses: the loads below are plain LDS
            const uint32_t st = smem_u32(smem) + ((g + i) & 1) * STAGE;
            const uint32_t sa = st + lane * 16;             // + j * 512: pair j of this lane's 8 rows
            const uint32_t sc = st + A_TILE + B_TILE;       // counts, then the index lists
            // all 8 of this warp's rows fully listed (extreme inputs): pair-major loop, each pair of A
            // words loaded once for the 8 rows instead of once per row
            const uint32_t c_lo = lds_u32(sc + warp * NPW), c_hi = lds_u32(sc + warp * NPW + 4);
            if (c_lo == 0x80808080u && c_hi == 0x80808080u) {
                const uint32_t sb0 = st + A_TILE + warp * NPW * CHUNK;
#pragma unroll 2
                for (uint32_t j = 0; j < CHUNK / 2; j += 2) {
                    const uint4 w1 = lds_v4(sa + (j << 9));
                    const uint4 w2 = lds_v4(sa + ((j + 1) << 9));
                    const uint32_t x1[4] = {w1.x, w1.y, w1.z, w1.w};
                    const uint32_t x2[4] = {w2.x, w2.y, w2.z, w2.w};
#pragma unroll
                    for (int nn = 0; nn < NPW; ++nn) {
                        const uint32_t bw = lds_u32(sb0 + nn * CHUNK + (j << 1));  // pairs j and j + 1
                        const uint32_t b1 = bw & 0xFFFFu, b2 = bw >> 16, b1h = bw << 16, b2h = bw & 0xFFFF0000u;
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            acc[nn][2 * q] = sat2_add(dp4a_us(x1[q], b1, 0), dp4a_us(x2[q], b2, 0), acc[nn][2 * q]);
                            acc[nn][2 * q + 1] =
                                sat2_add(dp4a_us(x1[q], b1h, 0), dp4a_us(x2[q], b2h, 0), acc[nn][2 * q + 1]);
                        }
                    }
                }
                __syncthreads();
                continue;
            }
#pragma unroll
            for (int nn = 0; nn < NPW; ++nn) {
                const int nl = warp * NPW + nn;
                const uint32_t sb = st + A_TILE + nl * CHUNK;  // + j * 2: the row's pair j of B
                const uint32_t sl = sc + TN + nl * (CHUNK / 2);
                const int cnt = static_cast<int>(lds_u8(sc + nl));
                // o1, o2: list entries = B byte offsets 2j; pair j of the lane's A rows sits at j * 512
                auto process = [&](uint32_t o1, uint32_t o2, bool two) {
                    const uint4 w1 = lds_v4(sa + (o1 << 8));
                    const uint4 w2 = lds_v4(sa + (o2 << 8));
                    const uint32_t b1 = lds_u16(sb + o1);
                    const uint32_t b2 = two ? lds_u16(sb + o2) : 0u;
                    const uint32_t b1h = b1 << 16, b2h = b2 << 16;
                    const uint32_t x1[4] = {w1.x, w1.y, w1.z, w1.w};
                    const uint32_t x2[4] = {w2.x, w2.y, w2.z, w2.w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        acc[nn][2 * q] = sat2_add(dp4a_us(x1[q], b1, 0), dp4a_us(x2[q], b2, 0), acc[nn][2 * q]);
                        acc[nn][2 * q + 1] = sat2_add(dp4a_us(x1[q], b1h, 0), dp4a_us(x2[q], b2h, 0), acc[nn][2 * q + 1]);
                    }
                };
                if (cnt == CHUNK / 2) {  // every pair of the row listed (extreme inputs): no list walk
#pragma unroll 4
                    for (uint32_t j = 0; j < CHUNK / 2; j += 2) {
                        const uint4 w1 = lds_v4(sa + (j << 9));
                        const uint4 w2 = lds_v4(sa + ((j + 1) << 9));
                        const uint32_t bw = lds_u32(sb + (j << 1));  // pairs j and j + 1 of B
                        const uint32_t b1 = bw & 0xFFFFu, b2 = bw >> 16, b1h = bw << 16, b2h = bw & 0xFFFF0000u;
                        const uint32_t x1[4] = {w1.x, w1.y, w1.z, w1.w};
                        const uint32_t x2[4] = {w2.x, w2.y, w2.z, w2.w};
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            acc[nn][2 * q] = sat2_add(dp4a_us(x1[q], b1, 0), dp4a_us(x2[q], b2, 0), acc[nn][2 * q]);
                            acc[nn][2 * q + 1] =
                                sat2_add(dp4a_us(x1[q], b1h, 0), dp4a_us(x2[q], b2h, 0), acc[nn][2 * q + 1]);
                        }
                    }
                } else {
                    // whole groups of four entries, then a tail of up to three (no per-pair guards)
                    const int full = cnt & ~3;
                    for (int e = 0; e < full; e += 4) {
                        const uint32_t idx = lds_u32(sl + e);
                        process(__byte_perm(idx, 0, 0x4440), __byte_perm(idx, 0, 0x4441), true);
                        process(__byte_perm(idx, 0, 0x4442), __byte_perm(idx, 0, 0x4443), true);
                    }
                    const int tail = cnt - full;
                    if (tail != 0) {
                        const uint32_t idx = lds_u32(sl + full);
                        process(__byte_perm(idx, 0, 0x4440), __byte_perm(idx, 0, 0x4441), tail >= 2);
                        if (tail == 3) process(__byte_perm(idx, 0, 0x4442), __byte_perm(idx, 0, 0x4442), false);
                    }
                }
            }
            __syncthreads();
        }
        g += static_cast<uint32_t>(nl_count);

        // Epilogue: box (row block t, column block w / 4) of 32 x 32 int32, SWIZZLE_128B: row r's
        // 16-byte chunk c sits at chunk c ^ (r & 7).  Lane l writes row l of 8 boxes (t = 0..7).
        uint8_t* cs = smem;
#pragma unroll
        for (int tt = 0; tt < 8; ++tt) {
            uint8_t* box = cs + (tt * (TN / 32) + (warp >> 2)) * 4096 + lane * 128;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int chunk = ((warp & 3) * 2 + h) ^ (lane & 7);
                *reinterpret_cast<int4*>(box + chunk * 16) =
                    make_int4(acc[4 * h + 0][tt], acc[4 * h + 1][tt], acc[4 * h + 2][tt], acc[4 * h + 3][tt]);
            }
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
            for (int bx = 0; bx < (TM / 32) * (TN / 32); ++bx) {
                const int rb = bx / (TN / 32), cb = bx % (TN / 32);
                tma_reduce_add_2d(&tma_c, cs + bx * 4096, static_cast<int32_t>(t * TN + cb * 32),
                                  static_cast<int32_t>(u * TM + rb * 32));
            }
            tma_store_commit();
            tma_store_wait_read<0>();  // smem must outlive the reads; the adds complete with the grid
        }
    }
}

}  // namespace ngemm_dev
