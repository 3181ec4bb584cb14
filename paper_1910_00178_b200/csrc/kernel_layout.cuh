// kernel_layout.cuh — device-side inverse of the reference PackedWeight layout.
//
// The reference packs the weight A [M x K] into tk x tm tiles traversed in the permutation's
// M/K order, v x h inner blocks K-first inside a tile, row-major (m*h + k) inside a block,
// zero padding to tm/tk multiples (layout.hpp:110-171).  The tensor cores want plain K-major
// rows, so a weight is repacked ONCE when it is made device-resident (the paper's offline
// prepack).  For 8-bit operands h = 4: every 4-byte word of the packed
// buffer is one row's K-group, so the kernel moves whole words.
#pragma once

#include "ptx.cuh"

namespace ngemm_dev {

struct PackedGeom {
    int32_t w, h, v, perm_m_before_k;
    int64_t tm, tk, m_pad, k_pad, m_orig, k_orig;
};

// PackedWeight::block_offset (layout.hpp:152-165), in elements.
__device__ __forceinline__ int64_t packed_block_offset(const PackedGeom& g, int64_t m_blk, int64_t k_blk) {
    const int64_t tile_m = m_blk * g.v / g.tm;
    const int64_t tile_k = k_blk * g.h / g.tk;
    const int64_t bm = m_blk - tile_m * (g.tm / g.v);
    const int64_t bk = k_blk - tile_k * (g.tk / g.h);
    const int64_t tiles_m = g.m_pad / g.tm;
    const int64_t tiles_k = g.k_pad / g.tk;
    const int64_t tile_lin = g.perm_m_before_k ? tile_m * tiles_k + tile_k : tile_k * tiles_m + tile_m;
    const int64_t blocks_per_tile = (g.tm / g.v) * (g.tk / g.h);
    return (tile_lin * blocks_per_tile + bm * (g.tk / g.h) + bk) * g.w;
}

// One thread per (row gm, 4-byte K-group kw) of the output; a warp covers 32 consecutive
// K-groups of one row, so the row-major writes are coalesced; the packed reads of consecutive
// K-groups of a row are w elements apart inside a tile and hit L2 lines that neighbouring rows
// reuse.  esize = 1 (u8, h = 4) or 2 (i16, h = 2): a K-group is always one 4-byte word.
__global__ void repack_kernel(PackedGeom g, const uint8_t* __restrict__ packed, uint8_t* __restrict__ a,
                              int64_t lda_bytes, int64_t kwords, int esize) {
    pdl_launch_dependents();
    pdl_wait();
    const int64_t total = g.m_orig * kwords;
    const int64_t k_bytes = g.k_orig * esize;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t gm = i / kwords, kw = i - gm * kwords;
        const int64_t off = (packed_block_offset(g, gm / g.v, kw) + (gm % g.v) * g.h) * esize;
        const uint32_t word = *reinterpret_cast<const uint32_t*>(packed + off);
        const int64_t gb = kw * 4;  // byte position in the row
        uint8_t* dst = a + gm * lda_bytes + gb;
        if (gb + 4 <= k_bytes && ((reinterpret_cast<uintptr_t>(dst) & 3) == 0)) {
            *reinterpret_cast<uint32_t*>(dst) = word;
        } else {
            for (int q = 0; q < 4 && gb + q < k_bytes; ++q) dst[q] = static_cast<uint8_t>(word >> (8 * q));
        }
    }
}

// Ragged operands -> TMA-describable copies (row pitch kp, a multiple of 16; bytes past k are
// zero): rows of A then rows of B in one launch, one thread per 16-byte output chunk.  Source
// rows with an unaligned pitch are read as aligned 4-byte words and realigned with funnel
// shifts (5 loads per 16 output bytes instead of 16 byte loads).
__global__ void stage_rows_kernel(const uint8_t* __restrict__ a, int64_t lda, int64_t ma,
                                  const uint8_t* __restrict__ b, int64_t ldb, int64_t nb, int64_t k, int64_t kp,
                                  uint8_t* __restrict__ da, uint8_t* __restrict__ db) {
    pdl_launch_dependents();
    pdl_wait();
    const int64_t cpr = kp / 16, total = (ma + nb) * cpr;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / cpr, c = i - r * cpr;
        const bool is_a = r < ma;
        const int64_t row = is_a ? r : r - ma;
        const uint8_t* src = is_a ? a + row * lda : b + row * ldb;
        uint8_t* dst = (is_a ? da : db) + row * kp + c * 16;
        const int64_t k0 = c * 16;
        const uintptr_t addr = reinterpret_cast<uintptr_t>(src + k0);
        uint32_t w[4] = {0, 0, 0, 0};
        if (k0 + 20 <= k && (k0 >= 4 || (addr & 3) == 0)) {  // the 20 bytes read stay inside the row
            const uint32_t* p = reinterpret_cast<const uint32_t*>(addr & ~uintptr_t(3));
            const uint32_t sh = static_cast<uint32_t>(addr & 3) * 8;
            uint32_t x[5];
#pragma unroll
            for (int q = 0; q < 5; ++q) x[q] = __ldg(p + q);
#pragma unroll
            for (int q = 0; q < 4; ++q) w[q] = __funnelshift_r(x[q], x[q + 1], sh);
        } else {
#pragma unroll
            for (int t = 0; t < 16; ++t)
                if (k0 + t < k) w[t >> 2] |= static_cast<uint32_t>(__ldg(src + k0 + t)) << (8 * (t & 3));
        }
        *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// Requantisation of an int32 C to int8 (the unfused form of the tcgen05 kernel's c_mode 4, same
// arithmetic): out[r][c] = clamp(rint(float(C[r][c] + bias[c]) * scale[c]) + zp, -128, 127).
__global__ void requant_kernel(const int32_t* __restrict__ c, int64_t ldc, int64_t m, int64_t n,
                               const float* __restrict__ scale, const int32_t* __restrict__ bias, int zp,
                               int8_t* __restrict__ out, int64_t ldo) {
    pdl_launch_dependents();
    pdl_wait();
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m * n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / n, col = i - r * n;
        out[r * ldo + col] = requant_s8(static_cast<uint32_t>(c[r * ldc + col]), bias ? bias[col] : 0, scale[col], zp);
    }
}

// Deterministic full-range operand fill for the tuner (splitmix64 of the element index).
__global__ void fill_random_kernel(uint8_t* __restrict__ p, int64_t rows, int64_t cols, int64_t ld, uint64_t seed) {
    const int64_t total = rows * cols;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        uint64_t z = seed + 0x9E3779B97F4A7C15ull * static_cast<uint64_t>(i + 1);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        const int64_t r = i / cols;
        p[r * ld + (i - r * cols)] = static_cast<uint8_t>(z >> 56);
    }
}

// Counts elements where x != y (the tuner's verify-before-time, tuner.hpp:155-161).
__global__ void count_mismatch_kernel(const int32_t* __restrict__ x, const int32_t* __restrict__ y, int64_t n,
                                      unsigned long long* __restrict__ bad) {
    unsigned long long local = 0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        local += (x[i] != y[i]) ? 1ull : 0ull;
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(bad, local);
}

// i16 operand -> two byte planes for the tensor cores: x = 256 * hi + lo with lo = x & 0xFF
// (u8) and hi = x >> 8 (s8), so sum_k a*b = 2^16 (ah.bh) + 2^8 (ah.bl + al.bh) + al.bl (mod 2^32)
// and each term is an int8 tensor-core GEMM.  Planes are K-major with row pitch kp (a multiple
// of 16, zero-filled past k) — the TMA operand layout.  One thread per 8 elements.
__global__ void split_i16_kernel(const int16_t* __restrict__ src, int64_t ld, int64_t rows, int64_t k, int64_t kp,
                                 uint8_t* __restrict__ lo, uint8_t* __restrict__ hi, int vec_ok) {
    pdl_launch_dependents();
    pdl_wait();
    const int64_t per_row = kp / 8;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < rows * per_row;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / per_row, c = (i - r * per_row) * 8;
        const int16_t* p = src + r * ld + c;
        uint32_t w[4];
        if (vec_ok && c + 8 <= k) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
            w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
        } else {
            uint16_t e[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) e[j] = (c + j < k) ? static_cast<uint16_t>(p[j]) : 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) w[j] = e[2 * j] | (static_cast<uint32_t>(e[2 * j + 1]) << 16);
        }
        // little-endian: bytes of w[j] are (lo0, hi0, lo1, hi1)
        const uint2 l = make_uint2(__byte_perm(w[0], w[1], 0x6420), __byte_perm(w[2], w[3], 0x6420));
        const uint2 h = make_uint2(__byte_perm(w[0], w[1], 0x7531), __byte_perm(w[2], w[3], 0x7531));
        *reinterpret_cast<uint2*>(lo + r * kp + c) = l;
        *reinterpret_cast<uint2*>(hi + r * kp + c) = h;
    }
}

}  // namespace ngemm_dev
