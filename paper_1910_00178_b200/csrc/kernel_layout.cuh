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

// Byte-wise max of A and (max, min) of B: the saturation-safety proof of the dispatcher.
// out[0] = max a, out[1] = max b, out[2] = -min b (all >= 0); out must be zeroed first.
__global__ void operand_range_kernel(const uint8_t* __restrict__ a, int64_t lda, int64_t m,
                                     const int8_t* __restrict__ b, int64_t ldb, int64_t n, int64_t k,
                                     int32_t* __restrict__ out) {
    int32_t amax = 0, bmax = 0, bneg = 0;
    const int64_t ta = m * k, tb = n * k;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < ta + tb;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (i < ta) {
            const int64_t r = i / k, c = i - r * k;
            amax = max(amax, static_cast<int32_t>(a[r * lda + c]));
        } else {
            const int64_t j = i - ta, r = j / k, c = j - r * k;
            const int32_t v = b[r * ldb + c];
            bmax = max(bmax, v);
            bneg = max(bneg, -v);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        amax = max(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        bmax = max(bmax, __shfl_xor_sync(0xffffffffu, bmax, o));
        bneg = max(bneg, __shfl_xor_sync(0xffffffffu, bneg, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&out[0], amax);
        atomicMax(&out[1], bmax);
        atomicMax(&out[2], bneg);
    }
}

}  // namespace ngemm_dev
