// ngemm/tuner.hpp — seeded operand generation in the "safe" range (reference
// tuner.hpp:22-43): u8 capped at 127 so no int16 pair sum can saturate, which makes
// HardwareSaturating and WideningExact agree and lets one oracle verify every timed run.
// (The reference's CPU tile search over (alpha, beta, tn, perm) has no meaning for tcgen05
// and is not part of this build.)
#pragma once

#include <cstdint>
#include <utility>

#include "ngemm/common.hpp"
#include "ngemm/gemm.hpp"
#include "ngemm/matrix.hpp"

namespace ngemm {

inline std::pair<std::int64_t, std::int64_t> safe_range(ElemKind kind) {
    if (kind == ElemKind::U8) return {0, 127};
    if (kind == ElemKind::I8) return {-128, 127};
    if (kind == ElemKind::I16) return {-32768, 32767};
    throw UnsupportedError("safe_range: no kernel path for i32");
}

inline MatrixBuf random_operand(ElemKind kind, std::int64_t rows, std::int64_t cols, std::uint64_t seed) {
    const auto [lo, hi] = safe_range(kind);
    return mat_random(kind, rows, cols, seed, lo, hi);
}

}  // namespace ngemm
