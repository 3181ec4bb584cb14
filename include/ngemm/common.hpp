// ngemm/common.hpp — element kinds, the error hierarchy and the int32/int16 arithmetic
// helpers of the drop-in API (same names and meaning as the reference's common.hpp:11-157;
// written for the B200 engine).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include "ngemm_cuda.h"

namespace ngemm {

// Operand/result domains: A is u8 (or i16), B is i8 (or i16), C is i32 (common.hpp:11-16).
enum class ElemKind : std::uint8_t { U8 = 0, I8 = 1, I16 = 2, I32 = 3 };

namespace kinds {
struct Info {
    int bits;
    bool is_signed;
    std::int64_t lo, hi;
    const char* name;
};
inline constexpr Info kTable[4] = {
    {8, false, 0, 255, "u8"},
    {8, true, -128, 127, "i8"},
    {16, true, -32768, 32767, "i16"},
    {32, true, -2147483647LL - 1, 2147483647LL, "i32"},
};
constexpr const Info& of(ElemKind k) { return kTable[static_cast<int>(k) & 3]; }
}  // namespace kinds

constexpr int elem_bits(ElemKind k) { return kinds::of(k).bits; }
constexpr int elem_size(ElemKind k) { return kinds::of(k).bits / 8; }
constexpr bool elem_signed(ElemKind k) { return kinds::of(k).is_signed; }
constexpr std::int64_t elem_min(ElemKind k) { return kinds::of(k).lo; }
constexpr std::int64_t elem_max(ElemKind k) { return kinds::of(k).hi; }
inline const char* elem_name(ElemKind k) { return kinds::of(k).name; }

// ---- errors (common.hpp:77-127): thrown before any device work is launched ---------------
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ShapeError : Error { using Error::Error; };
struct RangeError : Error { using Error::Error; };
struct IndexError : Error { using Error::Error; };
struct ConfigError : Error { using Error::Error; };
struct CorruptionError : Error { using Error::Error; };
struct UnsupportedError : Error { using Error::Error; };
struct FitError : Error { using Error::Error; };
struct TuneError : Error { using Error::Error; };
struct FormatError : Error {
    FormatError(const std::string& what, std::uint64_t offset)
        : Error(what + " (at byte offset " + std::to_string(offset) + ")"), byte_offset(offset) {}
    std::uint64_t byte_offset;
};
// A failure inside the CUDA runtime (no reference analogue: the reference never fails after
// validation).  Derives from Error so reference-style catch blocks still see it.
struct CudaError : Error { using Error::Error; };

// Maps a C-ABI status to the matching exception type (include/ngemm_cuda.h).
inline void throw_on_status(ngemm_status s) {
    if (s == NGEMM_OK) return;
    const std::string msg = ngemm_cuda_last_error();
    switch (s) {
    case NGEMM_ERR_SHAPE: throw ShapeError(msg);
    case NGEMM_ERR_UNSUPPORTED: throw UnsupportedError(msg);
    case NGEMM_ERR_CONFIG: throw ConfigError(msg);
    case NGEMM_ERR_RANGE: throw RangeError(msg);
    case NGEMM_ERR_CORRUPTION: throw CorruptionError(msg);
    case NGEMM_ERR_INDEX: throw IndexError(msg);
    case NGEMM_ERR_TUNE: throw TuneError(msg);
    default: throw CudaError(msg.empty() ? std::string("CUDA error") : msg);
    }
}

// ---- arithmetic helpers ------------------------------------------------------------------
// int32 accumulation is modulo 2^32 everywhere (common.hpp:129-135), which is what makes the
// GPU's reduction order (tensor-core K order, split-K atomics, warp folds) bit-exact.
constexpr std::int32_t wrap_add_i32(std::int32_t a, std::int32_t b) {
    return static_cast<std::int32_t>(static_cast<std::uint32_t>(a) + static_cast<std::uint32_t>(b));
}
constexpr std::int32_t wrap_i32(std::int64_t x) { return static_cast<std::int32_t>(static_cast<std::uint64_t>(x)); }
constexpr std::int16_t sat_i16(std::int32_t x) {
    return static_cast<std::int16_t>(x < -32768 ? -32768 : (x > 32767 ? 32767 : x));
}
constexpr std::int64_t round_up(std::int64_t x, std::int64_t multiple) {
    return ((x + multiple - 1) / multiple) * multiple;
}
constexpr int log2_exact(std::int64_t x) {
    int n = 0;
    for (std::int64_t p = 1; p < x; p <<= 1) ++n;
    return n;
}
constexpr bool is_pow2(std::int64_t x) { return x > 0 && (x & (x - 1)) == 0; }

}  // namespace ngemm
