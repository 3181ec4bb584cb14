// ngemm/gemm.hpp — the GEMM entry points of the drop-in API (reference gemm.hpp:34-409),
// served by the B200 engine through the C-ABI (include/ngemm_cuda.h).
//
//   gemm_conventional(a, b, shape, mode, engine)  -> ngemm_cuda_gemm_u8i8_host / _i16_host
//   gemm_ngemm(packed, b, mode, engine)            -> device-resident weight (uploaded and
//                                                     repacked once) + ngemm_cuda_gemm_packed
//   gemm_ref / gemm_sat_oracle                     -> the reference's scalar CPU oracles, kept
//                                                     as oracles (the checker, not a fallback)
//
// Semantics (bit-exact): WideningExact = sum_k a*b mod 2^32; HardwareSaturating = sum over
// even-aligned K pairs of sat16(a0*b0 + a1*b1) mod 2^32 (odd tail paired with 0); the 16-bit
// path has no saturation stage.  Errors are thrown before any launch with the reference's
// exception types; a CUDA failure raises CudaError.  There is no CPU fallback.
#pragma once

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "ngemm/common.hpp"
#include "ngemm/isa.hpp"
#include "ngemm/lanes.hpp"
#include "ngemm/layout.hpp"
#include "ngemm/matrix.hpp"

namespace ngemm {

namespace detail {

inline bool is_u8i8(ElemKind a, ElemKind b) { return a == ElemKind::U8 && b == ElemKind::I8; }
inline bool is_i16(ElemKind a, ElemKind b) { return a == ElemKind::I16 && b == ElemKind::I16; }

inline void require_gemm_operands(const MatrixBuf& a, const MatrixBuf& b) {
    if (!is_u8i8(a.kind(), b.kind()) && !is_i16(a.kind(), b.kind()))
        throw UnsupportedError(std::string("gemm: no kernel path for ") + elem_name(a.kind()) + " x " +
                               elem_name(b.kind()));
    if (a.cols() != b.cols())
        throw ShapeError("gemm: K mismatch, A is " + std::to_string(a.rows()) + "x" + std::to_string(a.cols()) +
                         " but B is " + std::to_string(b.rows()) + "x" + std::to_string(b.cols()) +
                         " (B is stored [N x K])");
}

// Engine -> C-ABI kernel id (include/ngemm_cuda.h); Native has no implementation here.
inline int engine_kernel(Engine e) {
    switch (e) {
    case Engine::Emulated: return NGEMM_KERNEL_SIMT;
    case Engine::Native: throw UnsupportedError("no native path for this shape/mode on this host "
                                                "(this build runs on the B200 engine: Engine::Cuda)");
    default: return NGEMM_KERNEL_AUTO;
    }
}

inline int abi_mode(SatMode m) { return m == SatMode::WideningExact ? NGEMM_SAT_EXACT : NGEMM_SAT_HARDWARE; }

template <typename TA, typename TB, bool kSat>
void scalar_gemm(const MatrixBuf& a, const MatrixBuf& b, MatrixBuf& c) {
    const std::int64_t k = a.cols();
    for (std::int64_t i = 0; i < a.rows(); ++i) {
        const TA* ar = a.row<TA>(i);
        std::int32_t* cr = c.row<std::int32_t>(i);
        for (std::int64_t j = 0; j < b.rows(); ++j) {
            const TB* br = b.row<TB>(j);
            std::uint32_t acc = 0;
            if constexpr (kSat) {
                for (std::int64_t q = 0; q < k; q += 2) {
                    const std::int32_t p = std::int32_t{ar[q]} * br[q] +
                                           (q + 1 < k ? std::int32_t{ar[q + 1]} * br[q + 1] : 0);
                    acc += static_cast<std::uint32_t>(static_cast<std::int32_t>(sat_i16(p)));
                }
            } else {
                for (std::int64_t q = 0; q < k; ++q) acc += static_cast<std::uint32_t>(std::int32_t{ar[q]} * br[q]);
            }
            cr[j] = static_cast<std::int32_t>(acc);
        }
    }
}

}  // namespace detail

// Scalar exact oracle (gemm.hpp:36-68): C = sum_k a*b, int32 wrapping.  CPU; the checker.
inline MatrixBuf gemm_ref(const MatrixBuf& a, const MatrixBuf& b) {
    detail::require_gemm_operands(a, b);
    MatrixBuf c(ElemKind::I32, a.rows(), b.rows());
    if (a.kind() == ElemKind::U8) detail::scalar_gemm<std::uint8_t, std::int8_t, false>(a, b, c);
    else detail::scalar_gemm<std::int16_t, std::int16_t, false>(a, b, c);
    return c;
}

inline MatrixBuf gemm_ref(const MatrixBuf& a, const MatrixBuf& b, const GemmProblem& p) {
    if (a.rows() != p.m || b.rows() != p.n || a.cols() != p.k || b.cols() != p.k || a.kind() != p.a_kind ||
        b.kind() != p.b_kind)
        throw ShapeError("gemm_ref: operands do not match the stated problem");
    return gemm_ref(a, b);
}

// Scalar saturating oracle (gemm.hpp:83-104).  CPU; the checker.
inline MatrixBuf gemm_sat_oracle(const MatrixBuf& a, const MatrixBuf& b) {
    detail::require_gemm_operands(a, b);
    if (a.kind() == ElemKind::I16) return gemm_ref(a, b);
    MatrixBuf c(ElemKind::I32, a.rows(), b.rows());
    detail::scalar_gemm<std::uint8_t, std::int8_t, true>(a, b, c);
    return c;
}

// Conventional entry on unpacked row-major A (gemm.hpp:327-369), computed on the GPU.
inline MatrixBuf gemm_conventional(const MatrixBuf& a, const MatrixBuf& b, const KernelShape& shape, SatMode mode,
                                   Engine engine = Engine::Auto) {
    detail::require_gemm_operands(a, b);
    if (shape.v * shape.h != shape.w || shape.h != (elem_bits(a.kind()) == 8 ? 4 : 2))
        throw ShapeError("gemm_conventional: kernel shape does not match operand kind");
    const int kernel = detail::engine_kernel(engine);
    MatrixBuf c(ElemKind::I32, a.rows(), b.rows());
    if (a.kind() == ElemKind::U8)
        throw_on_status(ngemm_cuda_gemm_u8i8_host(a.row<std::uint8_t>(0), b.row<std::int8_t>(0),
                                                  c.row<std::int32_t>(0), a.rows(), b.rows(), a.cols(),
                                                  detail::abi_mode(mode), kernel));
    else
        throw_on_status(ngemm_cuda_gemm_i16_host(a.row<std::int16_t>(0), b.row<std::int16_t>(0),
                                                 c.row<std::int32_t>(0), a.rows(), b.rows(), a.cols()));
    return c;
}

// NGEMM entry on a prepacked weight (gemm.hpp:373-409).  The weight is made device-resident
// once (repacked to K-major on the GPU) and cached on the PackedWeight; B and C cross the bus
// per call.  Engine::Emulated re-runs from the packed bytes through the CUDA-core kernel.
inline MatrixBuf gemm_ngemm(const PackedWeight& p, const MatrixBuf& b, SatMode mode, Engine engine = Engine::Auto) {
    if (!detail::is_u8i8(p.kind(), b.kind()) && !detail::is_i16(p.kind(), b.kind()))
        throw UnsupportedError(std::string("gemm_ngemm: no kernel path for ") + elem_name(p.kind()) + " x " +
                               elem_name(b.kind()));
    if (b.cols() != p.k_orig())
        throw ShapeError("gemm_ngemm: packed K=" + std::to_string(p.k_orig()) + " but B has K=" +
                         std::to_string(b.cols()));
    const int kernel = detail::engine_kernel(engine);
    MatrixBuf c(ElemKind::I32, p.m_orig(), b.rows());
    const ngemm_packed_meta meta = p.meta();
    if (kernel == NGEMM_KERNEL_AUTO && p.kind() == ElemKind::U8) {
        const std::shared_ptr<const DeviceWeight> w = p.device_weight();  // held for the whole call
        throw_on_status(ngemm_cuda_gemm_packed_resident_host(w->handle(), b.row<std::int8_t>(0),
                                                             c.row<std::int32_t>(0), b.rows(), detail::abi_mode(mode)));
    } else {
        throw_on_status(ngemm_cuda_gemm_packed_host(&meta, p.bytes(), p.byte_size(), b.bytes(),
                                                    c.row<std::int32_t>(0), b.rows(), detail::abi_mode(mode),
                                                    kernel));
    }
    return c;
}

}  // namespace ngemm
