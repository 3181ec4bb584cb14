// ngemm/isa.hpp — vector-profile descriptors and the Engine selector (reference isa.hpp:11-96).
//
// The profiles (scalar / V256 / V512) survive only as layout parameters: they fix the
// KernelShape (w, h, v) that PackedWeight is marshalled with.  The B200 engine consumes any
// profile's packing, so host SIMD detection is irrelevant to where the math runs:
//   Engine::Auto / Engine::Cuda -> libngemm_cuda.so dispatcher (tcgen05 / skinny / SIMT)
//   Engine::Emulated            -> the lane-faithful CUDA-core kernel (bit-identical oracle semantics)
//   Engine::Native              -> UnsupportedError: there is no x86 SIMD path and no CPU fallback.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <string>

#include "ngemm/common.hpp"

namespace ngemm {

enum class Isa : std::uint8_t { SCALAR = 0, V256 = 1, V512 = 2 };

struct IsaProfile {
    Isa name = Isa::SCALAR;
    int vector_bits = 128;

    static IsaProfile scalar() { return {Isa::SCALAR, 128}; }
    static IsaProfile v256() { return {Isa::V256, 256}; }
    static IsaProfile v512() { return {Isa::V512, 512}; }
    static IsaProfile of(Isa isa) {
        return isa == Isa::V512 ? v512() : (isa == Isa::V256 ? v256() : scalar());
    }
};

inline const char* isa_name(Isa isa) {
    constexpr const char* names[3] = {"scalar", "v256", "v512"};
    const int i = static_cast<int>(isa);
    return i >= 0 && i < 3 ? names[i] : "?";
}

inline Isa isa_from_name(const std::string& s) {
    for (Isa i : {Isa::SCALAR, Isa::V256, Isa::V512})
        if (s == isa_name(i)) return i;
    throw ConfigError("unknown isa \"" + s + "\" (expected scalar|v256|v512)");
}

// Which implementation services a call.  Cuda is appended so the reference values keep
// their numbering; Auto resolves to Cuda.
enum class Engine { Auto, Emulated, Native, Cuda };

// The layout profile used when a caller asks for the "host" profile: FORCE_ISA if set
// (isa.hpp:64-68), otherwise V512 — the widest packing, whose 16-row blocks tile the
// tensor-core operands evenly.  Detection never gates execution: the math runs on the GPU.
inline Isa host_isa() {
    static const Isa isa = [] {
        const char* f = std::getenv("FORCE_ISA");
        return f ? isa_from_name(f) : Isa::V512;
    }();
    return isa;
}

// No native x86 path exists in this build (Engine::Native always reports unsupported).
inline bool host_supports_native(Isa) { return false; }

}  // namespace ngemm
