// ngemm/prng.hpp — the deterministic generator every seeded input is drawn from.
// Same sequence as the reference's XorShift64Star (prng.hpp:13-43): one splitmix64 step turns
// the seed into a non-zero state, then xorshift64* with the 0x2545F4914F6CDD1D multiplier;
// range draws use plain modulo.  Golden digests in tests/golden depend on it bit for bit.
#pragma once

#include <cstdint>

#include "ngemm/common.hpp"

namespace ngemm {

class XorShift64Star {
public:
    explicit XorShift64Star(std::uint64_t seed) : s_(mix(seed)) {}

    std::uint64_t next() {
        s_ ^= s_ >> 12;
        s_ ^= s_ << 25;
        s_ ^= s_ >> 27;
        return s_ * 0x2545F4914F6CDD1Dull;
    }

    std::int64_t next_in(std::int64_t lo, std::int64_t hi) {
        if (hi < lo) throw RangeError("next_in: lo > hi");
        const std::uint64_t width = static_cast<std::uint64_t>(hi) - static_cast<std::uint64_t>(lo) + 1u;
        const std::uint64_t r = next();
        return width == 0 ? static_cast<std::int64_t>(r) : lo + static_cast<std::int64_t>(r % width);
    }

private:
    static std::uint64_t mix(std::uint64_t seed) {
        std::uint64_t z = seed + 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        return z ? z : 0x9E3779B97F4A7C15ull;
    }
    std::uint64_t s_;
};

}  // namespace ngemm
