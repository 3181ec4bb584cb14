// Our C++ suite for the drop-in API (include/ngemm): the reference's test patterns
// (test_gemm.cpp, test_layout.cpp) re-stated against the B200 engine, plus the device-
// resident weight cache.  Needs a GPU for the GEMM cases (run by tests/test_cpp_dropin.py).
#include <catch2/catch_amalgamated.hpp>

#include <atomic>
#include <cstdio>
#include <thread>
#include <vector>
#include <filesystem>

#include "ngemm/ngemm.hpp"

using namespace ngemm;

namespace {
MatrixBuf u8(std::int64_t r, std::int64_t c, std::uint64_t seed, std::int64_t hi = 255) {
    return mat_random(ElemKind::U8, r, c, seed, 0, hi);
}
MatrixBuf i8(std::int64_t r, std::int64_t c, std::uint64_t seed) { return mat_random(ElemKind::I8, r, c, seed, -128, 127); }
const KernelShape kS256{32, 4, 8};
const KernelShape kS512{64, 4, 16};
}  // namespace

TEST_CASE("dropin: 2x2 through every engine") {
    MatrixBuf a(ElemKind::U8, 2, 2), b(ElemKind::I8, 2, 2);
    a.set(0, 0, 1); a.set(0, 1, 2); a.set(1, 0, 3); a.set(1, 1, 4);
    b.set(0, 0, 5); b.set(0, 1, -1); b.set(1, 0, 2); b.set(1, 1, 0);
    for (Engine e : {Engine::Auto, Engine::Emulated, Engine::Cuda})
        for (SatMode m : {SatMode::WideningExact, SatMode::HardwareSaturating}) {
            MatrixBuf c = gemm_conventional(a, b, kS256, m, e);
            CHECK(c.get(0, 0) == 3);
            CHECK(c.get(0, 1) == 2);
            CHECK(c.get(1, 0) == 11);
            CHECK(c.get(1, 1) == 6);
            CHECK(gemm_ngemm(pack_weights(a, kS256, TileConfig{8, 1, 4, Perm::MNK}), b, m, e) == c);
        }
}

TEST_CASE("dropin: full-range random shapes match both oracles") {
    XorShift64Star rng(4242);
    for (int t = 0; t < 40; ++t) {
        const std::int64_t m = rng.next_in(1, 300), n = rng.next_in(1, 300), k = rng.next_in(1, 700);
        MatrixBuf a = u8(m, k, 100 + t), b = i8(n, k, 200 + t);
        const MatrixBuf exact = gemm_ref(a, b), sat = gemm_sat_oracle(a, b);
        CHECK(gemm_conventional(a, b, kS512, SatMode::WideningExact) == exact);
        CHECK(gemm_conventional(a, b, kS512, SatMode::HardwareSaturating) == sat);
        CHECK(gemm_conventional(a, b, kS256, SatMode::HardwareSaturating, Engine::Emulated) == sat);
        const Perm perm = static_cast<Perm>(t % 6);
        PackedWeight p = pack_weights(a, kS512, TileConfig{16 * (1 + t % 3), 64, 4 * (1 + t % 5), perm});
        CHECK(gemm_ngemm(p, b, SatMode::WideningExact) == exact);
        CHECK(gemm_ngemm(p, b, SatMode::HardwareSaturating) == sat);
        CHECK(gemm_ngemm(p, b, SatMode::HardwareSaturating, Engine::Emulated) == sat);
    }
}

TEST_CASE("dropin: saturating mode differs from exact on adversarial inputs") {
    MatrixBuf a(ElemKind::U8, 40, 64);
    MatrixBuf b(ElemKind::I8, 33, 64);
    XorShift64Star rng(55);
    for (std::int64_t r = 0; r < 40; ++r)
        for (std::int64_t c = 0; c < 64; ++c) a.set(r, c, 255);
    for (std::int64_t r = 0; r < 33; ++r)
        for (std::int64_t c = 0; c < 64; ++c) b.set(r, c, rng.next_in(0, 1) ? 127 : -128);
    const MatrixBuf sat = gemm_sat_oracle(a, b);
    CHECK_FALSE(sat == gemm_ref(a, b));
    CHECK(gemm_conventional(a, b, kS256, SatMode::HardwareSaturating) == sat);
    CHECK(gemm_ngemm(pack_weights(a, kS256, TileConfig{8, 1, 4, Perm::MNK}), b, SatMode::HardwareSaturating) == sat);
}

TEST_CASE("dropin: device-resident weight is reused and invalidated on mutation") {
    MatrixBuf a = u8(300, 260, 1), b = i8(100, 260, 2);
    PackedWeight p = pack_weights(a, kS512, TileConfig{16, 64, 64, Perm::NMK});
    CHECK(gemm_ngemm(p, b, SatMode::WideningExact) == gemm_ref(a, b));
    CHECK(gemm_ngemm(p, b, SatMode::WideningExact) == gemm_ref(a, b));  // cached device copy
    // poke one weight byte through the mutable accessor: the next call must see it
    p.data<std::uint8_t>()[p.elem_offset(5, 7)] = 0;
    a.set(5, 7, 0);
    CHECK(gemm_ngemm(p, b, SatMode::WideningExact) == gemm_ref(a, b));
}

TEST_CASE("dropin: concurrent gemm_ngemm on one const PackedWeight (reentrant device cache)") {
    // 8 threads x 50 calls race on the first upload and on the cached device copy; every result
    // must be bit-exact and the weight uploaded once (pure and reentrant).
    MatrixBuf a = u8(200, 384, 21), b = i8(96, 384, 22);
    const PackedWeight p = pack_weights(a, kS512, TileConfig{16, 64, 64, Perm::MNK});
    const MatrixBuf ref = gemm_ref(a, b), ref_sat = gemm_sat_oracle(a, b);
    std::atomic<int> good{0}, bad{0}, errors{0};
    std::vector<std::thread> ts;
    for (int t = 0; t < 8; ++t)
        ts.emplace_back([&, t] {
            for (int i = 0; i < 50; ++i) {
                try {
                    const bool sat = ((i + t) & 3) == 0;
                    const MatrixBuf c = gemm_ngemm(p, b, sat ? SatMode::HardwareSaturating : SatMode::WideningExact);
                    (c == (sat ? ref_sat : ref) ? good : bad).fetch_add(1);
                } catch (...) {
                    errors.fetch_add(1);
                }
            }
        });
    for (auto& th : ts) th.join();
    CHECK(errors.load() == 0);
    CHECK(bad.load() == 0);
    CHECK(good.load() == 400);
    const auto w1 = p.device_weight(), w2 = p.device_weight();
    CHECK(w1.get() == w2.get());  // one cached copy per device
}

TEST_CASE("dropin: NGPT file round trip feeds the GPU") {
    const std::string path = (std::filesystem::temp_directory_path() / "ngemm_dropin.ngpt").string();
    MatrixBuf a = u8(77, 129, 9), b = i8(31, 129, 10);
    PackedWeight p = pack_weights(a, kS256, TileConfig{16, 8, 12, Perm::KMN});
    packed_write(p, path);
    PackedWeight q = packed_read(path);
    CHECK(unpack_weights(q) == a);
    CHECK(gemm_ngemm(q, b, SatMode::WideningExact) == gemm_ref(a, b));
    std::filesystem::remove(path);
}

TEST_CASE("dropin: 16-bit path (no saturation stage)") {
    MatrixBuf a = mat_random(ElemKind::I16, 37, 45, 3, -32768, 32767);
    MatrixBuf b = mat_random(ElemKind::I16, 29, 45, 4, -32768, 32767);
    const MatrixBuf ref = gemm_ref(a, b);
    CHECK(gemm_conventional(a, b, KernelShape{16, 2, 8}, SatMode::HardwareSaturating) == ref);
    CHECK(gemm_ngemm(pack_weights(a, KernelShape{32, 2, 16}, TileConfig{16, 4, 6, Perm::NMK}), b,
                     SatMode::WideningExact) == ref);
}

TEST_CASE("dropin: errors are raised before dispatch") {
    MatrixBuf a = u8(4, 8, 1), b_badk = i8(4, 9, 2);
    CHECK_THROWS_AS(gemm_conventional(a, b_badk, kS256, SatMode::WideningExact), ShapeError);
    CHECK_THROWS_AS(gemm_conventional(a, i8(4, 8, 2), kS256, SatMode::WideningExact, Engine::Native),
                    UnsupportedError);
    CHECK_THROWS_AS(gemm_conventional(a, u8(4, 8, 3), kS256, SatMode::WideningExact), UnsupportedError);
    CHECK_THROWS_AS(gemm_conventional(a, i8(4, 8, 2), KernelShape{16, 2, 8}, SatMode::WideningExact), ShapeError);
    PackedWeight p = pack_weights(a, kS256, TileConfig{8, 1, 4, Perm::MNK});
    CHECK_THROWS_AS(gemm_ngemm(p, b_badk, SatMode::WideningExact), ShapeError);
}
