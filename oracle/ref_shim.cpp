// oracle/_ref shim — exposes the UNMODIFIED reference implementation (header-only C++20,
// /root/reference/proj/include/ngemm) through a small extern "C" surface so that the
// Python tests, the golden-fixture script and bench.py's reference arm can call it.
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile into oracle/_ref/libngemm_ref.so
// from the reference headers where they lie (never copied into this repo).  The product
// library never links it.
//
// The reference namespace is renamed (SURVEY.md §0 gotcha 4) so this translation unit
// could coexist with the drop-in headers of include/ngemm if both were ever linked together.
#define ngemm ngemm_ref
#include "ngemm/ngemm.hpp"
#undef ngemm

#include <cstring>
#include <memory>
#include <thread>
#include <vector>

using namespace ngemm_ref;

namespace {

MatrixBuf make_u8(const uint8_t* a, int64_t rows, int64_t cols) {
    MatrixBuf m(ElemKind::U8, rows, cols);
    std::memcpy(m.bytes(), a, static_cast<size_t>(rows * cols));
    return m;
}
MatrixBuf make_i8(const int8_t* b, int64_t rows, int64_t cols) {
    MatrixBuf m(ElemKind::I8, rows, cols);
    std::memcpy(m.bytes(), b, static_cast<size_t>(rows * cols));
    return m;
}
IsaProfile isa_of_bits(int bits) {
    return bits == 512 ? IsaProfile::v512() : bits == 256 ? IsaProfile::v256() : IsaProfile::scalar();
}
SatMode mode_of(int mode) { return mode == 0 ? SatMode::HardwareSaturating : SatMode::WideningExact; }
Engine engine_of(int e) { return e == 1 ? Engine::Emulated : e == 2 ? Engine::Native : Engine::Auto; }

// One row shard of a reference call: operands prebuilt outside any timed region.
struct Shard {
    int64_t r0, r1;
    MatrixBuf a;
    std::unique_ptr<PackedWeight> packed;
    MatrixBuf c{ElemKind::I32, 1, 1};
};

struct Session {
    int variant, mode, engine, isa_bits;
    int64_t m, n, k;
    MatrixBuf b{ElemKind::I8, 1, 1};
    std::vector<Shard> shards;
};

// variant: 0 gemm_ref, 1 gemm_sat_oracle, 2 gemm_conventional, 3 gemm_ngemm (pack per SURVEY 8(d) ii:
// tile {v, min(N,64), ceil4(K)}, MNK)
void run_shard(const Session& s, Shard& sh) {
    switch (s.variant) {
    case 0: sh.c = gemm_ref(sh.a, s.b); break;
    case 1: sh.c = gemm_sat_oracle(sh.a, s.b); break;
    case 2:
        sh.c = gemm_conventional(sh.a, s.b, kernel_shape(isa_of_bits(s.isa_bits), ElemKind::U8),
                                 mode_of(s.mode), engine_of(s.engine));
        break;
    default: sh.c = gemm_ngemm(*sh.packed, s.b, mode_of(s.mode), engine_of(s.engine)); break;
    }
}

} // namespace

extern "C" {

int ref_host_isa_bits() { return IsaProfile::of(host_isa()).vector_bits; }

void ref_mat_random(int kind, int64_t rows, int64_t cols, uint64_t seed, int64_t lo, int64_t hi,
                    void* out) {
    MatrixBuf m = mat_random(static_cast<ElemKind>(kind), rows, cols, seed, lo, hi);
    std::memcpy(out, m.bytes(), m.byte_size());
}

// Returns 0 on success, 1 UnsupportedError, 2 ShapeError, 3 other Error.
int ref_gemm(int variant, const uint8_t* a, const int8_t* b, int32_t* c, int64_t m, int64_t n,
             int64_t k, int mode, int engine, int isa_bits) {
    try {
        Session s{variant, mode, engine, isa_bits, m, n, k};
        s.b = make_i8(b, n, k);
        Shard sh{0, m, make_u8(a, m, k), nullptr};
        if (variant == 3) {
            KernelShape shape = kernel_shape(isa_of_bits(isa_bits), ElemKind::U8);
            TileConfig tile{shape.v, std::min<int64_t>(n, 64), round_up(k, 4), Perm::MNK};
            sh.packed = std::make_unique<PackedWeight>(pack_weights(sh.a, shape, tile));
        }
        run_shard(s, sh);
        std::memcpy(c, sh.c.bytes(), sh.c.byte_size());
        return 0;
    } catch (const UnsupportedError&) {
        return 1;
    } catch (const ShapeError&) {
        return 2;
    } catch (const Error&) {
        return 3;
    }
}

// i16 x i16 through the unmodified reference: variant 0 = gemm_ref, 2 = gemm_conventional
// (kernel shape for 16-bit lanes, WideningExact, Engine::Emulated).  Returns 0 on success.
int ref_gemm_i16(int variant, const int16_t* a, const int16_t* b, int32_t* c, int64_t m, int64_t n, int64_t k) {
    try {
        MatrixBuf am(ElemKind::I16, m, k), bm(ElemKind::I16, n, k);
        std::memcpy(am.bytes(), a, static_cast<size_t>(m * k) * 2);
        std::memcpy(bm.bytes(), b, static_cast<size_t>(n * k) * 2);
        MatrixBuf cm = variant == 0 ? gemm_ref(am, bm)
                                    : gemm_conventional(am, bm, kernel_shape(IsaProfile::v256(), ElemKind::I16),
                                                        SatMode::WideningExact, Engine::Emulated);
        std::memcpy(c, cm.bytes(), cm.byte_size());
        return 0;
    } catch (const Error&) {
        return 3;
    }
}

// pack_weights with an explicit tile; out has m_pad*k_pad bytes; returns byte size or -1.
int64_t ref_pack(const uint8_t* a, int64_t m, int64_t k, int w, int h, int v, int64_t tm, int64_t tn,
                 int64_t tk, int perm, uint8_t* out, int64_t out_cap) {
    try {
        MatrixBuf am = make_u8(a, m, k);
        PackedWeight p = pack_weights(am, KernelShape{w, h, v}, TileConfig{tm, tn, tk, static_cast<Perm>(perm)});
        if (static_cast<int64_t>(p.byte_size()) > out_cap) return -1;
        std::memcpy(out, p.bytes(), p.byte_size());
        return static_cast<int64_t>(p.byte_size());
    } catch (const Error&) {
        return -1;
    }
}

// gemm_ngemm on caller-provided packed bytes (reference emulated/native kernels).
int ref_gemm_ngemm_packed(const uint8_t* packed, int64_t nbytes, int w, int h, int v, int64_t tm,
                          int64_t tn, int64_t tk, int perm, int64_t m_orig, int64_t k_orig,
                          const int8_t* b, int64_t n, int32_t* c, int mode, int engine) {
    try {
        PackedWeight p(ElemKind::U8, KernelShape{w, h, v}, TileConfig{tm, tn, tk, static_cast<Perm>(perm)},
                       m_orig, k_orig);
        if (static_cast<int64_t>(p.byte_size()) != nbytes) return 2;
        std::memcpy(p.bytes(), packed, p.byte_size());
        MatrixBuf bm = make_i8(b, n, k_orig);
        MatrixBuf cm = gemm_ngemm(p, bm, mode_of(mode), engine_of(engine));
        std::memcpy(c, cm.bytes(), cm.byte_size());
        return 0;
    } catch (const UnsupportedError&) {
        return 1;
    } catch (const ShapeError&) {
        return 2;
    } catch (const Error&) {
        return 3;
    }
}

// Timed-harness session: A row-sharded over `threads` workers (our harness, not the
// reference's — the reference is single-threaded), each worker calling the
// unmodified reference entry point on its contiguous row block.
void* ref_session_create(const uint8_t* a, const int8_t* b, int64_t m, int64_t n, int64_t k, int variant,
                         int mode, int engine, int isa_bits, int threads) {
    auto* s = new Session{variant, mode, engine, isa_bits, m, n, k};
    s->b = make_i8(b, n, k);
    if (threads < 1) threads = 1;
    if (threads > m) threads = static_cast<int>(m);
    KernelShape shape = kernel_shape(isa_of_bits(isa_bits), ElemKind::U8);
    for (int t = 0; t < threads; ++t) {
        int64_t r0 = m * t / threads, r1 = m * (t + 1) / threads;
        Shard sh{r0, r1, make_u8(a + r0 * k, r1 - r0, k), nullptr};
        if (variant == 3) {
            TileConfig tile{shape.v, std::min<int64_t>(n, 64), round_up(k, 4), Perm::MNK};
            sh.packed = std::make_unique<PackedWeight>(pack_weights(sh.a, shape, tile));
        }
        s->shards.push_back(std::move(sh));
    }
    return s;
}

int ref_session_run(void* handle) {
    auto* s = static_cast<Session*>(handle);
    try {
        if (s->shards.size() == 1) {
            run_shard(*s, s->shards[0]);
            return 0;
        }
        std::vector<std::thread> workers;
        for (auto& sh : s->shards) workers.emplace_back([s, &sh] { run_shard(*s, sh); });
        for (auto& w : workers) w.join();
        return 0;
    } catch (const Error&) {
        return 3;
    }
}

void ref_session_result(void* handle, int32_t* c) {
    auto* s = static_cast<Session*>(handle);
    for (auto& sh : s->shards)
        std::memcpy(c + sh.r0 * s->n, sh.c.bytes(), sh.c.byte_size());
}

void ref_session_destroy(void* handle) { delete static_cast<Session*>(handle); }

} // extern "C"
