// ngemm — command-line front end of the B200 engine, following the reference CLI spec
// (the reference ships only tools/CMakeLists.txt, its source is absent).
//
//   ngemm rand  --kind u8|i8|i16 --rows R --cols C [--seed S] [--lo L --hi H] --out X.ngmm
//   ngemm pack  --in A.ngmm --out W.ngpt [--isa scalar|v256|v512] [--tile tm,tn,tk] [--perm mnk|...]
//   ngemm gemm  (--a A.ngmm | --packed W.ngpt) --b B.ngmm [--variant ref|conventional|ngemm]
//               [--mode sat|exact] [--out C.ngmm]
//   ngemm bench [--sizes MxNxK,...] [--kind u8i8|i16] [--mode sat|exact] [--repeats N] [--warmup N]
//               [--seed N] [--tile tm,tn,tk] [--perm P] [--out bench.csv]
//   ngemm tune  --sizes MxNxK,... [--mode sat|exact] [--repeats N] [--warmup N] [--store tune.txt]
//
// Every GEMM runs on the GPU (variant ref is the CPU oracle).  bench verifies each variant
// against gemm_ref before timing it (no unverified timing reaches the CSV, bench.hpp:243-247)
// and writes the reference's CSV schema `m,n,k,kind,isa,variant,median_ns,min_ns,trials,checksum`
// plus a geometric-mean footer; timings are wall-clock medians of the host-facing calls
// (operands cross PCIe per call; the ngemm weight stays device-resident).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "ngemm/ngemm.hpp"

using namespace ngemm;

namespace {

struct Args {
    std::string cmd;
    std::map<std::string, std::string> kv;
    std::string get(const std::string& k, const std::string& d = "") const {
        auto it = kv.find(k);
        return it == kv.end() ? d : it->second;
    }
    bool has(const std::string& k) const { return kv.count(k) != 0; }
};

Args parse(int argc, char** argv) {
    Args a;
    if (argc < 2) throw ConfigError("usage: ngemm rand|pack|gemm|bench|tune [--flag value ...]");
    a.cmd = argv[1];
    for (int i = 2; i < argc; ++i) {
        std::string f = argv[i];
        if (f.rfind("--", 0) != 0) throw ConfigError("unexpected argument \"" + f + "\"");
        if (i + 1 >= argc) throw ConfigError("flag " + f + " needs a value");
        a.kv[f.substr(2)] = argv[++i];
    }
    return a;
}

ElemKind kind_of(const std::string& s) {
    if (s == "u8") return ElemKind::U8;
    if (s == "i8") return ElemKind::I8;
    if (s == "i16") return ElemKind::I16;
    if (s == "i32") return ElemKind::I32;
    throw ConfigError("unknown kind \"" + s + "\"");
}

SatMode mode_of(const std::string& s) {
    if (s == "sat") return SatMode::HardwareSaturating;
    if (s == "exact") return SatMode::WideningExact;
    throw ConfigError("unknown mode \"" + s + "\" (sat|exact)");
}

struct Size {
    std::int64_t m, n, k;
};

std::vector<Size> parse_sizes(const std::string& spec) {
    std::vector<Size> out;
    std::stringstream ss(spec);
    std::string item;
    while (std::getline(ss, item, ',')) {
        Size z{};
        char x1 = 0, x2 = 0;
        std::stringstream is(item);
        if (!(is >> z.m >> x1 >> z.n >> x2 >> z.k) || x1 != 'x' || x2 != 'x' || z.m < 1 || z.n < 1 || z.k < 1)
            throw ConfigError("bad size \"" + item + "\" (expected MxNxK)");
        out.push_back(z);
    }
    if (out.empty()) throw ConfigError("empty size list");
    return out;
}

TileConfig tile_of(const Args& a, const KernelShape& s, std::int64_t n, std::int64_t k) {
    TileConfig t{s.v, std::min<std::int64_t>(64, n), s.h, Perm::MNK};  // bench.hpp defaults: alpha = beta = 1, tn = 64
    if (a.has("tile")) {
        char c1 = 0, c2 = 0;
        std::stringstream is(a.get("tile"));
        if (!(is >> t.tm >> c1 >> t.tn >> c2 >> t.tk) || c1 != ',' || c2 != ',')
            throw ConfigError("bad --tile (expected tm,tn,tk)");
    }
    (void)k;
    if (a.has("perm")) t.permutation = perm_from_name(a.get("perm"));
    return t;
}

IsaProfile isa_of(const Args& a) { return IsaProfile::of(a.has("isa") ? isa_from_name(a.get("isa")) : host_isa()); }

int cmd_rand(const Args& a) {
    const ElemKind kind = kind_of(a.get("kind", "u8"));
    const std::int64_t lo = a.has("lo") ? std::stoll(a.get("lo")) : elem_min(kind);
    const std::int64_t hi = a.has("hi") ? std::stoll(a.get("hi")) : elem_max(kind);
    MatrixBuf m = mat_random(kind, std::stoll(a.get("rows")), std::stoll(a.get("cols")),
                             std::stoull(a.get("seed", "0")), lo, hi);
    mat_write(m, a.get("out"));
    std::printf("wrote %s %lldx%lld checksum %lld\n", elem_name(kind), static_cast<long long>(m.rows()),
                static_cast<long long>(m.cols()), static_cast<long long>(m.checksum()));
    return 0;
}

int cmd_pack(const Args& a) {
    MatrixBuf m = mat_read(a.get("in"));
    const KernelShape s = kernel_shape(isa_of(a), m.kind());
    PackedWeight p = pack_weights(m, s, tile_of(a, s, 64, m.cols()));
    packed_write(p, a.get("out"));
    std::printf("packed w=%d h=%d v=%d tm=%lld tn=%lld tk=%lld perm=%s m_pad=%lld k_pad=%lld bytes=%zu\n", s.w, s.h,
                s.v, static_cast<long long>(p.tile().tm), static_cast<long long>(p.tile().tn),
                static_cast<long long>(p.tile().tk), perm_name(p.tile().permutation),
                static_cast<long long>(p.m_pad()), static_cast<long long>(p.k_pad()), p.byte_size());
    return 0;
}

int cmd_gemm(const Args& a) {
    const std::string variant = a.get("variant", a.has("packed") ? "ngemm" : "conventional");
    const SatMode mode = mode_of(a.get("mode", "exact"));
    MatrixBuf b = mat_read(a.get("b"));
    MatrixBuf c(ElemKind::I32, 1, 1);
    if (variant == "ngemm") {
        if (!a.has("packed")) throw ConfigError("variant ngemm needs --packed W.ngpt");
        c = gemm_ngemm(packed_read(a.get("packed")), b, mode);
    } else {
        if (a.has("packed")) throw ConfigError("variant " + variant + " takes an unpacked --a, not --packed");
        MatrixBuf am = mat_read(a.get("a"));
        if (variant == "ref")
            c = mode == SatMode::WideningExact ? gemm_ref(am, b) : gemm_sat_oracle(am, b);
        else if (variant == "conventional")
            c = gemm_conventional(am, b, kernel_shape(isa_of(a), am.kind()), mode);
        else
            throw ConfigError("unknown variant \"" + variant + "\" (ref|conventional|ngemm)");
    }
    if (a.has("out")) mat_write(c, a.get("out"));
    std::printf("%s %s %lldx%lld checksum %lld\n", variant.c_str(), sat_mode_name(mode),
                static_cast<long long>(c.rows()), static_cast<long long>(c.cols()),
                static_cast<long long>(c.checksum()));
    return 0;
}

template <typename Fn>
std::pair<double, double> time_fn(Fn&& fn, int repeats, int warmup) {  // bench.hpp:61-79 discipline
    for (int i = 0; i < warmup; ++i) fn();
    std::vector<double> t;
    for (int i = 0; i < repeats; ++i) {
        const auto t0 = std::chrono::steady_clock::now();
        fn();
        const auto t1 = std::chrono::steady_clock::now();
        t.push_back(static_cast<double>(std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count()));
    }
    std::sort(t.begin(), t.end());
    const std::size_t n = t.size();
    return {n % 2 ? t[n / 2] : 0.5 * (t[n / 2 - 1] + t[n / 2]), t.front()};
}

int cmd_bench(const Args& a) {
    std::vector<Size> sizes;
    if (a.has("sizes")) sizes = parse_sizes(a.get("sizes"));
    else
        for (std::int64_t mn : {64, 256})
            for (std::int64_t k : {128, 256, 512, 1024}) sizes.push_back({mn, mn, k});  // bench.hpp:47-53
    const std::string kind = a.get("kind", "u8i8");
    if (kind != "u8i8" && kind != "i16") throw ConfigError("unknown --kind (u8i8|i16)");
    const ElemKind ka = kind == "u8i8" ? ElemKind::U8 : ElemKind::I16;
    const ElemKind kb = kind == "u8i8" ? ElemKind::I8 : ElemKind::I16;
    const SatMode mode = mode_of(a.get("mode", "sat"));
    const int repeats = std::stoi(a.get("repeats", "7")), warmup = std::stoi(a.get("warmup", "2"));
    const std::uint64_t seed = std::stoull(a.get("seed", "42"));
    const IsaProfile isa = isa_of(a);
    std::ostringstream csv;
    csv << "m,n,k,kind,isa,variant,median_ns,min_ns,trials,checksum\n";
    double log_sum = 0;
    int pairs = 0;
    for (const Size& z : sizes) {
        const GemmProblem prob(z.m, z.n, z.k, ka, kb);
        MatrixBuf am = random_operand(ka, z.m, z.k, seed);      // safe range, tuner.hpp:26-43
        MatrixBuf bm = random_operand(kb, z.n, z.k, seed + 1);
        const MatrixBuf ref = gemm_ref(am, bm, prob);
        const KernelShape s = kernel_shape(isa, ka);
        PackedWeight p = pack_weights(am, s, tile_of(a, s, z.n, z.k));
        if (!(gemm_conventional(am, bm, s, mode) == ref))
            throw Error("bench: conventional kernel failed verification at " + std::to_string(z.m) + "x" +
                        std::to_string(z.n) + "x" + std::to_string(z.k));
        if (!(gemm_ngemm(p, bm, mode) == ref))
            throw Error("bench: ngemm kernel failed verification at " + std::to_string(z.m) + "x" +
                        std::to_string(z.n) + "x" + std::to_string(z.k));
        const auto tc = time_fn([&] { gemm_conventional(am, bm, s, mode); }, repeats, warmup);
        const auto tn = time_fn([&] { gemm_ngemm(p, bm, mode); }, repeats, warmup);
        for (int v = 0; v < 2; ++v) {
            const auto& t = v ? tn : tc;
            csv << z.m << ',' << z.n << ',' << z.k << ',' << kind << ",b200," << (v ? "ngemm" : "conventional") << ','
                << static_cast<long long>(t.first) << ',' << static_cast<long long>(t.second) << ',' << repeats << ','
                << ref.checksum() << '\n';
        }
        log_sum += std::log(tc.first / tn.first);
        ++pairs;
    }
    csv << "# geomean speedup ngemm/conventional: " << std::exp(log_sum / std::max(1, pairs)) << '\n';
    if (a.has("out")) {
        std::ofstream f(a.get("out"));
        f << csv.str();
    }
    std::cout << csv.str();
    return 0;
}

int cmd_tune(const Args& a) {
    const SatMode mode = mode_of(a.get("mode", "exact"));
    const int repeats = std::stoi(a.get("repeats", "5")), warmup = std::stoi(a.get("warmup", "2"));
    for (const Size& z : parse_sizes(a.get("sizes"))) {
        ngemm_tune_record r{};
        throw_on_status(ngemm_cuda_tune(z.m, z.n, z.k, mode == SatMode::WideningExact ? 1 : 0, repeats, warmup, &r));
        std::printf("%lldx%lldx%lld %s -> kernel=%d tc_cfg=%d splits=%d variant=%d median %.0f ns (min %.0f)\n",
                    static_cast<long long>(z.m), static_cast<long long>(z.n), static_cast<long long>(z.k),
                    sat_mode_name(mode), r.kernel, r.tc_cfg, r.tc_splits, r.skinny_variant, r.median_ns, r.min_ns);
    }
    if (a.has("store")) throw_on_status(ngemm_cuda_tune_store_save(a.get("store").c_str()));
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        const Args a = parse(argc, argv);
        if (a.cmd == "rand") return cmd_rand(a);
        if (a.cmd == "pack") return cmd_pack(a);
        if (a.cmd == "gemm") return cmd_gemm(a);
        if (a.cmd == "bench") return cmd_bench(a);
        if (a.cmd == "tune") return cmd_tune(a);
        throw ConfigError("unknown command \"" + a.cmd + "\" (rand|pack|gemm|bench|tune)");
    } catch (const std::exception& e) {
        std::fprintf(stderr, "ngemm: %s\n", e.what());
        return 1;
    }
}
