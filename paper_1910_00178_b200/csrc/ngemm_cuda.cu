// ngemm_cuda.cu — the C-ABI (include/ngemm_cuda.h) over the hand-written sm_100a kernels.
//
// Validation happens before any launch and maps 1:1 onto the reference exception types
// (gemm.hpp:19-30, 375-382; layout.hpp:92-102, 254-263).  There is no CPU path: if the
// device or the sm_100a image is missing, every entry returns NGEMM_ERR_CUDA.
#include "ngemm_cuda.h"

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <fstream>
#include <map>
#include <mutex>
#include <sstream>
#include <tuple>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#ifdef NGEMM_TRACE
// Trace build only (make trace -> libngemm_cuda_trace.so, scripts/probes/tc_trace.py): per
// launch and CTA, %globaltimer stamps of the tcgen05 kernel's phases.  The launch index comes
// from the host (TileMap::trace_id, one per captured launch), so recording a stamp is a single
// global store: no loads or atomics that would stall the traced thread.
constexpr int kTraceL = 64, kTraceCta = 160, kTraceP = 16;
__device__ unsigned long long g_tc_trace[kTraceL][kTraceCta][kTraceP];
int g_trace_next = 0;  // host: id of the next traced launch
__device__ __forceinline__ unsigned long long trace_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void trace_put(int L, int p, unsigned long long t) {
    if (L >= 0 && L < kTraceL && blockIdx.x < kTraceCta) g_tc_trace[L][blockIdx.x][p] = t;
}
#define TC_TRACE_KEEP(p) const unsigned long long _tck##p = trace_now();
#define TC_TRACE_NOW(p) trace_put(map.trace_id, p, trace_now())
#define TC_TRACE_FLUSH()                       \
    if (threadIdx.x == 0) {                    \
        trace_put(map.trace_id, 0, _tck0);     \
        trace_put(map.trace_id, 1, _tck1);     \
        trace_put(map.trace_id, 2, trace_now()); \
    }
#define TC_TRACE_END() \
    if (threadIdx.x == 0) trace_put(map.trace_id, 9, trace_now());
#endif

#include "kernel_layout.cuh"
#include "kernel_satfix.cuh"
#include "kernel_simt.cuh"
#include "kernel_skinny.cuh"
#include "kernel_tcgen05.cuh"

using namespace ngemm_dev;

namespace {

thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};

ngemm_status fail(ngemm_status s, const std::string& msg) {
    g_last_error = msg;
    return s;
}

#define NG_CUDA(expr)                                                                              \
    do {                                                                                           \
        cudaError_t e_ = (expr);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            return fail(NGEMM_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));       \
    } while (0)

#define NG_LAUNCHED()                                                                              \
    do {                                                                                           \
        cudaError_t e_ = cudaGetLastError();                                                       \
        if (e_ != cudaSuccess) return fail(NGEMM_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(e_)); \
        g_launches.fetch_add(1, std::memory_order_relaxed);                                        \
    } while (0)

int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

struct DevInfo {
    int sms = 0;
    int smem_optin = 0;
    int cc_major = 0, cc_minor = 0;
};

DevInfo dev_info(int dev) {
    static std::mutex mu;
    static DevInfo cache[64];
    static bool have[64] = {};
    std::lock_guard<std::mutex> lk(mu);
    if (dev >= 0 && dev < 64 && have[dev]) return cache[dev];
    DevInfo d;
    cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&d.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&d.cc_major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&d.cc_minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (dev >= 0 && dev < 64 && d.sms > 0) {
        cache[dev] = d;
        have[dev] = true;
    }
    return d;
}

// ---------------------------------------------------------------- experiment / test knobs
// Read ONCE from the environment (NGEMM_<NAME>) on first use and never again on the launch
// path; tests and the sweep scripts change them through ngemm_cuda_set_option.  -1 = unset
// (the planner decides).  None of them is needed in production.
enum Opt : int {
    O_PDL, O_L2_PREFETCH, O_SKINNY_FAST, O_SKINNY_SPLITS, O_SKINNY_RG, O_SKINNY_WARPS, O_SKINNY_VARIANT,
    O_TC_QUAD, O_TC_CFG, O_TC_SPLITS, O_TC_DIRECT, O_TC_PREISSUE, O_TC_L2HINT, O_TC_GROUP_M, O_TC_DBG,
    O_SAT_HYBRID, O_SATFIX_SKIP, O_I16_PATH, O_REQUANT_UNFUSED, O_TC_SCHED, O_SKINNY_XRED, O_N
};
struct OptDef {
    const char* name;
    int def;
};
constexpr OptDef kOpts[O_N] = {
    {"PDL", 1}, {"L2_PREFETCH", 1}, {"SKINNY_FAST", 1}, {"SKINNY_SPLITS", -1}, {"SKINNY_RG", -1},
    {"SKINNY_WARPS", -1}, {"SKINNY_VARIANT", -1}, {"TC_QUAD", 0}, {"TC_CFG", -1}, {"TC_SPLITS", -1},
    {"TC_DIRECT", 0}, {"TC_PREISSUE", 0}, {"TC_L2HINT", 7}, {"TC_GROUP_M", -1}, {"TC_DBG", 0},
    {"SAT_HYBRID", -1}, {"SATFIX_SKIP", 0}, {"I16_PATH", -1}, {"REQUANT_UNFUSED", 0}, {"TC_SCHED", -1},
    {"SKINNY_XRED", 1},
};
std::atomic<int> g_opt[O_N];
std::once_flag g_opt_once;

int env_opt(int i) {
    const std::string key = std::string("NGEMM_") + kOpts[i].name;
    const char* e = std::getenv(key.c_str());
    if (!e || !*e) return kOpts[i].def;
    if (i == O_I16_PATH) return std::strcmp(e, "tcgen05") == 0 ? 1 : 0;  // "tcgen05" | "simt"
    return std::atoi(e);
}
void load_opts() {
    for (int i = 0; i < O_N; ++i) g_opt[i].store(env_opt(i), std::memory_order_relaxed);
}
int opt(Opt o) {
    std::call_once(g_opt_once, load_opts);
    return g_opt[o].load(std::memory_order_relaxed);
}
int opt_index(const char* name) {
    if (!name) return -1;
    if (std::strncmp(name, "NGEMM_", 6) == 0) name += 6;
    for (int i = 0; i < O_N; ++i)
        if (std::strcmp(name, kOpts[i].name) == 0) return i;
    return -1;
}

// Stream-ordered scratch comes from the library's OWN pool per device (release threshold
// UINT64_MAX, so a host-entry call does not remap multi-GB buffers every time); the device's
// default pool — shared with the host application — is left untouched.  ngemm_cuda_trim()
// returns the cached bytes.  Inside a stream capture the allocation becomes a graph node.
cudaMemPool_t lib_pool(int dev) {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    static bool made[64] = {};
    if (dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> lk(mu);
    if (!made[dev]) {
        made[dev] = true;
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        if (cudaMemPoolCreate(&pools[dev], &props) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr);
        } else {
            cudaGetLastError();
            pools[dev] = nullptr;
        }
    }
    return pools[dev];
}

cudaError_t dev_alloc(void** p, size_t bytes, cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {
        cudaGetLastError();
        return cudaMallocAsync(p, bytes, st);
    }
    if (cs != cudaStreamCaptureStatusNone) return cudaMallocAsync(p, bytes, st);  // graph allocation node
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool = lib_pool(dev);
    return pool ? cudaMallocFromPoolAsync(p, bytes, pool, st) : cudaMallocAsync(p, bytes, st);
}
template <typename T>
cudaError_t dev_alloc(T** p, size_t bytes, cudaStream_t st) {
    return dev_alloc(reinterpret_cast<void**>(p), bytes, st);
}

void autoload_tune_store();

ngemm_status current_device(int* dev, DevInfo* info) {
    NG_CUDA(cudaGetDevice(dev));
    autoload_tune_store();
    *info = dev_info(*dev);
    if (info->sms <= 0) return fail(NGEMM_ERR_CUDA, "no CUDA device");
    if (info->cc_major != 10 || info->cc_minor != 0)
        return fail(NGEMM_ERR_UNSUPPORTED, "libngemm_cuda is built for sm_100a (B200); device is sm_" +
                                               std::to_string(info->cc_major) + std::to_string(info->cc_minor));
    return NGEMM_OK;
}

// ---------------------------------------------------------------- TMA descriptors
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<EncodeTiledFn>(nullptr);
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

// 2-D u8 tensor [outer x inner] with row stride `stride` bytes, box [box_outer x box_inner],
// SWIZZLE_128B, out-of-bounds elements read as zero.
ngemm_status make_tmap_u8(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t stride,
                          uint32_t box_inner, uint32_t box_outer) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return fail(NGEMM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {stride};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(NGEMM_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return NGEMM_OK;
}

// C through TMA (store / reduce-add epilogues): 16-byte aligned base and row pitch, and a row
// length that is a whole number of 16-byte granules — a box straddling the last column writes
// the whole trailing granule (measured: with N % 4 != 0 and ldc > N the bytes past column N-1
// of each row change, scripts/probes/probe_ldc.py), so such C goes through direct stores.
bool c_tma_ok(const int32_t* c, int64_t ldc, int64_t n) {
    return reinterpret_cast<uintptr_t>(c) % 16 == 0 && ldc % 4 == 0 && n % 4 == 0;
}

bool tma_ok(const void* p, int64_t ld) {
    return (reinterpret_cast<uintptr_t>(p) & 15) == 0 && ld % 16 == 0 && ld < (int64_t(1) << 39);
}

// ---------------------------------------------------------------- validation
ngemm_status validate(const void* a, int64_t lda, const void* b, int64_t ldb, const void* c, int64_t ldc, int64_t m,
                      int64_t n, int64_t k, int mode) {
    if (mode != NGEMM_SAT_HARDWARE && mode != NGEMM_SAT_EXACT)
        return fail(NGEMM_ERR_CONFIG, "sat_mode must be 0 (HardwareSaturating) or 1 (WideningExact)");
    if (m < 1 || n < 1 || k < 1)
        return fail(NGEMM_ERR_SHAPE, "gemm: dims must be >= 1, got " + std::to_string(m) + "x" + std::to_string(n) +
                                         "x" + std::to_string(k));
    if (lda < k || ldb < k || ldc < n) return fail(NGEMM_ERR_SHAPE, "gemm: leading dimension smaller than the row");
    if (!a || !b || !c) return fail(NGEMM_ERR_SHAPE, "gemm: null operand");
    if (m > INT32_MAX / 2 || n > INT32_MAX / 2) return fail(NGEMM_ERR_SHAPE, "gemm: dimension too large");
    return NGEMM_OK;
}

// ---------------------------------------------------------------- tuned choices
// A kernel choice for one (m, n, k, mode): set by ngemm_cuda_tune (or loaded from a tune
// store) and consulted by the dispatcher before its heuristics.  -1 = planner's default.
struct Choice {
    int kernel = NGEMM_KERNEL_AUTO;
    int tc_cfg = -1, tc_splits = -1, skinny_variant = -1;
};
thread_local Choice t_force;  // the choice in effect for the launch being issued on this thread

// ---------------------------------------------------------------- launchers
// Strided batch of independent GEMMs of one shape (count 1 = a single GEMM).
struct Batch {
    int count = 1;
    int64_t sa = 0, sb = 0, sc = 0;  // element strides between consecutive A / B / C
};
// Programmatic dependent launch: consecutive kernels on a stream overlap the next kernel's
// launch and prologue (barrier init, TMEM alloc, descriptor prefetch) with the tail of the
// previous one; every kernel calls griddepcontrol.wait before touching global memory, so
// stream order semantics are unchanged.  NGEMM_PDL=0 disables it.
bool pdl_enabled() { return opt(O_PDL) != 0; }

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, unsigned cx,
                     unsigned cy, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    unsigned na = 0;
    if (cx * cy > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = cx;
        attr[na].val.clusterDim.y = cy;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    if (pdl_enabled()) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

#define NG_LAUNCH(...)                                                                             \
    do {                                                                                           \
        cudaError_t e_ = launch_k(__VA_ARGS__);                                                    \
        if (e_ != cudaSuccess) return fail(NGEMM_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(e_)); \
        g_launches.fetch_add(1, std::memory_order_relaxed);                                        \
    } while (0)

template <typename K>
ngemm_status set_smem(K kernel, int bytes) {
    NG_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    // largest shared-memory carveout, so two lean CTAs (or a lean CTA and the next grid's) fit
    NG_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    return NGEMM_OK;
}

// Zero C before a split-K launch (the partial sums are wrap-added into it).
ngemm_status zero_c(int32_t* c, int64_t ldc, int64_t m, int64_t n, cudaStream_t st) {
    if (ldc == n) NG_CUDA(cudaMemsetAsync(c, 0, static_cast<size_t>(m * n) * 4, st));
    else NG_CUDA(cudaMemset2DAsync(c, static_cast<size_t>(ldc) * 4, 0, static_cast<size_t>(n) * 4, m, st));
    return NGEMM_OK;
}

// CUDA-core kernel launch: 128x128 tiles when they fill two waves of CTAs, else 64x64 tiles
// plus K splits (32-byte aligned) so that ~2 CTAs per SM are busy.  kbytes/lda/ldb in bytes.
template <int MODE>
ngemm_status launch_simt_bytes(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb, int32_t* c, int64_t ldc,
                               int64_t m, int64_t n, int64_t kbytes, const DevInfo& di, cudaStream_t st) {
    const int vec_ok = (reinterpret_cast<uintptr_t>(a) % 16 == 0 && reinterpret_cast<uintptr_t>(b) % 16 == 0 &&
                        lda % 16 == 0 && ldb % 16 == 0);
    const int c_vec = (reinterpret_cast<uintptr_t>(c) % 16 == 0 && ldc % 4 == 0);
    const int64_t tiles128 = ((m + 127) / 128) * ((n + 127) / 128);
    const int64_t target = 2 * di.sms;
    if (tiles128 >= target || (m + 63) / 64 > 65535) {
        dim3 grid(static_cast<unsigned>((n + 127) / 128), static_cast<unsigned>((m + 127) / 128), 1);
        if (grid.y > 65535) return fail(NGEMM_ERR_SHAPE, "simt: M too large");
        NG_LAUNCH(simt_gemm_kernel<MODE, 128>, grid, dim3(simt::THREADS), 0, st, 1, 1, a, lda, b, ldb, c, ldc, m, n,
                  kbytes, vec_ok, c_vec, kbytes, 0);
        return NGEMM_OK;
    }
    const int64_t tiles64 = ((m + 63) / 64) * ((n + 63) / 64);
    // K splits down to 128 bytes until ~8 CTAs per SM: few-tile shapes were latency bound
    // (128x1024x1024 sat 19.3 -> 12.2 us, others unchanged; profiles/r2/simt_split_r2.log)
    const int64_t tgt = 8 * static_cast<int64_t>(di.sms);
    int64_t splits = std::max<int64_t>(1, std::min<int64_t>((tgt + tiles64 - 1) / tiles64, kbytes / 128));
    const int64_t k_split = round_up((kbytes + splits - 1) / splits, 32);
    splits = (kbytes + k_split - 1) / k_split;
    if (splits > 1) {
        ngemm_status zs = zero_c(c, ldc, m, n, st);
        if (zs != NGEMM_OK) return zs;
    }
    dim3 grid(static_cast<unsigned>((n + 63) / 64), static_cast<unsigned>((m + 63) / 64), static_cast<unsigned>(splits));
    NG_LAUNCH(simt_gemm_kernel<MODE, 64>, grid, dim3(simt::THREADS), 0, st, 1, 1, a, lda, b, ldb, c, ldc, m, n, kbytes,
              vec_ok, c_vec, k_split, splits > 1 ? 1 : 0);
    return NGEMM_OK;
}

ngemm_status launch_simt(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb, int32_t* c, int64_t ldc,
                         int64_t m, int64_t n, int64_t k, int mode, cudaStream_t st) {
    int dev = 0;
    cudaGetDevice(&dev);
    const DevInfo di = dev_info(dev);
    return mode == NGEMM_SAT_EXACT ? launch_simt_bytes<1>(a, lda, b, ldb, c, ldc, m, n, k, di, st)
                                   : launch_simt_bytes<0>(a, lda, b, ldb, c, ldc, m, n, k, di, st);
}

// i16 x i16 -> i32 (the reference's 16-bit path, gemm.hpp:161-190, 245-281): SIMT kernel in
// MODE 2 over the operands viewed as bytes (2 bytes per element, K-groups of 2 per word).
ngemm_status launch_simt_i16(const int16_t* a, int64_t lda, const int16_t* b, int64_t ldb, int32_t* c, int64_t ldc,
                             int64_t m, int64_t n, int64_t k, cudaStream_t st) {
    int dev = 0;
    cudaGetDevice(&dev);
    return launch_simt_bytes<2>(reinterpret_cast<const uint8_t*>(a), lda * 2, reinterpret_cast<const int8_t*>(b),
                                ldb * 2, c, ldc, m, n, k * 2, dev_info(dev), st);
}

constexpr int kSkinnyMaxM = 16;
constexpr int64_t kSkinnySmemCap = 200 * 1024;

bool skinny_fits(int64_t m, int64_t k) {
    int mt = 1;
    while (mt < m) mt *= 2;
    return m <= kSkinnyMaxM && mt * round_up(k, 16) <= kSkinnySmemCap;
}

template <int MODE, int MT, int NR>
ngemm_status launch_skinny_t(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb, int32_t* c, int64_t ldc,
                             int64_t m, int64_t n, int64_t k, const DevInfo& di, cudaStream_t st) {
    const int64_t kpad = round_up(k, 16);
    const int smem = static_cast<int>(MT * kpad);
    auto kern = skinny_gemm_kernel<MODE, MT, NR>;
    if (smem > 48 * 1024) {
        ngemm_status s = set_smem(kern, smem);
        if (s != NGEMM_OK) return s;
    }
    const int b_vec = (reinterpret_cast<uintptr_t>(b) % 16 == 0 && ldb % 16 == 0);
    const int64_t groups = (n + NR - 1) / NR;
    int64_t blocks = (groups + skinny::WARPS - 1) / skinny::WARPS;
    blocks = std::min<int64_t>(blocks, static_cast<int64_t>(di.sms) * 8);
    NG_LAUNCH(kern, dim3(static_cast<unsigned>(blocks)), dim3(skinny::THREADS), smem, st, 1, 1, a, lda, b, ldb, c, ldc,
              static_cast<int>(m), n, k, kpad, b_vec);
    return NGEMM_OK;
}

template <int MODE>
ngemm_status launch_skinny_mode(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb, int32_t* c,
                                int64_t ldc, int64_t m, int64_t n, int64_t k, const DevInfo& di, cudaStream_t st) {
    if (m <= 1) return launch_skinny_t<MODE, 1, 8>(a, lda, b, ldb, c, ldc, m, n, k, di, st);
    if (m <= 2) return launch_skinny_t<MODE, 2, 8>(a, lda, b, ldb, c, ldc, m, n, k, di, st);
    if (m <= 4) return launch_skinny_t<MODE, 4, 4>(a, lda, b, ldb, c, ldc, m, n, k, di, st);
    if (m <= 8) return launch_skinny_t<MODE, 8, 4>(a, lda, b, ldb, c, ldc, m, n, k, di, st);
    return launch_skinny_t<MODE, 16, 4>(a, lda, b, ldb, c, ldc, m, n, k, di, st);
}

// Makes (a, lda) and (b, ldb) TMA-describable: ragged operands are copied by one
// stage_rows_kernel launch into a zero-padded scratch buffer with 16-byte row pitch (SURVEY.md
// §0 gotcha 3; padding K at the end is neutral).  Caller frees *scratch.
ngemm_status stage_tma_operands(const uint8_t*& a, int64_t& lda, int64_t m, const uint8_t*& b, int64_t& ldb,
                                int64_t n, int64_t k, uint8_t** scratch, cudaStream_t st) {
    *scratch = nullptr;
    const bool a_ok = tma_ok(a, lda), b_ok = tma_ok(b, ldb);
    if (a_ok && b_ok) return NGEMM_OK;
    const int64_t kp = round_up(k, 16);
    const int64_t ma = a_ok ? 0 : m, nb = b_ok ? 0 : n;
    NG_CUDA(dev_alloc(scratch, static_cast<size_t>((ma + nb) * kp), st));
    uint8_t* da = *scratch;
    uint8_t* db = *scratch + ma * kp;
    int dev = 0;
    cudaGetDevice(&dev);
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(((ma + nb) * (kp / 16) + 255) / 256,
                                                                   dev_info(dev).sms * 8));
    NG_LAUNCH(stage_rows_kernel, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, st, 1, 1, a, lda, ma, b, ldb, nb,
              k, kp, da, db);
    if (!a_ok) {
        a = da;
        lda = kp;
    }
    if (!b_ok) {
        b = db;
        ldb = kp;
    }
    return NGEMM_OK;
}

// Exact-mode skinny GEMM on the tensor cores (operands swapped, UMMA 128 x 16): 128-row tiles
// of B x a K-split cluster of up to 8 CTAs reduced through DSMEM.
ngemm_status launch_tc_skinny(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb, int32_t* c, int64_t ldc,
                              int64_t m, int64_t n, int64_t k, const DevInfo& di, cudaStream_t st) {
    if (m > tcs::MPAD) return fail(NGEMM_ERR_UNSUPPORTED, "tensor-core skinny path needs M <= 16");
    constexpr int STAGES = 4;
    using S = tcs::Smem<STAGES>;
    auto kern = tc_skinny_kernel<STAGES>;
    static std::once_flag once[64];
    int dev = 0;
    cudaGetDevice(&dev);
    ngemm_status s = NGEMM_OK;
    std::call_once(once[dev & 63], [&] { s = set_smem(kern, S::TOTAL); });
    if (s != NGEMM_OK) return s;
    const uint8_t* a_use = a;
    const uint8_t* b_use = reinterpret_cast<const uint8_t*>(b);
    int64_t lda_use = lda, ldb_use = ldb;
    uint8_t* scratch = nullptr;
    s = stage_tma_operands(a_use, lda_use, m, b_use, ldb_use, n, k, &scratch, st);
    if (s != NGEMM_OK) {
        if (scratch) cudaFreeAsync(scratch, st);
        return s;
    }
    const int n_tiles = static_cast<int>((n + tcs::BN_ROWS - 1) / tcs::BN_ROWS);
    const int num_kb = static_cast<int>((k + tcs::BK - 1) / tcs::BK);
    // cluster size along K: a power of two <= 8 (so 128 divides evenly), enough CTAs for ~2 waves
    // about one CTA per SM, each streaming several K blocks (measured best on the c2 shapes)
    int want = std::max(1, (di.sms + n_tiles - 1) / n_tiles);
    if (opt(O_SKINNY_SPLITS) > 0) want = opt(O_SKINNY_SPLITS);
    int ks = 1;
    while (ks * 2 <= std::min(8, std::min(want, num_kb))) ks *= 2;
    const int kb_per = (num_kb + ks - 1) / ks;
    CUtensorMap tb, ta;
    s = make_tmap_u8(&tb, b_use, k, n, ldb_use, tcs::BK, tcs::BN_ROWS);
    if (s == NGEMM_OK) s = make_tmap_u8(&ta, a_use, k, m, lda_use, tcs::BK, tcs::MPAD);
    if (s == NGEMM_OK) {
        cudaError_t e = launch_k(kern, dim3(n_tiles, ks), dim3(tcs::THREADS), S::TOTAL, st, 1, ks, tb, ta, c, ldc,
                                 static_cast<int>(m), static_cast<int>(n), num_kb, kb_per);
        if (e != cudaSuccess) s = fail(NGEMM_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(e));
        else g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    if (scratch) cudaFreeAsync(scratch, st);
    return s;
}

// Warp-MMA load-stream variant (skinny_mma_kernel, exact mode): 16 B-rows per row group, the
// CTA's 8/16/32 warps split K so that ~32 warps per SM are streaming; a grid K split (atomic
// wrap-add into a zeroed C) only when even 32 warps per row group are not enough.
// Skinny kernels' `vec_ok` argument: bit 0 = operands allow 16-byte vector loads, bit 1 = also
// warm L2 with the CTA's operand rows before the PDL dependency wait (NGEMM_L2_PREFETCH=0 off),
// bit 2 = whole in-range chunks take the branch-free load path (NGEMM_SKINNY_FAST=0 off).
bool l2_prefetch_enabled() { return opt(O_L2_PREFETCH) != 0; }

int skinny_vec_flags(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb, const Batch& bt) {
    const bool vec = reinterpret_cast<uintptr_t>(b) % 16 == 0 && ldb % 16 == 0 &&
                     reinterpret_cast<uintptr_t>(a) % 16 == 0 && lda % 16 == 0 && bt.sa % 16 == 0 && bt.sb % 16 == 0;
    const bool fast = opt(O_SKINNY_FAST) != 0;
    return vec ? (1 | (l2_prefetch_enabled() ? 2 : 0) | (fast ? 4 : 0)) : 0;
}

template <int MT, int WARPS, int RG = 1>
ngemm_status launch_skinny_mma_w(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb, int32_t* c,
                                 int64_t ldc, int64_t m, int64_t n, int64_t k, int64_t splits, const DevInfo& di,
                                 cudaStream_t st, const Batch& bt, const Requant& rq = Requant()) {
    const int64_t groups = (n + 16 * RG - 1) / (16 * RG);
    if (rq.out != nullptr) splits = 1;  // the requantised value needs the whole K sum
    const int64_t k_range = round_up((k + splits - 1) / splits, skinny_mma::CHUNK);
    splits = (k + k_range - 1) / k_range;
    // Two K splits of one row group run as a 2-CTA cluster and meet through DSMEM (no zeroing pass,
    // no atomics: 16x768x3072 4.95 -> 4.35 us); 4- and 8-CTA clusters schedule too slowly (16x256x16384
    // 8.6 vs 5.1 us, profiles/r2/skinny_xred_ab_r2.log), so more splits wrap-add into a zeroed C.
    // SKINNY_XRED=2 forces the cluster for up to 8 splits (tests).
    const bool xred = RG == 1 && splits > 1 && (splits == 2 || (splits <= 8 && opt(O_SKINNY_XRED) == 2)) &&
                      opt(O_SKINNY_XRED) != 0;
    for (int z = 0; z < bt.count && splits > 1 && !xred; ++z) {
        ngemm_status zs = zero_c(c + z * bt.sc, ldc, m, n, st);
        if (zs != NGEMM_OK) return zs;
    }
    const int vec = skinny_vec_flags(a, lda, b, ldb, bt);
    NG_LAUNCH(skinny_mma_kernel<MT, RG, WARPS>,
              dim3(static_cast<unsigned>(groups), static_cast<unsigned>(splits), static_cast<unsigned>(bt.count)),
              dim3(WARPS * 32), 0, st, 1, xred ? static_cast<unsigned>(splits) : 1u, a, lda, b, ldb, c, ldc,
              static_cast<int>(m), n, k, k_range, vec, xred ? 2 : (splits > 1 ? 1 : 0), bt.sa, bt.sb, bt.sc, rq);
    return NGEMM_OK;
}

template <int MT>
ngemm_status launch_skinny_mma_t(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb, int32_t* c,
                                 int64_t ldc, int64_t m, int64_t n, int64_t k, const DevInfo& di, cudaStream_t st,
                                 const Batch& bt = Batch(), const Requant& rq = Requant()) {
    const int64_t groups = (n + 15) / 16 * bt.count;  // CTAs of all GEMMs of the batch fill the SMs
    const int64_t chunks = (k + skinny_mma::CHUNK - 1) / skinny_mma::CHUNK;
    const int64_t warps_target = static_cast<int64_t>(di.sms) * 32;
    const int64_t ks = std::max<int64_t>(1, std::min<int64_t>(chunks, (warps_target + groups - 1) / groups));
    int64_t splits = 1;
    if (opt(O_SKINNY_SPLITS) > 0) splits = opt(O_SKINNY_SPLITS);
    // Row groups per CTA (RG, 8 warps): a single skinny GEMM has too few 16-row groups to fill
    // 148 SMs, so RG = 1 and the warps split K; a batch (or a very wide N) has CTAs to spare, so
    // each CTA takes RG groups and its warps stream longer K runs — fewer CTA launches and K
    // reductions per byte.  Measured on B200 (profiles/batched_skinny_r1.log): M > 8 wants the
    // largest RG that still leaves >= 4 CTAs per SM; M <= 8 wants ~128 KB of B per CTA.
    int rg = 1;
    {
        const int64_t row_groups = (n + 15) / 16 * bt.count;
        const int64_t min_ctas = 4 * static_cast<int64_t>(di.sms);
        for (int r : {2, 4, 8}) {
            if (row_groups / r < min_ctas) break;
            if (m <= 8 && static_cast<int64_t>(rg) * 16 * k >= (128 << 10)) break;
            rg = r;
        }
    }
    if (opt(O_SKINNY_RG) > 0) rg = opt(O_SKINNY_RG);  // experiments
    // MT = 16 in a 1024-thread CTA is capped at 64 registers and spills: 16 warps at most
    // (16 x 768 x 3072: 4.6 -> 3.85 us, profiles/sweep_skinny_warps_r1.log)
    int64_t ks_use = MT >= 16 ? std::min<int64_t>(ks, 16) : ks;
    if (opt(O_SKINNY_WARPS) > 0) ks_use = opt(O_SKINNY_WARPS);  // experiments: 8 / 16 / 32
    // warps capped below the K chunks wanted (MT = 16): split K over the grid instead, so deep-K /
    // narrow-N shapes (16 x 256 x 16384) still put ~32 streaming warps on every SM
    if (splits == 1 && rq.out == nullptr && ks_use < ks && ks_use >= 8 && ks_use <= 16 && opt(O_SKINNY_WARPS) <= 0)
        splits = (ks + ks_use - 1) / ks_use;
    if (rg == 2) return launch_skinny_mma_w<MT, 8, 2>(a, lda, b, ldb, c, ldc, m, n, k, splits, di, st, bt, rq);
    if (rg == 4) return launch_skinny_mma_w<MT, 8, 4>(a, lda, b, ldb, c, ldc, m, n, k, splits, di, st, bt, rq);
    if (rg == 8) return launch_skinny_mma_w<MT, 8, 8>(a, lda, b, ldb, c, ldc, m, n, k, splits, di, st, bt, rq);
    if (ks_use <= 8) return launch_skinny_mma_w<MT, 8>(a, lda, b, ldb, c, ldc, m, n, k, splits, di, st, bt, rq);
    if (ks_use <= 16) return launch_skinny_mma_w<MT, 16>(a, lda, b, ldb, c, ldc, m, n, k, splits, di, st, bt, rq);
    if (ks > 32 && splits == 1 && rq.out == nullptr) splits = (ks + 31) / 32;
    return launch_skinny_mma_w<MT, 32>(a, lda, b, ldb, c, ldc, m, n, k, splits, di, st, bt, rq);
}

// Saturating load-stream variant (skinny_sat_kernel): 16 B-rows per CTA, 8/16/32 warps split
// the K range; the work is CUDA-core (ALU) bound for larger M, so a grid K split (atomic
// wrap-add into a zeroed C) spreads it over every SM when there are few row groups.
template <int MT, int WARPS, bool MSPLIT>
ngemm_status launch_skinny_sat_w(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb, int32_t* c,
                                 int64_t ldc, int64_t m, int64_t n, int64_t k, int64_t splits, const DevInfo& di,
                                 cudaStream_t st, const Batch& bt) {
    const int64_t groups = (n + 15) / 16;
    const int64_t k_range = round_up((k + splits - 1) / splits, 128);
    splits = (k + k_range - 1) / k_range;
    for (int z = 0; z < bt.count && splits > 1; ++z) {
        ngemm_status zs = zero_c(c + z * bt.sc, ldc, m, n, st);
        if (zs != NGEMM_OK) return zs;
    }
    const int vec = skinny_vec_flags(a, lda, b, ldb, bt);
    // B-side pair masks (fewer instructions, more registers) for single latency-bound GEMMs;
    // A-side masks for one A row, 64-register CTAs and batches (occupancy-bound)
    constexpr bool bmask_ok = MT > 1 && !(MT <= 4 && WARPS >= 32);
    if (bmask_ok && bt.count == 1)
        NG_LAUNCH(skinny_sat_kernel<MT, WARPS, MSPLIT, bmask_ok>,
                  dim3(static_cast<unsigned>(groups), static_cast<unsigned>(splits), static_cast<unsigned>(bt.count)),
                  dim3(WARPS * 32), 0, st, 1, 1, a, lda, b, ldb, c, ldc, static_cast<int>(m), n, k, k_range, vec,
                  splits > 1 ? 1 : 0, bt.sa, bt.sb, bt.sc);
    else
        NG_LAUNCH(skinny_sat_kernel<MT, WARPS, MSPLIT, false>,
                  dim3(static_cast<unsigned>(groups), static_cast<unsigned>(splits), static_cast<unsigned>(bt.count)),
                  dim3(WARPS * 32), 0, st, 1, 1, a, lda, b, ldb, c, ldc, static_cast<int>(m), n, k, k_range, vec,
                  splits > 1 ? 1 : 0, bt.sa, bt.sb, bt.sc);
    return NGEMM_OK;
}

template <int MT>
ngemm_status launch_skinny_sat_t(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb, int32_t* c,
                                 int64_t ldc, int64_t m, int64_t n, int64_t k, const DevInfo& di, cudaStream_t st,
                                 const Batch& bt = Batch()) {
    const int64_t groups = (n + 15) / 16 * bt.count;
    const int64_t chunks = (k + 127) / 128;
    // Few 16-row groups x K chunks (< 4 warps per SM): split A's rows over warps too (MSPLIT),
    // else one warp per K slice (profiles/r2/skinny_sat_r2.log)
    if (MT > 4 && groups * chunks < 4 * static_cast<int64_t>(di.sms)) {
        constexpr int MS = MT > 4 ? MT / 4 : 1;
        const int64_t want = static_cast<int64_t>(di.sms) * 24;
        const int64_t ks = std::max<int64_t>(1, std::min<int64_t>(chunks, (want + groups * MS - 1) / (groups * MS)));
        int warps = ks * MS <= 8 ? 8 : 16;
        if (opt(O_SKINNY_WARPS) > 0) warps = opt(O_SKINNY_WARPS);  // experiments: 8 / 16 / 32
        const int64_t kw = warps / MS;
        const int64_t splits = std::max<int64_t>(1, (ks + kw - 1) / kw);
        if (warps >= 32) return launch_skinny_sat_w<MT, 32, true>(a, lda, b, ldb, c, ldc, m, n, k, splits, di, st, bt);
        if (warps >= 16) return launch_skinny_sat_w<MT, 16, true>(a, lda, b, ldb, c, ldc, m, n, k, splits, di, st, bt);
        return launch_skinny_sat_w<MT, 8, true>(a, lda, b, ldb, c, ldc, m, n, k, splits, di, st, bt);
    }
    const int64_t want = static_cast<int64_t>(di.sms) * (MT >= 8 ? 16 : 32);  // resident warps to fill
    const int64_t ks = std::max<int64_t>(1, std::min<int64_t>(chunks, (want + groups - 1) / groups));
    constexpr int WMAX = MT >= 8 ? 16 : 32;  // 1024-thread CTAs cap registers at 64: spills for MT >= 8
    if (ks <= 8) return launch_skinny_sat_w<MT, 8, false>(a, lda, b, ldb, c, ldc, m, n, k, 1, di, st, bt);
    if (ks <= 16 || WMAX == 16)
        return launch_skinny_sat_w<MT, 16, false>(a, lda, b, ldb, c, ldc, m, n, k, (ks + 15) / 16, di, st, bt);
    return launch_skinny_sat_w<MT, 32, false>(a, lda, b, ldb, c, ldc, m, n, k, (ks + 31) / 32, di, st, bt);
}

// Saturating tensor-core + sparse-fix variant (skinny_sathyb_kernel, 4 < M <= 16): one 16-row group
// of B per CTA, 8 or 16 warps splitting K like the exact warp-MMA stream, a grid K split when
// even 16 warps per row group leave SMs short of streaming warps.
template <int MT, int WARPS>
ngemm_status launch_skinny_sathyb_w(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb, int32_t* c,
                                    int64_t ldc, int64_t m, int64_t n, int64_t k, int64_t splits, cudaStream_t st,
                                    const Batch& bt) {
    using S = skinny_sathyb::Smem<MT, WARPS>;
    auto kern = skinny_sathyb_kernel<MT, WARPS>;
    static std::once_flag once[64];
    int dev = 0;
    cudaGetDevice(&dev);
    ngemm_status s = NGEMM_OK;
    // no shared-memory carveout preference: A is re-read through L1
    if (S::TOTAL > 48 * 1024)
        std::call_once(once[dev & 63], [&] {
            if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::TOTAL) != cudaSuccess)
                s = fail(NGEMM_ERR_CUDA, "cudaFuncSetAttribute(skinny_sathyb) failed");
        });
    if (s != NGEMM_OK) return s;
    const int64_t groups = (n + 15) / 16;
    const int64_t k_range = round_up((k + splits - 1) / splits, skinny_mma::CHUNK);
    splits = (k + k_range - 1) / k_range;
    // cluster reduction for two splits, as in the exact stream
    const bool xred = splits > 1 && (splits == 2 || (splits <= 8 && opt(O_SKINNY_XRED) == 2)) && opt(O_SKINNY_XRED) != 0;
    for (int z = 0; z < bt.count && splits > 1 && !xred; ++z) {
        ngemm_status zs = zero_c(c + z * bt.sc, ldc, m, n, st);
        if (zs != NGEMM_OK) return zs;
    }
    const int vec = skinny_vec_flags(a, lda, b, ldb, bt);
    NG_LAUNCH(kern, dim3(static_cast<unsigned>(groups), static_cast<unsigned>(splits), static_cast<unsigned>(bt.count)),
              dim3(WARPS * 32), S::TOTAL, st, 1, xred ? static_cast<unsigned>(splits) : 1u, a, lda, b, ldb, c, ldc,
              static_cast<int>(m), n, k, k_range, vec, xred ? 2 : (splits > 1 ? 1 : 0), bt.sa, bt.sb, bt.sc);
    return NGEMM_OK;
}

template <int MT>
ngemm_status launch_skinny_sathyb_t(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb, int32_t* c,
                                    int64_t ldc, int64_t m, int64_t n, int64_t k, const DevInfo& di, cudaStream_t st,
                                    const Batch& bt = Batch()) {
    const int64_t groups = (n + 15) / 16 * bt.count;
    const int64_t chunks = (k + skinny_mma::CHUNK - 1) / skinny_mma::CHUNK;
    const int64_t warps_target = static_cast<int64_t>(di.sms) * 32;
    const int64_t ks = std::max<int64_t>(1, std::min<int64_t>(chunks, (warps_target + groups - 1) / groups));
    int64_t splits = 1;
    if (opt(O_SKINNY_SPLITS) > 0) splits = opt(O_SKINNY_SPLITS);
    int64_t ks_use = std::min<int64_t>(ks, 16);
    if (opt(O_SKINNY_WARPS) > 0) ks_use = opt(O_SKINNY_WARPS);
    if (splits == 1 && ks_use < ks && opt(O_SKINNY_WARPS) <= 0) splits = (ks + ks_use - 1) / ks_use;
    if (ks_use <= 8) return launch_skinny_sathyb_w<MT, 8>(a, lda, b, ldb, c, ldc, m, n, k, splits, st, bt);
    return launch_skinny_sathyb_w<MT, 16>(a, lda, b, ldb, c, ldc, m, n, k, splits, st, bt);
}

// Lanes-own-rows variant (skinny_rows_kernel): 32-row tiles of B x K splits.
template <int MODE, int MT>
ngemm_status launch_skinny_rows_t(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb, int32_t* c,
                                  int64_t ldc, int64_t m, int64_t n, int64_t k, const DevInfo& di, cudaStream_t st) {
    const int64_t row_tiles = (n + 31) / 32;
    const int64_t max_splits = std::max<int64_t>(1, (k + 255) / 256);
    int64_t splits = std::min<int64_t>(max_splits, std::max<int64_t>(1, (2 * di.sms + row_tiles - 1) / row_tiles));
    int64_t k_range = round_up((k + splits - 1) / splits, 256);
    splits = (k + k_range - 1) / k_range;
    const int smem = static_cast<int>(std::max<int64_t>(MT * k_range, 8 * MT * 32 * 4));
    auto kern = skinny_rows_kernel<MODE, MT>;
    if (smem > 48 * 1024) {
        ngemm_status s = set_smem(kern, smem);
        if (s != NGEMM_OK) return s;
    }
    if (splits > 1) {
        if (ldc == n) NG_CUDA(cudaMemsetAsync(c, 0, static_cast<size_t>(m * n) * 4, st));
        else NG_CUDA(cudaMemset2DAsync(c, static_cast<size_t>(ldc) * 4, 0, static_cast<size_t>(n) * 4, m, st));
    }
    const int b_vec = (reinterpret_cast<uintptr_t>(b) % 16 == 0 && ldb % 16 == 0);
    dim3 grid(static_cast<unsigned>(row_tiles), static_cast<unsigned>(splits));
    NG_LAUNCH(kern, grid, dim3(skinny_rows::THREADS), smem, st, 1, 1, a, lda, b, ldb, c, ldc, static_cast<int>(m), n, k,
              k_range, b_vec, splits > 1 ? 1 : 0);
    return NGEMM_OK;
}

template <int MODE>
ngemm_status launch_skinny_rows_mode(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb, int32_t* c,
                                     int64_t ldc, int64_t m, int64_t n, int64_t k, const DevInfo& di,
                                     cudaStream_t st) {
    if (m <= 1) return launch_skinny_rows_t<MODE, 1>(a, lda, b, ldb, c, ldc, m, n, k, di, st);
    if (m <= 2) return launch_skinny_rows_t<MODE, 2>(a, lda, b, ldb, c, ldc, m, n, k, di, st);
    if (m <= 4) return launch_skinny_rows_t<MODE, 4>(a, lda, b, ldb, c, ldc, m, n, k, di, st);
    if (m <= 8) return launch_skinny_rows_t<MODE, 8>(a, lda, b, ldb, c, ldc, m, n, k, di, st);
    return launch_skinny_rows_t<MODE, 16>(a, lda, b, ldb, c, ldc, m, n, k, di, st);
}

ngemm_status launch_skinny(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb, int32_t* c, int64_t ldc,
                           int64_t m, int64_t n, int64_t k, int mode, const DevInfo& di, cudaStream_t st) {
    if (m > kSkinnyMaxM) return fail(NGEMM_ERR_UNSUPPORTED, "skinny path needs M <= 16");
    // Measured on B200 (profiles/sweep_r1_skinny*.log): exact -> the warp-MMA load stream (3),
    // fastest on 11 of the 12 c2 shapes (1.9-4.5 us; the tcgen05 swap-AB kernel (2) pays
    // ~1 us more for TMEM/mbarrier/cluster setup); saturating -> the dp4a load stream (4),
    // which since the pack-saturate step also beats the broadcast kernel (1) on every
    // M > 4, N < 2048 shape (profiles/sweep_r1_skinny_sat_variants.log).
    // Saturating, 8 < M <= 16: warp MMAs + sparse fix (5) — 1.4-1.8x faster than the dp4a stream on
    // weight-like B (config 2's sigma = 32: ~0.4 % of the pairs can clamp), 1.1-1.4x slower when
    // most pairs can (uniform int8 B takes its dense branch); NGEMM_SKINNY_VARIANT=4 or a tune-store
    // entry selects the dp4a stream (profiles/r2/skinny_sathyb_r2.log).
    int variant = mode == NGEMM_SAT_EXACT ? 3 : (m > 8 ? 5 : 4);
    if (opt(O_SKINNY_VARIANT) >= 0) variant = opt(O_SKINNY_VARIANT);  // experiments
    if (t_force.skinny_variant >= 0) variant = t_force.skinny_variant;
    if (variant == 2 && mode == NGEMM_SAT_EXACT) return launch_tc_skinny(a, lda, b, ldb, c, ldc, m, n, k, di, st);
    if (variant == 4 && mode != NGEMM_SAT_EXACT) {
        if (m <= 1) return launch_skinny_sat_t<1>(a, lda, b, ldb, c, ldc, m, n, k, di, st);
        if (m <= 4) return launch_skinny_sat_t<4>(a, lda, b, ldb, c, ldc, m, n, k, di, st);
        if (m <= 8) return launch_skinny_sat_t<8>(a, lda, b, ldb, c, ldc, m, n, k, di, st);
        return launch_skinny_sat_t<16>(a, lda, b, ldb, c, ldc, m, n, k, di, st);
    }
    if (variant == 5 && mode != NGEMM_SAT_EXACT)
        return m <= 8 ? launch_skinny_sathyb_t<8>(a, lda, b, ldb, c, ldc, m, n, k, di, st)
                      : launch_skinny_sathyb_t<16>(a, lda, b, ldb, c, ldc, m, n, k, di, st);
    if (variant == 3 && mode == NGEMM_SAT_EXACT)
        return m <= 8 ? launch_skinny_mma_t<8>(a, lda, b, ldb, c, ldc, m, n, k, di, st)
                      : launch_skinny_mma_t<16>(a, lda, b, ldb, c, ldc, m, n, k, di, st);
    if (variant == 0) {
        if (!skinny_fits(m, k)) return fail(NGEMM_ERR_UNSUPPORTED, "skinny butterfly variant needs A resident in smem");
        return mode == NGEMM_SAT_EXACT ? launch_skinny_mode<1>(a, lda, b, ldb, c, ldc, m, n, k, di, st)
                                       : launch_skinny_mode<0>(a, lda, b, ldb, c, ldc, m, n, k, di, st);
    }
    return mode == NGEMM_SAT_EXACT ? launch_skinny_rows_mode<1>(a, lda, b, ldb, c, ldc, m, n, k, di, st)
                                   : launch_skinny_rows_mode<0>(a, lda, b, ldb, c, ldc, m, n, k, di, st);
}

// 2-D int32 C [rows x cols] with row stride ldc elements, 32 x 32 boxes, SWIZZLE_128B (the
// epilogue's staging layout).
ngemm_status make_tmap_c(CUtensorMap* map, const int32_t* c, int64_t rows, int64_t cols, int64_t ldc) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return fail(NGEMM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldc) * 4};
    cuuint32_t box[2] = {32, 32};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, const_cast<int32_t*>(c), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(NGEMM_ERR_CUDA, "cuTensorMapEncodeTiled(C) failed: " + std::to_string(r));
    return NGEMM_OK;
}

// Tile configurations of the tcgen05 kernel (per CTA: 128 rows of A; cta_group::2 pairs two SMs).
enum TcCfg {
    TC_PAIR256 = 0, TC_1CTA256 = 1, TC_1CTA128 = 2, TC_1CTA64 = 3, TC_QUAD256 = 4, TC_LEAN128 = 5, TC_LEAN64 = 6,
    TC_MC128 = 7, TC_MC64 = 8,  // 1-CTA tiles in 2-CTA clusters sharing A by TMA multicast
    TC_PAIR512 = 9,             // 256x512 per pair, one accumulator over all 512 TMEM columns
    TC_NUM_CFG = 10
};
struct TcCfgInfo {
    int cg, bn, mc;
    double cycles_per_kb;  // MMA issue floor per 128-byte K slab, with the smem-bandwidth cap
    int lean;              // <= ~100 KB smem and <= 256 TMEM columns: two CTAs fit on an SM
};
constexpr TcCfgInfo kTcCfg[TC_NUM_CFG] = {
    {2, 256, 1, 512.0, 0},  // 256x256x128 int8 per pair at 8192 MAC/clk/SM
    {1, 256, 1, 520.0, 0},  // 128x256: 96 B/clk of smem operand reads
    {1, 128, 1, 300.0, 0},  // 128x128: 128 B/clk, at the smem port limit
    {1, 64, 1, 192.0, 0},   // 128x64 : smem-bound (192 B/clk needed)
    {2, 256, 2, 512.0, 0},  // two pairs sharing A (multicast): 256x512 per 4-CTA cluster
    {1, 128, 1, 450.0, 1},  // 128x128, 2 stages: latency-limited stream, but co-resident
    {1, 64, 1, 330.0, 1},   // 128x64, 3 stages
    {1, 128, 2, 300.0, 0},  // 128x128 x 2 CTAs sharing A: half the A traffic into each SM
    {1, 64, 2, 192.0, 0},   // 128x64 x 2 CTAs sharing A
    {2, 512, 1, 1024.0, 0}, // 256x512x128 per pair: 96 KB of operands per 16.8 M MACs (pairs of 256x256: 128 KB)
};
// Lean configurations fit two CTAs per SM, so under PDL the next grid's CTAs finish their setup
// while the previous grid runs — but their 2-3 stage pipelines lose more in the K loop than the
// overlap saves (profiles/tc_trace_r1.log, sweep_tc_cfg_r1.log): the planner skips them; the
// autotuner still tries them.

struct TcPlan {
    int cfg, splits;
};

// The 4-CTA A-multicast configuration is correct (tests force it) but measured 37% slower on
// 16384^3 (profiles/quad_bench_r1.log: 4-CTA clusters leave SMs idle — 132 of 148 usable — and
// the two pairs' pipelines run in lockstep), so the planner only considers it with
// NGEMM_TC_QUAD=1.
bool quad_disabled() { return opt(O_TC_QUAD) != 1; }

// Picks the configuration with the smallest estimated makespan (waves x K-loop + epilogue),
// then adds split-K (TMA reduce-add) while waves stay under one and K is deep.
TcPlan plan_tcgen05(int64_t m, int64_t n, int64_t k, int sms, int c_mode_ok) {
    const int64_t num_kb = (k + tc::BK - 1) / tc::BK;
    TcPlan best{TC_PAIR256, 1};
    double best_t = 1e30;
    for (int cfg = 0; cfg < TC_NUM_CFG; ++cfg) {
        const TcCfgInfo& ci = kTcCfg[cfg];
        const int64_t tiles_n = (n + ci.bn - 1) / ci.bn;
        if (ci.mc > 1 && (tiles_n % ci.mc != 0 || quad_disabled())) continue;
        if (ci.lean) continue;
        if (cfg == TC_PAIR512) continue;  // chosen by the rule below the loop
        const int64_t tiles = ((m + 128 * ci.cg - 1) / (128 * ci.cg)) * tiles_n / ci.mc;
        const int64_t units = sms / (ci.cg * ci.mc);
        for (int splits = 1; splits <= 16; splits *= 2) {
            if (splits > 1 && (!c_mode_ok || num_kb < 4 * splits || tiles * splits > units)) break;
            const int64_t work = tiles * splits;
            const int64_t waves = (work + units - 1) / units;
            const double kb = static_cast<double>((num_kb + splits - 1) / splits);
            double t = static_cast<double>(waves) * kb * ci.cycles_per_kb + 600.0 + ci.bn * 8.0;
            if (splits > 1) t += 1500.0;                 // zeroing C + reduce-add traffic
            // pairs: less L2->SM traffic per MAC, but ~1000 cycles more fixed cost (cluster launch
            // and sync) — 2048^3: 128x256 1-CTA tiles 11.7 us vs pairs 12.9 (profiles/r2/ab_tc_cfg_r2.log)
            if (ci.cg == 2) t = t * 0.97 + 1000.0;
            if (ci.mc == 2) t *= 0.98;                    // A multicast: a further 25% less
            if (t < best_t) {
                best_t = t;
                best = {cfg, splits};
            }
        }
    }
    // 256x512 pair tiles (one accumulator over all 512 TMEM columns): 25 % less L2->SM operand
    // traffic per MAC, but the epilogue no longer overlaps the next tile's MMAs (~7 us per tile) —
    // ahead for deep K and many waves (profiles/r2/pair512_ab_r2.log, pair512_ksweep_r2.log:
    // 16384^3 +5.5 %, 8192^3 +3 %, K = 4096 equal, K <= 2048 behind)
    if (best.cfg == TC_PAIR256 && best.splits == 1 && k >= 8192) {
        const int64_t units = sms / 2;
        const int64_t tm = (m + 255) / 256;
        const int64_t w256 = (tm * ((n + 255) / 256) + units - 1) / units;
        const int64_t w512 = (tm * ((n + 511) / 512) + units - 1) / units;
        if (w512 >= 4 && 2.0 * 0.95 * static_cast<double>(w512) < static_cast<double>(w256)) best.cfg = TC_PAIR512;
    }
    if (opt(O_TC_CFG) >= 0) best.cfg = opt(O_TC_CFG) % TC_NUM_CFG;  // experiments / tests

    if (opt(O_TC_SPLITS) > 0) best.splits = opt(O_TC_SPLITS);
    if (t_force.tc_cfg >= 0) best.cfg = t_force.tc_cfg % TC_NUM_CFG;
    if (t_force.tc_splits >= 1) best.splits = t_force.tc_splits;
    if (kTcCfg[best.cfg].mc > 1 && ((n + kTcCfg[best.cfg].bn - 1) / kTcCfg[best.cfg].bn) % kTcCfg[best.cfg].mc != 0)
        best.cfg = TC_PAIR256;  // multicast pairs need an even number of N tiles
    return best;
}

// Epilogue choice for an aligned, unsplit C: the TMA-store epilogue everywhere — direct 16-byte
// stores from registers (c_mode 3) measured 2-30 % slower even on single-wave grids
// (profiles/ab_direct_r1.log); NGEMM_TC_DIRECT=1 selects them for experiments.
bool direct_c_stores(int /*tiles*/, int /*units*/) { return opt(O_TC_DIRECT) != 0; }

// Operand formats and epilogue of one tcgen05 launch: the NGEMM path is u8 x s8 into C; the
// i16 path issues four launches over byte planes with mixed formats, shifting and adding into C.
struct TcOps {
    int a_signed = 0, b_signed = 1;
    int shift = 0;       // C (+)= acc << shift
    int accumulate = 0;  // 1: TMA reduce-add into C (C holds the previous planes' sum)
    // fused requantisation (c_mode 4): int8 out instead of C
    const float* rq_scale = nullptr;
    const int32_t* rq_bias = nullptr;
    int8_t* rq_out = nullptr;
    int64_t rq_ldo = 0;
    int rq_zp = 0;
};

template <int BN, int STAGES, int CG, int MC = 1>
ngemm_status launch_tc_t(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tbh, const CUtensorMap& tcmap, int32_t* c,
                         int64_t ldc, int64_t m, int64_t n, int64_t k, int splits, int c_mode, const DevInfo& di,
                         cudaStream_t st, const TcOps& ops) {
    using S = tc::Smem<BN, STAGES, CG>;
    auto kern = tc_gemm_kernel<BN, STAGES, CG, MC>;
    static std::once_flag once[64];
    int dev = 0;
    cudaGetDevice(&dev);
    ngemm_status s = NGEMM_OK;
    std::call_once(once[dev & 63], [&] { s = set_smem(kern, S::TOTAL); });
    if (s != NGEMM_OK) return s;
    TileMap map;
    map.tiles_m = static_cast<int>((m + tc::BM * CG - 1) / (tc::BM * CG));
    map.tiles_n = static_cast<int>((n + BN - 1) / BN) / MC;  // MC adjacent N tiles per cluster
    const int num_kb = static_cast<int>((k + tc::BK - 1) / tc::BK);
    const int tiles = map.tiles_m * map.tiles_n;
    // persistent units = clusters that can be resident at once: a cluster must fit in one GPC,
    // so with 4-CTA clusters (or 2-CTA ones on GPCs with an odd SM count) fewer than
    // SMs / cluster size are co-resident, and a grid sized SMs / cluster size would run its last
    // clusters as a second wave after the others finish
    static std::atomic<int> max_clusters[64] = {};
    int units = di.sms / (CG * MC);
    if (CG * MC > 1) {
        std::atomic<int>& mc = max_clusters[dev & 63];
        if (mc.load() == 0) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(static_cast<unsigned>(units * CG * MC));
            cfg.blockDim = dim3(tc::THREADS);
            cfg.dynamicSmemBytes = S::TOTAL;
            cudaLaunchAttribute attr;
            attr.id = cudaLaunchAttributeClusterDimension;
            attr.val.clusterDim.x = CG * MC;
            attr.val.clusterDim.y = 1;
            attr.val.clusterDim.z = 1;
            cfg.attrs = &attr;
            cfg.numAttrs = 1;
            int n_active = 0;
            if (cudaOccupancyMaxActiveClusters(&n_active, kern, &cfg) != cudaSuccess || n_active <= 0) {
                cudaGetLastError();
                n_active = units;
            }
            mc.store(n_active);
            if (std::getenv("NGEMM_VERBOSE"))
                std::fprintf(stderr, "ngemm: tc_gemm_kernel<%d,%d,%d,%d>: %d co-resident clusters of %d CTAs\n", BN,
                             STAGES, CG, MC, n_active, CG * MC);
        }
        units = std::min(units, mc.load());
    }
    // split-K needs the TMA reduce-add epilogue (C must be TMA-describable)
    map.splits = c_mode == 2 ? 1 : std::max(1, std::min(splits, num_kb));
    // raster group: as many M tiles as keep the group's A rows (group_m x 128*CG rows x K bytes)
    // within ~32 MiB of L2 — 16384^3: 8 (pairs), 8192^3: 16, K <= 4096: every M tile
    // (profiles/r2/ab_groupm_hint_r2.log: 8192^3 363 -> 356 us, 4096^3 55.6 -> 54.3 us, c5 unchanged)
    map.group_m = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>(map.tiles_m, (int64_t(32) << 20) / (static_cast<int64_t>(tc::BM) * CG * std::max<int64_t>(k, 1)))));
    // pre-issuing the first loads before the block sync measured slower (profiles/ab_preissue_r1.log)
    map.preissue = opt(O_TC_PREISSUE);  // experiments
    map.l2hint = opt(O_TC_L2HINT);      // experiments (default 7: A evict_last, B and C evict_first; profiles/r2/l2hint_r2.log)
    map.prefetch = l2_prefetch_enabled() ? 1 : 0;
    map.dbg = 0;
    map.trace_id = -1;
    map.a_signed = ops.a_signed;
    map.b_signed = ops.b_signed;
    map.shift = ops.shift;
    map.rq_scale = ops.rq_scale;
    map.rq_bias = ops.rq_bias;
    map.rq_out = ops.rq_out;
    map.rq_ldo = ops.rq_ldo;
    map.rq_zp = ops.rq_zp;
    if (ops.rq_out != nullptr) {
        c_mode = 4;  // the requantised value needs the whole K sum: no split
        map.splits = 1;
    }
#ifdef NGEMM_TRACE
    map.dbg = opt(O_TC_DBG);  // trace build only
    map.trace_id = g_trace_next++;
#endif
    if (opt(O_TC_GROUP_M) > 0) map.group_m = opt(O_TC_GROUP_M);  // experiments
    if (c_mode == 0 && map.splits == 1 && !ops.accumulate && direct_c_stores(tiles, units)) c_mode = 3;
    if (ops.accumulate) {
        c_mode = 1;  // C already holds a partial sum: every split reduce-adds into it
    } else if (map.splits > 1) {
        c_mode = 1;
        ngemm_status zs = zero_c(c, ldc, m, n, st);
        if (zs != NGEMM_OK) return zs;
    }
    // tail split (TileMap::full_tiles; TC_SCHED=1): a last wave less than half full runs as
    // half-width tiles.  Bit-exact, but measured neutral (4096^3 55.6 vs 55.7 us, c5 within noise,
    // profiles/r2/ab_tail_split_r2.log): the main waves are bound by L2->SM operand delivery, not
    // by per-SM MMA time, so the idle SMs of a short last wave cost little.  Off by default.
    map.full_tiles = tiles * map.splits;
    const int rem = tiles % units;
    if (MC == 1 && BN <= 256 && map.splits == 1 && rem > 0 && 2 * rem <= units && opt(O_TC_SCHED) == 1) map.full_tiles = tiles - rem;
    const int work = map.full_tiles + 2 * (tiles * map.splits - map.full_tiles);
    const int grid = std::min(work, units) * CG * MC;
    NG_LAUNCH(kern, dim3(grid), dim3(tc::THREADS), S::TOTAL, st, CG * MC, 1, ta, tb, tbh, tcmap, c, ldc,
              static_cast<int>(m), static_cast<int>(n), num_kb, map, c_mode);
    return NGEMM_OK;
}

ngemm_status launch_tcgen05(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb, int32_t* c, int64_t ldc,
                            int64_t m, int64_t n, int64_t k, const DevInfo& di, cudaStream_t st,
                            const TcOps& ops = TcOps()) {
    // TMA needs 16-byte aligned bases and strides (SURVEY.md §0 gotcha 3)
    const bool rq = ops.rq_out != nullptr;  // fused requantisation: no C, no split-K
    const bool c_tma = !rq && c_tma_ok(c, ldc, n);
    if (ops.accumulate && !c_tma) return fail(NGEMM_ERR_UNSUPPORTED, "tcgen05: accumulating epilogue needs a TMA-describable C");
    const uint8_t* a_use = a;
    const uint8_t* b_use = reinterpret_cast<const uint8_t*>(b);
    int64_t lda_use = lda, ldb_use = ldb;
    uint8_t* scratch = nullptr;
    {
        ngemm_status ss = stage_tma_operands(a_use, lda_use, m, b_use, ldb_use, n, k, &scratch, st);
        if (ss != NGEMM_OK) {
            if (scratch) cudaFreeAsync(scratch, st);
            return ss;
        }
    }
    const TcPlan plan = plan_tcgen05(m, n, k, di.sms, c_tma ? 1 : 0);
    const TcCfgInfo& ci = kTcCfg[plan.cfg];
    CUtensorMap ta, tb, tbh, tcm;
    std::memset(&tcm, 0, sizeof tcm);
    ngemm_status s = make_tmap_u8(&ta, a_use, k, m, lda_use, tc::BK, tc::BM / ci.mc);
    if (s == NGEMM_OK) s = make_tmap_u8(&tb, b_use, k, n, ldb_use, tc::BK, ci.bn / ci.cg);
    if (s == NGEMM_OK) s = make_tmap_u8(&tbh, b_use, k, n, ldb_use, tc::BK, ci.bn / (2 * ci.cg));  // tail half tiles
    if (s == NGEMM_OK && c_tma) s = make_tmap_c(&tcm, c, m, n, ldc);
    const int c_mode = c_tma ? 0 : 2;
    if (s == NGEMM_OK) {
        switch (plan.cfg) {
        case TC_PAIR256: s = launch_tc_t<256, 6, 2>(ta, tb, tbh, tcm, c, ldc, m, n, k, plan.splits, c_mode, di, st, ops); break;
        case TC_1CTA256: s = launch_tc_t<256, 4, 1>(ta, tb, tbh, tcm, c, ldc, m, n, k, plan.splits, c_mode, di, st, ops); break;
        case TC_1CTA128: s = launch_tc_t<128, 6, 1>(ta, tb, tbh, tcm, c, ldc, m, n, k, plan.splits, c_mode, di, st, ops); break;
        case TC_QUAD256: s = launch_tc_t<256, 6, 2, 2>(ta, tb, tbh, tcm, c, ldc, m, n, k, plan.splits, c_mode, di, st, ops); break;
        case TC_LEAN128: s = launch_tc_t<128, 2, 1>(ta, tb, tbh, tcm, c, ldc, m, n, k, plan.splits, c_mode, di, st, ops); break;
        case TC_LEAN64: s = launch_tc_t<64, 3, 1>(ta, tb, tbh, tcm, c, ldc, m, n, k, plan.splits, c_mode, di, st, ops); break;
        case TC_MC128: s = launch_tc_t<128, 6, 1, 2>(ta, tb, tbh, tcm, c, ldc, m, n, k, plan.splits, c_mode, di, st, ops); break;
        case TC_MC64: s = launch_tc_t<64, 8, 1, 2>(ta, tb, tbh, tcm, c, ldc, m, n, k, plan.splits, c_mode, di, st, ops); break;
        case TC_PAIR512: s = launch_tc_t<512, 4, 2>(ta, tb, tbh, tcm, c, ldc, m, n, k, plan.splits, c_mode, di, st, ops); break;
        default: s = launch_tc_t<64, 8, 1>(ta, tb, tbh, tcm, c, ldc, m, n, k, plan.splits, c_mode, di, st, ops); break;
        }
    }
    if (scratch) cudaFreeAsync(scratch, st);
    return s;
}

// Host rows of `k` bytes -> device rows of pitch `kp` (one 1-D copy when the pitches agree).
cudaError_t copy_rows_h2d(void* dst, int64_t kp, const void* src, int64_t k, int64_t rows, cudaStream_t st) {
    if (kp == k) return cudaMemcpyAsync(dst, src, static_cast<size_t>(rows * k), cudaMemcpyHostToDevice, st);
    return cudaMemcpy2DAsync(dst, kp, src, k, k, rows, cudaMemcpyHostToDevice, st);
}

// HardwareSaturating on the tensor cores (kernel_satfix.cuh), no host round trip:
//   1. sat_prep_a_kernel: max A -> guard[0], A in the fix kernel's pair-major tile layout
//   2. sat_prep_b_kernel: B_safe = B with the pairs that could clamp zeroed, B's tiles, the
//      per-row index lists of those pairs, per-tile-chunk counts, the total (guard[4..5])
//   3. tcgen05 on (A, B_safe): the exact sums of every pair that cannot clamp
//   4. sat_fix_kernel: adds the clamped sums of the listed pairs (exits at once if none)
// Used for M >= 256 and >= 1e9 MACs (profiles/sweep_sat_hybrid_r1.log): below that the chain's
// fixed cost (~20 us) loses to the dense CUDA-core kernel.  On uniform int8 B (~25 % of the
// pairs listed) it is 1.5-2.9x faster than the dense kernel, on weight-like B (sigma 32,
// ~0.4 %) 2.2-14x; rows whose pairs are all listed (config 4's extremes) take a list-free path
// (1.2x slower than the dense kernel there).
// NGEMM_SAT_HYBRID=1 forces the chain (tests), 0 disables it.
constexpr int64_t kSatHybridMinM = 256;
constexpr double kSatHybridMinWork = 1e9;
int sat_hybrid_env() { return opt(O_SAT_HYBRID); }

ngemm_status launch_sat_hybrid(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb, int32_t* c, int64_t ldc,
                               int64_t m, int64_t n, int64_t k, const DevInfo& di, cudaStream_t st) {
    using namespace satfix;
    const int64_t chunks = (k + CHUNK - 1) / CHUNK;
    const int64_t lds = chunks * CHUNK;  // B_safe pitch (TMA-describable, zero past k)
    const int64_t tn = (n + TN - 1) / TN, tm = (m + TM - 1) / TM;
    // one allocation: guard | flags (both zeroed) | L_t | A_pm | B_t | B_safe
    const size_t guard_b = 64, flags_b = round_up(static_cast<int64_t>(tn * chunks * 4), 256);
    const size_t lt_off = guard_b + flags_b, lt_b = static_cast<size_t>(tn * chunks) * L_TILE;
    const size_t apm_off = round_up(static_cast<int64_t>(lt_off + lt_b), 256), apm_b = static_cast<size_t>(tm * chunks) * A_TILE;
    const size_t bt_off = apm_off + apm_b, bt_b = static_cast<size_t>(tn * chunks) * B_TILE;
    const size_t bs_off = bt_off + bt_b, bs_b = static_cast<size_t>(n * lds);
    CUtensorMap tcm;
    ngemm_status s = make_tmap_c(&tcm, c, m, n, ldc);
    if (s != NGEMM_OK) return s;
    uint8_t* buf = nullptr;
    NG_CUDA(dev_alloc(&buf, bs_off + bs_b, st));
    int32_t* guard = reinterpret_cast<int32_t*>(buf);
    uint32_t* flags = reinterpret_cast<uint32_t*>(buf + guard_b);
    uint8_t* lt = buf + lt_off;
    uint32_t* apm = reinterpret_cast<uint32_t*>(buf + apm_off);
    uint8_t* bt = buf + bt_off;
    uint8_t* bsafe = buf + bs_off;
    if (cudaMemsetAsync(buf, 0, guard_b + flags_b, st) != cudaSuccess) s = fail(NGEMM_ERR_CUDA, "memset(guard) failed");
    const int va = (reinterpret_cast<uintptr_t>(a) % 16 == 0 && lda % 16 == 0);
    const int vb = (reinterpret_cast<uintptr_t>(b) % 16 == 0 && ldb % 16 == 0);
    auto launched = [&](cudaError_t e) {
        if (e != cudaSuccess) return fail(NGEMM_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(e));
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return NGEMM_OK;
    };
    // experiments only (timing probes): skip launches of the chain, results are then wrong
    const int skip = opt(O_SATFIX_SKIP);
    auto grid_for = [&](int64_t items) {
        return dim3(static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((items + 255) / 256, di.sms * 16))));
    };
    if (s == NGEMM_OK && !(skip & 1))
        s = launched(launch_k(sat_prep_a_kernel, grid_for(tm * chunks * 8 * (TM / 2)), dim3(256), 0, st, 1, 1, a, lda,
                              m, k, va, chunks, apm, guard));
    if (s == NGEMM_OK && !(skip & 2))
        s = launched(launch_k(sat_prep_b_kernel, grid_for(tn * chunks * TN * 16), dim3(256), 0, st, 1, 1, b, ldb, n, k,
                              vb, chunks, bsafe, lds, bt, lt, flags, guard));
    if (s == NGEMM_OK && !(skip & 8))
        s = launch_tcgen05(a, lda, reinterpret_cast<const int8_t*>(bsafe), lds, c, ldc, m, n, k, di, st);
    if (s == NGEMM_OK) {
        static std::once_flag once[64];
        int dev = 0;
        cudaGetDevice(&dev);
        std::call_once(once[dev & 63], [&] { s = set_smem(sat_fix_kernel, SMEM); });
    }
    if (s == NGEMM_OK && !(skip & 16)) {
        // Stream-K over (tile, chunk) units, one CTA per SM (kernel_satfix.cuh): every SM gets
        // the same number of chunk units whatever the tile count; a CTA's run may end one tile
        // and start the next, each segment closing with its own TMA reduce-add into C.
        const int64_t total = tn * tm * chunks;
        const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(total, di.sms));
        const int64_t total_pairs = tn * TN * chunks * (CHUNK / 2);  // listable (B row, pair) slots
        s = launched(launch_k(sat_fix_kernel, dim3(static_cast<unsigned>(grid)), dim3(THREADS), SMEM, st, 1, 1, tcm,
                              apm, bt, lt, flags, chunks, tn, total, total_pairs, guard));
    }
    cudaFreeAsync(buf, st);
    return s;
}

int pick(int64_t m, int64_t n, int64_t k, int mode) {
    if (m <= kSkinnyMaxM) return NGEMM_KERNEL_SKINNY;
    if (mode == NGEMM_SAT_EXACT) return NGEMM_KERNEL_TCGEN05;
    const int env = sat_hybrid_env();
    const bool big = m >= kSatHybridMinM && static_cast<double>(m) * n * k >= kSatHybridMinWork;
    return (env == 1 || (env != 0 && big)) ? NGEMM_KERNEL_SAT_HYBRID : NGEMM_KERNEL_SIMT;
}

bool tuned_lookup(int64_t m, int64_t n, int64_t k, int mode, Choice* out);

ngemm_status run_gemm(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb, int32_t* c, int64_t ldc, int64_t m,
                      int64_t n, int64_t k, int mode, int kernel, cudaStream_t st) {
    struct Restore {
        Choice saved = t_force;
        ~Restore() { t_force = saved; }
    } restore;
    if (kernel == NGEMM_KERNEL_AUTO) {
        Choice ch;
        if (tuned_lookup(m, n, k, mode, &ch)) {
            t_force = ch;
            kernel = ch.kernel;
        }
    }
    ngemm_status s = validate(a, lda, b, ldb, c, ldc, m, n, k, mode);
    if (s != NGEMM_OK) return s;
    int dev;
    DevInfo di;
    s = current_device(&dev, &di);
    if (s != NGEMM_OK) return s;
    const bool c_tma = c_tma_ok(c, ldc, n);  // the sat fix adds into C by TMA reduce
    if (kernel == NGEMM_KERNEL_AUTO) {
        kernel = pick(m, n, k, mode);
        if (kernel == NGEMM_KERNEL_SAT_HYBRID && !c_tma) kernel = NGEMM_KERNEL_SIMT;
    }
    switch (kernel) {
    case NGEMM_KERNEL_SAT_HYBRID:
        if (mode != NGEMM_SAT_HARDWARE) return fail(NGEMM_ERR_UNSUPPORTED, "sat_hybrid is the HardwareSaturating path");
        if (m <= kSkinnyMaxM) return fail(NGEMM_ERR_UNSUPPORTED, "sat_hybrid needs M > 16 (the skinny path covers M <= 16)");
        if (!c_tma) return fail(NGEMM_ERR_UNSUPPORTED, "sat_hybrid needs a 16-byte aligned C with ldc % 4 == 0 and N % 4 == 0");
        if (m > INT32_MAX - tc::BM || k > INT32_MAX - tc::BK) return fail(NGEMM_ERR_SHAPE, "sat_hybrid: dims too large");
        return launch_sat_hybrid(a, lda, b, ldb, c, ldc, m, n, k, di, st);
    case NGEMM_KERNEL_SIMT: return launch_simt(a, lda, b, ldb, c, ldc, m, n, k, mode, st);
    case NGEMM_KERNEL_SKINNY: return launch_skinny(a, lda, b, ldb, c, ldc, m, n, k, mode, di, st);
    case NGEMM_KERNEL_TCGEN05:
        if (mode != NGEMM_SAT_EXACT)
            return fail(NGEMM_ERR_UNSUPPORTED,
                        "tcgen05 computes exact int32 sums; HardwareSaturating needs the SIMT or skinny kernel");
        if (m > INT32_MAX - tc::BM || k > INT32_MAX - tc::BK) return fail(NGEMM_ERR_SHAPE, "tcgen05: dims too large");
        return launch_tcgen05(a, lda, b, ldb, c, ldc, m, n, k, di, st);
    default: return fail(NGEMM_ERR_CONFIG, "unknown kernel id " + std::to_string(kernel));
    }
}

// Strided batch: `count` independent GEMMs of one shape, operand z at base + z * stride.
// Skinny shapes (M <= 16) run as ONE launch whose grid.z walks the batch, so the CTAs of every
// GEMM fill the 148 SMs together and the launch latency is paid once (a single M <= 16 GEMM
// leaves most SMs idle and is latency-bound, profiles/floor_probe_r1.log); other shapes are
// issued back to back on the stream (each already fills the machine).  Strides of 0 on A or B
// broadcast one operand to the whole batch; C slices must not overlap.
ngemm_status run_gemm_batched(const uint8_t* a, int64_t lda, int64_t sa, const int8_t* b, int64_t ldb, int64_t sb,
                              int32_t* c, int64_t ldc, int64_t sc, int64_t count, int64_t m, int64_t n, int64_t k,
                              int mode, cudaStream_t st) {
    if (count < 0 || count > 65535) return fail(NGEMM_ERR_SHAPE, "batched: count must be in [0, 65535]");
    if (count == 0) return NGEMM_OK;
    ngemm_status s = validate(a, lda, b, ldb, c, ldc, m, n, k, mode);
    if (s != NGEMM_OK) return s;
    if (sa < 0 || sb < 0 || sc < 0) return fail(NGEMM_ERR_SHAPE, "batched: strides must be >= 0");
    if ((sa != 0 && sa < (m - 1) * lda + k) || (sb != 0 && sb < (n - 1) * ldb + k))
        return fail(NGEMM_ERR_SHAPE, "batched: a non-zero operand stride is smaller than one operand");
    if (count > 1 && sc < (m - 1) * ldc + n) return fail(NGEMM_ERR_SHAPE, "batched: C slices overlap");
    int dev;
    DevInfo di;
    s = current_device(&dev, &di);
    if (s != NGEMM_OK) return s;
    Choice ch;
    const bool tuned = tuned_lookup(m, n, k, mode, &ch);
    const int kernel = tuned ? ch.kernel : pick(m, n, k, mode);
    if (count > 1 && kernel == NGEMM_KERNEL_SKINNY && m <= kSkinnyMaxM && k <= INT32_MAX) {
        const Batch bt{static_cast<int>(count), sa, sb, sc};
        if (mode == NGEMM_SAT_EXACT)
            return m <= 8 ? launch_skinny_mma_t<8>(a, lda, b, ldb, c, ldc, m, n, k, di, st, bt)
                          : launch_skinny_mma_t<16>(a, lda, b, ldb, c, ldc, m, n, k, di, st, bt);
        if (m <= 1) return launch_skinny_sat_t<1>(a, lda, b, ldb, c, ldc, m, n, k, di, st, bt);
        if (m <= 4) return launch_skinny_sat_t<4>(a, lda, b, ldb, c, ldc, m, n, k, di, st, bt);
        if (m <= 8) return launch_skinny_sat_t<8>(a, lda, b, ldb, c, ldc, m, n, k, di, st, bt);
        if (opt(O_SKINNY_VARIANT) == 4) return launch_skinny_sat_t<16>(a, lda, b, ldb, c, ldc, m, n, k, di, st, bt);
        return launch_skinny_sathyb_t<16>(a, lda, b, ldb, c, ldc, m, n, k, di, st, bt);
    }
    for (int64_t z = 0; z < count; ++z) {
        s = run_gemm(a + z * sa, lda, b + z * sb, ldb, c + z * sc, ldc, m, n, k, mode, NGEMM_KERNEL_AUTO, st);
        if (s != NGEMM_OK) return s;
    }
    return NGEMM_OK;
}

// ---------------------------------------------------------------- packed weights
ngemm_status validate_meta(const ngemm_packed_meta* p) {
    if (!p) return fail(NGEMM_ERR_CONFIG, "null packed metadata");
    if (p->v * p->h != p->w || (p->h != 4 && p->h != 2) || p->v < 1)
        return fail(NGEMM_ERR_CONFIG, "pack: shape (w=" + std::to_string(p->w) + ",h=" + std::to_string(p->h) +
                                          ",v=" + std::to_string(p->v) + ") matches neither the u8 (h=4) nor the i16 (h=2) path");
    if (p->tm < p->v || p->tm % p->v != 0)
        return fail(NGEMM_ERR_CONFIG, "tile: tm=" + std::to_string(p->tm) + " is not a positive multiple of v");
    if (p->tk < p->h || p->tk % p->h != 0)
        return fail(NGEMM_ERR_CONFIG, "tile: tk=" + std::to_string(p->tk) + " is not a positive multiple of h");
    if (p->tn < 1) return fail(NGEMM_ERR_CONFIG, "tile: tn must be >= 1");
    if (p->perm < 0 || p->perm > 5) return fail(NGEMM_ERR_CONFIG, "unknown permutation tag");
    if (p->m_orig < 1 || p->k_orig < 1) return fail(NGEMM_ERR_SHAPE, "packed: dims must be >= 1");
    if (p->m_pad != round_up(p->m_orig, p->tm) || p->k_pad != round_up(p->k_orig, p->tk))
        return fail(NGEMM_ERR_SHAPE, "packed: padded dims disagree with tile metadata");
    return NGEMM_OK;
}

PackedGeom geom_of(const ngemm_packed_meta* p) {
    PackedGeom g;
    g.w = p->w;
    g.h = p->h;
    g.v = p->v;
    g.perm_m_before_k = (p->perm == 0 || p->perm == 1 || p->perm == 2) ? 1 : 0;
    g.tm = p->tm;
    g.tk = p->tk;
    g.m_pad = p->m_pad;
    g.k_pad = p->k_pad;
    g.m_orig = p->m_orig;
    g.k_orig = p->k_orig;
    return g;
}

ngemm_status repack_on(const ngemm_packed_meta* meta, const uint8_t* d_packed, uint8_t* d_a, int64_t lda,
                       cudaStream_t st) {
    ngemm_status s = validate_meta(meta);
    if (s != NGEMM_OK) return s;
    if (lda < meta->k_orig) return fail(NGEMM_ERR_SHAPE, "repack: lda < K");
    if (reinterpret_cast<uintptr_t>(d_packed) % 4 != 0) return fail(NGEMM_ERR_SHAPE, "repack: packed buffer must be 4-byte aligned");
    const int esize = meta->h == 4 ? 1 : 2;  // K-group of h elements = one 4-byte word
    const int64_t kwords = (meta->k_orig + meta->h - 1) / meta->h;
    const int64_t total = meta->m_orig * kwords;
    const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 32);
    NG_LAUNCH(repack_kernel, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, st, 1, 1, geom_of(meta), d_packed, d_a,
              lda * esize, kwords, esize);
    return NGEMM_OK;
}

// ---------------------------------------------------------------- tuned table
// NGEMM_TUNE_STORE=<path>: records saved by an earlier `ngemm tune` are loaded on first use.
struct TuneKey {
    int64_t m, n, k;
    int mode;
    bool operator<(const TuneKey& o) const {
        return std::tie(m, n, k, mode) < std::tie(o.m, o.n, o.k, o.mode);
    }
};
std::mutex g_tune_mu;
std::map<TuneKey, std::pair<Choice, ngemm_tune_record>> g_tuned;

bool tuned_lookup(int64_t m, int64_t n, int64_t k, int mode, Choice* out) {
    std::lock_guard<std::mutex> lk(g_tune_mu);
    if (g_tuned.empty()) return false;
    auto it = g_tuned.find(TuneKey{m, n, k, mode});
    if (it == g_tuned.end()) return false;
    *out = it->second.first;
    return true;
}

ngemm_status load_store_file(const char* path, int* loaded);

void autoload_tune_store() {
    static std::once_flag once;
    std::call_once(once, [] {
        const char* p = std::getenv("NGEMM_TUNE_STORE");
        if (p && *p) {
            std::ifstream probe(p);
            if (probe) load_store_file(p, nullptr);
        }
    });
}

void tuned_put(const ngemm_tune_record& r) {
    Choice ch;
    ch.kernel = r.kernel;
    ch.tc_cfg = r.tc_cfg;
    ch.tc_splits = r.tc_splits;
    ch.skinny_variant = r.skinny_variant;
    std::lock_guard<std::mutex> lk(g_tune_mu);
    g_tuned[TuneKey{r.m, r.n, r.k, r.sat_mode}] = {ch, r};
}

}  // namespace

struct ngemm_packed_dev {
    int device;
    uint8_t* d_a;
    int64_t lda, m, k;  // lda and k in elements
    int esize;          // 1 = u8 weight (u8 x i8 path), 2 = i16 weight (16-bit path)
};

namespace {

// i16 x i16 on the tensor cores: split both operands into byte planes (split_i16_kernel), then
// four int8 tcgen05 GEMMs with per-launch operand formats —
//   C  = lo(A).lo(B)                 u8 x u8
//   C += (lo(A).hi(B)) << 8          u8 x s8   (TMA reduce-add epilogue)
//   C += (hi(A).lo(B)) << 8          s8 x u8
//   C += (hi(A).hi(B)) << 16         s8 x s8
// exact mod 2^32 like the reference's wrapping pair accumulation (gemm.hpp:161-190).
ngemm_status launch_i16_tc(const int16_t* a, int64_t lda, const int16_t* b, int64_t ldb, int32_t* c, int64_t ldc,
                           int64_t m, int64_t n, int64_t k, const DevInfo& di, cudaStream_t st) {
    const int64_t kp = round_up(k, 16);
    uint8_t* planes = nullptr;
    NG_CUDA(dev_alloc(&planes, static_cast<size_t>(2 * (m + n) * kp), st));
    uint8_t* al = planes;
    uint8_t* ah = al + m * kp;
    uint8_t* bl = ah + m * kp;
    uint8_t* bh = bl + n * kp;
    ngemm_status s = NGEMM_OK;
    auto split = [&](const int16_t* x, int64_t ld, int64_t rows, uint8_t* lo, uint8_t* hi) {
        if (s != NGEMM_OK) return;
        const int vec = reinterpret_cast<uintptr_t>(x) % 16 == 0 && ld % 8 == 0;
        const int64_t work = rows * (kp / 8);
        const int blocks = static_cast<int>(std::min<int64_t>((work + 255) / 256, 8LL * di.sms));
        cudaError_t e = launch_k(split_i16_kernel, dim3(blocks), dim3(256), 0, st, 1, 1, x, ld, rows, k, kp, lo, hi, vec);
        if (e != cudaSuccess) s = fail(NGEMM_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(e));
        else g_launches.fetch_add(1, std::memory_order_relaxed);
    };
    split(a, lda, m, al, ah);
    split(b, ldb, n, bl, bh);
    struct Term {
        const uint8_t* x;
        const uint8_t* y;
        TcOps ops;
    };
    const Term terms[4] = {{al, bl, {0, 0, 0, 0}}, {al, bh, {0, 1, 8, 1}}, {ah, bl, {1, 0, 8, 1}}, {ah, bh, {1, 1, 16, 1}}};
    for (const Term& t : terms) {
        if (s != NGEMM_OK) break;
        s = launch_tcgen05(t.x, kp, reinterpret_cast<const int8_t*>(t.y), kp, c, ldc, m, n, kp, di, st, t.ops);
    }
    cudaFreeAsync(planes, st);
    return s;
}

// i16 GEMMs with at least this many MACs (and M > 16, TMA-describable C) use the tensor cores.
constexpr double kI16TensorMinWork = 1 << 22;

ngemm_status run_i16(const int16_t* a, int64_t lda, const int16_t* b, int64_t ldb, int32_t* c, int64_t ldc, int64_t m,
                     int64_t n, int64_t k, cudaStream_t st) {
    ngemm_status s = validate(a, lda, b, ldb, c, ldc, m, n, k, NGEMM_SAT_EXACT);
    if (s != NGEMM_OK) return s;
    int dev;
    DevInfo di;
    s = current_device(&dev, &di);
    if (s != NGEMM_OK) return s;
    const bool c_tma = c_tma_ok(c, ldc, n);
    bool tensor = c_tma && m > kSkinnyMaxM && static_cast<double>(m) * n * k >= kI16TensorMinWork &&
                  m <= INT32_MAX / 2 && k <= INT32_MAX / 4;
    if (opt(O_I16_PATH) >= 0) tensor = c_tma && opt(O_I16_PATH) == 1;  // tests
    if (tensor) return launch_i16_tc(a, lda, b, ldb, c, ldc, m, n, k, di, st);
    return launch_simt_i16(a, lda, b, ldb, c, ldc, m, n, k, st);
}

bool is_pinned(const void* p) {
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return attr.type == cudaMemoryTypeHost;
}

}  // namespace

#include "host_pipeline.cuh"

namespace {

// Host operands -> pooled device buffers (rows padded to 16 bytes for TMA) -> optional device
// repack of a packed weight -> GEMM -> host C.  esize selects the u8 x i8 or i16 x i16 path.
ngemm_status host_gemm(int esize, const ngemm_packed_meta* meta, const void* a_or_packed, size_t packed_bytes,
                       const void* b, int32_t* c, int64_t m, int64_t n, int64_t k, int sat_mode, int kernel) {
    int dev;
    DevInfo di;
    ngemm_status s = current_device(&dev, &di);
    if (s != NGEMM_OK) return s;
    const int64_t kb = k * esize;            // row bytes
    const int64_t kpb = round_up(kb, 16);    // padded row bytes
    const int64_t kp = kpb / esize;          // padded row elements
    const size_t p_bytes = meta ? packed_bytes : 0;
    const size_t a_bytes = static_cast<size_t>(m * kpb), b_bytes = static_cast<size_t>(n * kpb);
    const size_t c_bytes = static_cast<size_t>(m * n) * 4;
    const size_t a_off = round_up(static_cast<int64_t>(p_bytes), 256), b_off = a_off + round_up(a_bytes, 256),
                 c_off = b_off + round_up(b_bytes, 256);
    cudaStream_t st = cudaStreamPerThread;
    uint8_t* buf = nullptr;
    NG_CUDA(dev_alloc(&buf, c_off + c_bytes, st));
    bool ok = true;
    if (meta) {
        ok = cudaMemcpyAsync(buf, a_or_packed, p_bytes, cudaMemcpyHostToDevice, st) == cudaSuccess;
    } else {
        ok = copy_rows_h2d(buf + a_off, kpb, a_or_packed, kb, m, st) == cudaSuccess;
    }
    ok = ok && copy_rows_h2d(buf + b_off, kpb, b, kb, n, st) == cudaSuccess;
    s = ok ? NGEMM_OK : fail(NGEMM_ERR_CUDA, "host gemm: H2D copy failed");
    if (s == NGEMM_OK && meta) s = repack_on(meta, buf, buf + a_off, kp, st);
    if (s == NGEMM_OK) {
        int32_t* dc = reinterpret_cast<int32_t*>(buf + c_off);
        if (esize == 1)
            s = run_gemm(buf + a_off, kp, reinterpret_cast<const int8_t*>(buf + b_off), kp, dc, n, m, n, k, sat_mode,
                         kernel, st);
        else
            s = run_i16(reinterpret_cast<const int16_t*>(buf + a_off), kp,
                        reinterpret_cast<const int16_t*>(buf + b_off), kp, dc, n, m, n, k, st);
    }
    if (s == NGEMM_OK && cudaMemcpyAsync(c, buf + c_off, c_bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess)
        s = fail(NGEMM_ERR_CUDA, "host gemm: D2H copy failed");
    cudaFreeAsync(buf, st);
    if (cudaStreamSynchronize(st) != cudaSuccess && s == NGEMM_OK)
        s = fail(NGEMM_ERR_CUDA, std::string("host gemm: ") + cudaGetErrorString(cudaGetLastError()));
    return s;
}

}  // namespace

extern "C" {

int ngemm_cuda_abi_version(void) { return NGEMM_CUDA_ABI_VERSION; }

const char* ngemm_cuda_status_name(int s) {
    switch (s) {
    case NGEMM_OK: return "ok";
    case NGEMM_ERR_SHAPE: return "ShapeError";
    case NGEMM_ERR_UNSUPPORTED: return "UnsupportedError";
    case NGEMM_ERR_CONFIG: return "ConfigError";
    case NGEMM_ERR_RANGE: return "RangeError";
    case NGEMM_ERR_CORRUPTION: return "CorruptionError";
    case NGEMM_ERR_INDEX: return "IndexError";
    case NGEMM_ERR_CUDA: return "CudaError";
    case NGEMM_ERR_TUNE: return "TuneError";
    default: return "unknown";
    }
}

const char* ngemm_cuda_last_error(void) { return g_last_error.c_str(); }

uint64_t ngemm_cuda_launch_count(void) { return g_launches.load(); }

int ngemm_cuda_pick_kernel(int64_t m, int64_t n, int64_t k, int sat_mode) { return pick(m, n, k, sat_mode); }

ngemm_status ngemm_cuda_gemm_u8i8(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb, int32_t* c,
                                  int64_t ldc, int64_t m, int64_t n, int64_t k, int sat_mode, void* stream) {
    return run_gemm(a, lda, b, ldb, c, ldc, m, n, k, sat_mode, NGEMM_KERNEL_AUTO, static_cast<cudaStream_t>(stream));
}

ngemm_status ngemm_cuda_gemm_u8i8_strided_batched(const uint8_t* a, int64_t lda, int64_t stride_a, const int8_t* b,
                                                  int64_t ldb, int64_t stride_b, int32_t* c, int64_t ldc,
                                                  int64_t stride_c, int64_t batch, int64_t m, int64_t n, int64_t k,
                                                  int sat_mode, void* stream) {
    return run_gemm_batched(a, lda, stride_a, b, ldb, stride_b, c, ldc, stride_c, batch, m, n, k, sat_mode,
                            static_cast<cudaStream_t>(stream));
}

ngemm_status ngemm_cuda_gemm_u8i8_ex(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb, int32_t* c,
                                     int64_t ldc, int64_t m, int64_t n, int64_t k, int sat_mode, int kernel,
                                     void* stream) {
    return run_gemm(a, lda, b, ldb, c, ldc, m, n, k, sat_mode, kernel, static_cast<cudaStream_t>(stream));
}

ngemm_status ngemm_cuda_gemm_u8i8_requant(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb, int8_t* out,
                                          int64_t ldo, int64_t m, int64_t n, int64_t k, const float* scale,
                                          const int32_t* bias, int zero_point, int sat_mode, void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    ngemm_status s = validate(a, lda, b, ldb, out, ldo, m, n, k, sat_mode);
    if (s != NGEMM_OK) return s;
    if (!scale) return fail(NGEMM_ERR_SHAPE, "requant: null scale");
    int dev;
    DevInfo di;
    s = current_device(&dev, &di);
    if (s != NGEMM_OK) return s;
    const bool unfused = opt(O_REQUANT_UNFUSED) == 1;  // experiments: time the unfused form
    if (sat_mode == NGEMM_SAT_EXACT && m > kSkinnyMaxM && m <= INT32_MAX - tc::BM && k <= INT32_MAX - tc::BK &&
        !unfused) {
        TcOps ops;
        ops.rq_scale = scale;
        ops.rq_bias = bias;
        ops.rq_out = out;
        ops.rq_ldo = ldo;
        ops.rq_zp = zero_point;
        return launch_tcgen05(a, lda, b, ldb, nullptr, n, m, n, k, di, st, ops);
    }
    if (sat_mode == NGEMM_SAT_EXACT && m <= kSkinnyMaxM && !unfused) {
        Requant rq;
        rq.scale = scale;
        rq.bias = bias;
        rq.out = out;
        rq.ldo = ldo;
        rq.zp = zero_point;
        return m <= 8 ? launch_skinny_mma_t<8>(a, lda, b, ldb, nullptr, n, m, n, k, di, st, Batch(), rq)
                      : launch_skinny_mma_t<16>(a, lda, b, ldb, nullptr, n, m, n, k, di, st, Batch(), rq);
    }
    // the saturating mode: C in scratch, then the same arithmetic unfused
    int32_t* cbuf = nullptr;
    NG_CUDA(dev_alloc(&cbuf, static_cast<size_t>(m * n) * 4, st));
    s = run_gemm(a, lda, b, ldb, cbuf, n, m, n, k, sat_mode, NGEMM_KERNEL_AUTO, st);
    if (s == NGEMM_OK) {
        const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((m * n + 255) / 256, di.sms * 8));
        cudaError_t e = launch_k(requant_kernel, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, st, 1, 1, cbuf, n,
                                 m, n, scale, bias, zero_point, out, ldo);
        if (e != cudaSuccess) s = fail(NGEMM_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(e));
        else g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    cudaFreeAsync(cbuf, st);
    return s;
}

ngemm_status ngemm_cuda_packed_validate(const ngemm_packed_meta* meta) { return validate_meta(meta); }

ngemm_status ngemm_cuda_repack(const ngemm_packed_meta* meta, const uint8_t* d_packed, uint8_t* d_a, int64_t lda,
                               void* stream) {
    return repack_on(meta, d_packed, d_a, lda, static_cast<cudaStream_t>(stream));
}


ngemm_status ngemm_cuda_gemm_i16(const int16_t* a, int64_t lda, const int16_t* b, int64_t ldb, int32_t* c,
                                 int64_t ldc, int64_t m, int64_t n, int64_t k, void* stream) {
    return run_i16(a, lda, b, ldb, c, ldc, m, n, k, static_cast<cudaStream_t>(stream));
}

ngemm_status ngemm_cuda_packed_upload(const ngemm_packed_meta* meta, const uint8_t* host_packed, size_t nbytes,
                                      ngemm_packed_handle* out) {
    ngemm_status s = validate_meta(meta);
    if (s != NGEMM_OK) return s;
    if (!out || !host_packed) return fail(NGEMM_ERR_SHAPE, "packed_upload: null pointer");
    const int esize = meta->h == 4 ? 1 : 2;
    if (nbytes != static_cast<size_t>(meta->m_pad * meta->k_pad * esize))
        return fail(NGEMM_ERR_SHAPE, "packed_upload: byte size disagrees with m_pad*k_pad");
    int dev;
    DevInfo di;
    s = current_device(&dev, &di);
    if (s != NGEMM_OK) return s;
    const int64_t lda = round_up(meta->k_orig * esize, 16) / esize;
    const size_t a_bytes = static_cast<size_t>(meta->m_orig * lda * esize);
    uint8_t* d_packed = nullptr;
    uint8_t* d_a = nullptr;
    NG_CUDA(cudaMalloc(&d_packed, nbytes));
    if (cudaMalloc(&d_a, a_bytes) != cudaSuccess) {
        cudaFree(d_packed);
        return fail(NGEMM_ERR_CUDA, "packed_upload: out of device memory");
    }
    cudaStream_t st = nullptr;
    s = NGEMM_OK;
    if (cudaMemsetAsync(d_a, 0, a_bytes, st) != cudaSuccess ||
        cudaMemcpyAsync(d_packed, host_packed, nbytes, cudaMemcpyHostToDevice, st) != cudaSuccess)
        s = fail(NGEMM_ERR_CUDA, "packed_upload: copy failed");
    if (s == NGEMM_OK) s = repack_on(meta, d_packed, d_a, lda, st);
    if (s == NGEMM_OK && cudaStreamSynchronize(st) != cudaSuccess) s = fail(NGEMM_ERR_CUDA, "packed_upload: sync failed");
    cudaFree(d_packed);
    if (s != NGEMM_OK) {
        cudaFree(d_a);
        return s;
    }
    *out = new ngemm_packed_dev{dev, d_a, lda, meta->m_orig, meta->k_orig, esize};
    return NGEMM_OK;
}

ngemm_status ngemm_cuda_packed_from_device(const uint8_t* d_src, int64_t lda_src, int64_t m, int64_t k,
                                           ngemm_packed_handle* out) {
    if (!out || !d_src) return fail(NGEMM_ERR_SHAPE, "packed_from_device: null pointer");
    if (m < 1 || k < 1 || lda_src < k) return fail(NGEMM_ERR_SHAPE, "packed_from_device: bad shape");
    int dev;
    DevInfo di;
    ngemm_status s = current_device(&dev, &di);
    if (s != NGEMM_OK) return s;
    const int64_t lda = round_up(k, 16);
    uint8_t* d_a = nullptr;
    NG_CUDA(cudaMalloc(&d_a, static_cast<size_t>(m * lda)));
    if (cudaMemset(d_a, 0, static_cast<size_t>(m * lda)) != cudaSuccess ||
        cudaMemcpy2D(d_a, lda, d_src, lda_src, k, m, cudaMemcpyDeviceToDevice) != cudaSuccess) {
        cudaFree(d_a);
        return fail(NGEMM_ERR_CUDA, "packed_from_device: copy failed");
    }
    *out = new ngemm_packed_dev{dev, d_a, lda, m, k, 1};
    return NGEMM_OK;
}

ngemm_status ngemm_cuda_packed_free(ngemm_packed_handle h) {
    if (!h) return NGEMM_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(h->device);
    cudaFree(h->d_a);
    cudaSetDevice(prev);
    delete h;
    return NGEMM_OK;
}

ngemm_status ngemm_cuda_packed_info(ngemm_packed_handle h, const uint8_t** d_a, int64_t* lda, int64_t* m, int64_t* k,
                                    int* device) {
    if (!h) return fail(NGEMM_ERR_SHAPE, "null handle");
    if (d_a) *d_a = h->d_a;
    if (lda) *lda = h->lda;
    if (m) *m = h->m;
    if (k) *k = h->k;
    if (device) *device = h->device;
    return NGEMM_OK;
}

ngemm_status ngemm_cuda_gemm_packed(ngemm_packed_handle h, const int8_t* b, int64_t ldb, int32_t* c, int64_t ldc,
                                    int64_t n, int sat_mode, void* stream) {
    if (!h) return fail(NGEMM_ERR_SHAPE, "null handle");
    if (h->esize != 1) return fail(NGEMM_ERR_UNSUPPORTED, "gemm_packed: i16 weight needs an i16 input (gemm_packed_i16)");
    return run_gemm(h->d_a, h->lda, b, ldb, c, ldc, h->m, n, h->k, sat_mode, NGEMM_KERNEL_AUTO,
                    static_cast<cudaStream_t>(stream));
}

ngemm_status ngemm_cuda_gemm_packed_i16(ngemm_packed_handle h, const int16_t* b, int64_t ldb, int32_t* c, int64_t ldc,
                                        int64_t n, void* stream) {
    if (!h) return fail(NGEMM_ERR_SHAPE, "null handle");
    if (h->esize != 2) return fail(NGEMM_ERR_UNSUPPORTED, "gemm_packed_i16: u8 weight needs an i8 input");
    return run_i16(reinterpret_cast<const int16_t*>(h->d_a), h->lda, b, ldb, c, ldc, h->m, n, h->k,
                   static_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------- host-pointer entries
ngemm_status ngemm_cuda_gemm_u8i8_host(const uint8_t* a, const int8_t* b, int32_t* c, int64_t m, int64_t n, int64_t k,
                                       int sat_mode, int kernel) {
    ngemm_status s = validate(a, k, b, k, c, n, m, n, k, sat_mode);
    if (s != NGEMM_OK) return s;
    int dev;
    DevInfo di;
    s = current_device(&dev, &di);
    if (s != NGEMM_OK) return s;
    // big problems: overlap H2D / compute / D2H over a grid of C tiles (pageable operands move
    // through pinned staging slots)
    if (pipeline_worth(m, n, k)) {
        HostGemm g;
        g.a_host = a;
        g.b_host = b;
        g.c_host = c;
        g.a_pinned = is_pinned(a);
        g.b_pinned = is_pinned(b);
        g.c_pinned = is_pinned(c);
        g.m = m;
        g.n = n;
        g.k = k;
        g.mode = sat_mode;
        g.kernel = kernel;
        s = host_pipeline(g);
        if (s != NGEMM_ERR_UNSUPPORTED) return s;
    }
    return host_gemm(1, nullptr, a, 0, b, c, m, n, k, sat_mode, kernel);
}

ngemm_status ngemm_cuda_gemm_packed_resident_host(ngemm_packed_handle h, const int8_t* b, int32_t* c, int64_t n,
                                                  int sat_mode) {
    if (!h) return fail(NGEMM_ERR_SHAPE, "null handle");
    if (h->esize != 1) return fail(NGEMM_ERR_UNSUPPORTED, "gemm_packed_resident_host: u8 weights only");
    ngemm_status s = validate(h->d_a, h->lda, b, h->k, c, n, h->m, n, h->k, sat_mode);
    if (s != NGEMM_OK) return s;
    int dev;
    DevInfo di;
    s = current_device(&dev, &di);
    if (s != NGEMM_OK) return s;
    if (dev != h->device) return fail(NGEMM_ERR_UNSUPPORTED, "weight handle lives on another device");
    if (pipeline_worth(h->m, n, h->k)) {  // B streams in by column blocks, C tiles stream out
        HostGemm g;
        g.a_dev = h->d_a;
        g.lda_dev = h->lda;
        g.b_host = b;
        g.c_host = c;
        g.b_pinned = is_pinned(b);
        g.c_pinned = is_pinned(c);
        g.m = h->m;
        g.n = n;
        g.k = h->k;
        g.mode = sat_mode;
        g.kernel = NGEMM_KERNEL_AUTO;
        s = host_pipeline(g);
        if (s != NGEMM_ERR_UNSUPPORTED) return s;
    }
    const int64_t k = h->k, m = h->m, kp = round_up(k, 16);
    const size_t b_bytes = static_cast<size_t>(n * kp), c_bytes = static_cast<size_t>(m * n) * 4;
    const size_t c_off = round_up(b_bytes, 256);
    cudaStream_t st = cudaStreamPerThread;
    uint8_t* buf = nullptr;
    NG_CUDA(dev_alloc(&buf, c_off + c_bytes, st));
    s = copy_rows_h2d(buf, kp, b, k, n, st) == cudaSuccess ? NGEMM_OK : fail(NGEMM_ERR_CUDA, "H2D copy failed");
    if (s == NGEMM_OK)
        s = run_gemm(h->d_a, h->lda, reinterpret_cast<const int8_t*>(buf), kp, reinterpret_cast<int32_t*>(buf + c_off),
                     n, m, n, k, sat_mode, NGEMM_KERNEL_AUTO, st);
    if (s == NGEMM_OK && cudaMemcpyAsync(c, buf + c_off, c_bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess)
        s = fail(NGEMM_ERR_CUDA, "D2H copy failed");
    cudaFreeAsync(buf, st);
    if (cudaStreamSynchronize(st) != cudaSuccess && s == NGEMM_OK)
        s = fail(NGEMM_ERR_CUDA, std::string("gemm_packed_resident_host: ") + cudaGetErrorString(cudaGetLastError()));
    return s;
}

ngemm_status ngemm_cuda_device(int* device) {
    if (!device) return fail(NGEMM_ERR_SHAPE, "null pointer");
    NG_CUDA(cudaGetDevice(device));
    return NGEMM_OK;
}

ngemm_status ngemm_cuda_gemm_i16_host(const int16_t* a, const int16_t* b, int32_t* c, int64_t m, int64_t n,
                                      int64_t k) {
    ngemm_status s = validate(a, k, b, k, c, n, m, n, k, NGEMM_SAT_EXACT);
    if (s != NGEMM_OK) return s;
    return host_gemm(2, nullptr, a, 0, b, c, m, n, k, NGEMM_SAT_EXACT, NGEMM_KERNEL_SIMT);
}

ngemm_status ngemm_cuda_gemm_packed_host(const ngemm_packed_meta* meta, const uint8_t* host_packed, size_t nbytes,
                                         const void* b, int32_t* c, int64_t n, int sat_mode, int kernel) {
    ngemm_status s = validate_meta(meta);
    if (s != NGEMM_OK) return s;
    const int esize = meta->h == 4 ? 1 : 2;
    if (nbytes != static_cast<size_t>(meta->m_pad * meta->k_pad * esize))
        return fail(NGEMM_ERR_SHAPE, "gemm_packed_host: byte size disagrees with m_pad*k_pad");
    const int64_t m = meta->m_orig, k = meta->k_orig;
    s = validate(host_packed, k, b, k, c, n, m, n, k, esize == 1 ? sat_mode : NGEMM_SAT_EXACT);
    if (s != NGEMM_OK) return s;
    return host_gemm(esize, meta, host_packed, nbytes, b, c, m, n, k, sat_mode,
                     esize == 1 ? kernel : NGEMM_KERNEL_SIMT);
}

// ---------------------------------------------------------------- multi-GPU M-shard driver
ngemm_status ngemm_cuda_shard_rows(int64_t m, int ndev, int64_t align, int64_t* row_start) {
    if (m < 1 || ndev < 1 || align < 1 || !row_start) return fail(NGEMM_ERR_CONFIG, "shard_rows: bad arguments");
    const int64_t per = round_up((m + ndev - 1) / ndev, align);
    for (int d = 0; d <= ndev; ++d) row_start[d] = std::min<int64_t>(m, per * d);
    return NGEMM_OK;
}

}  // extern "C"

namespace {

// Peer access between every pair of distinct devices in the list (NVLink / NVSwitch), once per
// process and pair; a pair without P2P keeps working (copies are then staged by the driver).
void enable_peers(const int* devices, int ndev) {
    static std::mutex mu;
    static std::vector<std::pair<int, int>> done;
    std::lock_guard<std::mutex> lk(mu);
    int prev = 0;
    cudaGetDevice(&prev);
    for (int i = 0; i < ndev; ++i)
        for (int j = 0; j < ndev; ++j) {
            const int a = devices[i], b = devices[j];
            if (a == b || std::find(done.begin(), done.end(), std::make_pair(a, b)) != done.end()) continue;
            done.push_back({a, b});
            int can = 0;
            if (cudaDeviceCanAccessPeer(&can, a, b) != cudaSuccess || !can) {
                cudaGetLastError();
                continue;
            }
            cudaSetDevice(a);
            if (cudaDeviceEnablePeerAccess(b, 0) != cudaSuccess) cudaGetLastError();  // already enabled is fine
        }
    cudaSetDevice(prev);
}

// Replicas of one host buffer (rows x k bytes, row pitch kp on the devices) on every device: ONE
// host-to-device copy into devices[0], then a chunked relay devices[0] -> [1] -> ... over NVLink
// (each chunk is forwarded as soon as it lands), so PCIe carries B once and the replication costs
// about one chunk per extra device.  ready[d] is recorded on device d once its replica is whole.
struct Replicas {
    std::vector<uint8_t*> ptr;
    std::vector<cudaStream_t> st;
    std::vector<cudaEvent_t> ready;
};
ngemm_status replicate_rows(const int* devices, int ndev, const void* host, int64_t rows, int64_t k, int64_t kp,
                            Replicas* r) {
    r->ptr.assign(ndev, nullptr);
    r->st.assign(ndev, nullptr);
    r->ready.assign(ndev, nullptr);
    const int64_t chunk = std::max<int64_t>(1, (16 << 20) / kp);
    const int64_t nchunks = (rows + chunk - 1) / chunk;
    std::vector<std::vector<cudaEvent_t>> landed(ndev, std::vector<cudaEvent_t>(static_cast<size_t>(nchunks), nullptr));
    ngemm_status s = NGEMM_OK;
    for (int d = 0; d < ndev && s == NGEMM_OK; ++d) {
        if (cudaSetDevice(devices[d]) != cudaSuccess ||
            cudaStreamCreateWithFlags(&r->st[d], cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&r->ready[d], cudaEventDisableTiming) != cudaSuccess ||
            dev_alloc(&r->ptr[d], static_cast<size_t>(rows * kp), r->st[d]) != cudaSuccess) {
            s = fail(NGEMM_ERR_CUDA, "replicate: device setup failed on device " + std::to_string(devices[d]));
            break;
        }
        for (auto& e : landed[d])
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) s = fail(NGEMM_ERR_CUDA, "event");
    }
    for (int64_t c = 0; c < nchunks && s == NGEMM_OK; ++c) {
        const int64_t r0 = c * chunk, nr = std::min(chunk, rows - r0);
        for (int d = 0; d < ndev && s == NGEMM_OK; ++d) {
            cudaSetDevice(devices[d]);
            cudaError_t e;
            if (d == 0) {
                e = copy_rows_h2d(r->ptr[0] + r0 * kp, kp, static_cast<const uint8_t*>(host) + r0 * k, k, nr, r->st[0]);
            } else {
                cudaStreamWaitEvent(r->st[d], landed[d - 1][c], 0);
                e = cudaMemcpyPeerAsync(r->ptr[d] + r0 * kp, devices[d], r->ptr[d - 1] + r0 * kp, devices[d - 1],
                                        static_cast<size_t>(nr * kp), r->st[d]);
            }
            if (e != cudaSuccess) s = fail(NGEMM_ERR_CUDA, std::string("replicate: ") + cudaGetErrorString(e));
            else cudaEventRecord(landed[d][c], r->st[d]);
        }
    }
    for (int d = 0; d < ndev && s == NGEMM_OK; ++d) {
        cudaSetDevice(devices[d]);
        cudaEventRecord(r->ready[d], r->st[d]);
    }
    // chunk events may be destroyed right after their records are enqueued (the driver releases
    // them once they complete); on failure drain the relay before the caller frees the replicas
    for (int d = 0; d < ndev; ++d) {
        if (!r->st[d]) continue;
        cudaSetDevice(devices[d]);
        if (s != NGEMM_OK) cudaStreamSynchronize(r->st[d]);
        for (auto& e : landed[d])
            if (e) cudaEventDestroy(e);
    }
    return s;
}

void free_replicas(const int* devices, int ndev, Replicas* r) {
    for (int d = 0; d < ndev && d < static_cast<int>(r->ptr.size()); ++d) {
        cudaSetDevice(devices[d]);
        if (r->ptr[d]) cudaFreeAsync(r->ptr[d], r->st[d]);
        if (r->st[d]) {
            cudaStreamSynchronize(r->st[d]);
            cudaStreamDestroy(r->st[d]);
        }
        if (r->ready[d]) cudaEventDestroy(r->ready[d]);
    }
}

// One host thread per device running the host pipeline on its row shard (A rows streamed in,
// the replicated B resident, C rows streamed out to the host and/or peer-copied to the gather
// buffer).  `a_dev` (per device) replaces the host A for resident sharded weights.
ngemm_status run_multi(const int* devices, int ndev, const std::vector<int64_t>& rs, const uint8_t* a_host,
                       const std::vector<const uint8_t*>& a_dev, const std::vector<int64_t>& lda_dev, const int8_t* b,
                       int32_t* c, int64_t n, int64_t k, int sat_mode, int gather_device, int32_t* full) {
    enable_peers(devices, ndev);
    if (gather_device >= 0) {
        std::vector<int> all(devices, devices + ndev);
        all.push_back(gather_device);
        enable_peers(all.data(), ndev + 1);
    }
    const int64_t kp = round_up(k, 16);
    Replicas rep;
    ngemm_status s = replicate_rows(devices, ndev, b, n, k, kp, &rep);
    std::vector<ngemm_status> st(static_cast<size_t>(ndev), NGEMM_OK);
    std::vector<std::string> msg(static_cast<size_t>(ndev));
    if (s == NGEMM_OK) {
        const bool a_pinned = a_host && is_pinned(a_host), b_pinned = is_pinned(b), c_pinned = c && is_pinned(c);
        std::vector<std::thread> workers;
        for (int d = 0; d < ndev; ++d) {
            workers.emplace_back([&, d] {
                const int64_t r0 = rs[d], rows = rs[d + 1] - rs[d];
                if (rows <= 0) return;
                if (cudaSetDevice(devices[d]) != cudaSuccess) {
                    st[d] = fail(NGEMM_ERR_CUDA, "cudaSetDevice failed");
                    msg[d] = ngemm_cuda_last_error();
                    return;
                }
                HostGemm g;
                if (!a_dev.empty()) {
                    g.a_dev = a_dev[d];
                    g.lda_dev = lda_dev[d];
                } else {
                    g.a_host = a_host + r0 * k;
                    g.a_pinned = a_pinned;
                }
                g.b_dev = reinterpret_cast<const int8_t*>(rep.ptr[d]);
                g.ldb_dev = kp;
                g.b_ready = rep.ready[d];
                g.b_pinned = b_pinned;
                g.c_host = c ? c + r0 * n : nullptr;
                g.c_pinned = c_pinned;
                g.c_gather = full ? full + r0 * n : nullptr;
                g.gather_dev = gather_device;
                g.m = rows;
                g.n = n;
                g.k = k;
                g.mode = sat_mode;
                g.kernel = NGEMM_KERNEL_AUTO;
                st[d] = host_pipeline(g);
                if (st[d] != NGEMM_OK) msg[d] = st[d] == NGEMM_ERR_UNSUPPORTED ? "row too long for staging" : ngemm_cuda_last_error();
            });
        }
        for (auto& w : workers) w.join();
    }
    free_replicas(devices, ndev, &rep);
    if (s != NGEMM_OK) return s;
    for (int d = 0; d < ndev; ++d)
        if (st[d] != NGEMM_OK) return fail(st[d], "device " + std::to_string(devices[d]) + ": " + msg[d]);
    return NGEMM_OK;
}

}  // namespace

extern "C" {

ngemm_status ngemm_cuda_gemm_u8i8_multi(const int* devices, int ndev, const uint8_t* a, const int8_t* b, int32_t* c,
                                        int64_t m, int64_t n, int64_t k, int sat_mode, int gather_device,
                                        int32_t** gathered) {
    if (!devices || ndev < 1) return fail(NGEMM_ERR_CONFIG, "multi: empty device list");
    const bool want_gather = gather_device >= 0 && gathered != nullptr;
    if (!c && !want_gather) return fail(NGEMM_ERR_SHAPE, "multi: no output (host C and gather both absent)");
    ngemm_status s = validate(a, k, b, k, c ? static_cast<const void*>(c) : static_cast<const void*>(a), n, m, n, k,
                              sat_mode);
    if (s != NGEMM_OK) return s;
    if (round_up(k, 16) > static_cast<int64_t>(kSlotBytes)) return fail(NGEMM_ERR_SHAPE, "multi: K too large");
    std::vector<int64_t> rs(static_cast<size_t>(ndev) + 1);
    ngemm_cuda_shard_rows(m, ndev, tc::BM, rs.data());
    int prev = 0;
    cudaGetDevice(&prev);
    int32_t* full = nullptr;
    if (want_gather) {
        NG_CUDA(cudaSetDevice(gather_device));
        NG_CUDA(cudaMalloc(&full, static_cast<size_t>(m * n) * 4));
    }
    s = run_multi(devices, ndev, rs, a, {}, {}, b, c, n, k, sat_mode, want_gather ? gather_device : -1, full);
    if (full) {  // gather copies ran on the workers' streams, which host_pipeline synchronised
        cudaSetDevice(gather_device);
        if (s != NGEMM_OK) {
            cudaFree(full);
            full = nullptr;
        }
    }
    cudaSetDevice(prev);
    if (s != NGEMM_OK) return s;
    if (want_gather) *gathered = full;
    return NGEMM_OK;
}

// Sharded resident weight: the packed weight's rows split over `devices` in tile-aligned blocks
// of whole tm-strips (ngemm_cuda_shard_rows with align = lcm(tm, 128)).  With an M-before-K
// permutation each strip is one contiguous byte range (layout.hpp:159-161), so a shard is a plain
// copy of the packed bytes; with K-before-M each K tile row contributes one contiguous run of the
// shard's strips, gathered on the host.  Each shard is then repacked on its device.
ngemm_status ngemm_cuda_packed_upload_sharded(const ngemm_packed_meta* meta, const uint8_t* host_packed, size_t nbytes,
                                              const int* devices, int ndev, ngemm_packed_handle* out) {
    ngemm_status s = validate_meta(meta);
    if (s != NGEMM_OK) return s;
    if (!devices || ndev < 1 || !out || !host_packed) return fail(NGEMM_ERR_CONFIG, "upload_sharded: bad arguments");
    if (meta->h != 4) return fail(NGEMM_ERR_UNSUPPORTED, "upload_sharded: u8 weights only");
    if (nbytes != static_cast<size_t>(meta->m_pad * meta->k_pad))
        return fail(NGEMM_ERR_SHAPE, "upload_sharded: byte size disagrees with m_pad*k_pad");
    const int64_t tm = meta->tm, tk = meta->tk;
    int64_t align = 128;
    while (align % tm) align += 128;  // lcm(tm, 128)
    std::vector<int64_t> rs(static_cast<size_t>(ndev) + 1);
    ngemm_cuda_shard_rows(meta->m_orig, ndev, align, rs.data());
    const bool m_first = meta->perm == 0 || meta->perm == 1 || meta->perm == 2;
    const int64_t n_tm = meta->m_pad / tm, n_tk = meta->k_pad / tk, tile_bytes = tm * tk;
    int prev = 0;
    cudaGetDevice(&prev);
    for (int d = 0; d < ndev; ++d) out[d] = nullptr;
    std::vector<uint8_t> gathered;
    for (int d = 0; d < ndev && s == NGEMM_OK; ++d) {
        const int64_t rows = rs[d + 1] - rs[d];
        if (rows <= 0) continue;
        const int64_t s0 = rs[d] / tm, s1 = (rs[d] + round_up(rows, tm)) / tm;  // strips [s0, s1)
        ngemm_packed_meta sm = *meta;
        sm.m_orig = rows;
        sm.m_pad = (s1 - s0) * tm;
        const uint8_t* src;
        if (m_first) {
            src = host_packed + s0 * n_tk * tile_bytes;
        } else {
            gathered.resize(static_cast<size_t>(sm.m_pad * meta->k_pad));
            for (int64_t t = 0; t < n_tk; ++t)
                std::memcpy(gathered.data() + t * (s1 - s0) * tile_bytes, host_packed + (t * n_tm + s0) * tile_bytes,
                            static_cast<size_t>((s1 - s0) * tile_bytes));
            src = gathered.data();
        }
        if (cudaSetDevice(devices[d]) != cudaSuccess) s = fail(NGEMM_ERR_CUDA, "cudaSetDevice failed");
        if (s == NGEMM_OK) s = ngemm_cuda_packed_upload(&sm, src, static_cast<size_t>(sm.m_pad * sm.k_pad), &out[d]);
    }
    cudaSetDevice(prev);
    if (s != NGEMM_OK)
        for (int d = 0; d < ndev; ++d) {
            ngemm_cuda_packed_free(out[d]);
            out[d] = nullptr;
        }
    return s;
}

// gemm_ngemm over a sharded resident weight: B replicated by one H2D + NVLink relay, every
// device computes its rows of C from its resident shard, C rows stream back to the host.
ngemm_status ngemm_cuda_gemm_packed_multi(const ngemm_packed_handle* shards, int ndev, const int8_t* b, int32_t* c,
                                          int64_t n, int sat_mode) {
    if (!shards || ndev < 1 || !b || !c) return fail(NGEMM_ERR_SHAPE, "packed_multi: bad arguments");
    std::vector<int> devices;
    std::vector<const uint8_t*> a_dev;
    std::vector<int64_t> lda, rs{0};
    int64_t k = -1;
    for (int d = 0; d < ndev; ++d) {
        if (!shards[d]) continue;  // an empty shard (more devices than row blocks)
        if (shards[d]->esize != 1) return fail(NGEMM_ERR_UNSUPPORTED, "packed_multi: u8 weights only");
        if (k >= 0 && shards[d]->k != k) return fail(NGEMM_ERR_SHAPE, "packed_multi: shards disagree on K");
        k = shards[d]->k;
        devices.push_back(shards[d]->device);
        a_dev.push_back(shards[d]->d_a);
        lda.push_back(shards[d]->lda);
        rs.push_back(rs.back() + shards[d]->m);
    }
    if (devices.empty()) return fail(NGEMM_ERR_SHAPE, "packed_multi: no shards");
    ngemm_status s = validate(a_dev[0], lda[0], b, k, c, n, rs.back(), n, k, sat_mode);
    if (s != NGEMM_OK) return s;
    int prev = 0;
    cudaGetDevice(&prev);
    s = run_multi(devices.data(), static_cast<int>(devices.size()), rs, nullptr, a_dev, lda, b, c, n, k, sat_mode, -1,
                  nullptr);
    cudaSetDevice(prev);
    return s;
}

// ---------------------------------------------------------------- GPU autotuner (tuner.hpp:132-245)
// Exhaustive search over the engine's own knobs for one (m, n, k, mode) on the current device:
// seeded full-range operands, every candidate verified bit-for-bit against the CUDA-core
// kernel (the lane-faithful Engine::Emulated path) before its timing counts; median of
// `repeats` CUDA-event timings after `warmup` runs; the winner is recorded in the in-process
// table the dispatcher consults (and can be persisted with ngemm_cuda_tune_store_save).
ngemm_status ngemm_cuda_tune(int64_t m, int64_t n, int64_t k, int sat_mode, int repeats, int warmup,
                             ngemm_tune_record* out) {
    if (repeats < 3 || warmup < 1) return fail(NGEMM_ERR_CONFIG, "tune: repeats must be >= 3 and warmup >= 1");
    int dev;
    DevInfo di;
    ngemm_status s = current_device(&dev, &di);
    if (s != NGEMM_OK) return s;
    s = validate(reinterpret_cast<void*>(1), k, reinterpret_cast<void*>(1), k, reinterpret_cast<void*>(1), n, m, n, k,
                 sat_mode);
    if (s != NGEMM_OK) return s;
    const int64_t kp = round_up(k, 16);
    const size_t a_b = static_cast<size_t>(m * kp), b_b = static_cast<size_t>(n * kp), c_b = static_cast<size_t>(m * n) * 4;
    const size_t b_off = round_up(static_cast<int64_t>(a_b), 256), c0 = b_off + round_up(static_cast<int64_t>(b_b), 256),
                 c1 = c0 + round_up(static_cast<int64_t>(c_b), 256), bad_off = c1 + round_up(static_cast<int64_t>(c_b), 256);
    uint8_t* buf = nullptr;
    NG_CUDA(cudaMalloc(&buf, bad_off + 64));
    cudaStream_t st = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    uint8_t* da = buf;
    int8_t* db = reinterpret_cast<int8_t*>(buf + b_off);
    int32_t* cref = reinterpret_cast<int32_t*>(buf + c0);
    int32_t* ctry = reinterpret_cast<int32_t*>(buf + c1);
    auto* bad = reinterpret_cast<unsigned long long*>(buf + bad_off);
    cudaMemset(buf, 0, bad_off + 64);
    fill_random_kernel<<<di.sms * 4, 256, 0, st>>>(da, m, k, kp, 0x4E47454D4D31ull);
    fill_random_kernel<<<di.sms * 4, 256, 0, st>>>(reinterpret_cast<uint8_t*>(db), n, k, kp, 0x4E47454D4D32ull);
    g_launches.fetch_add(2, std::memory_order_relaxed);
    s = run_gemm(da, kp, db, kp, cref, n, m, n, k, sat_mode, NGEMM_KERNEL_SIMT, st);  // the reference result

    std::vector<Choice> cands;
    if (m <= kSkinnyMaxM) {
        for (int v = 0; v < 6; ++v) {
            if (sat_mode == NGEMM_SAT_EXACT ? v >= 4 : (v == 2 || v == 3)) continue;
            Choice c;
            c.kernel = NGEMM_KERNEL_SKINNY;
            c.skinny_variant = v;
            cands.push_back(c);
        }
    } else if (sat_mode == NGEMM_SAT_EXACT) {
        for (int cfg = 0; cfg < TC_NUM_CFG; ++cfg) {
            const TcCfgInfo& ci = kTcCfg[cfg];
            if (ci.mc > 1 && ((n + ci.bn - 1) / ci.bn) % ci.mc != 0) continue;
            for (int sp : {1, 2, 4}) {
                if (sp > 1 && (k + tc::BK - 1) / tc::BK < 4 * sp) continue;
                Choice c;
                c.kernel = NGEMM_KERNEL_TCGEN05;
                c.tc_cfg = cfg;
                c.tc_splits = sp;
                cands.push_back(c);
            }
        }
    }
    {
        Choice c;
        c.kernel = NGEMM_KERNEL_SIMT;
        cands.push_back(c);
        if (sat_mode != NGEMM_SAT_EXACT && m > kSkinnyMaxM) {
            Choice p;  // tensor cores + sparse fix of the pairs that can clamp
            p.kernel = NGEMM_KERNEL_SAT_HYBRID;
            cands.push_back(p);
        }
    }
    ngemm_tune_record best{};
    best.median_ns = 1e30;
    for (const Choice& c : cands) {
        if (s != NGEMM_OK) break;
        struct Restore {
            Choice saved = t_force;
            ~Restore() { t_force = saved; }
        } restore;
        t_force = c;
        auto once = [&]() { return run_gemm(da, kp, db, kp, ctry, n, m, n, k, sat_mode, c.kernel, st); };
        cudaMemsetAsync(ctry, 0x5A, c_b, st);
        s = once();
        if (s != NGEMM_OK) break;
        cudaMemsetAsync(bad, 0, 8, st);
        count_mismatch_kernel<<<di.sms * 4, 256, 0, st>>>(cref, ctry, m * n, bad);
        unsigned long long nbad = 0;
        cudaMemcpy(&nbad, bad, 8, cudaMemcpyDeviceToHost);
        if (nbad) {
            s = fail(NGEMM_ERR_TUNE, "tune: candidate kernel=" + std::to_string(c.kernel) + " cfg=" +
                                         std::to_string(c.tc_cfg) + " splits=" + std::to_string(c.tc_splits) +
                                         " variant=" + std::to_string(c.skinny_variant) + " disagrees with the "
                                         "reference kernel on " + std::to_string(nbad) + " elements");
            break;
        }
        for (int w = 0; w < warmup && s == NGEMM_OK; ++w) s = once();
        std::vector<float> t;
        for (int r = 0; r < repeats && s == NGEMM_OK; ++r) {
            cudaEventRecord(e0, st);
            s = once();
            cudaEventRecord(e1, st);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            t.push_back(ms);
        }
        if (s != NGEMM_OK) break;
        std::sort(t.begin(), t.end());
        const double med = (t.size() % 2 ? t[t.size() / 2] : 0.5 * (t[t.size() / 2 - 1] + t[t.size() / 2])) * 1e6;
        if (med < best.median_ns) {
            best.kernel = c.kernel;
            best.tc_cfg = c.tc_cfg;
            best.tc_splits = c.tc_splits;
            best.skinny_variant = c.skinny_variant;
            best.median_ns = med;
            best.min_ns = t.front() * 1e6;
        }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(buf);
    if (s != NGEMM_OK) return s;
    best.m = m;
    best.n = n;
    best.k = k;
    best.sat_mode = sat_mode;
    best.trials = repeats;
    best.timestamp = static_cast<int64_t>(std::chrono::duration_cast<std::chrono::seconds>(
                                              std::chrono::system_clock::now().time_since_epoch())
                                              .count());
    tuned_put(best);
    if (out) *out = best;
    return NGEMM_OK;
}

// Tune store (tuner.hpp:177-245 style): one record per line, fixed field order, append-only,
// last record for a key wins:  m n k mode kernel tc_cfg tc_splits skinny_variant median_ns min_ns trials timestamp
ngemm_status ngemm_cuda_tune_store_save(const char* path) {
    if (!path) return fail(NGEMM_ERR_CONFIG, "tune store: null path");
    std::ofstream f(path, std::ios::app);
    if (!f) return fail(NGEMM_ERR_CONFIG, std::string("tune store: cannot open ") + path);
    std::lock_guard<std::mutex> lk(g_tune_mu);
    for (const auto& kv : g_tuned) {
        const ngemm_tune_record& r = kv.second.second;
        f << r.m << ' ' << r.n << ' ' << r.k << ' ' << r.sat_mode << ' ' << r.kernel << ' ' << r.tc_cfg << ' '
          << r.tc_splits << ' ' << r.skinny_variant << ' ' << r.median_ns << ' ' << r.min_ns << ' ' << r.trials << ' '
          << r.timestamp << '\n';
    }
    return f ? NGEMM_OK : fail(NGEMM_ERR_CONFIG, "tune store: write failed");
}

ngemm_status ngemm_cuda_tune_store_load(const char* path, int* loaded) { return load_store_file(path, loaded); }

}  // extern "C"

namespace {
ngemm_status load_store_file(const char* path, int* loaded) {
    if (!path) return fail(NGEMM_ERR_CONFIG, "tune store: null path");
    std::ifstream f(path);
    if (!f) return fail(NGEMM_ERR_CONFIG, std::string("tune store: cannot open ") + path);
    std::string line;
    int count = 0, lineno = 0;
    while (std::getline(f, line)) {
        ++lineno;
        if (line.empty() || line[0] == '#') continue;
        std::istringstream is(line);
        ngemm_tune_record r{};
        if (!(is >> r.m >> r.n >> r.k >> r.sat_mode >> r.kernel >> r.tc_cfg >> r.tc_splits >> r.skinny_variant >>
              r.median_ns >> r.min_ns >> r.trials >> r.timestamp) ||
            r.m < 1 || r.n < 1 || r.k < 1 || (r.sat_mode != 0 && r.sat_mode != 1) || r.kernel < 0 || r.kernel > 4)
            return fail(NGEMM_ERR_CONFIG, "tune store: malformed record at line " + std::to_string(lineno));
        tuned_put(r);
        ++count;
    }
    if (loaded) *loaded = count;
    return NGEMM_OK;
}
}  // namespace

extern "C" {

ngemm_status ngemm_cuda_set_option(const char* name, int value) {
    const int i = opt_index(name);
    if (i < 0) return fail(NGEMM_ERR_CONFIG, std::string("unknown option ") + (name ? name : "(null)"));
    std::call_once(g_opt_once, load_opts);
    g_opt[i].store(value, std::memory_order_relaxed);
    return NGEMM_OK;
}

int ngemm_cuda_get_option(const char* name) {
    const int i = opt_index(name);
    return i < 0 ? INT32_MIN : opt(static_cast<Opt>(i));
}

ngemm_status ngemm_cuda_reset_options(void) {
    std::call_once(g_opt_once, load_opts);
    load_opts();
    return NGEMM_OK;
}

ngemm_status ngemm_cuda_trim(void) {
    int dev = 0;
    NG_CUDA(cudaGetDevice(&dev));
    if (cudaMemPool_t pool = lib_pool(dev)) {
        NG_CUDA(cudaDeviceSynchronize());
        NG_CUDA(cudaMemPoolTrimTo(pool, 0));
    }
    return NGEMM_OK;
}

ngemm_status ngemm_cuda_tune_clear(void) {
    std::lock_guard<std::mutex> lk(g_tune_mu);
    g_tuned.clear();
    return NGEMM_OK;
}

ngemm_status ngemm_cuda_free(void* p) {
    if (p) NG_CUDA(cudaFree(p));
    return NGEMM_OK;
}

}  // extern "C"

#ifdef NGEMM_TRACE
extern "C" int ngemm_trace_reset(void) {  // zero the stamps; the next traced launch gets id 0
    static unsigned long long zeros[kTraceL * kTraceCta * kTraceP];
    g_trace_next = 0;
    return cudaMemcpyToSymbol(g_tc_trace, zeros, sizeof(zeros)) == cudaSuccess ? 0 : 1;
}
extern "C" int ngemm_trace_read(void* dst, size_t bytes) {
    if (bytes > sizeof(g_tc_trace)) bytes = sizeof(g_tc_trace);
    return cudaMemcpyFromSymbol(dst, g_tc_trace, bytes) == cudaSuccess ? 0 : 1;
}
#endif
